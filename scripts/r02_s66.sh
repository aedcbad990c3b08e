# round-2 pass 66: does the plan's single-CTA scan wait for the gather to end?
# (256 x 58-register CTA > the 12 K registers a u8 gather CTA leaves) —
# scan128 / scan64 vs base: timelines and c2 benches.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s66
mkdir -p $O
export PYTHONUNBUFFERED=1
B="python bench.py --no-e2e --no-cpu-baseline --steps 50"
for v in nmsbase scan128 scan64; do
 for fmt in 1 0; do
  MP_LIB=build/ab/$v.so CFG=c2_1080p_sparse DEPTH=3 FMT=$fmt timeout -s KILL 300 python scripts/timeline.py > $O/tl_c2_fmt${fmt}_$v.txt 2>&1
 done
done
for rep in 1 2; do
 for v in nmsbase scan128 scan64; do
  MP_LIB=build/ab/$v.so timeout -s KILL 300 $B --config c2_1080p_sparse --fmt u8 > $O/u8_c2_${v}_$rep.log 2>&1
  MP_LIB=build/ab/$v.so timeout -s KILL 300 $B --config c2_1080p_sparse > $O/f32_c2_${v}_$rep.log 2>&1
 done
done
ls $O
