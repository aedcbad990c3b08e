# round-2 pass 71: u8 c2/c3 — a 4-warp NMS tiny tier (co-resides with a u8
# gather CTA) at k = 0 / 1 vs the current build.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s71
mkdir -p $O
export PYTHONUNBUFFERED=1
B="python bench.py --no-e2e --no-cpu-baseline --steps 50 --fmt u8"
for rep in 1 2; do
 for v in cur tiny4; do
  for k in 0 1; do
   MP_LIB=build/ab/$v.so timeout -s KILL 300 $B --config c2_1080p_sparse --gather-sm-reserve $k > $O/u8_c2_${v}_k${k}_$rep.log 2>&1
  done
 done
done
for v in cur tiny4; do
  MP_LIB=build/ab/$v.so RSV=0 CFG=c2_1080p_sparse DEPTH=3 FMT=1 timeout -s KILL 300 python scripts/timeline.py > $O/tl_c2_u8_${v}_k0.txt 2>&1
  MP_LIB=build/ab/$v.so timeout -s KILL 300 python bench.py --no-e2e --no-cpu-baseline --steps 50 --config c2_1080p_sparse > $O/f32_c2_${v}.log 2>&1
done
ls $O
