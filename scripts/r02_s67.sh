# round-2 pass 67: plan/NMS scan geometry (threads, register cap) and the NMS
# tiny tier's CTA size — c2 f32 / u8 benches (2 reps) and timelines.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s67
mkdir -p $O
export PYTHONUNBUFFERED=1
B="python bench.py --no-e2e --no-cpu-baseline --steps 50"
for v in nmsbase scan128 scan256r48 scan128r48 scan128t4; do
 for fmt in 1 0; do
  MP_LIB=build/ab/$v.so CFG=c2_1080p_sparse DEPTH=3 FMT=$fmt timeout -s KILL 300 python scripts/timeline.py > $O/tl_c2_fmt${fmt}_$v.txt 2>&1
 done
done
for rep in 1 2; do
 for v in nmsbase scan128 scan256r48 scan128r48 scan128t4; do
  MP_LIB=build/ab/$v.so timeout -s KILL 300 $B --config c2_1080p_sparse --fmt u8 > $O/u8_c2_${v}_$rep.log 2>&1
  MP_LIB=build/ab/$v.so timeout -s KILL 300 $B --config c2_1080p_sparse > $O/f32_c2_${v}_$rep.log 2>&1
 done
done
ls $O
