# round-2 pass 60: plan alone and the depth-3 pipelined timeline, base vs
# int16-box planner (c4 u8 step 2.65 -> 2.74 ms in pass 59: why).
cd $GRAFT_REPO_ROOT
O=gpurun_out/s60
mkdir -p $O
export PYTHONUNBUFFERED=1
for v in base box16; do
 for fmt in 1 0; do
  MP_LIB=build/ab/$v.so CFG=c4_4k_drone DEPTH=3 FMT=$fmt timeout -s KILL 300 python scripts/timeline.py > $O/tl_c4_fmt${fmt}_$v.txt 2>&1
 done
 MP_LIB=build/ab/$v.so CFG=c3_1080p_dense DEPTH=3 FMT=1 timeout -s KILL 300 python scripts/timeline.py > $O/tl_c3_fmt1_$v.txt 2>&1
done
ls $O
