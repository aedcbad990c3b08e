# round-2 pass 72: f32 lines, 4-warp NMS tiny tier vs current (3 interleaved reps).
cd $GRAFT_REPO_ROOT
O=gpurun_out/s72
mkdir -p $O
export PYTHONUNBUFFERED=1
B="python bench.py --no-e2e --no-cpu-baseline --steps 100"
for rep in 1 2 3; do
 for v in cur tiny4; do
  MP_LIB=build/ab/$v.so timeout -s KILL 300 $B --config c2_1080p_sparse > $O/f32_c2_${v}_$rep.log 2>&1
 done
done
for v in cur tiny4; do
  MP_LIB=build/ab/$v.so timeout -s KILL 300 $B --config c3_1080p_dense --steps 30 > $O/f32_c3_${v}.log 2>&1
  MP_LIB=build/ab/$v.so timeout -s KILL 300 $B --config c2_1080p_sparse --src nv12 > $O/nv12_c2_${v}.log 2>&1
  MP_LIB=build/ab/$v.so timeout -s KILL 300 $B --config c1_540p > $O/f32_c1_${v}.log 2>&1
done
ls $O
