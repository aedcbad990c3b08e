# round-2 pass 13: ncu of the side kernels as they are now.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s13
mkdir -p $O
export PYTHONUNBUFFERED=1
D="python bench.py --no-e2e --no-cpu-baseline --depth 1 --steps 2 --warmup 3"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"nms_small_kernel" -s 2 -c 1 -o $O/prof_nms_small_c3 -f $D --config c3_1080p_dense > $O/p1.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"plan_fast_kernel" -s 2 -c 1 -o $O/prof_plan_fast_c3 -f $D --config c3_1080p_dense > $O/p2.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"nms_large_kernel" -s 2 -c 1 -o $O/prof_nms_large_c4 -f $D --config c4_4k_drone > $O/p3.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"plan_full_kernel" -s 2 -c 1 -o $O/prof_plan_full_c4 -f $D --config c4_4k_drone > $O/p4.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" -s 3 -c 1 -o $O/prof_gather_c3 -f $D --config c3_1080p_dense > $O/p5.log 2>&1
ls -la $O
