# round-2 first evidence pass: baseline ncu --set full of the side kernels
# (plan_full_kernel, nms_large_kernel at c4) and of the u8 gather at c2.
cd $GRAFT_REPO_ROOT
O=gpurun_out/p1
mkdir -p $O
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
B="python bench.py --no-e2e --no-cpu-baseline --depth 1 --steps 2 --warmup 3"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"plan_full_kernel" -s 2 -c 1 -o $O/prof_plan_full -f $B --config c4_4k_drone > $O/prof_plan.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"nms_large_kernel" -s 2 -c 1 -o $O/prof_nms_large -f $B --config c4_4k_drone > $O/prof_nms.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" -s 3 -c 1 -o $O/prof_gather_u8 -f $B --fmt u8 > $O/prof_u8.log 2>&1
timeout -s KILL 600 python bench.py --fmt u8 --no-e2e --no-cpu-baseline --steps 50 > $O/bench_u8.log 2>&1
timeout -s KILL 600 python bench.py --config c4_4k_drone --no-e2e --no-cpu-baseline --steps 50 > $O/bench_c4.log 2>&1
ls -la $O
