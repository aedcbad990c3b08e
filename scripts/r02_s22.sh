# round-2 pass 22: side kernels at c2 (ncu), u8 gather (current code) ncu.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s22
mkdir -p $O
export PYTHONUNBUFFERED=1
D="python bench.py --no-e2e --no-cpu-baseline --depth 1 --steps 2 --warmup 3"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"plan_fast_kernel|nms_tiny_kernel|plan_full_kernel|nms_small_kernel|nms_large_kernel" -s 10 -c 5 -o $O/prof_side_c2 -f $D > $O/p1.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" -s 3 -c 1 -o $O/prof_gather_u8 -f $D --fmt u8 > $O/p2.log 2>&1
ls -la $O
