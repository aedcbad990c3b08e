cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for pv in 0 1 2 3; do MP_GATHER_L2PROMO=$pv timeout -s KILL 600 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_p$pv.log 2>&1; done
MP_GATHER_L2PROMO=0 timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" -s 3 -c 1 -o gpurun_out/prof_gather python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof_bench.log 2>&1
