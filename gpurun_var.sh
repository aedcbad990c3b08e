cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
timeout -s KILL 600 python bench.py --mode wsel --steps 3 --warmup 1 > gpurun_out/bench_wsel.log 2>&1
timeout -s KILL 600 python bench.py --mode sweep --steps 10 --warmup 3 > gpurun_out/bench_sweep.log 2>&1
