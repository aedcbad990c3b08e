cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_nv12.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_nv12.log 2>&1
WHAT=proxy_nv12,proxy_rgb timeout -s KILL 300 python scripts/time_gather.py > gpurun_out/var.log 2>&1
timeout -s KILL 600 python bench.py --steps 100 --warmup 5 --src nv12 > gpurun_out/bench_nv12.log 2>&1
timeout -s KILL 600 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1
