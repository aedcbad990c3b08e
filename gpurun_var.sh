cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nv12.py -q -x > gpurun_out/pytest_u8.log 2>&1
timeout -s KILL 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --fmt u8 > gpurun_out/b_u8.log 2>&1
timeout -s KILL 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/b_f32.log 2>&1
