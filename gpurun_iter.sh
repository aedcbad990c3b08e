cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout -s KILL 600 python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/bench.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" -s 3 -c 1 -o gpurun_out/prof_gather python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof_bench.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
