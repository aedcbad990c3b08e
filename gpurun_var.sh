cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
for d in 1 2 3; do timeout -s KILL 600 python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu-baseline --depth $d > gpurun_out/bench_d$d.log 2>&1; done
