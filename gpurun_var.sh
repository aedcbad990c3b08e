cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
for d in 1 2; do timeout -s KILL 600 python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu-baseline --depth $d > gpurun_out/bench_d$d.log 2>&1; done
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"plan_|gather_|nms_" -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 > gpurun_out/launches_bench.log 2>&1
