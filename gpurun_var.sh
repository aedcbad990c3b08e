cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
timeout -s KILL 600 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1
for c in c3_1080p_dense c4_4k_drone; do timeout -s KILL 600 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 30 > gpurun_out/bench_$c.log 2>&1; done
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"plan_|gather_|nms_" -c 30 --csv --log-file gpurun_out/launches_c4.csv python bench.py --config c4_4k_drone --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 > /dev/null 2>&1
