cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/var.log
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_proxy_sweep.py tests/test_window_sets.py -q -x -m gpu > gpurun_out/pytest_plan.log 2>&1
for c in c4_4k_drone c3_1080p_dense c2_1080p_sparse; do
  timeout -s KILL 300 python bench.py --config $c --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/b.log 2>&1
  echo "$c $(tail -1 gpurun_out/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'], d['roofline']['launch_ms'])")" >> gpurun_out/var.log
done
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"plan_" -c 8 --csv --log-file gpurun_out/plan_c4.csv python bench.py --config c4_4k_drone --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 --graphs 0 > /dev/null 2>&1
