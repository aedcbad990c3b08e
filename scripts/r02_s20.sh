# round-2 pass 20: plan grids up to 65536 cells.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s20
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_proxy_sweep.py tests/test_window_sets.py -m gpu -q -x -k "plan or fuzz or sweep or window" > $O/plan_tests.log 2>&1; echo "rc=$?" >> $O/plan_tests.log
timeout -s KILL 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "8k_grid" > $O/san_memcheck_8k.log 2>&1; echo "rc=$?" >> $O/san_memcheck_8k.log
timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --steps 50 --config c4_4k_drone > $O/bench_c4.log 2>&1
ls -la $O
