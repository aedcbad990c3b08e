cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout -s KILL 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_assign.py -q -x -k "large or synth" > $O/san_racecheck_assign.log 2>&1; echo "rc=$?" >> $O/san_racecheck_assign.log
timeout -s KILL 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_assign.py -q -x -k "large" > $O/san_synccheck_assign.log 2>&1; echo "rc=$?" >> $O/san_synccheck_assign.log
timeout -s KILL 900 python -m pytest tests/test_gpu_assign.py -q > $O/pytest_assign.log 2>&1
timeout -s KILL 600 python bench.py --mode assign --steps 50 --warmup 5 > $O/bench_assign.log 2>&1
