cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout -s KILL 900 compute-sanitizer --tool memcheck --print-limit 20 python __graft_entry__.py smoke > gpurun_out/san_memcheck_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/san_memcheck_smoke.log
timeout -s KILL 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "c1_540p or nms_parity_frame_sizes or adversarial and 200" > gpurun_out/san_memcheck_tests.log 2>&1; echo "rc=$?" >> gpurun_out/san_memcheck_tests.log
timeout -s KILL 900 compute-sanitizer --tool racecheck --print-limit 20 python __graft_entry__.py smoke > gpurun_out/san_racecheck_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/san_racecheck_smoke.log
timeout -s KILL 900 compute-sanitizer --tool synccheck --print-limit 20 python __graft_entry__.py smoke > gpurun_out/san_synccheck_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/san_synccheck_smoke.log
timeout -s KILL 900 compute-sanitizer --tool initcheck --print-limit 20 python __graft_entry__.py smoke > gpurun_out/san_initcheck_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/san_initcheck_smoke.log
