cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -k adversarial > gpurun_out/pytest_adv.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_adv.log
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"plan_|gather_|nms_" -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" -s 3 -c 1 -o gpurun_out/prof_gather python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof_bench.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"plan_frames|nms_small" -s 2 -c 2 -o gpurun_out/prof_plan_nms python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof_bench2.log 2>&1
ls -la gpurun_out
