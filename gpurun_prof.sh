cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python bench.py > gpurun_out/bench_full.log 2>&1
timeout -s KILL 600 python bench.py --fmt u8 --no-e2e --no-cpu-baseline > gpurun_out/bench_u8.log 2>&1
for c in c1_540p c3_1080p_dense c4_4k_drone; do timeout -s KILL 600 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 50 > gpurun_out/bench_$c.log 2>&1; done
timeout -s KILL 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"plan_|gather_|nms_" -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 > gpurun_out/launches_bench.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" -s 3 -c 1 -o gpurun_out/prof_gather python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 > gpurun_out/prof_bench.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"plan_frames|nms_tiny|gather_prep" -s 3 -c 3 -o gpurun_out/prof_small python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 > gpurun_out/prof_bench2.log 2>&1
