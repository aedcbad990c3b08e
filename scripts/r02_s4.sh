# round-2 session-2 pass 4: dead-flag cooperative merge; evidence captures.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s4
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_proxy_sweep.py tests/test_window_sets.py -m gpu -q -x -k "plan or fuzz or sweep or window" > $O/plan_tests.log 2>&1; echo "rc=$?" >> $O/plan_tests.log
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $O/all.log 2>&1; echo "rc=$?" >> $O/all.log
CFG=c4_4k_drone DEPTH=3 timeout -s KILL 600 python scripts/timeline.py > $O/timeline_c4.txt 2>&1
B="python bench.py --no-e2e --no-cpu-baseline --steps 50"
for c in c2_1080p_sparse c4_4k_drone c3_1080p_dense c1_540p; do timeout -s KILL 600 $B --config $c > $O/bench_$c.log 2>&1; done
timeout -s KILL 600 $B --fmt u8 > $O/bench_u8.log 2>&1
timeout -s KILL 600 python bench.py --mode sweep > $O/bench_sweep.log 2>&1
timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --steps 5 --warmup 3 --trace $O/trace_c2.json > $O/trace_c2.log 2>&1
timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 --config c1_540p --trace $O/trace_c1.json > $O/trace_c1.log 2>&1
D="python bench.py --no-e2e --no-cpu-baseline --depth 1 --steps 2 --warmup 3"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"plan_full_kernel" -s 2 -c 1 -o $O/prof_plan_full -f $D --config c4_4k_drone > $O/prof_plan.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"nms_large_kernel" -s 2 -c 1 -o $O/prof_nms_large -f $D --config c4_4k_drone > $O/prof_nms.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" -s 3 -c 1 -o $O/prof_gather_nv12 -f $D --src nv12 > $O/prof_nv12.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_c1.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --config c1_540p --step-graph 0 > $O/launches_c1.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"plan_|gather_|nms_" -c 60 --csv --log-file $O/launches_c4.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 --config c4_4k_drone > $O/launches_c4.log 2>&1
ls -la $O
