# round-2 pass 5: plan tiers full (shared memory, LDS) / huge (global scratch).
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_proxy_sweep.py tests/test_window_sets.py -m gpu -q -x -k "plan or fuzz or sweep or window" > $O/plan_tests.log 2>&1; echo "rc=$?" >> $O/plan_tests.log
CFG=c4_4k_drone DEPTH=3 timeout -s KILL 600 python scripts/timeline.py > $O/timeline_c4.txt 2>&1
B="python bench.py --no-e2e --no-cpu-baseline --steps 50"
for c in c4_4k_drone c2_1080p_sparse c3_1080p_dense; do timeout -s KILL 600 $B --config $c > $O/bench_$c.log 2>&1; done
timeout -s KILL 600 $B --config c4_4k_drone --depth 4 --side-streams 2 > $O/bench_c4_d4s2.log 2>&1
D="python bench.py --no-e2e --no-cpu-baseline --depth 1 --steps 2 --warmup 3"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"plan_full_kernel" -s 2 -c 1 -o $O/prof_plan_full -f $D --config c4_4k_drone > $O/prof_plan.log 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $O/all.log 2>&1; echo "rc=$?" >> $O/all.log
ls -la $O
