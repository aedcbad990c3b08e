# round-2 evidence pass: default bench (all legs), reference arm, every
# config / format / NEXT mode, sanitizers on the round-2 code paths, smoke.
cd $GRAFT_REPO_ROOT
O=gpurun_out/ev
mkdir -p $O
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout -s KILL 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout -s KILL 900 python bench.py > $O/bench_default.log 2>&1
timeout -s KILL 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref.log 2>&1
B="python bench.py --no-e2e --no-cpu-baseline --steps 50"
for c in c1_540p c3_1080p_dense c4_4k_drone; do timeout -s KILL 600 $B --config $c > $O/bench_$c.log 2>&1; done
for c in c2_1080p_sparse c3_1080p_dense c4_4k_drone; do timeout -s KILL 600 $B --config $c --fmt u8 > $O/bench_u8_$c.log 2>&1; done
timeout -s KILL 600 python bench.py --src nv12 --no-cpu-baseline > $O/bench_nv12.log 2>&1
timeout -s KILL 900 python bench.py --mode sweep > $O/bench_sweep.log 2>&1
timeout -s KILL 900 python bench.py --mode wsel --steps 5 --warmup 3 > $O/bench_wsel.log 2>&1
timeout -s KILL 600 python bench.py --mode assign --steps 50 --warmup 5 > $O/bench_assign.log 2>&1
timeout -s KILL 900 python bench.py --mode refine --steps 20 --warmup 3 > $O/bench_refine.log 2>&1
timeout -s KILL 1200 python bench.py --mode clips --clips 24 --steps 1 --warmup 1 > $O/bench_clips24.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"plan_|gather_|nms_" -c 60 --csv --log-file $O/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 > $O/launches_bench.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" -s 3 -c 1 -o $O/prof_gather -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 > $O/prof_bench.log 2>&1
timeout -s KILL 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_edges.py -q -x -k "grid_path and (giant or stacked) or beyond_shared" > $O/san_memcheck_nms.log 2>&1; echo "rc=$?" >> $O/san_memcheck_nms.log
timeout -s KILL 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_edges.py -q -x -k "grid_path and spread and 500" > $O/san_racecheck_nms.log 2>&1; echo "rc=$?" >> $O/san_racecheck_nms.log
timeout -s KILL 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "largest_grid or adversarial and 3840" > $O/san_memcheck_plan.log 2>&1; echo "rc=$?" >> $O/san_memcheck_plan.log
timeout -s KILL 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "largest_grid or adversarial and 3840" > $O/san_racecheck_plan.log 2>&1; echo "rc=$?" >> $O/san_racecheck_plan.log
timeout -s KILL 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "largest_grid" > $O/san_synccheck_plan.log 2>&1; echo "rc=$?" >> $O/san_synccheck_plan.log
timeout -s KILL 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_proxy_sweep.py -q -x -k "single_pass" > $O/san_memcheck_sweep.log 2>&1; echo "rc=$?" >> $O/san_memcheck_sweep.log
timeout -s KILL 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "scales_and_edges and 0.7" > $O/san_memcheck_gather_u8.log 2>&1; echo "rc=$?" >> $O/san_memcheck_gather_u8.log
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
ls -la $O
