cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
export PYTHONUNBUFFERED=1
O=gpurun_out/final
timeout -s KILL 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout -s KILL 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout -s KILL 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_nv12.py -q -x -k "proxy_input or invalid or grey" > $O/san_memcheck_nv12.log 2>&1; echo "rc=$?" >> $O/san_memcheck_nv12.log
timeout -s KILL 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_assign.py -q -x > $O/san_memcheck_assign.log 2>&1; echo "rc=$?" >> $O/san_memcheck_assign.log
timeout -s KILL 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_refine.py -q -x -k "degenerate or invalid" > $O/san_memcheck_refine.log 2>&1; echo "rc=$?" >> $O/san_memcheck_refine.log
timeout -s KILL 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_assign.py -q -x -k "large" > $O/san_racecheck_assign.log 2>&1; echo "rc=$?" >> $O/san_racecheck_assign.log
timeout -s KILL 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_refine.py -q -x -k "degenerate" > $O/san_racecheck_refine.log 2>&1; echo "rc=$?" >> $O/san_racecheck_refine.log
timeout -s KILL 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_nv12.py -q -x -k "grey" > $O/san_racecheck_nv12.log 2>&1; echo "rc=$?" >> $O/san_racecheck_nv12.log
for tool in memcheck racecheck synccheck; do timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "scales_and_edges and 0.7 or capacity_and_invalid" > $O/san_${tool}_gather.log 2>&1; echo "rc=$?" >> $O/san_${tool}_gather.log; done
timeout -s KILL 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_zero_copy.py -q -x -k "edges and 0.37" > $O/san_memcheck_zero_copy.log 2>&1; echo "rc=$?" >> $O/san_memcheck_zero_copy.log
timeout -s KILL 900 python bench.py > $O/bench_full.log 2>&1
timeout -s KILL 600 python bench.py --fmt u8 --no-e2e --no-cpu-baseline > $O/bench_u8.log 2>&1
timeout -s KILL 600 python bench.py --src nv12 > $O/bench_nv12.log 2>&1
for c in c1_540p c3_1080p_dense c4_4k_drone; do timeout -s KILL 600 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 50 > $O/bench_$c.log 2>&1; done
for c in c3_1080p_dense c4_4k_drone; do timeout -s KILL 600 python bench.py --config $c --fmt u8 --no-e2e --no-cpu-baseline --steps 50 > $O/bench_u8_$c.log 2>&1; done
timeout -s KILL 600 python scripts/zero_copy_probe.py > $O/zero_copy_probe.log 2>&1
timeout -s KILL 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"plan_|gather_|nms_" -c 60 --csv --log-file $O/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 > $O/launches_bench.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" -s 3 -c 1 -o $O/prof_gather -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 > $O/prof_bench.log 2>&1
timeout -s KILL 600 python bench.py --mode assign --steps 50 --warmup 5 > $O/bench_assign.log 2>&1
timeout -s KILL 900 python bench.py --mode refine --steps 20 --warmup 3 > $O/bench_refine.log 2>&1
timeout -s KILL 900 python bench.py --mode sweep > $O/bench_sweep.log 2>&1
timeout -s KILL 900 python bench.py --mode wsel --steps 5 --warmup 3 > $O/bench_wsel.log 2>&1
