# round-2c u8 evidence after the one-SM reserve (bench auto rule): smoke, GPU
# suite, every u8 line, the u8 e2e line, the default line.
cd $GRAFT_REPO_ROOT
O=gpurun_out/ev2f
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout -s KILL 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
B="python bench.py --no-e2e --no-cpu-baseline --steps 50"
for c in c2_1080p_sparse c3_1080p_dense c4_4k_drone; do timeout -s KILL 600 $B --config $c --fmt u8 > $O/bench_u8_$c.log 2>&1; done
timeout -s KILL 600 python bench.py --fmt u8 --no-cpu-baseline > $O/bench_u8_e2e.log 2>&1
timeout -s KILL 900 python bench.py > $O/bench_default.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"plan_|gather_|nms_" -c 60 --csv --log-file $O/launches_u8.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 --fmt u8 > $O/launches_bench.log 2>&1
ls -la $O
