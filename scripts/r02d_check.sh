# round-2 session-4 check of HEAD: smoke, GPU suite, default bench line.
cd $GRAFT_REPO_ROOT
O=gpurun_out/ev2d
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout -s KILL 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout -s KILL 900 python bench.py > $O/bench_default.log 2>&1
B="python bench.py --no-e2e --no-cpu-baseline --steps 50"
for c in c2_1080p_sparse c4_4k_drone; do timeout -s KILL 600 $B --config $c --fmt u8 > $O/bench_u8_$c.log 2>&1; done
ls -la $O
