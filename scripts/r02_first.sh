# round-2 (re-entry) first GPU pass: whole -m gpu suite, smoke, default bench,
# and ncu --set full baselines of the side kernels (plan_full, nms_large at c4)
# and of the u8 gather at c2.
cd $GRAFT_REPO_ROOT
O=gpurun_out/f1
mkdir -p $O
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x > $O/all.log 2>&1; echo "rc=$?" >> $O/all.log
timeout -s KILL 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout -s KILL 600 python bench.py --no-cpu-baseline > $O/bench.log 2>&1
timeout -s KILL 600 python bench.py --fmt u8 --no-e2e --no-cpu-baseline --steps 50 > $O/bench_u8.log 2>&1
timeout -s KILL 600 python bench.py --config c4_4k_drone --no-e2e --no-cpu-baseline --steps 50 > $O/bench_c4.log 2>&1
timeout -s KILL 600 python bench.py --config c1_540p --no-e2e --no-cpu-baseline --steps 50 > $O/bench_c1.log 2>&1
B="python bench.py --no-e2e --no-cpu-baseline --depth 1 --steps 2 --warmup 3"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"plan_full_kernel" -s 2 -c 1 -o $O/prof_plan_full -f $B --config c4_4k_drone > $O/prof_plan.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"nms_large_kernel" -s 2 -c 1 -o $O/prof_nms_large -f $B --config c4_4k_drone > $O/prof_nms.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" -s 3 -c 1 -o $O/prof_gather_u8 -f $B --fmt u8 > $O/prof_u8.log 2>&1
ls -la $O
