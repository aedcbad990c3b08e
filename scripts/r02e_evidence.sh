# round-2c final evidence pass (int16-box planner, gather SM reserve, batched 128-thread scans): smoke, default bench (all
# legs), reference arm, every config / format line, NV12, clips, launch list
# and ncu of the default bench's gather, the GPU suite on the in-tree library.
cd $GRAFT_REPO_ROOT
O=gpurun_out/ev2e
mkdir -p $O
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout -s KILL 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout -s KILL 900 python bench.py > $O/bench_default.log 2>&1
timeout -s KILL 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref.log 2>&1
B="python bench.py --no-e2e --no-cpu-baseline --steps 50"
for c in c1_540p c3_1080p_dense c4_4k_drone; do timeout -s KILL 600 $B --config $c > $O/bench_$c.log 2>&1; done
for c in c2_1080p_sparse c3_1080p_dense c4_4k_drone; do timeout -s KILL 600 $B --config $c --fmt u8 > $O/bench_u8_$c.log 2>&1; done
timeout -s KILL 600 python bench.py --fmt u8 --no-cpu-baseline > $O/bench_u8_e2e.log 2>&1
timeout -s KILL 600 python bench.py --src nv12 --no-cpu-baseline > $O/bench_nv12.log 2>&1
timeout -s KILL 1200 python bench.py --mode clips --clips 24 --steps 1 --warmup 1 > $O/bench_clips24.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"plan_|gather_|nms_" -c 60 --csv --log-file $O/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 > $O/launches_bench.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" -s 3 -c 1 -o $O/prof_gather -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 > $O/prof_bench.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"plan_full_kernel" -s 2 -c 1 -o $O/prof_plan_full_c4 -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 --config c4_4k_drone --fmt u8 > $O/prof_plan_bench.log 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
ls -la $O
