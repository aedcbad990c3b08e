# round-2 pass 40: evidence for the u8 consumer rewrite — bench lines (u8
# c2/c3/c4 + default f32 headline), launch list + ncu --set full of the u8
# gather in the bench's launch configuration, sanitizers on the fixed-tap
# path (memcheck, racecheck: warp row buffers + __syncwarp ordering).
cd $GRAFT_REPO_ROOT
O=gpurun_out/s40
mkdir -p $O
export PYTHONUNBUFFERED=1
B="python bench.py --no-e2e --no-cpu-baseline --steps 50"
for c in c2_1080p_sparse c3_1080p_dense c4_4k_drone; do timeout -s KILL 600 $B --config $c --fmt u8 > $O/bench_u8_$c.log 2>&1; done
timeout -s KILL 900 python bench.py > $O/bench_default.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"plan_|gather_|nms_" -c 60 --csv --log-file $O/launches_u8.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 --fmt u8 > $O/launches_u8.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" -s 3 -c 1 -o $O/prof_gather_u8 -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 --fmt u8 > $O/prof_u8.log 2>&1
timeout -s KILL 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "fixed_tap or (configs and c1_540p)" > $O/san_memcheck_r43.log 2>&1; echo "rc=$?" >> $O/san_memcheck_r43.log
timeout -s KILL 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "fixed_tap and tma" > $O/san_racecheck_r43.log 2>&1; echo "rc=$?" >> $O/san_racecheck_r43.log
timeout -s KILL 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "fixed_tap and tma" > $O/san_synccheck_r43.log 2>&1; echo "rc=$?" >> $O/san_synccheck_r43.log
ls -la $O
