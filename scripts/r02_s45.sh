# round-2 pass 45: r43 tiling with equal row tiles (no staged rows past a
# short last tile) and a stage budget that keeps the side reserve beside the
# row buffers (bal) vs pass 44 (cw); gather alone, GPU suite, pipelined bench
# lines (u8 c2/c3/c4 and the default f32 headline, c3/c4 f32).
cd $GRAFT_REPO_ROOT
O=gpurun_out/s45
mkdir -p $O
export PYTHONUNBUFFERED=1
for rep in 1 2; do
 for cfg in c2_1080p_sparse c3_1080p_dense c4_4k_drone; do
  for fmt in 1 0; do
   for v in cw bal; do
    MP_LIB=build/ab/$v.so REP=$rep TAG=$v CFG=$cfg FMT=$fmt WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
   done
  done
 done
done
MP_LIB=build/ab/bal.so timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_bal.log 2>&1; tail -3 $O/pytest_bal.log
for c in c2_1080p_sparse c3_1080p_dense c4_4k_drone; do MP_LIB=build/ab/bal.so timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --steps 50 --config $c --fmt u8 > $O/bench_u8_$c.log 2>&1; done
for c in c3_1080p_dense c4_4k_drone; do MP_LIB=build/ab/bal.so timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --steps 50 --config $c > $O/bench_$c.log 2>&1; done
MP_LIB=build/ab/bal.so timeout -s KILL 900 python bench.py > $O/bench_default.log 2>&1
MP_LIB=build/ab/bal.so CFG=c2_1080p_sparse FMT=1 WHAT=crops_rgb timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" -s 3 -c 1 -o $O/prof_u8bal -f python scripts/time_gather.py > $O/ncu.log 2>&1
tail -2 $O/ncu.log
