# round-2 pass 44: 12 consumer warps for the u8 instantiation only (cw_of),
# one row buffer per warp (ring + buffers leave the 56-KB side reserve):
# gather alone vs the 8-warp build (cur); GPU suite; pipelined u8 bench.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s44
mkdir -p $O
export PYTHONUNBUFFERED=1
for rep in 1 2; do
 for cfg in c2_1080p_sparse c3_1080p_dense c4_4k_drone c1_540p; do
  for fmt in 1 0; do
   for v in cur cw; do
    MP_LIB=build/ab/$v.so REP=$rep TAG=$v CFG=$cfg FMT=$fmt WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
   done
  done
 done
done
MP_LIB=build/ab/cw.so timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_cw.log 2>&1; tail -3 $O/pytest_cw.log
for c in c2_1080p_sparse c3_1080p_dense c4_4k_drone; do MP_LIB=build/ab/cw.so timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --steps 50 --config $c --fmt u8 > $O/bench_u8_$c.log 2>&1; done
MP_LIB=build/ab/cw.so CFG=c2_1080p_sparse FMT=1 WHAT=crops_rgb timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" -s 3 -c 1 -o $O/prof_u8cw -f python scripts/time_gather.py > $O/ncu.log 2>&1
tail -2 $O/ncu.log
