# round-2 pass 48: own TMA box for a short last row tile (no staged rows below
# the window) vs HEAD; gather alone u8/f32, GPU suite, u8 c2 bench line, ncu.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s48
mkdir -p $O
export PYTHONUNBUFFERED=1
for rep in 1 2; do
 for cfg in c2_1080p_sparse c3_1080p_dense c4_4k_drone; do
  for fmt in 1 0; do
   for v in head last; do
    MP_LIB=build/ab/$v.so REP=$rep TAG=$v CFG=$cfg FMT=$fmt WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
   done
  done
 done
done
MP_LIB=build/ab/last.so timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_last.log 2>&1; tail -3 $O/pytest_last.log
for v in head last; do MP_LIB=build/ab/$v.so timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --steps 50 --fmt u8 > $O/bench_u8_c2_$v.log 2>&1; done
MP_LIB=build/ab/last.so CFG=c2_1080p_sparse FMT=1 WHAT=crops_rgb timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" -s 3 -c 1 -o $O/prof_u8last -f python scripts/time_gather.py > $O/ncu.log 2>&1
tail -2 $O/ncu.log
