# round-2 pass 54: u8 fixed-tap consumer with the lambda = 1/2 shortcuts
# (j = 1 columns: m + n; row 3m+1: T + B; the 1/2s in the rounding's exact
# scale) vs HEAD: gather alone, u8 bench c2, GPU suite through the
# bounds-checked build of the variant.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s54
mkdir -p $O
export PYTHONUNBUFFERED=1
for rep in 1 2 3; do
 for cfg in c2_1080p_sparse c3_1080p_dense c4_4k_drone; do
  for v in head half; do
   MP_LIB=build/ab/$v.so REP=$rep TAG=$v CFG=$cfg FMT=1 WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
  done
 done
done
for v in head half; do MP_LIB=build/ab/$v.so timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --steps 50 --fmt u8 > $O/bench_u8_c2_$v.log 2>&1; done
MP_LIB=build/ab/halfb.so timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_halfb.log 2>&1; echo "rc=$?" >> $O/pytest_halfb.log; tail -3 $O/pytest_halfb.log
