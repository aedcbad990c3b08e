# round-2 pass 56: fixed-tap task indices by shift (ncg is a power of two)
# vs HEAD, all three fixed-tap consumers; GPU suite through the bounds build.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s56
mkdir -p $O
export PYTHONUNBUFFERED=1
for rep in 1 2; do
 for cfg in c2_1080p_sparse c3_1080p_dense c4_4k_drone; do
  for v in head shift; do
   MP_LIB=build/ab/$v.so REP=$rep TAG=$v CFG=$cfg FMT=1 WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
   MP_LIB=build/ab/$v.so REP=$rep TAG=$v CFG=$cfg FMT=0 WHAT=crops_rgb,crops_nv12 timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
  done
 done
done
MP_LIB=build/ab/shiftb.so timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_shiftb.log 2>&1; echo "rc=$?" >> $O/pytest_shiftb.log; tail -3 $O/pytest_shiftb.log
