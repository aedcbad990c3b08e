# round-2 pass 57: own TMA box for a short last row tile, re-measured on the
# final consumers (time, DRAM bytes by ncu), GPU suite through the bounds build.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s57
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
for v in head last; do
 MP_LIB=build/ab/$v.so CFG=c2_1080p_sparse FMT=1 WHAT=crops_rgb timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gather_kernel" -s 3 -c 1 --csv python scripts/time_gather.py > $O/ncu_u8_$v.csv 2>&1
done
MP_LIB=build/ab/lastb.so timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_lastb.log 2>&1; echo "rc=$?" >> $O/pytest_lastb.log; tail -3 $O/pytest_lastb.log
