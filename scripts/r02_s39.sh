# round-2 pass 39: r43 consumer with all four source runs loaded up front (pf)
# vs the committed r43 and HEAD~1 (base); GPU suite (incl. the new fixed-tap
# test) through pf; ncu of its c2 launch.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s39
mkdir -p $O
export PYTHONUNBUFFERED=1
for rep in 1 2; do
 for cfg in c2_1080p_sparse c3_1080p_dense c4_4k_drone; do
  for v in base r43 pf; do
   MP_LIB=build/ab/$v.so REP=$rep TAG=$v CFG=$cfg FMT=1 WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
  done
 done
done
MP_LIB=build/ab/pf.so timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_pf.log 2>&1; tail -3 $O/pytest_pf.log
MP_LIB=build/ab/pf.so CFG=c2_1080p_sparse FMT=1 WHAT=crops_rgb timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" -s 3 -c 1 -o $O/prof_u8pf -f python scripts/time_gather.py > $O/ncu.log 2>&1
tail -2 $O/ncu.log
