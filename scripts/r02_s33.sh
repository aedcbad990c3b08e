# round-2 pass 33: u8 output rows staged in shared memory and written with one
# bulk copy per row (cp.async.bulk shared->global): GPU tests through the
# variant library, then gather-alone A/B against the in-tree library.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s33
mkdir -p $O
export PYTHONUNBUFFERED=1
MP_LIB=build/ab/bulk.so timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_bulk.log 2>&1; tail -3 $O/pytest_bulk.log
for rep in 1 2 3; do
 for cfg in c2_1080p_sparse c3_1080p_dense c4_4k_drone; do
  for v in base bulk; do
   lib=""; [ $v != base ] && lib=build/ab/$v.so
   MP_LIB=$lib REP=$rep TAG=$v CFG=$cfg FMT=1 WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
  done
 done
done
MP_LIB=build/ab/bulk.so CFG=c2_1080p_sparse FMT=1 WHAT=crops_rgb timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" -s 3 -c 1 -o $O/prof_u8bulk -f python scripts/time_gather.py > $O/ncu.log 2>&1
tail -2 $O/ncu.log
