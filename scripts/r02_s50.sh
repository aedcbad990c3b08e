# round-2 pass 50: the GPU suite through the bounds-checked dev build
# (-DMP_BOUNDS_CHECK: every shared-memory access of the round-2b consumers
# inside its stage box / warp row buffer, every global store inside its
# class's output tensor; a violation traps), and gather-alone timing of the
# production build with the checks compiled out (head2) vs HEAD.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s50
mkdir -p $O
export PYTHONUNBUFFERED=1
for cfg in c2_1080p_sparse c3_1080p_dense c4_4k_drone; do
 for fmt in 1 0; do
  for v in head head2; do
   MP_LIB=build/ab/$v.so REP=1 TAG=$v CFG=$cfg FMT=$fmt WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
  done
 done
done
MP_LIB=build/ab/bounds.so timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_bounds.log 2>&1; echo "rc=$?" >> $O/pytest_bounds.log; tail -3 $O/pytest_bounds.log
grep -c MP_BOUNDS_CHECK $O/pytest_bounds.log
