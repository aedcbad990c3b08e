# round-2 pass 31: u8 RGB consumer v2 (broadcast-lambda pairs, 1.0-bias bytes,
# single-emit downscale loop) — parity of the u8 tests through the variant
# library, then gather-alone A/B against the in-tree (round-2) library.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s31
mkdir -p $O
export PYTHONUNBUFFERED=1
MP_LIB=build/ab/u8v2.so timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_v2.log 2>&1; tail -3 $O/pytest_v2.log
for rep in 1 2 3; do
 for cfg in c2_1080p_sparse c3_1080p_dense c4_4k_drone; do
  for v in base u8v2; do
   lib=""; [ $v != base ] && lib=build/ab/$v.so
   MP_LIB=$lib REP=$rep TAG=$v CFG=$cfg FMT=1 WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
  done
 done
done
cat $O/ab.jsonl
