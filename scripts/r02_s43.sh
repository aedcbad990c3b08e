# round-2 pass 43: consumer-warp count with the fixed-tap consumers: the
# whole library built with 12 consumer warps (-DMP_KCW=12: 384 tasks per r43
# tile, 128 registers) and 16 (96 registers, spills) vs 8, gather alone.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s43
mkdir -p $O
export PYTHONUNBUFFERED=1
for rep in 1 2; do
 for cfg in c2_1080p_sparse c3_1080p_dense c4_4k_drone; do
  for fmt in 1 0; do
   for v in cur kcw12 kcw16; do
    MP_LIB=build/ab/$v.so REP=$rep TAG=$v CFG=$cfg FMT=$fmt WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
   done
  done
 done
done
cat $O/err.log | tail -5
