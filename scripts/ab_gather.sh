# A/B the gather alone over every variant in build/ab/*.so (and the in-tree
# library as "base"), alternating variants per repetition, f32 and u8, c2/c3/c4.
cd $GRAFT_REPO_ROOT
O=gpurun_out/ab_${AB_TAG:-x}
mkdir -p $O
export PYTHONUNBUFFERED=1
for rep in 1 2 3; do
 for cfg in ${AB_CFGS:-c2_1080p_sparse c3_1080p_dense c4_4k_drone}; do
  for fmt in ${AB_FMTS:-0 1}; do
   for v in build/ab/*.so; do
     lib=""; [ "$v" != base ] && lib=$v
     MP_LIB=$lib REP=$rep TAG=$(basename $v .so) CFG=$cfg FMT=$fmt WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
   done
  done
 done
done
