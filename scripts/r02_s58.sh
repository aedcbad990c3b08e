# round-2 pass 58: 10 vs 12 consumer warps for the u8 instantiation — gather
# alone and the pipelined c2 / c3 / c4 u8 steps (c4 is plan-bound beside the
# 12-warp gather).
cd $GRAFT_REPO_ROOT
O=gpurun_out/s58
mkdir -p $O
export PYTHONUNBUFFERED=1
for rep in 1 2; do
 for cfg in c2_1080p_sparse c3_1080p_dense c4_4k_drone; do
  for v in cw12 cw10; do
   MP_LIB=build/ab/$v.so REP=$rep TAG=$v CFG=$cfg FMT=1 WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
   MP_LIB=build/ab/$v.so timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --steps 50 --config $cfg --fmt u8 > $O/bench_${cfg}_${v}_$rep.log 2>&1
  done
 done
done
