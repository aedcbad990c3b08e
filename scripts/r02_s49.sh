# round-2 pass 49: mbarrier wait mode of the 12-warp u8 consumers (they spin
# on the full barrier: 16 M try_wait + 16 M YIELD per c2 launch): plain
# try_wait (0) vs consumers sleeping (2) vs both sides sleeping (3); and the
# ring depth (MP_GATHER_STAGES=3 with a 52-KB budget) — gather alone.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s49
mkdir -p $O
export PYTHONUNBUFFERED=1
for rep in 1 2; do
 for cfg in c2_1080p_sparse c3_1080p_dense c4_4k_drone; do
  for fmt in 1 0; do
   for wm in 0 2 3; do
    MP_LIB=build/ab/knobs.so MP_GATHER_WAIT=$wm REP=$rep TAG=wait$wm CFG=$cfg FMT=$fmt WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
   done
  done
  MP_LIB=build/ab/knobs.so MP_GATHER_STAGES=3 MP_GATHER_BUDGET_KB=52 REP=$rep TAG=st3b52 CFG=$cfg FMT=1 WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
 done
done
