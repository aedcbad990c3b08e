# round-2 pass 26: u8 tile geometry sweep for the dominant c2 class (ow = 192).
cd $GRAFT_REPO_ROOT
O=gpurun_out/s26
mkdir -p $O
export PYTHONUNBUFFERED=1
for rep in 1 2; do
  MP_LIB=build/ab/knobs.so REP=$rep TAG=default CFG=c2_1080p_sparse FMT=1 WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/sweep.jsonl 2>>$O/err.log
  for t in 192,4 192,5 192,6 192,7 192,8 96,8 96,12 64,8 128,8 128,6; do
    MP_LIB=build/ab/knobs.so MP_GATHER_TILE=192,$t REP=$rep TAG=t$t CFG=c2_1080p_sparse FMT=1 WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/sweep.jsonl 2>>$O/err.log
  done
done
cat $O/sweep.jsonl | head -30
