# round-2 pass 27: taller u8 tiles for the dominant c2 class (Rw 9/10/12).
cd $GRAFT_REPO_ROOT
O=gpurun_out/s27
mkdir -p $O
export PYTHONUNBUFFERED=1
for rep in 1 2; do
  MP_LIB=build/ab/knobs.so REP=$rep TAG=default CFG=c2_1080p_sparse FMT=1 WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/sweep.jsonl 2>>$O/err.log
  for t in 192,9 192,10 192,12; do
    MP_LIB=build/ab/knobs.so MP_GATHER_TILE=192,$t REP=$rep TAG=t$t CFG=c2_1080p_sparse FMT=1 WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/sweep.jsonl 2>>$O/err.log
    MP_LIB=build/ab/knobs.so MP_GATHER_TILE=192,$t MP_GATHER_BUDGET_KB=100 REP=$rep TAG=t${t}b100 CFG=c2_1080p_sparse FMT=1 WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/sweep.jsonl 2>>$O/err.log
  done
done
cat $O/sweep.jsonl
