# round-2 pass 53: configs[0] (30 x 540p frames) gather latency vs ring shape:
# stage budget 16/24/32 KB x 2-4 stages (knobs build), f32 and u8, alone.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s53
mkdir -p $O
export PYTHONUNBUFFERED=1
for rep in 1 2; do
 for fmt in 0 1; do
  MP_LIB=build/ab/knobs.so REP=$rep TAG=default CFG=c1_540p FMT=$fmt WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
  for b in 12 16 24 32; do
   for st in 2 3 4; do
    MP_LIB=build/ab/knobs.so MP_GATHER_BUDGET_KB=$b MP_GATHER_STAGES=$st REP=$rep TAG=b${b}s$st CFG=c1_540p FMT=$fmt WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
   done
  done
 done
done
