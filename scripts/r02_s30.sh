# round-2 pass 30: u8 gather diagnosis — copies-only / compute-only split
# (knobs build, MP_GATHER_DEBUG=1: no compute, =2: no pixel copies) and one
# ncu --set full capture with source counters of the u8 c2 launch.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s30
mkdir -p $O
export PYTHONUNBUFFERED=1
for rep in 1 2; do
 for cfg in c2_1080p_sparse c4_4k_drone; do
  for dbg in 0 1 2; do
   MP_LIB=build/ab/knobs.so MP_GATHER_DEBUG=$dbg REP=$rep TAG=dbg$dbg CFG=$cfg FMT=1 WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/dbg.jsonl 2>>$O/err.log
  done
 done
done
cat $O/dbg.jsonl
D="python bench.py --no-e2e --no-cpu-baseline --depth 1 --steps 2 --warmup 3"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" -s 3 -c 1 -o $O/prof_gather_u8 -f $D --fmt u8 > $O/p2.log 2>&1
ls -la $O
