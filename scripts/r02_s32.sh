# round-2 pass 32: why did the u8 v2 consumer (fewer instructions) not speed
# up?  Store-path diagnosis: v2 with no stores (st1), one byte per pixel
# (st2), the generic consumer (gen); each with and without pixel copies
# (MP_GATHER_DEBUG=2); plus ncu of the v2 launch.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s32
mkdir -p $O
export PYTHONUNBUFFERED=1
for rep in 1 2; do
 for cfg in c2_1080p_sparse c4_4k_drone; do
  for v in gen u8v2 st1 st2; do
   for dbg in 0 2; do
    MP_LIB=build/ab/$v.so MP_GATHER_DEBUG=$dbg REP=$rep TAG=$v.d$dbg CFG=$cfg FMT=1 WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
   done
  done
 done
done
MP_LIB=build/ab/u8v2.so CFG=c2_1080p_sparse FMT=1 WHAT=crops_rgb timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" -s 3 -c 1 -o $O/prof_u8v2 -f python scripts/time_gather.py > $O/ncu.log 2>&1
tail -3 $O/ncu.log
