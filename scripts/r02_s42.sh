# round-2 pass 42: f32 fixed-tap 4:3 consumer with warp-staged plane rows (consume_tile_r43f: LDS.128
# source runs, 16-B plane-row stores) vs the round-2 HEAD (base) and the u8-only
# r43 build; GPU suite through r43f; ncu of its c2 f32 launch.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s42
mkdir -p $O
export PYTHONUNBUFFERED=1
for rep in 1 2; do
 for cfg in c2_1080p_sparse c3_1080p_dense c4_4k_drone c1_540p; do
  for v in base r43 r43f; do
   MP_LIB=build/ab/$v.so REP=$rep TAG=$v CFG=$cfg FMT=0 WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
  done
  MP_LIB=build/ab/r43f.so REP=$rep TAG=r43f CFG=$cfg FMT=1 WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab_u8.jsonl 2>>$O/err.log
 done
done
MP_LIB=build/ab/r43f.so timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_r43f.log 2>&1; tail -3 $O/pytest_r43f.log
MP_LIB=build/ab/r43f.so CFG=c2_1080p_sparse FMT=0 WHAT=crops_rgb timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" -s 3 -c 1 -o $O/prof_f32r43 -f python scripts/time_gather.py > $O/ncu.log 2>&1
tail -2 $O/ncu.log
