# round-2 pass 36: fixed-tap 4:3 u8 consumer (consume_tile_r43), direct STG.32 rows vs the
# round-2 HEAD library (base, built from git HEAD into build/ab); A/B BEFORE
# the GPU tests (a GPU test rebuilds the in-tree library), then the GPU suite
# through the variant, then ncu of its c2 launch.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s36
mkdir -p $O
export PYTHONUNBUFFERED=1
for rep in 1 2 3; do
 for cfg in c2_1080p_sparse c3_1080p_dense c4_4k_drone c1_540p; do
  for v in base r43; do
   MP_LIB=build/ab/$v.so REP=$rep TAG=$v CFG=$cfg FMT=1 WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
  done
 done
done
MP_LIB=build/ab/r43.so timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_r43.log 2>&1; tail -3 $O/pytest_r43.log
MP_LIB=build/ab/r43.so CFG=c2_1080p_sparse FMT=1 WHAT=crops_rgb timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" -s 3 -c 1 -o $O/prof_u8r43 -f python scripts/time_gather.py > $O/ncu.log 2>&1
tail -2 $O/ncu.log
