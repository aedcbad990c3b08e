# round-2 pass 38: r43 consumer (warp-staged 16-B row stores, trimmed copy-out)
# vs HEAD; ring variants through the knobs build: 3 stages of <= 40 / 44 KB
# (fewer row groups per tile) against the default 2 x ~53 KB.  A/B before
# the GPU suite (a GPU test rebuilds the in-tree library).
cd $GRAFT_REPO_ROOT
O=gpurun_out/s38
mkdir -p $O
export PYTHONUNBUFFERED=1
for rep in 1 2; do
 for cfg in c2_1080p_sparse c3_1080p_dense c4_4k_drone c1_540p; do
  MP_LIB=build/ab/base.so REP=$rep TAG=base CFG=$cfg FMT=1 WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
  MP_LIB=build/ab/r43.so REP=$rep TAG=r43 CFG=$cfg FMT=1 WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
  MP_LIB=build/ab/r43k.so MP_GATHER_STAGES=3 MP_GATHER_BUDGET_KB=40 REP=$rep TAG=r43_3x40 CFG=$cfg FMT=1 WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
  MP_LIB=build/ab/r43k.so MP_GATHER_STAGES=3 MP_GATHER_BUDGET_KB=44 REP=$rep TAG=r43_3x44 CFG=$cfg FMT=1 WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
 done
done
for cfg in c2_1080p_sparse c3_1080p_dense; do
  MP_LIB=build/ab/base.so REP=1 TAG=base CFG=$cfg FMT=0 WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab_f32.jsonl 2>>$O/err.log
  MP_LIB=build/ab/r43.so REP=1 TAG=r43 CFG=$cfg FMT=0 WHAT=crops_rgb timeout 300 python scripts/time_gather.py >> $O/ab_f32.jsonl 2>>$O/err.log
done
MP_LIB=build/ab/r43.so timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_r43.log 2>&1; tail -3 $O/pytest_r43.log
MP_LIB=build/ab/r43.so CFG=c2_1080p_sparse FMT=1 WHAT=crops_rgb timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" -s 3 -c 1 -o $O/prof_u8r43 -f python scripts/time_gather.py > $O/ncu.log 2>&1
tail -2 $O/ncu.log
