# round-2 pass 51: NV12 fixed-tap consumer (consume_tile_r43nv) vs HEAD:
# NV12 crop gather alone (2 and 3 stages), the NV12 bench line, the GPU suite
# through the bounds-checked build of the variant.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s51
mkdir -p $O
export PYTHONUNBUFFERED=1
for rep in 1 2; do
 for cfg in c2_1080p_sparse c3_1080p_dense c4_4k_drone; do
  for v in head nv; do
   MP_LIB=build/ab/$v.so REP=$rep TAG=$v CFG=$cfg FMT=0 WHAT=crops_nv12 timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
  done
  MP_LIB=build/ab/nvk.so MP_GATHER_STAGES=3 REP=$rep TAG=nv_st3 CFG=$cfg FMT=0 WHAT=crops_nv12 timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
 done
done
for v in head nv; do MP_LIB=build/ab/$v.so timeout -s KILL 600 python bench.py --src nv12 --no-cpu-baseline --no-e2e > $O/bench_nv12_$v.log 2>&1; done
MP_LIB=build/ab/nvb.so timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_nvb.log 2>&1; echo "rc=$?" >> $O/pytest_nvb.log; tail -3 $O/pytest_nvb.log
grep -m3 MP_BOUNDS_CHECK $O/pytest_nvb.log || true
