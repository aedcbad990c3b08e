# round-2 pass 52: NV12 fixed-tap classes on a three-stage ring (nv3) —
# NV12 GPU tests through it, crops alone vs nv (2 stages), NV12 bench line.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s52
mkdir -p $O
export PYTHONUNBUFFERED=1
MP_LIB=build/ab/nv3.so timeout 900 python -m pytest tests/test_gpu_nv12.py tests/test_gpu_parity.py -q -m gpu > $O/pytest_nv3.log 2>&1; echo "rc=$?" >> $O/pytest_nv3.log
for rep in 1 2; do
 for cfg in c2_1080p_sparse c3_1080p_dense c4_4k_drone; do
  for v in nv nv3; do
   MP_LIB=build/ab/$v.so REP=$rep TAG=$v CFG=$cfg FMT=0 WHAT=crops_nv12,proxy_nv12 timeout 300 python scripts/time_gather.py >> $O/ab.jsonl 2>>$O/err.log
  done
 done
done
MP_LIB=build/ab/nv3.so timeout -s KILL 600 python bench.py --src nv12 --no-cpu-baseline > $O/bench_nv12_nv3.log 2>&1
