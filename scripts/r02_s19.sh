# round-2 pass 19: same-box A/B of the pipelined step (head vs overlap pre-test), capture_steps test.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s19
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout -s KILL 600 python -m pytest tests/test_gpu_pipeline.py -q -x > $O/pipe_tests.log 2>&1; echo "rc=$?" >> $O/pipe_tests.log
for rep in 1 2 3; do
 for c in c2_1080p_sparse c3_1080p_dense c4_4k_drone; do
  for v in head ovl; do
   MP_LIB=build/ab/$v.so timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --steps 50 --config $c > $O/ab_${v}_${c}_$rep.log 2>&1
  done
 done
done
ls -la $O | head
