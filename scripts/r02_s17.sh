# round-2 pass 17: full-tile specialization A/B (gather alone, f32 + u8), parity.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s17
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nv12.py -m gpu -q -x -k "gather or full_size or nv12" > $O/gather_tests.log 2>&1; echo "rc=$?" >> $O/gather_tests.log
AB_TAG=s17 bash scripts/ab_gather.sh
mv gpurun_out/ab_s17 $O/ab
ls -la $O
