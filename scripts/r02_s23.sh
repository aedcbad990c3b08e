# round-2 pass 23: lambda pairs through shared memory (A/B, gather alone, f32 + u8).
cd $GRAFT_REPO_ROOT
O=gpurun_out/s23
mkdir -p $O
export PYTHONUNBUFFERED=1
AB_TAG=s23 bash scripts/ab_gather.sh
mv gpurun_out/ab_s23 $O/ab
MP_LIB=build/ab/lam.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "gather" > $O/lam_tests.log 2>&1; echo "rc=$?" >> $O/lam_tests.log
ls -la $O
