cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/var.log
run() { env "$@" WHAT=proxy_nv12,proxy_rgb,crops_nv12,crops_rgb timeout -s KILL 300 python scripts/time_gather.py >> gpurun_out/var.log 2>&1; }
run TAG=base
run TAG=st3b64 MP_GATHER_STAGES=3 MP_GATHER_BUDGET_KB=64
run TAG=st2b64 MP_GATHER_STAGES=2 MP_GATHER_BUDGET_KB=64
run TAG=st2b96 MP_GATHER_STAGES=2 MP_GATHER_BUDGET_KB=96
run TAG=dbg1 MP_GATHER_DEBUG=1
run TAG=dbg2 MP_GATHER_DEBUG=2
timeout -s KILL 900 python -m pytest tests/test_gpu_nv12.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_nv12.log 2>&1
