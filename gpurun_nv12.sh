cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_refine.py -q -x > gpurun_out/pytest_refine.log 2>&1
