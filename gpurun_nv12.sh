cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_nv12.py -q -x -k full_size > gpurun_out/pytest_nv12full.log 2>&1
