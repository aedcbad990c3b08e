# round-2 pass 63: production mp_gather_set_sm_reserve + int16-box planner:
# whole GPU suite, c4 u8 (auto reserve 16) and the default line.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s63
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
B="python bench.py --no-e2e --no-cpu-baseline --steps 50"
timeout -s KILL 300 $B --config c4_4k_drone --fmt u8 > $O/u8_c4.log 2>&1
timeout -s KILL 300 $B --config c2_1080p_sparse --fmt u8 > $O/u8_c2.log 2>&1
timeout -s KILL 300 $B --config c4_4k_drone > $O/f32_c4.log 2>&1
ls $O
