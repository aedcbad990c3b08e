cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -k "gather or full_size" > gpurun_out/pytest_gpu.log 2>&1
timeout -s KILL 600 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --depth 1 > gpurun_out/bench_c2.log 2>&1
for c in c1_540p c3_1080p_dense c4_4k_drone; do timeout -s KILL 600 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 30 --depth 1 > gpurun_out/bench_$c.log 2>&1; done
MP_GATHER_TILE=2880,160,5 timeout -s KILL 600 python bench.py --config c4_4k_drone --no-e2e --no-cpu-baseline --steps 30 --depth 1 > gpurun_out/bench_t160.log 2>&1
MP_GATHER_TILE=720,240,3 timeout -s KILL 600 python bench.py --config c1_540p --no-e2e --no-cpu-baseline --steps 30 --depth 1 > gpurun_out/bench_t720.log 2>&1
