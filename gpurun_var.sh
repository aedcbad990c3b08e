cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -k "gather or full_size" > gpurun_out/pytest_gpu.log 2>&1
for d in 1 2; do timeout -s KILL 600 python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu-baseline --depth $d > gpurun_out/bench_d$d.log 2>&1; done
timeout -s KILL 600 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 --config c3_1080p_dense > gpurun_out/bench_c3.log 2>&1
timeout -s KILL 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"gather_kernel" -s 3 -c 1 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 > gpurun_out/ncu_bytes.log 2>&1
