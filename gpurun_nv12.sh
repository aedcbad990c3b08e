cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python bench.py --mode refine --steps 20 --warmup 3 > gpurun_out/bench_refine.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"track_|dbscan|cluster_|refine_|scan_kernel" -c 30 --csv --log-file gpurun_out/refine_ncu.csv python bench.py --mode refine --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
