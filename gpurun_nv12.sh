cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 600 python bench.py --mode assign --steps 50 --warmup 5 > gpurun_out/bench_assign.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"hung_" -c 9 --csv --log-file gpurun_out/assign_ncu.csv python bench.py --mode assign --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
