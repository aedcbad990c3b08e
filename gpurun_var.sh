cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for d in 1 2; do for g in 0 1; do timeout -s KILL 600 python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu-baseline --depth $d --graphs $g > gpurun_out/bench_d${d}g$g.log 2>&1; done; done
