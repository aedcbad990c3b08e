cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/var.log
for c in c4_4k_drone c3_1080p_dense c2_1080p_sparse; do for m in 0 1; do
  timeout -s KILL 300 python bench.py --config $c --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --merge-on-gather $m > gpurun_out/b.log 2>&1
  echo "$c mog=$m $(tail -1 gpurun_out/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['launch_ms'])")" >> gpurun_out/var.log
done; done
MOG=1 CFG=c4_4k_drone timeout -s KILL 300 python scripts/timeline.py > gpurun_out/timeline.log 2>&1
