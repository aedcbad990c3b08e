cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/var.log
cp paper_2103_14695_b200/libmp_b200.so /tmp/orig.so
for v in base2 w32 base2 w32; do
  cp .variants/lib_$v.so paper_2103_14695_b200/libmp_b200.so
  TAG=$v WHAT=crops_rgb timeout -s KILL 300 python scripts/time_gather.py >> gpurun_out/var.log 2>&1
  for f in f32 u8; do
  timeout -s KILL 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --fmt $f > gpurun_out/b.log 2>&1
  echo "$v $f $(tail -1 gpurun_out/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'], d['roofline']['launch_ms'], d['roofline']['frac'])")" >> gpurun_out/var.log
  done
done
cp /tmp/orig.so paper_2103_14695_b200/libmp_b200.so
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gather or full_size" > gpurun_out/pytest_w32.log 2>&1
