cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cp paper_2103_14695_b200/libmp_b200.so /tmp/base.so
for f in .variants/lib_*.so; do v=$(basename $f .so); cp $f paper_2103_14695_b200/libmp_b200.so
  timeout -s KILL 600 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_$v.log 2>&1
done
cp /tmp/base.so paper_2103_14695_b200/libmp_b200.so
