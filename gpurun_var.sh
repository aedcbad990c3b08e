cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/var.log
cp paper_2103_14695_b200/libmp_b200.so /tmp/orig.so
for k in 8 12 16; do
  cp .variants/lib_kcw$k.so paper_2103_14695_b200/libmp_b200.so
  TAG=kcw$k WHAT=crops_rgb,crops_nv12,proxy_nv12 timeout -s KILL 300 python scripts/time_gather.py >> gpurun_out/var.log 2>&1
  timeout -s KILL 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/b_kcw$k.log 2>&1
  timeout -s KILL 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --fmt u8 > gpurun_out/bu8_kcw$k.log 2>&1
done
cp /tmp/orig.so paper_2103_14695_b200/libmp_b200.so
