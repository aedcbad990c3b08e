# round-2 pass 70: a few SMs left free for the side kernels' tail (scan /
# scatter / NMS tiny that cannot co-reside with a u8 gather CTA) — c2 u8 and
# f32, c3 u8, k = 0 / 1 / 2 / 4; timelines at k = 0 / 2.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s70
mkdir -p $O
export PYTHONUNBUFFERED=1
B="python bench.py --no-e2e --no-cpu-baseline --steps 50"
for rep in 1 2; do
 for k in 0 1 2 4; do
  timeout -s KILL 300 $B --config c2_1080p_sparse --fmt u8 --gather-sm-reserve $k > $O/u8_c2_k${k}_$rep.log 2>&1
  timeout -s KILL 300 $B --config c2_1080p_sparse --gather-sm-reserve $k > $O/f32_c2_k${k}_$rep.log 2>&1
 done
done
for k in 0 2; do
  timeout -s KILL 300 $B --config c3_1080p_dense --fmt u8 --gather-sm-reserve $k > $O/u8_c3_k${k}.log 2>&1
done
ls $O
for k in 0 2; do
  for fmt in 1 0; do
    RSV=$k CFG=c2_1080p_sparse DEPTH=3 FMT=$fmt timeout -s KILL 300 python scripts/timeline.py > $O/tl_c2_fmt${fmt}_k$k.txt 2>&1
  done
done
