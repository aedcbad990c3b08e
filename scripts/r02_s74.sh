# round-2 pass 74: NV12 line (crops + proxy-input downscale, f32 out) with
# k = 0 / 1 / 2 SMs left out of the gathers' grids.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s74
mkdir -p $O
export PYTHONUNBUFFERED=1
B="python bench.py --no-e2e --no-cpu-baseline --steps 50 --src nv12"
for rep in 1 2; do
 for k in 0 1 2 8; do
  timeout -s KILL 300 $B --gather-sm-reserve $k > $O/nv12_k${k}_$rep.log 2>&1
 done
done
ls $O
