# round-2 pass 69: c4 u8 — instead of leaving SMs to the planner, plan further
# ahead (depth 4, two plan streams: plans of two batches overlap two gathers).
cd $GRAFT_REPO_ROOT
O=gpurun_out/s69
mkdir -p $O
export PYTHONUNBUFFERED=1
B="python bench.py --no-e2e --no-cpu-baseline --steps 40 --config c4_4k_drone --fmt u8"
for rep in 1 2; do
 for k in 0 8 16; do
  for d in 3 4; do
   timeout -s KILL 300 $B --gather-sm-reserve $k --depth $d --side-streams 2 > $O/u8_c4_k${k}_d${d}_ss2_$rep.log 2>&1
  done
  timeout -s KILL 300 $B --gather-sm-reserve $k --depth 3 --side-streams 1 > $O/u8_c4_k${k}_d3_ss1_$rep.log 2>&1
 done
done
ls $O
