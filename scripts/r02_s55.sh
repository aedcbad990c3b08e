# round-2 pass 55: c4 u8 step is plan-bound (the 172-KB u8 ring leaves room
# for one 34-KB plan CTA per SM).  Smaller u8 stages (knob budget 66 / 60 KB:
# ~150 KB ring, two plan CTAs beside it) vs the default — pipelined bench
# lines for c4 and c2 u8, plus the c4 timeline.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s55
mkdir -p $O
export PYTHONUNBUFFERED=1
for rep in 1 2; do
 for c in c4_4k_drone c2_1080p_sparse; do
  MP_LIB=build/ab/knobs.so timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --steps 50 --config $c --fmt u8 > $O/bench_${c}_default_$rep.log 2>&1
  for b in 66 60; do
   MP_LIB=build/ab/knobs.so MP_GATHER_BUDGET_KB=$b timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --steps 50 --config $c --fmt u8 > $O/bench_${c}_b${b}_$rep.log 2>&1
  done
 done
done
