# round-2 pass 21: c1 stage budget sweep (tile size for small batches).
cd $GRAFT_REPO_ROOT
O=gpurun_out/s21
mkdir -p $O
export PYTHONUNBUFFERED=1
B="python bench.py --no-e2e --no-cpu-baseline --steps 200 --config c1_540p"
for rep in 1 2; do
  MP_LIB=build/ab/knobs.so timeout -s KILL 300 $B > $O/c1_base_$rep.log 2>&1
  for kb in 12 16 24 32; do MP_LIB=build/ab/knobs.so MP_GATHER_BUDGET_KB=$kb timeout -s KILL 300 $B > $O/c1_b${kb}_$rep.log 2>&1; done
  for st in 3 4; do MP_LIB=build/ab/knobs.so MP_GATHER_BUDGET_KB=16 MP_GATHER_STAGES=$st timeout -s KILL 300 $B > $O/c1_b16s${st}_$rep.log 2>&1; done
done
ls $O
