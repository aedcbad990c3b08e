# round-2 pass 8: u8 word taps; c4 plan co-running vs free shared memory.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s8
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $O/all.log 2>&1; echo "rc=$?" >> $O/all.log
B="python bench.py --no-e2e --no-cpu-baseline --steps 50"
timeout -s KILL 600 $B --fmt u8 > $O/bench_u8.log 2>&1
for kb in 40 48; do
  MP_LIB=build/ab/knobs.so MP_GATHER_BUDGET_KB=$kb CFG=c4_4k_drone DEPTH=3 timeout -s KILL 600 python scripts/timeline.py > $O/timeline_c4_b$kb.txt 2>&1
  MP_LIB=build/ab/knobs.so MP_GATHER_BUDGET_KB=$kb timeout -s KILL 600 $B --config c4_4k_drone > $O/bench_c4_b$kb.log 2>&1
done
MP_LIB=build/ab/knobs.so timeout -s KILL 600 $B --config c4_4k_drone > $O/bench_c4_knobbase.log 2>&1
ls -la $O
