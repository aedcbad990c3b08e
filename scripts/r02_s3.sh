# round-2 session-2 pass 3: plan full tier 128 threads x 4/SM, plan streams at
# high priority, single-pass proxy sweep; c4 timeline; A/Bs.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $O/all.log 2>&1; echo "rc=$?" >> $O/all.log
CFG=c4_4k_drone DEPTH=3 timeout -s KILL 600 python scripts/timeline.py > $O/timeline_c4.txt 2>&1
B="python bench.py --no-e2e --no-cpu-baseline --steps 50"
for c in c2_1080p_sparse c4_4k_drone c3_1080p_dense c1_540p; do timeout -s KILL 600 $B --config $c > $O/bench_$c.log 2>&1; done
for c in c2_1080p_sparse c4_4k_drone c3_1080p_dense; do timeout -s KILL 600 $B --config $c --plan-priority 0 > $O/bench_noprio_$c.log 2>&1; done
timeout -s KILL 600 $B --fmt u8 > $O/bench_u8.log 2>&1
for kb in 56 64 72; do MP_LIB=build/ab/knobs.so MP_GATHER_BUDGET_KB=$kb timeout -s KILL 600 $B --fmt u8 > $O/ab_u8_b$kb.log 2>&1; done
timeout -s KILL 600 python bench.py --mode sweep > $O/bench_sweep.log 2>&1
ls -la $O
