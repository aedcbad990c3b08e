# round-2 session-2 pass: side-kernel co-residency (plan full tier 35 KB with
# global fallback, NMS large tier 256 threads / 53 KB, gather ring leaving 56 KB
# per SM), whole-step graphs for small batches, CUPTI host-sync trace.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s2
mkdir -p $O
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x > $O/all.log 2>&1; echo "rc=$?" >> $O/all.log
B="python bench.py --no-e2e --no-cpu-baseline --steps 50"
for c in c2_1080p_sparse c4_4k_drone c3_1080p_dense c1_540p; do timeout -s KILL 600 $B --config $c > $O/bench_$c.log 2>&1; done
timeout -s KILL 600 $B --fmt u8 > $O/bench_u8.log 2>&1
timeout -s KILL 600 $B --config c1_540p --step-graph 0 > $O/bench_c1_nograph.log 2>&1
# A/B: experiment-knob build (same code) with the former 3-stage f32 ring, and 56-KB f32 stages
for c in c2_1080p_sparse c4_4k_drone c3_1080p_dense; do
  MP_LIB=build/ab/knobs.so timeout -s KILL 600 $B --config $c > $O/ab_knobs_base_$c.log 2>&1
  MP_LIB=build/ab/knobs.so MP_GATHER_STAGES=3 timeout -s KILL 600 $B --config $c > $O/ab_stages3_$c.log 2>&1
  MP_LIB=build/ab/knobs.so MP_GATHER_BUDGET_KB=56 timeout -s KILL 600 $B --config $c > $O/ab_b56_$c.log 2>&1
done
timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --steps 5 --warmup 3 --trace $O/trace_c2.json > $O/trace_c2.log 2>&1
timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 --config c1_540p --trace $O/trace_c1.json > $O/trace_c1.log 2>&1
CFG=c4_4k_drone DEPTH=3 timeout -s KILL 600 python scripts/timeline.py > $O/timeline_c4.txt 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"plan_|gather_|nms_" -c 60 --csv --log-file $O/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 > $O/launches_bench.log 2>&1
ls -la $O
