# round-2 pass 10: max shared-memory carveout for every hot-path kernel.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s10
mkdir -p $O
export PYTHONUNBUFFERED=1
for c in c4_4k_drone c3_1080p_dense c2_1080p_sparse; do CFG=$c DEPTH=3 timeout -s KILL 600 python scripts/timeline.py > $O/timeline_$c.txt 2>&1; done
B="python bench.py --no-e2e --no-cpu-baseline --steps 50"
for c in c4_4k_drone c3_1080p_dense c2_1080p_sparse c1_540p; do timeout -s KILL 600 $B --config $c > $O/bench_$c.log 2>&1; done
timeout -s KILL 600 $B --fmt u8 > $O/bench_u8.log 2>&1
timeout -s KILL 600 $B --fmt u8 --config c4_4k_drone > $O/bench_u8_c4.log 2>&1
timeout -s KILL 600 $B --fmt u8 --config c3_1080p_dense > $O/bench_u8_c3.log 2>&1
MP_LIB=build/ab/prof.so timeout -s KILL 300 python scripts/plan_prof.py > $O/plan_prof.txt 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $O/all.log 2>&1; echo "rc=$?" >> $O/all.log
ls -la $O
