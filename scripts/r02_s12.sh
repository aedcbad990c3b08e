# round-2 pass 12: single-CTA scans at 256 threads (co-reside with the gather).

cd $GRAFT_REPO_ROOT
O=gpurun_out/s12
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_proxy_sweep.py -m gpu -q -x > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for c in c4_4k_drone c3_1080p_dense c2_1080p_sparse; do CFG=$c DEPTH=3 timeout -s KILL 600 python scripts/timeline.py > $O/timeline_$c.txt 2>&1; done
B="python bench.py --no-e2e --no-cpu-baseline --steps 50"
for c in c4_4k_drone c3_1080p_dense c2_1080p_sparse; do timeout -s KILL 600 $B --config $c > $O/bench_$c.log 2>&1; done
timeout -s KILL 600 $B --fmt u8 --config c4_4k_drone > $O/bench_u8_c4.log 2>&1
timeout -s KILL 600 $B --fmt u8 --config c3_1080p_dense > $O/bench_u8_c3.log 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $O/all.log 2>&1; echo "rc=$?" >> $O/all.log
ls -la $O
