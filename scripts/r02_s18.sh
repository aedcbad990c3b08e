# round-2 pass 18: exact overlap pre-test in every NMS path; NV12 step bytes.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s18
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -q -x -k "nms or remap or fuzz" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
B="python bench.py --no-e2e --no-cpu-baseline --steps 50"
for c in c2_1080p_sparse c3_1080p_dense c4_4k_drone; do timeout -s KILL 600 $B --config $c > $O/bench_$c.log 2>&1; done
timeout -s KILL 600 $B --src nv12 > $O/bench_nv12.log 2>&1
ls -la $O
