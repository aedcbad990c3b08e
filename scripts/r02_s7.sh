# round-2 pass 7: adaptive NMS grid, 128-thread NMS tiers; word-tap A/B.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s7
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -q -x -k "nms or remap or fuzz" > $O/nms_tests.log 2>&1; echo "rc=$?" >> $O/nms_tests.log
CFG=c4_4k_drone DEPTH=3 timeout -s KILL 600 python scripts/timeline.py > $O/timeline_c4.txt 2>&1
CFG=c3_1080p_dense DEPTH=3 timeout -s KILL 600 python scripts/timeline.py > $O/timeline_c3.txt 2>&1
B="python bench.py --no-e2e --no-cpu-baseline --steps 50"
for c in c4_4k_drone c3_1080p_dense c2_1080p_sparse; do timeout -s KILL 600 $B --config $c > $O/bench_$c.log 2>&1; done
AB_TAG=s7 bash scripts/ab_gather.sh
mv gpurun_out/ab_s7 $O/ab
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $O/all.log 2>&1; echo "rc=$?" >> $O/all.log
ls -la $O
