# round-2 pass 6: spatial-grid NMS path.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s6
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -q -x -k "nms or remap or fuzz" > $O/nms_tests.log 2>&1; echo "rc=$?" >> $O/nms_tests.log
CFG=c4_4k_drone DEPTH=3 timeout -s KILL 600 python scripts/timeline.py > $O/timeline_c4.txt 2>&1
CFG=c3_1080p_dense DEPTH=3 timeout -s KILL 600 python scripts/timeline.py > $O/timeline_c3.txt 2>&1
B="python bench.py --no-e2e --no-cpu-baseline --steps 50"
for c in c4_4k_drone c3_1080p_dense c2_1080p_sparse; do timeout -s KILL 600 $B --config $c > $O/bench_$c.log 2>&1; done
D="python bench.py --no-e2e --no-cpu-baseline --depth 1 --steps 2 --warmup 3"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"nms_large_kernel" -s 2 -c 1 -o $O/prof_nms_large -f $D --config c4_4k_drone > $O/prof_nms.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"nms_small_kernel" -s 2 -c 1 -o $O/prof_nms_small -f $D --config c3_1080p_dense > $O/prof_nms_small.log 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $O/all.log 2>&1; echo "rc=$?" >> $O/all.log
ls -la $O
