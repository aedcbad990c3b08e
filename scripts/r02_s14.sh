# round-2 pass 14: single-pass NMS grid adjacency (hit masks, exact overlap reject).
cd $GRAFT_REPO_ROOT
O=gpurun_out/s14
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -q -x -k "nms or remap or fuzz" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for c in c3_1080p_dense c4_4k_drone; do CFG=$c DEPTH=3 timeout -s KILL 600 python scripts/timeline.py > $O/timeline_$c.txt 2>&1; done
B="python bench.py --no-e2e --no-cpu-baseline --steps 50"
for c in c3_1080p_dense c4_4k_drone c2_1080p_sparse; do timeout -s KILL 600 $B --config $c > $O/bench_$c.log 2>&1; done
D="python bench.py --no-e2e --no-cpu-baseline --depth 1 --steps 2 --warmup 3"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"nms_small_kernel" -s 2 -c 1 -o $O/prof_nms_small_c3 -f $D --config c3_1080p_dense > $O/p1.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"nms_large_kernel" -s 2 -c 1 -o $O/prof_nms_large_c4 -f $D --config c4_4k_drone > $O/p3.log 2>&1
ls -la $O
