# round-2 pass 16: u8 lane regroup A/B (gather alone), u8 parity, NMS racecheck.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s16
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_zero_copy.py -m gpu -q -x -k "gather or full_size or zero" > $O/gather_tests.log 2>&1; echo "rc=$?" >> $O/gather_tests.log
timeout -s KILL 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_edges.py -q -x -k "grid_path and spread and 500" > $O/san_racecheck_nms.log 2>&1; echo "rc=$?" >> $O/san_racecheck_nms.log
AB_TAG=s16 AB_FMTS=1 bash scripts/ab_gather.sh
mv gpurun_out/ab_s16 $O/ab
timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --steps 50 --fmt u8 > $O/bench_u8.log 2>&1
D="python bench.py --no-e2e --no-cpu-baseline --depth 1 --steps 2 --warmup 3"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" -s 3 -c 1 -o $O/prof_gather_u8 -f $D --fmt u8 > $O/p1.log 2>&1
ls -la $O
