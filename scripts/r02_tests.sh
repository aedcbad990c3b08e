# round-2 GPU test pass: new tests first, then the whole -m gpu suite, plus
# memcheck on the capacity-overflow and unbounded-NMS paths.
cd $GRAFT_REPO_ROOT
O=gpurun_out/t2
mkdir -p $O
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout -s KILL 1500 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_edges.py -q -x > $O/new.log 2>&1; echo "rc=$?" >> $O/new.log
timeout -s KILL 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_pipeline.py -q -x -k "overflow" > $O/san_overflow.log 2>&1; echo "rc=$?" >> $O/san_overflow.log
timeout -s KILL 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_edges.py -q -x -k "mixed_tiers or 2049" > $O/san_nms.log 2>&1; echo "rc=$?" >> $O/san_nms.log
timeout -s KILL 2400 python -m pytest tests -m gpu -q > $O/all.log 2>&1; echo "rc=$?" >> $O/all.log
timeout -s KILL 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $O/bench.log 2>&1
