# memcheck per GPU test file (one process each: device memory does not
# accumulate across files under the sanitizer), minus the c4 full-size test.
cd $GRAFT_REPO_ROOT
O=gpurun_out/san3
mkdir -p $O
export PYTHONUNBUFFERED=1
for f in tests/test_gpu_*.py tests/test_proxy_sweep.py tests/test_window_sets.py tests/test_c_abi_demo.py; do
  b=$(basename $f .py)
  timeout -s KILL 1500 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest $f -m gpu -q -k "not (full_size_pipelined and c4)" > $O/memcheck_$b.log 2>&1; echo "rc=$?" >> $O/memcheck_$b.log
done
grep -H "ERROR SUMMARY\|passed\|failed\|rc=" $O/*.log
