# round-2 pass 25: merge-heavy plan fuzz + the whole GPU suite.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s25
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -k "merge_heavy" > $O/fuzz.log 2>&1; echo "rc=$?" >> $O/fuzz.log
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $O/all.log 2>&1; echo "rc=$?" >> $O/all.log
tail -3 $O/*.log
