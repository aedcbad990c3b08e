# round-2 pass 64: are the u8 steps merge-bound? side streams (merges of
# consecutive batches overlap) and depth, c2/c3/c4 u8; c2 u8 timeline.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s64
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_pipeline.py -m gpu -q > $O/pytest_pipeline.log 2>&1; echo "rc=$?" >> $O/pytest_pipeline.log
B="python bench.py --no-e2e --no-cpu-baseline --steps 40"
for cfg in c3_1080p_dense c2_1080p_sparse c4_4k_drone; do
 for ss in 1 2 3; do
  timeout -s KILL 300 $B --config $cfg --fmt u8 --side-streams $ss > $O/u8_${cfg}_ss$ss.log 2>&1
 done
 timeout -s KILL 300 $B --config $cfg --fmt u8 --side-streams 2 --depth 4 > $O/u8_${cfg}_ss2_d4.log 2>&1
done
timeout -s KILL 300 $B --config c3_1080p_dense --side-streams 2 > $O/f32_c3_ss2.log 2>&1
timeout -s KILL 300 $B --config c3_1080p_dense --side-streams 1 > $O/f32_c3_ss1.log 2>&1
CFG=c2_1080p_sparse DEPTH=3 FMT=1 timeout -s KILL 300 python scripts/timeline.py > $O/tl_c2_u8.txt 2>&1
ls $O
