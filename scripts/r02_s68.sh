# round-2 pass 68: single-CTA scans reading their runs in batches of 8
# independent loads (ub256 / ub128 threads) vs base — c2 f32 / u8 benches and
# timelines, c3/c4 f32 and u8 lines; GPU suite on ub128.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s68
mkdir -p $O
export PYTHONUNBUFFERED=1
B="python bench.py --no-e2e --no-cpu-baseline --steps 50"
for v in nmsbase ub256 ub128; do
 for fmt in 1 0; do
  MP_LIB=build/ab/$v.so CFG=c2_1080p_sparse DEPTH=3 FMT=$fmt timeout -s KILL 300 python scripts/timeline.py > $O/tl_c2_fmt${fmt}_$v.txt 2>&1
 done
done
for rep in 1 2; do
 for v in nmsbase ub256 ub128; do
  MP_LIB=build/ab/$v.so timeout -s KILL 300 $B --config c2_1080p_sparse --fmt u8 > $O/u8_c2_${v}_$rep.log 2>&1
  MP_LIB=build/ab/$v.so timeout -s KILL 300 $B --config c2_1080p_sparse > $O/f32_c2_${v}_$rep.log 2>&1
 done
done
for v in nmsbase ub128; do
  MP_LIB=build/ab/$v.so timeout -s KILL 300 $B --config c3_1080p_dense > $O/f32_c3_${v}.log 2>&1
  MP_LIB=build/ab/$v.so timeout -s KILL 300 $B --config c3_1080p_dense --fmt u8 > $O/u8_c3_${v}.log 2>&1
  MP_LIB=build/ab/$v.so timeout -s KILL 300 $B --config c4_4k_drone --fmt u8 > $O/u8_c4_${v}.log 2>&1
  MP_LIB=build/ab/$v.so timeout -s KILL 300 $B --config c1_540p > $O/f32_c1_${v}.log 2>&1
done
MP_LIB=build/ab/ub128.so timeout -s KILL 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu_ub128.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_ub128.log
ls $O
