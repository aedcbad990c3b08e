# round-2 pass 59: int16 component boxes in the planner (full tier ~33 -> ~26 KB
# of shared memory: two plan CTAs beside the u8 ring) — GPU suite on the new
# library, then pipelined steps base vs box16 (u8 c2/c3/c4, f32 c4).
cd $GRAFT_REPO_ROOT
O=gpurun_out/s59
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for rep in 1 2; do
 for v in base box16; do
  for cfg in c4_4k_drone c3_1080p_dense c2_1080p_sparse; do
   MP_LIB=build/ab/$v.so timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --steps 50 --config $cfg --fmt u8 > $O/bench_u8_${cfg}_${v}_$rep.log 2>&1
  done
  MP_LIB=build/ab/$v.so timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --steps 50 --config c4_4k_drone > $O/bench_f32_c4_${v}_$rep.log 2>&1
 done
done
ls $O
