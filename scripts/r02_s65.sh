# round-2 pass 65: NMS side-kernel geometry beside the u8 gather — nmsA (small
# tier cap 448 at 48 registers: two CTAs beside a u8 gather CTA; tiny tier 4
# warps per CTA), nmsB (tiny 4 warps only) vs nmsbase; GPU suite on nmsA.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s65
mkdir -p $O
export PYTHONUNBUFFERED=1
MP_LIB=build/ab/nmsA.so timeout -s KILL 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu_nmsA.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_nmsA.log
B="python bench.py --no-e2e --no-cpu-baseline --steps 40"
for rep in 1 2; do
 for v in nmsbase nmsA nmsB; do
  MP_LIB=build/ab/$v.so timeout -s KILL 300 $B --config c3_1080p_dense --fmt u8 > $O/u8_c3_${v}_$rep.log 2>&1
  MP_LIB=build/ab/$v.so timeout -s KILL 300 $B --config c2_1080p_sparse --fmt u8 > $O/u8_c2_${v}_$rep.log 2>&1
  MP_LIB=build/ab/$v.so timeout -s KILL 300 $B --config c3_1080p_dense > $O/f32_c3_${v}_$rep.log 2>&1
  MP_LIB=build/ab/$v.so timeout -s KILL 300 $B --config c2_1080p_sparse > $O/f32_c2_${v}_$rep.log 2>&1
 done
done
ls $O
