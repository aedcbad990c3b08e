# round-2 pass 73: u8 gather register cap (120 / 112, spills) so the side
# kernels' tail co-resides without an SM reserve — u8 c2 / c3 at k = 0 / 1.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s73
mkdir -p $O
export PYTHONUNBUFFERED=1
B="python bench.py --no-e2e --no-cpu-baseline --steps 50 --fmt u8"
for rep in 1 2; do
 for v in cur r120 r112; do
  for k in 0 1; do
   MP_LIB=build/ab/$v.so timeout -s KILL 300 $B --config c2_1080p_sparse --gather-sm-reserve $k > $O/u8_c2_${v}_k${k}_$rep.log 2>&1
  done
 done
done
for v in cur r120; do
  MP_LIB=build/ab/$v.so timeout -s KILL 300 $B --config c3_1080p_dense --gather-sm-reserve 0 > $O/u8_c3_${v}_k0.log 2>&1
  MP_LIB=build/ab/$v.so timeout -s KILL 300 $B --config c3_1080p_dense --gather-sm-reserve 1 > $O/u8_c3_${v}_k1.log 2>&1
done
ls $O
