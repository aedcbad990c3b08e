# round-2 pass 47: as pass 46 with one plane-row buffer per f32 warp (fin1) vs the
# fixed-tap consumers (fin): c2/c3/c4 f32 and c4 u8 bench lines, plus the
# per-stream timeline of c4 (plan / gather / merge intervals).
cd $GRAFT_REPO_ROOT
O=gpurun_out/s47
mkdir -p $O
export PYTHONUNBUFFERED=1
for rep in 1; do
 for v in base fin1; do
  for c in c2_1080p_sparse c3_1080p_dense c4_4k_drone; do
   MP_LIB=build/ab/$v.so timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --steps 50 --config $c > $O/bench_${v}_${c}_$rep.log 2>&1
  done
  MP_LIB=build/ab/$v.so timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --steps 50 --config c4_4k_drone --fmt u8 > $O/bench_${v}_u8_c4_$rep.log 2>&1
 done
done
for v in base fin1; do MP_LIB=build/ab/$v.so CFG=c4_4k_drone DEPTH=3 timeout -s KILL 600 python scripts/timeline.py > $O/timeline_c4_$v.txt 2>&1; done
