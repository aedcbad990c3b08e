# round-2 pass 62: gather SM reserve sweep at c4 u8, int16-box planner
# (knobs) vs int32-box planner (knobs_base), two reps.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s62
mkdir -p $O
export PYTHONUNBUFFERED=1
B="python bench.py --no-e2e --no-cpu-baseline --steps 30"
for rep in 1 2; do
 for v in knobs knobs_base; do
  for k in 0 12 16 20; do
   MP_GATHER_SM_RESERVE=$k MP_LIB=build/ab/$v.so timeout -s KILL 300 $B --config c4_4k_drone --fmt u8 > $O/u8_c4_${v}_k${k}_$rep.log 2>&1
  done
 done
done
for v in knobs knobs_base; do
 MP_GATHER_SM_RESERVE=16 MP_LIB=build/ab/$v.so timeout -s KILL 300 $B --config c3_1080p_dense --fmt u8 > $O/u8_c3_${v}_k16.log 2>&1
done
MP_GATHER_SM_RESERVE=0 MP_LIB=build/ab/knobs.so timeout -s KILL 300 $B --config c3_1080p_dense --fmt u8 > $O/u8_c3_knobs_k0.log 2>&1
ls $O
