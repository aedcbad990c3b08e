# round-2 pass 61: gather grid leaving k SMs to the planner (knob build,
# int16-box planner): c4 u8 step (plan-bound), c4 f32 / c2 u8 cost.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s61
mkdir -p $O
export PYTHONUNBUFFERED=1
B="python bench.py --no-e2e --no-cpu-baseline --steps 30"
for k in 0 8 16 24 40; do
  MP_GATHER_SM_RESERVE=$k MP_LIB=build/ab/knobs.so timeout -s KILL 300 $B --config c4_4k_drone --fmt u8 > $O/u8_c4_k$k.log 2>&1
done
for k in 0 16; do
  MP_GATHER_SM_RESERVE=$k MP_LIB=build/ab/knobs.so timeout -s KILL 300 $B --config c2_1080p_sparse --fmt u8 > $O/u8_c2_k$k.log 2>&1
  MP_GATHER_SM_RESERVE=$k MP_LIB=build/ab/knobs.so timeout -s KILL 300 $B --config c4_4k_drone > $O/f32_c4_k$k.log 2>&1
done
MP_GATHER_SM_RESERVE=16 MP_LIB=build/ab/knobs.so CFG=c4_4k_drone DEPTH=3 FMT=1 timeout -s KILL 300 python scripts/timeline.py > $O/tl_c4_u8_k16.txt 2>&1
ls $O
