# round-2 final sanity of HEAD's bench paths: clips mode (f32 and u8), default, reference arm.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s75
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout -s KILL 1200 python bench.py --mode clips --clips 24 --steps 1 --warmup 1 > $O/bench_clips24.log 2>&1; echo "rc=$?" >> $O/bench_clips24.log
timeout -s KILL 1200 python bench.py --mode clips --clips 24 --steps 1 --warmup 1 --fmt u8 > $O/bench_clips24_u8.log 2>&1; echo "rc=$?" >> $O/bench_clips24_u8.log
timeout -s KILL 900 python bench.py > $O/bench_default.log 2>&1; echo "rc=$?" >> $O/bench_default.log
timeout -s KILL 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref.log 2>&1; echo "rc=$?" >> $O/bench_ref.log
ls $O
