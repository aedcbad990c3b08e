cd $GRAFT_REPO_ROOT
O=gpurun_out/d23
mkdir -p $O
for rep in 1 2; do
for d in 2 3; do
  timeout 300 python bench.py --depth $d --no-e2e --no-cpu-baseline --steps 200 > $O/c2_d${d}_$rep.json 2>>$O/err
  timeout 300 python bench.py --depth $d --fmt u8 --no-e2e --no-cpu-baseline --steps 200 > $O/u8_d${d}_$rep.json 2>>$O/err
  timeout 300 python bench.py --depth $d --src nv12 --no-e2e --no-cpu-baseline --steps 100 > $O/nv12_d${d}_$rep.json 2>>$O/err
done
done
