cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in crops_rgb; do
WHAT=$w FRAMES=600 timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:gather_kernel -s 2 -c 1 -o gpurun_out/prof_$w -f python scripts/time_gather.py > gpurun_out/prof_$w.log 2>&1
done
