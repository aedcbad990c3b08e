# round-2 pass 24: consumer warps 8 (base) / 10 / 12, gather alone, f32 + u8.
cd $GRAFT_REPO_ROOT
O=gpurun_out/s24
mkdir -p $O
export PYTHONUNBUFFERED=1
AB_TAG=s24 bash scripts/ab_gather.sh
mv gpurun_out/ab_s24 $O/ab
ls -la $O
