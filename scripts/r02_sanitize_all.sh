# round-2: compute-sanitizer memcheck over the whole GPU suite, racecheck /
# synccheck over the pipeline, gather and NMS tests.
cd $GRAFT_REPO_ROOT
O=gpurun_out/san
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout -s KILL 3000 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests -m gpu -q -x > $O/memcheck_all.log 2>&1; echo "rc=$?" >> $O/memcheck_all.log
timeout -s KILL 1500 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_pipeline.py -q -x -k "capture_steps or new_inputs and eager and 2" > $O/racecheck_pipeline.log 2>&1; echo "rc=$?" >> $O/racecheck_pipeline.log
timeout -s KILL 1500 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "scales_and_edges and 0.7 or full_size_pipelined and c4" > $O/racecheck_gather.log 2>&1; echo "rc=$?" >> $O/racecheck_gather.log
timeout -s KILL 1500 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_edges.py -q -x -k "grid_path or beyond_shared or mixed_tiers" > $O/racecheck_nms.log 2>&1; echo "rc=$?" >> $O/racecheck_nms.log
timeout -s KILL 1500 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py -q -x -k "grid_path and 500 or plan_parity_configs or nms_parity_frame_sizes" > $O/synccheck_side.log 2>&1; echo "rc=$?" >> $O/synccheck_side.log
timeout -s KILL 1500 compute-sanitizer --tool initcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "plan_parity_configs or remap_nms_parity_configs" > $O/initcheck_side.log 2>&1; echo "rc=$?" >> $O/initcheck_side.log
grep -H "ERROR SUMMARY\|RACECHECK SUMMARY\|passed\|failed\|rc=" $O/*.log
