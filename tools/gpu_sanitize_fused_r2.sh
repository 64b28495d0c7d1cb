# compute-sanitizer (memcheck, synccheck) over the fused decode tests incl. the bench geometries.
set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for tool in memcheck synccheck; do
  timeout 2400 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
     python -m pytest tests/test_gpu_decode.py tests/test_gpu_geometries.py -m gpu -q -x \
     -k "test_fused_step_vs_oracle and (2051 or GQA or 1500) or test_fused_graph_replay_outgrows or test_cfg2_geometry or test_cfg4 or test_cfg5 or test_decode_step_host" \
     > gpurun_out/sanitize_fused_r2_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_fused_r2_$tool.log
  tail -4 gpurun_out/sanitize_fused_r2_$tool.log
done
