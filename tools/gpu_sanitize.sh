# compute-sanitizer over a representative subset of the fused-step GPU tests.
set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SEL="test_fused_step_vs_oracle and (2051 or 32800 or GQA or 5000 or 1500) or test_fused_multi_step or test_fused_graph_replay_outgrows or test_decode_step_host_consecutive"
for tool in memcheck synccheck; do
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
     python -m pytest tests/test_gpu_decode.py tests/test_gpu_attention.py -m gpu -q -x -k "$SEL" \
     > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
done
