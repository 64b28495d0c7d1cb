# compute-sanitizer over the round-2 kernels: grouped (mma) attention + group top-K, register
# top-K rows, the new estimate kernels, vectorised prefill, attend with staged page lists,
# and the bench-geometry fused tests.  memcheck, synccheck and racecheck.
set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SEL="test_grouped_step_vs_oracle or test_grouped_separable or test_grouped_heavy or test_grouped_errors or test_wide_gqa_estimate or test_estimate or test_select or test_prefill or test_sparse or test_dense or test_batched_quest_step"
for tool in memcheck synccheck racecheck; do
  timeout 2400 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
     python -m pytest tests/test_gpu_grouped.py tests/test_gpu_selection.py tests/test_gpu_kv_store.py tests/test_gpu_attention.py -m gpu -q -x -k "$SEL" \
     > gpurun_out/sanitize_r2_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_r2_$tool.log
  tail -4 gpurun_out/sanitize_r2_$tool.log
done
