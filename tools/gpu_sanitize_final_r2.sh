# compute-sanitizer memcheck + racecheck over the kernels changed last in round 2: the row-pair
# top-K, the launch-sized attention splits, the 256-thread prefill, the prefetching MHA
# estimate and the cp.async-staged GQA estimate.
set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SEL="mixed_modes or bench_page_counts or random_geometry or operator_chain or prefill or dense or sparse or estimate or select or grouped_step"
for tool in memcheck racecheck; do
  timeout 2400 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
     python -m pytest tests/test_gpu_geometries.py tests/test_gpu_random_ops.py tests/test_gpu_kv_store.py \
     tests/test_gpu_attention.py tests/test_gpu_selection.py tests/test_gpu_grouped.py -m gpu -q -x -k "$SEL" \
     > gpurun_out/sanitize_final_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_final_$tool.log
  tail -4 gpurun_out/sanitize_final_$tool.log
done
