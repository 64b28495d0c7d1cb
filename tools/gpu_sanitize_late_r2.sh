# compute-sanitizer memcheck over the late round-2 paths: qk_cache_reserve growth, host-step
# buffers read/written in place (qk_host_alloc), the random-geometry sweeps (fused step,
# grouped step, separate operators) and the 256 x 8 fused selection.
set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 \
   python -m pytest tests/test_gpu_kv_store.py tests/test_gpu_attention.py tests/test_gpu_random_ops.py \
   tests/test_gpu_decode.py tests/test_gpu_grouped.py -m gpu -q -x \
   -k "grows or reserve or quest_cache_capacity or pinned or host_alloc or random_geometry" \
   > gpurun_out/sanitize_late_memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/sanitize_late_memcheck.log
tail -4 gpurun_out/sanitize_late_memcheck.log
