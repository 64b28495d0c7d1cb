set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 10 \
   python -m pytest tests/test_gpu_decode.py tests/test_gpu_attention.py tests/test_gpu_trace.py -m gpu -q -x \
   > gpurun_out/sanitize_full.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/sanitize_full.log
