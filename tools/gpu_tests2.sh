set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention_api.py tests/test_cpp_layer.py -q --timeout=600 -rf -x > gpurun_out/pytest_api.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_api.log
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 -rf > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -30 gpurun_out/pytest_api.log; tail -8 gpurun_out/pytest_gpu.log
