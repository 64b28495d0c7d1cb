cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_decode.py -m gpu -q -x --timeout=900 > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
bash tools/ab_bench.sh 2
for v in base pipe; do QK_LIB=$PWD/ab/$v.so timeout 600 python bench.py --config cfg3 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/cfg3_$v.json 2>/dev/null; done
