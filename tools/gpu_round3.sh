set +e
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q --timeout=600 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
QK_PROBE=1 timeout 300 python tools/probe_fused.py > gpurun_out/probe2.txt 2>&1
QK_PROBE=1 timeout 300 python tools/probe_fused.py --ctx 8192 --budget 1024 >> gpurun_out/probe2.txt 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo "bench rc=$?" >> gpurun_out/bench3.err
echo done
