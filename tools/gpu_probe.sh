set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout=600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
QK_PROBE=1 timeout 300 python tools/probe_fused.py --reps 1 > gpurun_out/probe.txt 2>&1
QK_PROBE=1 timeout 300 python tools/probe_fused.py --reps 1 --ctx 8192 --budget 1024 >> gpurun_out/probe.txt 2>&1
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
echo done
