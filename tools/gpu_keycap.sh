set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout=600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --config cfg3 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_cfg3.json 2>> gpurun_out/bench.err
QK_PROBE=1 QK_PROBE_GRAPH=1 timeout 300 python tools/probe_fused.py --reps 1 --layers 32 --graph-steps 50 --fresh-q 2>&1 | grep -v '"ctas"' > gpurun_out/gp.txt
echo done
