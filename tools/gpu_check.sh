# GPU tests + one ncu capture of the fused kernel (source-level) + bench.
set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout=600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_fused -s 40 -c 1 -o gpurun_out/prof_check python bench.py --steps 3 --warmup 3 --layers 8 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_check.log 2>&1
echo done
