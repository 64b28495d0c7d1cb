set +e
cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q --timeout=600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "bench rc=$?" >> gpurun_out/bench2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches2.csv python bench.py --steps 3 --warmup 1 --layers 8 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_bench2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_fused -s 12 -c 1 -o gpurun_out/prof_fused python bench.py --steps 3 --warmup 1 --layers 8 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_fused.log 2>&1
echo done
