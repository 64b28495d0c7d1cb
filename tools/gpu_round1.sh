set +e
cd $GRAFT_REPO_ROOT
nvidia-smi -L > gpurun_out/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q -x --timeout=600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench rc=$?" >> gpurun_out/bench1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --layers 4 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:estimate_kernel -s 8 -c 1 -o gpurun_out/prof_estimate python bench.py --steps 2 --warmup 1 --layers 4 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_est.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attend_kernel -s 8 -c 1 -o gpurun_out/prof_attend python bench.py --steps 2 --warmup 1 --layers 4 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_att.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:topk_kernel -s 8 -c 1 -o gpurun_out/prof_topk python bench.py --steps 2 --warmup 1 --layers 4 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_topk.log 2>&1
echo done
