set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_grouped.py -q --timeout=600 -rf -x > gpurun_out/pytest_grouped.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_grouped.log
timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --group-select max > gpurun_out/bench_cfg4_gmax.json 2> gpurun_out/bench_cfg4_gmax.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"append_kernel|estimate_kernel|group_topk|grouped_attend" -c 16 --csv --log-file gpurun_out/launches_cfg4g.csv python bench.py --config cfg4 --steps 1 --warmup 3 --layers 2 --no-cpu-baseline --e2e-steps 1 --group-select max > gpurun_out/ncu_cfg4g.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_attend -s 2 -c 1 -o gpurun_out/prof_grouped python bench.py --config cfg4 --steps 1 --warmup 3 --layers 2 --no-cpu-baseline --e2e-steps 1 --group-select max > gpurun_out/ncu_grouped.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:estimate_kernel -s 2 -c 1 -o gpurun_out/prof_estimate_g4 python bench.py --config cfg4 --steps 1 --warmup 3 --layers 2 --no-cpu-baseline --e2e-steps 1 --group-select max > gpurun_out/ncu_est.log 2>&1
tail -3 gpurun_out/pytest_grouped.log; python -c "import json;d=json.load(open('gpurun_out/bench_cfg4_gmax.json'));print(d['value'],d['roofline']['frac'])"; tail -2 gpurun_out/bench_cfg4_gmax.err
