set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_selection.py tests/test_gpu_grouped.py -q -x > gpurun_out/pt_sel.log 2>&1; tail -1 gpurun_out/pt_sel.log
timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
python -c "import json;d=json.load(open('gpurun_out/bench_cfg4.json'));print('cfg4', d['value'],d['roofline']['frac'])"
timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --group-select max > gpurun_out/bench_cfg4_gmax.json 2> gpurun_out/bench_cfg4_gmax.err
python -c "import json;d=json.load(open('gpurun_out/bench_cfg4_gmax.json'));print('grouped', d['value'],d['roofline']['frac'])"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"append_kernel|estimate_|topk|attend_kernel" -c 12 --csv --log-file gpurun_out/launches_cfg4u.csv python bench.py --config cfg4 --steps 1 --warmup 3 --layers 2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_cfg4u.log 2>&1
