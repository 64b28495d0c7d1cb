# Iteration pass: full GPU suite, cfg2 bench breakdown, cfg4 fused vs unfused vs grouped, launch list.
set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['roofline']['frac'],d['kernel_breakdown_us'])"; tail -2 gpurun_out/bench.err
for path in auto unfused; do
QK_DECODE_PATH=${path/auto/} timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_cfg4_$path.json 2> gpurun_out/bench_cfg4_$path.err
python -c "import json;d=json.load(open('gpurun_out/bench_cfg4_$path.json'));print('$path', d['value'],d['roofline']['frac'])"
done
timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --group-select max > gpurun_out/bench_cfg4_gmax.json 2> gpurun_out/bench_cfg4_gmax.err
python -c "import json;d=json.load(open('gpurun_out/bench_cfg4_gmax.json'));print('grouped', d['value'],d['roofline']['frac'])"
QK_DECODE_PATH=unfused timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"append_kernel|estimate_|topk|attend_kernel" -c 12 --csv --log-file gpurun_out/launches_cfg4u.csv python bench.py --config cfg4 --steps 1 --warmup 3 --layers 2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_cfg4u.log 2>&1
