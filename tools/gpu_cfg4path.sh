set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for path in fused unfused; do
QK_DECODE_PATH=$path timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_cfg4_$path.json 2> gpurun_out/bench_cfg4_$path.err
python -c "import json;d=json.load(open('gpurun_out/bench_cfg4_$path.json'));print('$path', d['value'],d['roofline']['frac'])"
done
QK_DECODE_PATH=unfused timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"append_kernel|estimate_|topk|attend_kernel" -c 12 --csv --log-file gpurun_out/launches_cfg4u.csv python bench.py --config cfg4 --steps 1 --warmup 3 --layers 2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_cfg4u.log 2>&1
