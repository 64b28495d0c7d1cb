# Grouped measurement: cfg4 bench per-head vs group-shared, recall study,
# ncu of the tensor-core group attention and of the per-head fused kernel at cfg4.
set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --group-select max > gpurun_out/bench_cfg4_gmax.json 2> gpurun_out/bench_cfg4_gmax.err
timeout 600 python tools/group_recall.py > gpurun_out/group_recall.jsonl 2> gpurun_out/group_recall.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_cfg4g.csv python bench.py --config cfg4 --steps 1 --warmup 3 --layers 2 --no-cpu-baseline --e2e-steps 1 --group-select max > gpurun_out/ncu_cfg4g.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_attend -s 2 -c 1 -o gpurun_out/prof_grouped python bench.py --config cfg4 --steps 1 --warmup 3 --layers 2 --no-cpu-baseline --e2e-steps 1 --group-select max > gpurun_out/ncu_grouped.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fused -s 2 -c 1 -o gpurun_out/prof_fused_cfg4 python bench.py --config cfg4 --steps 1 --warmup 3 --layers 2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_fused_cfg4.log 2>&1
cat gpurun_out/bench_cfg4_gmax.json; tail -3 gpurun_out/bench_cfg4_gmax.err; cat gpurun_out/group_recall.jsonl; tail -3 gpurun_out/group_recall.err; tail -2 gpurun_out/ncu_grouped.log
