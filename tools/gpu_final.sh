# Round-2 full measurement pass: tests, smoke, every bench config (+ grouped, budget sweep,
# reference arm), ncu launch lists and full captures of the kernels the docs cite.
set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for c in cfg1 cfg3 cfg4 cfg5; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --group-select max > gpurun_out/bench_cfg4_gmax.json 2> gpurun_out/bench_cfg4_gmax.err
timeout 600 python bench.py --config cfg3 --shard heads --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3h.json 2> gpurun_out/bench_cfg3h.err
for B in 256 512 1024 4096; do timeout 300 python bench.py --budget $B --no-cpu-baseline --e2e-steps 1 --steps 20 --warmup 5 > gpurun_out/bench_b$B.json 2>/dev/null; done
timeout 300 python tools/group_recall.py > gpurun_out/group_recall.jsonl 2> gpurun_out/group_recall.err
timeout 300 python tools/prefill_bench.py > gpurun_out/prefill.json 2>&1
QK_PROBE=1 QK_PROBE_GRAPH=1 timeout 300 python tools/probe_fused.py --reps 1 --layers 8 --graph-steps 4 --fresh-q > gpurun_out/probe_graph.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 40 -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --layers 8 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"append_kernel|estimate_|topk|attend_kernel|decode_fused" -c 24 --csv --log-file gpurun_out/launches_cfg4.csv python bench.py --config cfg4 --steps 1 --warmup 3 --layers 2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_cfg4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"decode_fused" -c 8 --csv --log-file gpurun_out/launches_cfg5.csv python bench.py --config cfg5 --steps 1 --warmup 3 --layers 2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_cfg5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_fused -s 40 -c 1 -o gpurun_out/prof_fused python bench.py --steps 3 --warmup 3 --layers 8 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_fused.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"estimate_mha|topk_rows|attend_kernel" -c 3 -o gpurun_out/prof_sepops python bench.py --steps 1 --warmup 3 --layers 2 --e2e-steps 1 > gpurun_out/ncu_sepops.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"grouped_attend|estimate_gqa" -s 2 -c 2 -o gpurun_out/prof_grouped python bench.py --config cfg4 --steps 1 --warmup 3 --layers 2 --no-cpu-baseline --e2e-steps 1 --group-select max > gpurun_out/ncu_grouped.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
for f in bench bench_ref bench_cfg1 bench_cfg3 bench_cfg4 bench_cfg5 bench_cfg4_gmax bench_cfg3h bench_b256 bench_b512 bench_b1024 bench_b4096; do python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f', d.get('value'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'))" 2>&1 | tail -1; done
