# Round-2 first GPU pass: smoke, every GPU test, bench (cfg2 + ref arm + cfg3/4/5), launch list.
set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/nvsmi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1; nproc >> gpurun_out/lscpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q --timeout=900 -rf --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for c in cfg1 cfg3 cfg4 cfg5; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 40 -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --layers 8 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_bench.log 2>&1
tail -25 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log | tail -3
for f in bench bench_ref bench_cfg1 bench_cfg3 bench_cfg4 bench_cfg5; do echo "== $f"; cat gpurun_out/$f.json; tail -3 gpurun_out/$f.err; done
