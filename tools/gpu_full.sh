# Full GPU pass: tests, smoke, bench (default + budget sweep), ncu launch list + full
# capture of the fused kernel.  Outputs land in gpurun_out/.
set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/nvsmi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1; nproc >> gpurun_out/lscpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q --timeout=600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for B in 256 512 1024 4096; do timeout 300 python bench.py --budget $B --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_b$B.json 2>/dev/null; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 40 -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --layers 8 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_fused -s 40 -c 1 -o gpurun_out/prof_fused python bench.py --steps 3 --warmup 3 --layers 8 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_fused.log 2>&1
QK_PROBE=1 timeout 300 python tools/probe_fused.py --reps 1 > gpurun_out/probe.txt 2>&1
echo done
