# Every BASELINE.json config through bench.py (cfg2 is the default / headline).
set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for C in cfg1 cfg3 cfg4; do
  timeout 900 python bench.py --config $C --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_$C.json 2> gpurun_out/bench_$C.err
done
timeout 900 python bench.py --config cfg5 --layers 16 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
for B in 256 512 1024 4096; do timeout 300 python bench.py --budget $B --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_b$B.json 2>/dev/null; done
echo done
