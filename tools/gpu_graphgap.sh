set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for L in 4 8 32; do timeout 300 python bench.py --layers $L --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_L$L.json 2>/dev/null; done
QK_NO_PDL=1 timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_nopdl.json 2>/dev/null
echo done
