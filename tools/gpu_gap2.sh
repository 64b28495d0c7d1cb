set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in 32700 32768 32900; do timeout 300 python bench.py --ctx $c --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_ctx$c.json 2>/dev/null; done
QK_PROBE=1 QK_PROBE_GRAPH=1 timeout 300 python tools/probe_fused.py --reps 1 --layers 32 --ctx 32700 > gpurun_out/probe_g32_32700.txt 2>&1
QK_PROBE=1 QK_PROBE_GRAPH=1 timeout 300 python tools/probe_fused.py --reps 1 --layers 32 --ctx 32900 > gpurun_out/probe_g32_32900.txt 2>&1
echo done
