set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
QK_PROBE=1 timeout 300 python tools/probe_fused.py --reps 1 --layers 1 > gpurun_out/probe_warm.txt 2>&1
QK_PROBE=1 QK_NO_PREFETCH=1 timeout 300 python tools/probe_fused.py --reps 1 --layers 4 > gpurun_out/probe_nopf.txt 2>&1
echo done
