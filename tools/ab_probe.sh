# Probe timeline of every ab/*.so (one line per variant: the median layer's stamps).
set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/ab_probe.txt
for v in ab/*.so; do
  echo "== $v" >> gpurun_out/ab_probe.txt
  QK_PROBE=1 QK_LIB=$PWD/$v timeout 300 python tools/probe_fused.py --reps 1 "$@" 2>&1 | head -2 >> gpurun_out/ab_probe.txt
done
