cd $GRAFT_REPO_ROOT
for a in "--graph-steps 1" "--graph-steps 50" "--graph-steps 50 --fresh-q"; do
  echo "== $a"
  QK_PROBE=1 QK_PROBE_GRAPH=1 timeout 300 python tools/probe_fused.py --reps 1 --layers 32 $a 2>&1 | grep -v '"ctas"'
done
