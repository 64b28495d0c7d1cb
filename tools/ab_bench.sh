# A/B the kernel builds in ab/*.so on one box: bench.py (cfg2) alternating between
# variants, R rounds.   usage: bash tools/ab_bench.sh [R] [extra bench args]
set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
R=${1:-3}
shift
: > gpurun_out/ab.txt
for r in $(seq 1 $R); do
  for v in ab/*.so; do
    QK_LIB=$PWD/$v timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 "$@" > gpurun_out/ab_one.json 2>/dev/null
    python -c "import json,sys; d=json.load(open('gpurun_out/ab_one.json')); print('$v', d['value'], d['roofline']['frac'])" >> gpurun_out/ab.txt
  done
done
python - <<'PY'
import collections
d = collections.defaultdict(list)
for l in open('gpurun_out/ab.txt'):
    v, x, f = l.split()
    d[v].append(float(x))
for v, xs in sorted(d.items()):
    xs.sort()
    print(f"{v:40s} median {xs[len(xs)//2]:.3f}  all {xs}")
PY
