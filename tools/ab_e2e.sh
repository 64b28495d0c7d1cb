# A/B of ab/*.so on one box for the device value AND the C++ end-to-end leg (bench.py cfg2),
# R rounds: each variant is copied over the in-tree library of this (scratch) box copy, so
# both the Python bench and the native e2e binary load it.   usage: bash tools/ab_e2e.sh [R]
set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
R=${1:-3}
LIB=paper_2406_10774_b200/libquestkv_b200.so
cp $LIB /tmp/lib_keep.so
: > gpurun_out/ab_e2e.txt
for r in $(seq 1 $R); do
  for v in ab/*.so; do
    cp $v $LIB
    timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab_one.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab_one.json')); e=d['e2e']; print('$v', d['value'], e['value'], e.get('pageable_host_buffers'))" >> gpurun_out/ab_e2e.txt
  done
done
cp /tmp/lib_keep.so $LIB
cat gpurun_out/ab_e2e.txt
