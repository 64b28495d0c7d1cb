set +e
cd $GRAFT_REPO_ROOT
for v in 0 1; do
  if [ $v = 1 ]; then export QK_TOPK_ROWS=1; else unset QK_TOPK_ROWS; fi
  timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /tmp/c4.json 2>/tmp/c4.err
  python -c "import json;d=json.load(open('/tmp/c4.json'));print('topk_rows_forced=$v', d['value'], d['roofline']['frac'])"
done
unset QK_TOPK_ROWS
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"topk" -c 4 --csv --log-file gpurun_out/l_topk.csv python bench.py --config cfg4 --steps 1 --warmup 3 --layers 2 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
grep -o '"gpu__time_duration.sum","[a-z]*","[0-9.,]*"' gpurun_out/l_topk.csv
