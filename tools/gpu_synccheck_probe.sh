set +e
cd $GRAFT_REPO_ROOT
for env in "QK_X=1" "QK_NO_PDL=1" "QK_NO_PREFETCH=1"; do
  env $env timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool synccheck --print-limit 2 python tools/synccheck_cases.py 16 16 1 20000 > /tmp/sc.log 2>&1
  echo "== $env: $(grep -m1 'ERROR SUMMARY' /tmp/sc.log) $(grep -m1 -o '^ok.*' /tmp/sc.log)"
done
