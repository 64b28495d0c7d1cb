# GPU pass for the GQA group-shared variant: its parity tests, then a grouped bench line.
set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_grouped.py -q --timeout=600 -rf -x > gpurun_out/pytest_grouped.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_grouped.log
tail -30 gpurun_out/pytest_grouped.log
