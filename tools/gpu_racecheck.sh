set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 --print-limit 10 \
   python -m pytest tests/test_gpu_decode.py -m gpu -q -x -k "test_fused_selection_modes or (test_fused_step_vs_oracle and (GQA or 32767 or 8191))" \
   > gpurun_out/racecheck.log 2>&1
echo "racecheck rc=$?" >> gpurun_out/racecheck.log
