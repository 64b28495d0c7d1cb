# GPU parity suite (first: the new bench-geometry tests), then a short bench.
set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_geometries.py -q --timeout=900 -rf > gpurun_out/pytest_geom.log 2>&1; echo "geom rc=$?" >> gpurun_out/pytest_geom.log
timeout 1200 python -m pytest tests -m gpu -q --timeout=600 -rf --deselect tests/test_gpu_geometries.py > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/pytest_geom.log gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json
