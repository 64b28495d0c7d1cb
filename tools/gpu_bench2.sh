set +e
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shard.py -q --timeout=800 -rf > gpurun_out/pytest_shard.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_shard.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-native-e2e > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 600 python bench.py --config cfg3 --shard heads --steps 10 --warmup 3 > gpurun_out/bench_cfg3h.json 2> gpurun_out/bench_cfg3h.err
tail -3 gpurun_out/pytest_shard.log; for f in bench bench_ref bench_cfg4 bench_cfg3h; do echo "== $f"; cat gpurun_out/$f.json; tail -3 gpurun_out/$f.err; done
