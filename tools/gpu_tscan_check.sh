cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tscan.py -x -q > gpurun_out/tscan_tests.log 2>&1; echo exit=$? >> gpurun_out/tscan_tests.log
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --stream-batches '' --stream-config '' > gpurun_out/bench_tc.log 2>&1
