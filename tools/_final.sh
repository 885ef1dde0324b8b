cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 400 python bench.py > gpurun_out/bench.log 2>gpurun_out/bench.err; tail -1 gpurun_out/bench.log | cut -c1-300
timeout 200 python bench.py --config c3 --steps 10 --warmup 3 > gpurun_out/bench_c3.log 2>/dev/null; tail -1 gpurun_out/bench_c3.log | cut -c1-200
timeout 200 python bench.py --index trained > gpurun_out/bench_trained.log 2>/dev/null; tail -1 gpurun_out/bench_trained.log | cut -c1-200
timeout 200 python bench.py --config c1 > gpurun_out/bench_c1.log 2>/dev/null; tail -1 gpurun_out/bench_c1.log | cut -c1-200
