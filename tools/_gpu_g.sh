cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_synth.py tests/test_gpu_golden.py tests/test_gpu_configs.py -x -q > gpurun_out/g_tests.log 2>&1; echo exit=$? >> gpurun_out/g_tests.log
timeout 300 python bench.py --no-cpu-baseline --steps 1 --warmup 1 --batch 16 --stream-batches '1,2,3,4' > gpurun_out/g_ws4.log 2>&1
