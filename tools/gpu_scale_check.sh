cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/multi_tests.log 2>&1; echo exit=$? >> gpurun_out/multi_tests.log
timeout 1500 python -m pytest tests/test_gpu_scale.py -x -q -k "config2 or config5" --durations=0 > gpurun_out/scale_tests.log 2>&1; echo exit=$? >> gpurun_out/scale_tests.log
timeout 1800 python -m pytest tests/test_gpu_scale.py -x -q -k "config4" --durations=0 > gpurun_out/scale_c4.log 2>&1; echo exit=$? >> gpurun_out/scale_c4.log
