cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_filter.py tests/test_gpu_configs.py -x -q > gpurun_out/i_tests.log 2>&1; echo exit=$? >> gpurun_out/i_tests.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_i.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --stream-batches '' --stream-config '' > gpurun_out/ncu_launch_i.log 2>&1
