cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --stream-batches '' --stream-config '' > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:scan_topk -c 1 -o gpurun_out/scan_filter python tools/prof_search.py --config c2 > gpurun_out/ncu_full.log 2>&1
