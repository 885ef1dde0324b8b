cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_train.py -x -q > gpurun_out/t_tests.log 2>&1; echo exit=$? >> gpurun_out/t_tests.log
for a in "--method apcpq --quantize --n 20000" "--method apcpq --quantize --n 100000 --no-ref"; do python tools/bench_train.py $a >> gpurun_out/t_bench.log 2>&1; done
