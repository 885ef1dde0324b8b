cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q > gpurun_out/l_tests.log 2>&1; echo exit=$? >> gpurun_out/l_tests.log
python tools/lat_b1.py > gpurun_out/lat.log 2>&1; python tools/lat_b1.py --config c1 >> gpurun_out/lat.log 2>&1
