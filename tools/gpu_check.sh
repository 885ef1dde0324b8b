# Quick GPU check (bash tools/gpu_check.sh on the box): GPU tests, smoke, bench, reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt
free -g >> gpurun_out/smi.txt; nproc >> gpurun_out/smi.txt; df -h /tmp . >> gpurun_out/smi.txt
python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
