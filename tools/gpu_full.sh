# Full GPU pass (bash tools/gpu_full.sh on the box): GPU tests, smoke, bench line,
# reference arm, launch list, the trained-index bench -> gpurun_out/
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt
nproc >> gpurun_out/smi.txt
timeout 3000 python -m pytest tests -m gpu -x -q --durations=15 ${PYTEST_ARGS:-} > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo exit=$? >> gpurun_out/smoke.log
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --stream-batches '' --stream-config '' --index trained > gpurun_out/bench_trained.log 2>&1
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --stream-batches '' --stream-config '' > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --stream-batches '' --stream-config '' > gpurun_out/ncu_launch.log 2>&1
