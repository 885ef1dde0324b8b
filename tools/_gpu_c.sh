cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --config c4 --n 12500000 --batch 4096 --steps 2 --warmup 1 --no-cpu-baseline --stream-batches '' --stream-config '' > gpurun_out/bench_c4.log 2>&1
timeout 600 python bench.py --config c3 --steps 3 --warmup 2 --no-cpu-baseline --stream-batches '' --stream-config '' > gpurun_out/bench_c3.log 2>&1
