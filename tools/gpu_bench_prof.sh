# bench line + reference arm + launch list + one ncu --set full capture of the
# K2-T filter kernel (bash tools/gpu_bench_prof.sh on the box)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --stream-batches '' --stream-config '' > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --stream-batches '' --stream-config '' > gpurun_out/ncu_launch.log 2>&1
