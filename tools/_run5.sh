cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tscan.py tests/test_gpu_round2_paths.py tests/test_gpu_scale.py -m gpu -x -q -k "not config4_full and not c5 and not 1_000_000" 2>&1 | tail -3
for c in c1 c2 c3; do timeout 200 python tools/stage_midbatch.py $c 2>&1 | tail -4; done
python bench.py --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['detail']['stage_ms'])"
