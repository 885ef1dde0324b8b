cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_topk -s 1 -c 1 -o gpurun_out/scan_filter_b10k python tools/prof_search.py --config c2 > gpurun_out/ncu_full10k.log 2>&1
for c in c1; do
  python bench.py --config $c --no-cpu-baseline --stream-batches '' --stream-config '' > gpurun_out/bench_$c.log 2>&1
  PCPQG_SCAN_FILTER=0 python bench.py --config $c --no-cpu-baseline --stream-batches '' --stream-config '' > gpurun_out/bench_${c}_nof.log 2>&1
done
