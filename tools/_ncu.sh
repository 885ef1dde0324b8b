cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_topk -s 1 -c 1 -o gpurun_out/scan_filter python tools/prof_search.py --config c2 --batch 2048 > gpurun_out/ncu_full.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_full.log
