cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_topk -s 1 -c 1 -o gpurun_out/c3_b4 python tools/prof_search.py --config c3 --batch 4 > gpurun_out/ncu_c3b4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_topk -s 1 -c 1 -o gpurun_out/c3_b2 python tools/prof_search.py --config c3 --batch 2 > gpurun_out/ncu_c3b2.log 2>&1
