"""K2-T stage times (prep + seed, filter, finish) at mid batch sizes."""
import os, sys, statistics
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_2112_02179_b200 as P
from paper_2112_02179_b200 import datagen
cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = datagen.CONFIGS[cfgname]
dev = torch.device("cuda:0")
data = datagen.synth_index(cfg, seed=1, device=dev)
idx = P.deserialize(data, device=0)
Q = datagen.queries(cfg, 512, seed=2, device=dev)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
P.set_option("scan_tc_min_work", 0)
for bs in [int(x) for x in os.environ.get("BATCHES", "16,64,128").split(",")]:
    qs = Q[:bs].contiguous()
    for _ in range(3):
        P.search_device(idx, qs, cfg.topn)
    P.set_profiling(True)
    t = []
    for _ in range(10):
        flush.add_(1.0)
        torch.cuda.synchronize()
        P.search_device(idx, qs, cfg.topn)
        t.append(P.last_timings())
    P.set_profiling(False)
    print(cfgname, "B", bs, P.plan_info(idx, bs, cfg.topn).get("filter"), "stages ms",
          [round(statistics.median(x[i] for x in t), 4) for i in range(3)], flush=True)
