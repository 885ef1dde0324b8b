import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_2112_02179_b200 as P
from paper_2112_02179_b200 import datagen
cfg = datagen.CONFIGS["c2"]
dev = torch.device("cuda:0")
data = datagen.synth_index(cfg, seed=1, device=dev)
Q = datagen.queries(cfg, 512, seed=2, device=dev)
idx = P.deserialize(data, device=0)
P.set_option("scan_tc", 0)
P.set_option("scan_filter", int(sys.argv[2]))
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
for bs in [int(v) for v in sys.argv[1].split(",")]:
    print("B", bs, "plan", P.plan_info(idx, bs, cfg.topn), flush=True)
    for it in range(40):
        flush.add_(1.0)
        torch.cuda.synchronize()
        r = P.search_device(idx, Q[:bs].contiguous(), cfg.topn)
        torch.cuda.synchronize()
    print("  ok", flush=True)
