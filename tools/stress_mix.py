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
for _o in sys.argv[1:]:
    P.set_option(_o.split("=")[0], int(_o.split("=")[1]))
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
for rep in range(3):
  for bs in [1, 2, 4, 6, 8, 12, 16, 32, 64, 128, 255]:
    for it in range(13):
        flush.add_(1.0)
        torch.cuda.synchronize()
        r = P.search_device(idx, Q[:bs].contiguous(), cfg.topn)
        torch.cuda.synchronize()
    print("B", bs, "ok", flush=True)
