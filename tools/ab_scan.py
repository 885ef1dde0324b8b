"""A/B of the fused search on one index: run with PCPQG_LIB=<lib> to compare
builds.  Prints the median LUT/scan/merge times of `--iters` searches."""
import argparse, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2112_02179_b200 as P
from paper_2112_02179_b200 import datagen

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--iters", type=int, default=5)
a = ap.parse_args()
cfg = datagen.CONFIGS[a.config]
dev = torch.device("cuda:0")
data = datagen.synth_index(cfg, seed=1, device=dev)
idx = P.deserialize(data, device=0)
B = a.batch or cfg.batch
Q = datagen.queries(cfg, B, seed=2, device=dev)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
P.search_device(idx, Q, cfg.topn)
P.set_profiling(True)
t = []
for _ in range(a.iters):
    flush.add_(1.0)
    torch.cuda.synchronize()
    P.search_device(idx, Q, cfg.topn)
    t.append(P.last_timings())
print(os.environ.get("PCPQG_LIB", "current"), "lut/scan/merge ms",
      [round(statistics.median(x[i] for x in t), 3) for i in range(3)])
