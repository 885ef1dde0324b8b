"""Minimal driver for ncu: build a config-shaped index, run `--iters` fused
searches of `--batch` queries (after one warm-up search)."""
import argparse, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2112_02179_b200 as P
from paper_2112_02179_b200 import datagen

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--iters", type=int, default=1)
ap.add_argument("--topn", type=int, default=0)
a = ap.parse_args()
cfg = datagen.CONFIGS[a.config]
data = datagen.synth_index(cfg, seed=1, n=a.n or cfg.n, device=torch.device("cuda:0"))
B = a.batch or cfg.batch
Q = datagen.queries(cfg, B, seed=2, device=torch.device("cuda:0"), mixture_seed=1)
idx = P.deserialize(data, device=0)
topn = a.topn or cfg.topn
P.search_device(idx, Q, topn)
torch.cuda.synchronize()
P.set_profiling(True)
for _ in range(a.iters):
    P.search_device(idx, Q, topn)
    print("lut/scan/merge ms", P.last_timings())
torch.cuda.synchronize()
