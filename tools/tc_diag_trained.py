"""K2-T / K2-F / exact scan on the CONFIGURED index: config 2's data, the index
built by the repo's byte-identical GPU apcpq trainer (not datagen.synth_image);
queries from the same mixture.  Prints the K2-T list statistics and the stage
times of every scan path."""
import argparse
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2112_02179_b200 as P
from paper_2112_02179_b200 import datagen

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--iters", type=int, default=20)
args = ap.parse_args()
cfg = datagen.CONFIGS[args.config]
n = args.n or cfg.n
B = args.batch or cfg.batch
centers, w = datagen.mixture_params(cfg, 1)
X = datagen.mixture_chunk(cfg, centers, w, 0, n, 1).numpy()
t0 = time.perf_counter()
img = P.build_pq_index(X, P.PQConfig(method=cfg.method, quantize_scalars=cfg.s > 0, m=cfg.m, k=cfg.k, s=max(cfg.s, 1),
                                     t_frac=cfg.t_frac, max_iters=args.iters, seed=1))
print("trained in %.1f s" % (time.perf_counter() - t0), P.train_phases(), flush=True)
from paper_2112_02179_b200 import pcpqidx
ix = pcpqidx.deserialize(img)
lam = np.asarray(ix.scalar_codebooks)
print("scale codebooks: |lambda| max per section (first 8)", np.abs(lam).max(axis=1)[:8], "median level", np.median(np.abs(lam)), flush=True)
Q = datagen.queries(cfg, B, seed=2, device="cuda", mixture_seed=1).contiguous()
idx = P.deserialize(np.frombuffer(img, np.uint8), device=0)
print("plan", P.plan_info(idx, B, cfg.topn), flush=True)
P.set_option("scan_tc_diag", 1)
P.search_device(idx, Q, cfg.topn)
P.set_option("scan_tc_diag", 0)
P.set_profiling(True)
for name, opts in (("K2-T", {}), ("K2-F", {"scan_tc": 0}), ("exact", {"scan_tc": 0, "scan_filter": 0})):
    for k, v in opts.items():
        P.set_option(k, v)
    for _ in range(2):
        P.search_device(idx, Q, cfg.topn)
        torch.cuda.synchronize()
    print(name, "stages ms:", P.last_timings(), flush=True)
    P.set_option("scan_tc", 1)
    P.set_option("scan_filter", 1)
