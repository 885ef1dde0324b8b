"""Exact ground truth throughput: pcpqg_brute_force_topn
(device arrays, CUDA events) vs the reference's brute_force_topn
(oracle/_ref, proj/core/src/eval.cpp:36-49) on all host cores over a bounded
query sample; C2-shaped synthetic data (config 2 mixture).  One JSON line."""
import argparse, json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2112_02179_b200 as P
from paper_2112_02179_b200 import datagen

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--batch", type=int, default=1000)
ap.add_argument("--topn", type=int, default=100)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--ref-sample", type=int, default=16)
a = ap.parse_args()
cfg = datagen.CONFIGS[a.config]
n = a.n or cfg.n
dev = torch.device("cuda:0")
X = datagen.mixture_chunk(cfg, *datagen.mixture_params(cfg, 1, dev), 0, n, 1, dev).float().contiguous()
Q = datagen.queries(cfg, a.batch, seed=2, device=dev).contiguous()
P.brute_force_topn_device(X, Q[:8], a.topn)
torch.cuda.synchronize()
ms = []
for _ in range(a.iters):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ids, sc = P.brute_force_topn_device(X, Q, a.topn)
    e1.record()
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
t = statistics.median(ms)
out = {"metric": "exact ground-truth queries/s", "config": {"workload": f"{cfg.name} data n={n} d={cfg.d}",
       "batch": a.batch, "topn": a.topn}, "ms_per_batch": t, "queries_per_s": a.batch / (t * 1e-3),
       "dot_products_per_s": a.batch * n / (t * 1e-3)}
try:
    from oracle.oracle import Ref
    if Ref.available():
        R = Ref()
        Xh, Qh = X.cpu().numpy(), Q[: a.ref_sample].cpu().numpy()
        thr = os.cpu_count() or 1
        t0 = time.perf_counter()
        rid, rsc = R.brute_force_topn(Xh, Qh, a.topn, threads=thr)
        dt = time.perf_counter() - t0
        out["reference"] = {"queries_per_s": a.ref_sample / dt, "threads": thr, "sample": a.ref_sample,
                            "parity_ids": bool(np.array_equal(rid, ids[: a.ref_sample].cpu().numpy())),
                            "parity_scores": bool(np.array_equal(rsc, sc[: a.ref_sample].cpu().numpy()))}
        out["speedup_vs_reference"] = out["queries_per_s"] / out["reference"]["queries_per_s"]
except Exception as e:
    out["reference"] = {"unavailable": str(e)}
print(json.dumps(out))
