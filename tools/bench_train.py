"""Index build time: the GPU trainer
(build_pq_index -> pcpqg_train_*) vs the reference's build_pq_index
(oracle/_ref, one thread, as the reference runs) on C2-shaped synthetic data;
the two images must be byte-identical.  One JSON line with the GPU trainer's
phase split (prep incl. weights, Lloyd, scales, serialize)."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2112_02179_b200 as P
from paper_2112_02179_b200 import datagen

ap = argparse.ArgumentParser()
ap.add_argument("--method", default="kmeans")
ap.add_argument("--quantize", action="store_true")
ap.add_argument("--n", type=int, default=200_000)
ap.add_argument("--m", type=int, default=50)
ap.add_argument("--k", type=int, default=16)
ap.add_argument("--s", type=int, default=8)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--no-ref", action="store_true")
a = ap.parse_args()
cfg = datagen.CONFIGS["c2"]
X = datagen.mixture_chunk(cfg, *datagen.mixture_params(cfg, 1), 0, a.n, 1).numpy()
s = a.s if a.method in ("pcpq", "apcpq") else 1
pc = P.PQConfig(method=a.method, quantize_scalars=a.quantize, m=a.m, k=a.k, s=s, max_iters=a.iters, seed=7)
P.build_pq_index(X[:2000], P.PQConfig(method=a.method, quantize_scalars=a.quantize, m=a.m, k=a.k, s=s,
                                      max_iters=2, seed=7))  # warm-up
t0 = time.perf_counter()
img = P.build_pq_index(X, pc)
tg = time.perf_counter() - t0
out = {"metric": f"{a.method} index build seconds", "config": {"n": a.n, "d": cfg.d, "m": a.m, "k": a.k, "s": s,
       "quantize": a.quantize, "max_iters": a.iters, "data": "c2 mixture (synthetic)"}, "gpu_s": tg,
       "gpu_phases_s": P.train_phases(), "host_threads": os.cpu_count(), "image_bytes": len(img)}
if not a.no_ref:
    from oracle.oracle import Ref
    if Ref.available():
        t0 = time.perf_counter()
        ref = Ref().build_index(X, method=a.method, quantize=a.quantize, m=a.m, k=a.k, s=s, t_frac=0.2,
                                max_iters=a.iters, tol=1e-6, seed=7)
        tr = time.perf_counter() - t0
        out["reference"] = {"s": tr, "threads": 1, "kind": "reference"}
        out["identical_image"] = img == ref
        out["speedup"] = tr / tg
print(json.dumps(out))
