"""Index build time, method kmeans: the GPU trainer
(pcpqg_train_kmeans) vs the reference's build_pq_index (oracle/_ref, one
thread, as the reference runs) on C2-shaped synthetic data; the two images
must be byte-identical.  One JSON line."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2112_02179_b200 as P
from paper_2112_02179_b200 import datagen

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=200_000)
ap.add_argument("--m", type=int, default=50)
ap.add_argument("--k", type=int, default=16)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--no-ref", action="store_true")
a = ap.parse_args()
cfg = datagen.CONFIGS["c2"]
X = datagen.mixture_chunk(cfg, *datagen.mixture_params(cfg, 1), 0, a.n, 1).numpy()
pc = P.PQConfig(method="kmeans", m=a.m, k=a.k, s=1, max_iters=a.iters, seed=7)
P.build_pq_index(X[:2000], P.PQConfig(method="kmeans", m=a.m, k=a.k, s=1, max_iters=2, seed=7))  # warm-up
t0 = time.perf_counter()
img = P.build_pq_index(X, pc)
tg = time.perf_counter() - t0
out = {"metric": "kmeans index build seconds", "config": {"n": a.n, "d": cfg.d, "m": a.m, "k": a.k,
       "max_iters": a.iters}, "gpu_s": tg, "image_bytes": len(img)}
if not a.no_ref:
    from oracle.oracle import Ref
    if Ref.available():
        t0 = time.perf_counter()
        ref = Ref().build_index(X, method="kmeans", quantize=False, m=a.m, k=a.k, s=1, t_frac=0.2,
                                max_iters=a.iters, tol=1e-6, seed=7)
        tr = time.perf_counter() - t0
        out["reference"] = {"s": tr, "threads": 1, "kind": "reference"}
        out["identical_image"] = img == ref
        out["speedup"] = tr / tg
print(json.dumps(out))
