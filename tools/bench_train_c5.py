"""Config 5 (encode/train) end to end on one GPU: build_pq_index(apcpq,
m = 32, k = 16, s = 16, t_frac = 0.2, 10 iterations, seed 7) of the first n
points of config 5's data with the repo's GPU trainer (real anisotropic
weights, k-means++-seeded and Lloyd-trained centers, the score-aware scale
quantizer) — the index the reference builds with pcpq::build_pq_index
(proj/core/src/pq_index.cpp:62-168; the Lloyd loop of
proj/core/src/clustering.cpp:624-733).  At n = 1e6 (and 20K) the image's
SHA-256 is checked against tests/golden/c5_*_ref.json, made by the
unmodified reference.  Prints one JSON line with the phase split.

    python tools/bench_train_c5.py [--n 1000000]
"""
import argparse
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2112_02179_b200 as P  # noqa: E402
from tests.golden.make_c5_ref import PARAMS, data  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--devices", type=str, default="0", help="comma list, e.g. 0,1,2,3 (sections are dealt round-robin)")
a = ap.parse_args()
x = data(a.n)
cfg = P.PQConfig(method=PARAMS["method"], quantize_scalars=PARAMS["quantize"], m=PARAMS["m"], k=PARAMS["k"],
                 s=PARAMS["s"], t_frac=PARAMS["t_frac"], max_iters=PARAMS["max_iters"], seed=PARAMS["seed"])
t0 = time.perf_counter()
devs = [int(v) for v in a.devices.split(",")]
img = P.build_pq_index(x, cfg, device=devs)
wall = time.perf_counter() - t0
ph = P.train_phases()
sha = hashlib.sha256(img).hexdigest()
golden = {1_000_000: "c5_1m_ref.json"}.get(a.n, f"c5_{a.n}_ref.json")
gpath = os.path.join(ROOT, "tests", "golden", golden)
ref = None
if os.path.exists(gpath):
    with open(gpath) as f:
        g = json.load(f)
    ref = {"sha256_match": g["sha256"] == sha, "reference_build_s": g.get("reference_build_s"),
           "speedup_vs_1thread_reference": (g.get("reference_build_s") or 0) / wall}
print(json.dumps({"workload": f"c5 apcpq build: n={a.n} d=128 m=32 k=16 s=16 t_frac=0.2 iters=10",
                  "devices": devs, "weights_on_gpu": P.train_weights_on_gpu(), "wall_s": wall, "phases_s": ph, "point_sections_per_s": a.n * 32 / wall,
                  "image_bytes": len(img), "sha256": sha, "reference": ref}), flush=True)
