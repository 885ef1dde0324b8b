"""Config-5 encode/train reference (VERDICT r01 'next' 1): the unmodified
reference trainer (oracle/_ref: pcpq::build_pq_index + serialize,
proj/core/src/pq_index.cpp:62-168, :372-407; the score-aware Lloyd loop of
proj/core/src/clustering.cpp:624-733) builds the apcpq index of config 5's
data — the first 1e6 points of the seeded config-3/5 mixture (d = 128,
4096 components; datagen.mixture_chunk(seed 5)) — with m = 32, k = 16,
s = 16, t_frac = 0.2, 10 iterations, seed 7 (BASELINE.json config 5 leaves s
and t unspecified; SURVEY §8(d) C5 fixes them so).  The image is 64 MB, so
only its SHA-256, size and every 9973rd code row are committed
(tests/golden/c5_1m_ref.json); tests/test_gpu_scale.py trains the same data
with the repo's GPU trainer and must reproduce the hash.

    python tests/golden/make_c5_ref.py [n]      (~40 min single-threaded)
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2112_02179_b200 import datagen, pcpqidx  # noqa: E402
from oracle.oracle import Ref  # noqa: E402

PARAMS = dict(method="apcpq", quantize=True, m=32, k=16, s=16, t_frac=0.2, max_iters=10, seed=7)


def data(n: int) -> np.ndarray:
    cfg = datagen.CONFIGS["c3"]
    centers, w = datagen.mixture_params(cfg, 5)
    return datagen.mixture_chunk(cfg, centers, w, 0, n, 5).numpy()


def summary(img: bytes, n: int) -> dict:
    ix = pcpqidx.deserialize(img)
    rows = list(range(0, n, 9973))
    return {"n": n, "d": 128, "params": PARAMS, "data": "datagen.CONFIGS['c3'] mixture, seed 5, points [0, n)",
            "bytes": len(img), "sha256": hashlib.sha256(img).hexdigest(),
            "sample_rows": rows,
            "center_codes": ix.center_codes[rows].tolist(), "scale_codes": ix.scalar_codes[rows].tolist()}


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    x = data(n)
    t0 = time.time()
    img = Ref().build_index(x, **PARAMS)
    out = summary(img, n)
    out["reference_build_s"] = time.time() - t0
    name = "c5_1m_ref.json" if n == 1_000_000 else f"c5_{n}_ref.json"
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), name), "w") as f:
        json.dump(out, f)
    print(name, out["sha256"], out["reference_build_s"])
