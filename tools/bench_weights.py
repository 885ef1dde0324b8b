"""Anisotropic weights: the GPU kernel (pcpqg_aniso_weights_gpu)
against the host-thread path (pcpqg_aniso_weights) on config-5-shaped rows
(unit vectors of d = 128 cut into 32 sections of 4, t = 0.2).  One JSON line.

    python tools/bench_weights.py [--rows 4000000] [--host-rows 200000]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_02179_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=4_000_000)
ap.add_argument("--host-rows", type=int, default=200_000)
a = ap.parse_args()
rng = np.random.default_rng(1)
x = rng.standard_normal((a.rows // 32, 128)).astype(np.float32)
x /= np.linalg.norm(x, axis=1, keepdims=True)
rows = np.ascontiguousarray(x.reshape(-1, 4))
P.aniso_weights(rows[:1000], 0.2, device=0)  # self-check + context
t0 = time.perf_counter()
g = P.aniso_weights(rows, 0.2, device=0)
tg = time.perf_counter() - t0
t0 = time.perf_counter()
h = P.aniso_weights(rows[:a.host_rows], 0.2)
th = time.perf_counter() - t0
same = g[0][:a.host_rows].tobytes() == h[0].tobytes() and g[1][:a.host_rows].tobytes() == h[1].tobytes()
print(json.dumps({"workload": f"aniso_weights: {rows.shape[0]} rows of dbar 4, t 0.2 (2 x 1025 sin per row)",
                  "gpu_wall_s": tg, "gpu_rows_per_s": rows.shape[0] / tg, "gpu_sin_per_s": rows.shape[0] * 1025 / tg,
                  "host_rows": a.host_rows, "host_threads": os.cpu_count(), "host_wall_s": th,
                  "host_rows_per_s": a.host_rows / th, "speedup": (rows.shape[0] / tg) / (a.host_rows / th),
                  "bit_identical": bool(same)}), flush=True)
