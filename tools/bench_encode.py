"""Config 5 (encode / Lloyd step) throughput on one GPU: n points, 32
sections of 4 dims, k = 16 centers.  Per Lloyd iteration and section:
anisotropic assignment with the keep-previous fallback, center statistics
(exact member-order sums), and at the end the score-aware alpha codes.
Weights are computed on the device here (timing only; the bit-exact path
feeds the reference's host-computed weights).  Also times the
reference's assign_anisotropic on a bounded CPU sample.  Prints one JSON line."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2112_02179_b200 as P  # noqa: E402
from paper_2112_02179_b200 import datagen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
cfg = datagen.CONFIGS["c3"]  # config 5 uses config 3's data shape (d=128, m=32, k=16)
dev = torch.device("cuda", 0)
m, dbar, k = 32, 4, 16
centers_mix, w = datagen.mixture_params(cfg, 9, dev)
x = datagen.mixture_chunk(cfg, centers_mix, w, 0, a.n, 9, dev)            # (n, 128)
xs = x.view(a.n, m, dbar).permute(1, 0, 2).contiguous()                   # (m, n, dbar)
del x
nrm = xs.double().square().sum(-1).sqrt()
theta = (0.2 / nrm.clamp_min(1e-30)).clamp(max=np.pi / 2)
h_bot = (theta ** 5) / 5.0                                                  # smooth stand-in weights
h_par = torch.maximum(3 * ((theta ** 3) / 3 - h_bot), h_bot)
g = torch.Generator(device=dev)
g.manual_seed(3)
cents = torch.randn(m, k, dbar, generator=g, device=dev)
prev = [None] * m
torch.cuda.synchronize()
times = []
for it in range(a.iters + 1):
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    assigns, alphas = [], []
    for j in range(m):
        aj, alj, _ = P.assign_anisotropic(xs[j], cents[j], h_par[j], h_bot[j], prev=prev[j])
        assigns.append(aj)
        alphas.append(alj)
        prev[j] = aj
    stats = P.center_stats(xs, torch.stack(assigns), torch.stack(alphas), h_par, h_bot, k)
    t1.record()
    torch.cuda.synchronize()
    if it > 0:
        times.append(t0.elapsed_time(t1))
values = torch.linspace(-1, 1, 16, device=dev)
t0 = torch.cuda.Event(enable_timing=True)
t1 = torch.cuda.Event(enable_timing=True)
t0.record()
for j in range(m):
    P.aniso_alpha_codes(xs[j], cents[j], prev[j], h_par[j], h_bot[j], values)
t1.record()
torch.cuda.synchronize()
codes_ms = t0.elapsed_time(t1)
ms = float(np.median(times))
# reference CPU assign on a bounded sample (one section)
ref = None
try:
    from oracle.oracle import Ref
    if Ref.available():
        R = Ref()
        S = 200_000
        xc = xs[0, :S].cpu().numpy()
        t = time.perf_counter()
        R.assign_anisotropic(xc, cents[0].cpu().numpy(), h_par[0, :S].cpu().numpy(), h_bot[0, :S].cpu().numpy())
        el = time.perf_counter() - t
        ref = {"value": S / el, "unit": "point-sections/s", "cores": 1, "kind": "reference",
               "sample": f"assign_anisotropic, {S} points of one section, 1 thread, {el:.2f} s"}
except Exception as e:  # noqa: BLE001
    ref = {"unavailable": str(e)}
print(json.dumps({"metric": "encode Lloyd iteration (assign + center stats), point-sections/s",
                  "config": {"workload": f"c5: n={a.n} d=128 m=32 k=16 (aniso assign w/ prev fallback + stats)"},
                  "ms_per_iteration": ms, "value": a.n * m / (ms * 1e-3), "unit": "point-sections/s",
                  "alpha_codes_ms_all_sections": codes_ms, "cpu_reference": ref}))
