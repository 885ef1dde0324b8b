"""IVF query throughput: the batched GPU query_ivf
(pcpqg_ivf_query_device) against the reference's own query_ivf
(oracle/_ref, proj/core/src/ivf.cpp:89-153) on all host cores, on a seeded
synthetic PCPQIVF1 container (datagen.synth_ivf: Zipf-skewed cells, raw
singleton cells, per-cell PQ over residuals).  Prints one JSON line.

  device  queries/s with queries and results resident in HBM (CUDA events)
  e2e     queries/s through the host API (H2D queries, D2H ids + scores)
  ref     queries/s of the reference on a bounded query sample, all cores
The GPU results on the reference's sample are checked bit-for-bit."""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2112_02179_b200 as P  # noqa: E402
from paper_2112_02179_b200 import datagen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_183_514)
ap.add_argument("--d", type=int, default=100)
ap.add_argument("--kbar", type=int, default=1024)
ap.add_argument("--m", type=int, default=50)
ap.add_argument("--k", type=int, default=16)
ap.add_argument("--s", type=int, default=8)
ap.add_argument("--method", default="apcpq")
ap.add_argument("--kprobe", type=int, default=64)
ap.add_argument("--topn", type=int, default=100)
ap.add_argument("--batch", type=int, default=1000)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--ref-sample", type=int, default=200)
ap.add_argument("--seed", type=int, default=1)
a = ap.parse_args()

dev = torch.device("cuda:0")
t0 = time.time()
data = datagen.synth_ivf(a.n, a.d, a.kbar, a.m, a.k, a.s, seed=a.seed, method=a.method)
t_gen = time.time() - t0
t0 = time.time()
iv = P.deserialize_ivf(data)
t_load = time.time() - t0
g = torch.Generator().manual_seed(a.seed + 1)
Qh = torch.randn(a.batch, a.d, generator=g).float()
Q = Qh.to(dev)

# device-resident
for _ in range(2):
    P.query_ivf_device(iv, Q, a.kprobe, a.topn)
torch.cuda.synchronize()
ms = []
for _ in range(a.iters):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ids_d, sc_d, cnt_d, _, _ = P.query_ivf_device(iv, Q, a.kprobe, a.topn)
    e1.record()
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
dev_ms = statistics.median(ms)
P.set_profiling(True)
P.query_ivf_device(iv, Q, a.kprobe, a.topn)
stages = P.last_timings()  # probe selection / scoring / top-n, ms
P.set_profiling(False)

# end to end through the host API
Qn = Qh.numpy()
P.query_ivf_batch(iv, Qn, a.kprobe, a.topn)
e2e = []
for _ in range(a.iters):
    t0 = time.perf_counter()
    r = P.query_ivf_batch(iv, Qn, a.kprobe, a.topn)
    e2e.append((time.perf_counter() - t0) * 1e3)
e2e_ms = statistics.median(e2e)
out = {"metric": "ivf_queries_per_s", "config": {"n": a.n, "d": a.d, "kbar": a.kbar, "m": a.m, "k": a.k,
                                                 "s": a.s, "method": a.method, "k_probe": a.kprobe,
                                                 "topn": a.topn, "batch": a.batch},
       "container_bytes": len(data), "device_code_bytes": iv.code_bytes, "raw_cells": iv.n_raw_cells,
       "gen_s": round(t_gen, 2), "load_s": round(t_load, 3),
       "device": {"ms_per_batch": dev_ms, "queries_per_s": a.batch / (dev_ms * 1e-3),
                  "stage_ms": {"probes": stages[0], "score": stages[1], "select": stages[2]}},
       "e2e": {"ms_per_batch": e2e_ms, "queries_per_s": a.batch / (e2e_ms * 1e-3)}}

try:
    from oracle.oracle import Ref
    if Ref.available():
        R = Ref()
        h = R.ivf_open(data)
        ns = min(a.ref_sample, a.batch)
        thr = os.cpu_count() or 1
        R.ivf_query_h(h, Qn[:min(ns, 8)], a.kprobe, a.topn, threads=thr)
        t0 = time.perf_counter()
        rid, rsc = R.ivf_query_h(h, Qn[:ns], a.kprobe, a.topn, threads=thr)
        dt = time.perf_counter() - t0
        R.ivf_close(h)
        same_ids = bool(np.array_equal(rid, r["ids"][:ns]))
        same_sc = bool(np.array_equal(np.nan_to_num(rsc, nan=7.0), np.nan_to_num(r["scores"][:ns], nan=7.0)))
        out["reference"] = {"queries_per_s": ns / dt, "threads": thr, "sample": ns, "kind": "reference",
                            "parity_ids": same_ids, "parity_scores": same_sc}
        out["speedup_e2e_vs_reference"] = out["e2e"]["queries_per_s"] / out["reference"]["queries_per_s"]
except Exception as e:  # keep the GPU line
    out["reference"] = {"unavailable": str(e)}
print(json.dumps(out))
