"""Single-query latency through the host API (the reference CLI's per-query
loop, tools/main.cpp:229-243): mean wall time of P.search(idx, q, topn) per
query vs the device time of its LUT + scan + merge."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2112_02179_b200 as P
from paper_2112_02179_b200 import datagen

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--queries", type=int, default=300)
a = ap.parse_args()
cfg = datagen.CONFIGS[a.config]
data = datagen.synth_index(cfg, seed=1)
idx = P.deserialize(data, device=0)
Q = datagen.queries(cfg, a.queries, seed=2).numpy()
for i in range(20):
    P.search(idx, Q[i:i + 1], cfg.topn)
t = time.perf_counter()
for i in range(a.queries):
    P.search(idx, Q[i:i + 1], cfg.topn)
wall = (time.perf_counter() - t) / a.queries
P.set_profiling(True)
dev = []
for i in range(50):
    P.search(idx, Q[i:i + 1], cfg.topn)
    dev.append(sum(P.last_timings()))
P.set_profiling(False)
print(json.dumps({"config": cfg.name, "topn": cfg.topn, "wall_us_per_query": wall * 1e6,
                  "device_us_per_query": float(np.median(dev)) * 1e3}))
