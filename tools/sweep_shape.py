"""Scan-shape sweep for the small-batch HBM streaming mode: for each forced
(threads, ppt, stages) shape, time the scan of `--config` at B = 1, 2, 4
(CUDA events inside the library, median of 10, L2 flushed between runs)."""
import argparse, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2112_02179_b200 as P
from paper_2112_02179_b200 import datagen

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--batches", default="1,2,4")
ap.add_argument("--ws", default="1,0")
ap.add_argument("--shapes", default="0,5120202,5120103,5120104,5120105,2560203,2560204,2560103,2560104,2560106,1280106")
a = ap.parse_args()
cfg = datagen.CONFIGS[a.config]
dev = torch.device("cuda:0")
data = datagen.synth_index(cfg, seed=1, device=dev)
idx = P.deserialize(data, device=0)
del data
Q = datagen.queries(cfg, 8, seed=2, device=dev)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
code_bytes = idx.n_local * idx.bytes_per_point
ref = {}
import itertools
for ws, shape in itertools.product([int(w) for w in a.ws.split(",")], [int(s) for s in a.shapes.split(",")]):
    P.set_option("scan_shape", shape)
    P.set_option("scan_ws", ws)
    for bs in [int(b) for b in a.batches.split(",")]:
        qs = Q[:bs].contiguous()
        try:
            ids, sc = P.search_device(idx, qs, cfg.topn)[:2]
        except P.PcpqError as e:
            print(f"shape {shape} B={bs}: {e}")
            continue
        got = ids.cpu()
        if bs in ref:
            assert torch.equal(ref[bs], got), f"shape {shape} B={bs}: ids differ"
        else:
            ref[bs] = got
        P.set_profiling(True)
        for _ in range(3):
            P.search_device(idx, qs, cfg.topn)
        sm, mg = [], []
        for _ in range(10):
            flush.add_(1.0)
            torch.cuda.synchronize()
            P.search_device(idx, qs, cfg.topn)
            t = P.last_timings()
            sm.append(t[1])
            mg.append(t[2])
        P.set_profiling(False)
        s = statistics.median(sm)
        print(f"ws {ws} shape {shape:>9} B={bs}: scan {s*1e3:8.1f} us  {code_bytes/(s*1e-3)/1e9:7.1f} GB/s  "
              f"merge {statistics.median(mg)*1e3:6.1f} us", flush=True)
P.set_option("scan_shape", 0)
