"""Stage split of the C3 small-batch search: whole search timed by events vs the library's per-stage events."""
import os, sys, statistics
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_2112_02179_b200 as P
from paper_2112_02179_b200 import datagen
cfg = datagen.CONFIGS["c3"]
dev = torch.device("cuda:0")
data = datagen.synth_index(cfg, seed=1, device=dev)
idx = P.deserialize(data, device=0)
del data
Q = datagen.queries(cfg, 8, seed=2, device=dev)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
nit = int(os.environ.get("NIT", "20"))
for bs in (1, 2, 4):
    qs = Q[:bs].contiguous()
    for _ in range(3): P.search_device(idx, qs, cfg.topn)
    tt = []
    for _ in range(nit):
        flush.add_(1.0)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); P.search_device(idx, qs, cfg.topn); e1.record(); torch.cuda.synchronize()
        tt.append(e0.elapsed_time(e1))
    P.set_profiling(True)
    st = []
    for _ in range(nit):
        flush.add_(1.0); torch.cuda.synchronize()
        P.search_device(idx, qs, cfg.topn); st.append(P.last_timings())
    P.set_profiling(False)
    print("B", bs, "whole (events, no profiling) ms", round(statistics.median(tt), 4),
          "stages lut/scan/merge", [round(statistics.median(x[i] for x in st), 4) for i in range(3)])
