"""C3 small-batch search, whole call timed by events (no profiling): PDL and
the one-shot merge on/off."""
import os, sys, statistics
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_2112_02179_b200 as P
from paper_2112_02179_b200 import datagen
cfgname = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = datagen.CONFIGS[cfgname]
dev = torch.device("cuda:0")
data = datagen.synth_index(cfg, seed=1, device=dev)
idx = P.deserialize(data, device=0)
del data
Q = datagen.queries(cfg, 8, seed=2, device=dev)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
nit = int(os.environ.get("NIT", "30"))
code_bytes = idx.n_local * idx.bytes_per_point
for pdl, one, lf in ((0, 0, 0), (1, 1, 0), (1, 1, 1)):
    P.set_option("scan_lut_fused", lf)
    P.set_option("pdl", pdl)
    P.set_option("merge_oneshot", one)
    for bs in (1, 2, 4):
        qs = Q[:bs].contiguous()
        for _ in range(3):
            P.search_device(idx, qs, cfg.topn)
        tt = []
        for _ in range(nit):
            flush.add_(1.0)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            P.search_device(idx, qs, cfg.topn)
            e1.record()
            torch.cuda.synchronize()
            tt.append(e0.elapsed_time(e1))
        t = statistics.median(tt)
        print(f"pdl {pdl} oneshot {one} lutfused {lf} B {bs}: whole search {t*1e3:.1f} us = {code_bytes/(t*1e-3)/1e9:.0f} GB/s", flush=True)
P.set_option("pdl", 1)
P.set_option("merge_oneshot", 1)
