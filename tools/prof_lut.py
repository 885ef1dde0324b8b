"""LUT build at config 4's batch (B=4096, m=64, k=256, dbar=4): exact
CUDA-core kernel vs tcgen05 kernel (option lut_tensor_cores)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2112_02179_b200 as P
from paper_2112_02179_b200 import datagen
cfg = datagen.CONFIGS["c4"]
data = datagen.synth_index(cfg, seed=1, n=int(sys.argv[1]) if len(sys.argv) > 1 else 40000)
Q = datagen.queries(cfg, 4096, seed=2).cuda()
idx = P.deserialize(data, device=0)
P.set_profiling(True)
for tc in (0, 1):
    P.set_option("lut_tensor_cores", tc)
    for it in range(3):
        P.search_device(idx, Q, cfg.topn)
        t = P.last_timings()
    print("tensor_cores" if tc else "exact", "lut/scan/merge ms", t)
