"""C4 at n = 1e8 on one GPU: K2-T stage times for several seed caps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2112_02179_b200 as P
from paper_2112_02179_b200 import datagen
cfg = datagen.CONFIGS["c4"]
data = datagen.synth_image(cfg, seed=1, device="cuda")
Q = datagen.queries(cfg, cfg.batch, seed=2, device="cuda").contiguous()
idx = P.deserialize(data, device=0, ingest="gpu")
del data
torch.cuda.empty_cache()
P.set_profiling(True)
for cap in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "8388608,1048576,262144").split(",")]:
    P.set_option("scan_tc_seed_max", cap)
    for _ in range(3):
        P.search_device(idx, Q, cfg.topn)
        torch.cuda.synchronize()
    t = P.last_timings()
    print("seed cap", cap, "stages ms (prep+seed, filter, finish):", t, "total", sum(t), flush=True)
