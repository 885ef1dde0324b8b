"""K2-T diagnostics on a config workload: stage times and list statistics."""
import argparse
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2112_02179_b200 as P
from paper_2112_02179_b200 import datagen

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--cpu-data", action="store_true")
ap.add_argument("--seed-target", type=int, default=16)
args = ap.parse_args()
cfg = datagen.CONFIGS[args.config]
n = args.n or cfg.n
B = args.batch or cfg.batch
dev = "cpu" if args.cpu_data else "cuda"
data = datagen.synth_index(cfg, seed=1, n=n, device=dev)
Q = datagen.queries(cfg, B, seed=2, device=dev).contiguous().cuda()
idx = P.deserialize(data, device=0)
print("plan", P.plan_info(idx, B, cfg.topn), flush=True)
P.set_option("scan_tc_seed", args.seed_target)
P.set_option("scan_tc_diag", 1)
P.search_device(idx, Q, cfg.topn)
P.set_option("scan_tc_diag", 0)
P.set_profiling(True)
for _ in range(args.reps):
    P.search_device(idx, Q, cfg.topn)
    torch.cuda.synchronize()
    print("stages ms (prep, filter, finish):", P.last_timings(), flush=True)
