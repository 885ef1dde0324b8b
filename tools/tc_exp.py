"""K2-T limiter experiments (results are wrong by design): filter time with
the epilogue reduced to wait+release (exp 1) and without candidate appends
(exp 2), against the full kernel."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2112_02179_b200 as P
from paper_2112_02179_b200 import datagen

cfg = datagen.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n
data = datagen.synth_index(cfg, seed=1, n=n, device="cuda")
Q = datagen.queries(cfg, cfg.batch, seed=2, device="cuda").contiguous()
idx = P.deserialize(data, device=0)
P.set_profiling(True)
for exp in [int(v) for v in os.environ.get('EXPS', '0,1,2,3,4,0').split(',')]:
    P.set_option("scan_tc_exp", exp)
    for _ in range(3):
        P.search_device(idx, Q, cfg.topn)
        torch.cuda.synchronize()
    print("exp", exp, "stages ms (prep, filter, finish):", P.last_timings(), flush=True)
P.set_option("scan_tc_exp", 0)
