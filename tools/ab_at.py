"""K2-T: query operand in shared memory vs TMEM (option scan_tc_at) on a long-K config."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2112_02179_b200 as P
from paper_2112_02179_b200 import datagen
cfg = datagen.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n
data = datagen.synth_index(cfg, seed=1, n=n, device="cuda")
Q = datagen.queries(cfg, cfg.batch, seed=2, device="cuda", mixture_seed=1).contiguous()
idx = P.deserialize(data, device=0)
del data
P.set_profiling(True)
res = {}
for at in (0, 1, 0, 1):
    P.set_option("scan_tc_at", at)
    for _ in range(3):
        ids, sc, _ = P.search_device(idx, Q, cfg.topn)
        torch.cuda.synchronize()
    print("at", at, "plan", P.plan_info(idx, cfg.batch, cfg.topn), "stages ms (prep, filter, finish):", P.last_timings(), flush=True)
    res[at] = (ids.clone(), sc.clone())
print("equal:", bool(torch.equal(res[0][0], res[1][0]) and torch.equal(res[0][1], res[1][1])))
P.set_option("scan_tc_at", 1)
