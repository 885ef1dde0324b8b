"""A/B of one library option on a config workload (stage times + result equality):
    python tools/ab_opt.py <option> <config> [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2112_02179_b200 as P
from paper_2112_02179_b200 import datagen
opt = sys.argv[1]
cfg = datagen.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "c2"]
n = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.n
data = datagen.synth_index(cfg, seed=1, n=n, device="cuda")
Q = datagen.queries(cfg, cfg.batch, seed=2, device="cuda", mixture_seed=1).contiguous()
idx = P.deserialize(data, device=0)
del data
P.set_profiling(True)
res = {}
for v in (0, 1, 0, 1):
    P.set_option(opt, v)
    P.set_option("scan_tc_diag", 1)
    P.search_device(idx, Q, cfg.topn)
    P.set_option("scan_tc_diag", 0)
    for _ in range(3):
        ids, sc, _ = P.search_device(idx, Q, cfg.topn)
        torch.cuda.synchronize()
    print(opt, v, "stages ms (prep, filter, finish):", P.last_timings(), flush=True)
    res[v] = (ids.clone(), sc.clone())
print("equal:", bool(torch.equal(res[0][0], res[1][0]) and torch.equal(res[0][1], res[1][1])))
P.set_option(opt, 1)
