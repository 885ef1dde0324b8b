"""Whole search (one event pair, L2 flushed) across batch sizes: the planner's
CUDA-core paths (K2-T off) against K2-T forced from B = 1 (scan_tc_min_batch), with and
without the decoded operand cache.  python tools/ab_midbatch.py [c3|c2] """
import os, sys, statistics
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_2112_02179_b200 as P
from paper_2112_02179_b200 import datagen
cfgname = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = datagen.CONFIGS[cfgname]
dev = torch.device("cuda:0")
data = datagen.synth_index(cfg, seed=1, device=dev)
Q = datagen.queries(cfg, 512, seed=2, device=dev)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
nit = int(os.environ.get("NIT", "15"))
batches = [int(x) for x in os.environ.get("BATCHES", "1,2,4,8,16,32,64,128,192,256,512").split(",")]
modes = (("cuda-core", 1 << 30, 40), ("tc-cached", 1, 40), ("tc-decode", 1, 0))
if os.environ.get("MODES"):
    modes = tuple(m for m in modes if m[0] in os.environ["MODES"].split(","))
for label, minb, cache in modes:
    P.set_option("scan_tc_min_batch", minb)
    P.set_option("scan_tc_min_work", 0)
    P.set_option("scan_tc_cache_pct", cache)
    idx = P.deserialize(data, device=0)
    for bs in batches:
        qs = Q[:bs].contiguous()
        try:
            plan = P.plan_info(idx, bs, cfg.topn)
            ref = None
            for _ in range(3):
                ref = P.search_device(idx, qs, cfg.topn)
        except Exception as e:  # noqa: BLE001
            print(f"{label} B {bs}: {e}", flush=True)
            continue
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
        print(f"{label} B {bs}: {t*1e3:.1f} us  ({t*1e3/bs:.1f} us/query) filter={plan.get('filter')} nq={plan.get('nq')}", flush=True)
    del idx
    torch.cuda.empty_cache()
