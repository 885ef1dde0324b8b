"""Index load time: host-threaded parse + repack
(pcpqg_index_load) vs GPU ingest (pcpqg_index_load_gpu) on a config-shaped
image held in host memory, and from a file (pcpqg_index_load_file[_gpu]).
Prints one JSON line; both loads must give identical device code streams."""
import argparse, json, os, sys, tempfile, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2112_02179_b200 as P
from paper_2112_02179_b200 import datagen

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--file", action="store_true")
a = ap.parse_args()
cfg = datagen.CONFIGS[a.config]
data = datagen.synth_index(cfg, seed=1, n=a.n or cfg.n, device=torch.device("cuda:0"))
out = {"metric": "index load GB/s (image bytes / wall time)", "config": {"workload": a.config, "n": a.n or cfg.n},
       "image_bytes": len(data)}
for mode in ("host", "gpu"):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    idx = P.deserialize(data, ingest=mode)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    out[mode] = {"s": dt, "GBps": len(data) / dt / 1e9}
    if mode == "host":
        ref = P.index_codes(idx)
    else:
        out["identical_codes"] = bool(np.array_equal(ref, P.index_codes(idx)))
    del idx
if a.file:
    with tempfile.NamedTemporaryFile(suffix=".idx", delete=False) as f:
        f.write(data)
        path = f.name
    for mode in ("host", "gpu"):
        t0 = time.perf_counter()
        idx = P.read_pq_index(path, ingest=mode)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        out["file_" + mode] = {"s": dt, "GBps": len(data) / dt / 1e9}
        del idx
    os.unlink(path)
out["speedup"] = out["host"]["s"] / out["gpu"]["s"]
print(json.dumps(out))
