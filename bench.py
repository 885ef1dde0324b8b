#!/usr/bin/env python3
"""Benchmark of the PCPQ query-time scoring path (BASELINE.json metric:
scored query x point pairs/s for LUT build + fused scan + top-k).

Workload (BASELINE.json configs[1], "c2"): n = 1,183,514 points, d = 100,
m = 50 sections, k = 16 centers, s = 8 alpha levels (4-bit center | 3-bit
alpha per byte), batch of 10,000 queries, top-100.  Seeded synthetic mixture
(1000 Gaussians, Zipf(1.1) weights, std 0.25, unit-normalised) stands in for
the paper's Glove-100-shaped data; the index is synthesised deterministically
(paper_2112_02179_b200/datagen.py) and both arms read the same PCPQIDX1 bytes.

One step = one full batch: LUT build + fused scan/top-n + merge (+ NCCL
all-gather and merge of per-shard lists when N > 1, points sharded by rank).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c2] [--batch B]

Output: one JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2112_02179_b200 import datagen  # noqa: E402

L2_BYTES = 126 * 1024 * 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=list(datagen.CONFIGS) + ["c5"],
                    help="c5: the encode/train config (one apcpq build per step; --n to shrink it)")
    ap.add_argument("--batch", type=int, default=0, help="override the config's query batch")
    ap.add_argument("--n", type=int, default=0, help="override the config's point count")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--index", default="synth", choices=["synth", "trained"],
                    help="synth: the deterministic index of datagen.synth_image (both arms read the same bytes); "
                         "trained: the config's index built by the repo's byte-identical GPU trainer "
                         "(ours arm, N = 1, configs the trainer can build: c1, c2)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--stream-batches", default="1,2,4",
                    help="extra small-batch (HBM streaming) measurements, '' to skip")
    ap.add_argument("--stream-config", default="c3",
                    help="config whose code stream (> L2) is scanned at the stream batches, '' to skip")
    return ap.parse_args()


L2_NOTE = ("GPU arm: L2 flushed between steps (256 MiB write outside the timed events); "
           "reference arm: CPU run on the host cores")


def config_of(cfg, n, B):
    """The `config` object, identical in both arms (arm-specific facts go to `detail`)."""
    return {"workload": f"{cfg.name}: n={n} d={cfg.d} m={cfg.m} k={cfg.k} s={cfg.s} B={B} top{cfg.topn}",
            "global_batch": B, "l2": L2_NOTE}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(cfg, args, device=None, rows=None):
    """The config's PCPQIDX1 image (uint8 array; rows=(b, e): a part image
    with only those rows, built by this rank alone) and its query batch."""
    n = args.n or cfg.n
    B = args.batch or cfg.batch
    # large synthetic indexes (config 3/4 scale) are generated on the GPU; the
    # mixture is seeded per row chunk, so a part's rows equal the full image's
    dev = device or ("cuda" if torch.cuda.is_available() and n * cfg.m > 10 ** 8 else "cpu")
    if getattr(args, "index", "synth") == "trained" and rows is None and args.impl == "ours":
        # the configured index itself: the reference's trainer restated on the GPU
        # (byte-identical images, tests/test_gpu_train.py, tests/test_gpu_scale.py)
        import paper_2112_02179_b200 as P
        centers, w = datagen.mixture_params(cfg, args.seed)
        X = datagen.mixture_chunk(cfg, centers, w, 0, n, args.seed).numpy()
        t0 = time.perf_counter()
        img = P.build_pq_index(X, P.PQConfig(method=cfg.method, quantize_scalars=cfg.s > 0, m=cfg.m, k=cfg.k,
                                             s=max(cfg.s, 1), t_frac=cfg.t_frac, max_iters=20, seed=args.seed))
        args.train_s = time.perf_counter() - t0
        data = np.frombuffer(img, dtype=np.uint8)
        Q = datagen.queries(cfg, B, seed=args.seed + 1, device="cpu", mixture_seed=args.seed).cpu().numpy()
        return data, Q, n, B
    data = datagen.synth_image(cfg, seed=args.seed, n=n, device=dev, rows=rows)
    # queries from the same mixture as the points (config 2: "drawn from the same mixture")
    Q = datagen.queries(cfg, B, seed=args.seed + 1, device=dev, mixture_seed=args.seed).cpu().numpy()
    return data, Q, n, B


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: an NVML
    thread (every ~2 ms; the timed region of a few batches lasts tens of
    milliseconds, shorter than nvidia-smi's loop period), nvidia-smi -lms as the
    fallback when pynvml is not importable."""

    BITS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []          # (sm_mhz, reasons bitmask)
        self.smax = None
        self.stop = threading.Event()
        self.thread = None
        self.f = None
        self.p = None
        try:
            import pynvml
            pynvml.nvmlInit()
            # LOCAL_RANK indexes the visible devices: map through CUDA_VISIBLE_DEVICES when it lists ordinals
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            phys = gpu
            if vis and all(v.strip().isdigit() for v in vis.split(",")) and gpu < len(vis.split(",")):
                phys = int(vis.split(",")[gpu])
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            self.smax = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self.nv = None

    def _loop(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                try:
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.rows.append((float(mhz), int(rs)))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv is not None:
            self.thread = threading.Thread(target=self._loop, daemon=True)
            self.thread.start()
            return self
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "20"], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.thread:
            self.stop.set()
            self.thread.join(timeout=2)
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        if self.nv is not None:
            if not self.rows:
                return {"sm_mhz": None, "sm_max_mhz": self.smax, "reasons": ["unsampled"]}
            reasons = sorted({n for _, rs in self.rows for n in names if rs & self.BITS[n]})
            return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": self.smax,
                    "reasons": reasons, "samples": len(self.rows), "source": "nvml"}
        rows = []
        if self.f:
            self.f.flush()
            with open(self.f.name) as fh:
                for line in fh:
                    parts = [x.strip() for x in line.split(",")]
                    if len(parts) >= 8:
                        rows.append(parts)
            os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        smax = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows), "source": "nvidia-smi"}


def _ref_index(data):
    from oracle.oracle import Port, Ref
    kind = "reference" if Ref.available() else "port"
    return kind, (Ref().open(data) if kind == "reference" else Port().parse(data))


def _time_sample(ix, Q, topn, threads, budget_s):
    """Time the reference's score_query + partial_sort loop
    (proj/tools/main.cpp:229-243) on `threads` host threads over the largest
    query prefix that fits `budget_s` (a multiple of the thread count)."""
    t0 = time.perf_counter()
    ix.search(Q[:1], topn, threads=1)
    t1 = max(time.perf_counter() - t0, 1e-4)
    S = int(min(len(Q), max(threads, budget_s * threads / t1)))
    S = max(1, (S // threads) * threads) if S >= threads else S
    t0 = time.perf_counter()
    ix.search(Q[:S], topn, threads=threads)
    return S, time.perf_counter() - t0


def cpu_baseline(data, Q, topn, budget_s=15.0, budget_1t=6.0, ix=None):
    """Reference CPU path (oracle/_ref = the unmodified reference library when
    built, else the C restatement) on the host cores, bounded sample; plus the
    literal single-thread loop of proj/tools/main.cpp:230-243."""
    kind, ix = ix if ix is not None else _ref_index(data)
    cores = os.cpu_count() or 1
    S, wall = _time_sample(ix, Q, topn, cores, budget_s)
    n = ix.n
    out = {"value": S * n / wall, "unit": "pairs/s", "cores": cores, "kind": kind,
           "sample": f"{S} of the batch's queries x all {n} points, score_query + partial_sort "
                     f"(proj/tools/main.cpp:229-243) on a {cores}-thread pool, {wall:.2f} s wall",
           "qps": S / wall, "sample_wall_s": wall}
    if budget_1t:
        S1, wall1 = _time_sample(ix, Q, topn, 1, budget_1t)
        out["single_thread"] = {"value": S1 * n / wall1, "unit": "pairs/s", "cores": 1, "kind": kind,
                                "sample": f"{S1} queries x all {n} points, 1 thread, {wall1:.2f} s wall",
                                "qps": S1 / wall1}
    return out


def run_reference(args, cfg):
    """The reference arm: the unmodified reference library (oracle/_ref) on
    the host cores.  Never maps libpcpqg.so (the package API is lazy and only
    its data tools are imported here).  One step = one bounded query sample
    of the workload (the whole batch would take minutes per step on the CPU);
    ms_per_step is that sample's measured wall time."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    data, Q, n, B = workload(cfg, args, device="cpu")
    kind, ix = _ref_index(data)
    cores = os.cpu_count() or 1
    # the step's query sample: a multiple of the thread count worth ~6 s, less when
    # many steps are asked for (the whole run stays within a few minutes)
    per_step = max(1.0, min(6.0, 120.0 / max(1, args.steps + args.warmup)))
    S, _ = _time_sample(ix, Q, cfg.topn, cores, per_step)
    walls, samples = [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        ix.search(Q[:S], cfg.topn, threads=cores)
        wall = time.perf_counter() - t0
        if i >= args.warmup:
            walls.append(wall)
            samples.append(S)
    pairs = sum(samples) * ix.n
    v = pairs / sum(walls)
    S1, wall1 = _time_sample(ix, Q, cfg.topn, 1, 6.0)
    cb = {"value": v, "unit": "pairs/s", "cores": cores, "kind": kind,
          "sample": f"per step {samples[0]} of the batch's {B} queries x all {ix.n} points, score_query + "
                    f"partial_sort (proj/tools/main.cpp:229-243) on a {cores}-thread pool",
          "single_thread": {"value": S1 * ix.n / wall1, "unit": "pairs/s", "cores": 1, "kind": kind,
                            "sample": f"{S1} queries x all {ix.n} points, 1 thread, {wall1:.2f} s wall"}}
    line = {"metric": "scored query x point pairs/s (LUT build + scan + top-k)", "value": v, "unit": "pairs/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": statistics.mean(walls) * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_of(cfg, n, B),
            "detail": {"parallelism": f"{cores} host threads, one query per task",
                       "step": f"{samples[0]} queries (bounded sample of the B={B} batch) x all points"},
            "impl": "reference", "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, cfg):
    import paper_2112_02179_b200 as P
    from paper_2112_02179_b200.sharded import ShardedSearcher
    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        # each rank synthesises and loads only its own rows (a part image)
        from paper_2112_02179_b200.sharded import shard_range
        b, e = shard_range(args.n or cfg.n, rank, world)
        data, Q, n, B = workload(cfg, args, rows=(b, e))
        sh = ShardedSearcher.from_index(P.deserialize_part(data, b, device=local), n, rank, world)
        del data
        data = None
    else:
        data, Q, n, B = workload(cfg, args)
        sh = ShardedSearcher(data, rank, world, device=local)
    topn = cfg.topn
    idx = sh.index
    dQ = torch.from_numpy(Q).to(dev)
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize(dev)

    P.set_profiling(True)
    for _ in range(args.warmup):
        flush.add_(1.0)
        sh.search_device(dQ, topn)
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kt = []
    with ClockSampler(local) as clk:
        barrier()
        for i in range(args.steps):
            flush.add_(1.0)  # > L2: evict the code stream between steps (outside the timed events)
            ev[i][0].record(stream)
            sh.search_device(dQ, topn)
            ev[i][1].record(stream)
            kt.append(P.last_timings())
        barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    dev_ms = sum(step_ms)
    lut_ms = statistics.mean(t[0] for t in kt)
    scan_ms = statistics.mean(t[1] for t in kt)
    merge_ms = statistics.mean(t[2] for t in kt)
    t = torch.tensor([dev_ms, scan_ms], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms, scan_max = float(t[0]), float(t[1])
    ms_per_step = dev_ms / args.steps
    pairs = B * n
    value = pairs / (ms_per_step * 1e-3)

    # ---- end to end through the public API: pinned host queries in, ids/scores out
    Qh = torch.from_numpy(Q).pin_memory()
    ids_h = torch.empty((B, topn), dtype=torch.int32).pin_memory()
    sc_h = torch.empty((B, topn), dtype=torch.float32).pin_memory()
    P.set_profiling(False)
    barrier()
    e2e_ms = []
    for i in range(args.warmup + args.steps):
        flush.add_(1.0)
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        dq = Qh.to(dev, non_blocking=True)
        ids, sc = sh.search_device(dq, topn)
        if rank == 0:
            ids_h.copy_(ids, non_blocking=True)
            sc_h.copy_(sc, non_blocking=True)
        t1.record(stream)
        torch.cuda.synchronize(dev)
        if i >= args.warmup:
            e2e_ms.append(t0.elapsed_time(t1))
    te = torch.tensor([statistics.mean(e2e_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = pairs / (float(te[0]) * 1e-3)

    # ---- small-batch HBM streaming mode (same index, B = 1, 2, 4)
    stream_modes = []
    if args.stream_batches:
        for bs in [int(x) for x in args.stream_batches.split(",") if x]:
            qs = dQ[:bs].contiguous()
            P.set_profiling(True)
            for _ in range(3):
                flush.add_(1.0)
                sh.search_device(qs, topn)
            sm = []
            for _ in range(10):
                flush.add_(1.0)
                torch.cuda.synchronize(dev)
                sh.search_device(qs, topn)
                sm.append(P.last_timings()[1])
            s_ms = statistics.median(sm)
            code_bytes = idx.n_local * idx.bytes_per_point
            stream_modes.append({"batch": bs, "scan_ms": s_ms, "code_GBps": code_bytes / (s_ms * 1e-3) / 1e9})
        P.set_profiling(False)

    # ---- mid-size batches on the same index (K2-T from 8 queries and 8e6 pairs up):
    # the whole search by one event pair, L2 flushed between calls
    mid_batches = []
    if args.stream_batches and rank == 0:
        for bs in (16, 128):
            if bs > dQ.shape[0]:
                continue
            qs = dQ[:bs].contiguous()
            for _ in range(3):
                sh.search_device(qs, topn)
            tt = []
            for _ in range(10):
                flush.add_(1.0)
                torch.cuda.synchronize(dev)
                m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                m0.record()
                sh.search_device(qs, topn)
                m1.record()
                torch.cuda.synchronize(dev)
                tt.append(m0.elapsed_time(m1))
            mid_batches.append({"batch": bs, "search_ms": statistics.median(tt),
                                "path": {0: "cuda-core", 1: "K2-F", 2: "K2-T"}.get(P.plan_info(idx, bs, topn)["filter"])})

    # ---- HBM streaming mode on a config whose code stream exceeds L2 (C3: 800 MB)
    stream_c3 = []
    if args.stream_config and args.stream_batches and rank == 0:
        scfg = datagen.CONFIGS[args.stream_config]
        sdata = datagen.synth_index(scfg, seed=args.seed, device=dev)
        sidx = P.deserialize(sdata, device=local)
        del sdata
        sq = datagen.queries(scfg, 8, seed=args.seed + 1, device=dev)
        code_bytes = sidx.n_local * sidx.bytes_per_point
        for bs in [int(x) for x in args.stream_batches.split(",") if x]:
            qs = sq[:bs].contiguous()
            P.set_profiling(True)
            for _ in range(3):
                P.search_device(sidx, qs, scfg.topn)
            sm, tot = [], []
            for _ in range(10):
                flush.add_(1.0)
                torch.cuda.synchronize(dev)
                P.search_device(sidx, qs, scfg.topn)
                t3 = P.last_timings()
                sm.append(t3[1])
                tot.append(sum(t3))
            s_ms = statistics.median(sm)
            gbps = code_bytes / (s_ms * 1e-3) / 1e9
            # the whole search by ONE event pair around the call, stage events off (they sit
            # between the kernels and serialise the programmatic dependent launches)
            P.set_profiling(False)
            whole = []
            for _ in range(12):
                flush.add_(1.0)
                torch.cuda.synchronize(dev)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                P.search_device(sidx, qs, scfg.topn)
                e1.record(stream)
                torch.cuda.synchronize(dev)
                whole.append(e0.elapsed_time(e1))
            w_ms = statistics.median(whole)
            stream_c3.append({"batch": bs, "scan_ms": s_ms, "search_ms": statistics.median(tot),
                              "search_one_event_pair_ms": w_ms,
                              "search_GBps": code_bytes / (w_ms * 1e-3) / 1e9,
                              "code_bytes": code_bytes, "code_GBps": gbps})
        P.set_profiling(False)
        del sidx

    if rank != 0:
        return
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    peak_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    clocks = clk.summary()
    for r in stream_c3:
        r["hbm_frac"] = r["code_GBps"] / hbm_peak
        r["search_hbm_frac"] = r["search_GBps"] / hbm_peak
    # algorithmic bytes of one scan launch: logical code bytes once per
    # batch + queries + results
    logical_bpp = P.logical_payload_bits(1, idx.m, idx.k, idx.scales) / 8.0
    alg_bytes = idx.n_local * logical_bpp + B * idx.d * 4 + B * topn * 8
    achieved = alg_bytes / (scan_max * 1e-3) / 1e9
    # shared-memory LUT pipe: 32 fp32 lookups / clk / SM
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    f_sm = (clocks.get("sm_mhz") or 1965.0) * 1e6
    lookups = B * idx.n_local * idx.m
    lut_peak = sms * 32 * f_sm
    lut_rate = lookups / (scan_max * 1e-3)
    cb = None
    if not args.no_cpu_baseline and world == 1:
        try:
            cb = cpu_baseline(data, Q, topn)
        except Exception as e:  # keep the GPU line even if the checker is missing
            cb = {"value": None, "unit": "pairs/s", "cores": 0, "kind": "port", "sample": f"unavailable: {e}"}
    plan = P.plan_info(idx, B, topn)
    tc = plan["filter"] == 2  # K2-T: tensor-core pre-score filter + exact re-score
    if tc:
        # prep, seed-pass GEMM, seed select, filter GEMM, exact re-score/top-K, the two
        # parallel-fallback kernels (they return at once when no query needs the exact
        # scan) (+ cross-shard merge)
        launches = 7 + (1 if world > 1 else 0)
    else:
        # lut, [3 filter-table kernels], scan, sorted merge (+ cross-shard merge)
        launches = (3 if world == 1 else 4) + (3 if plan["filter"] else 0)
    # DRAM traffic of the dominant kernel from the committed ncu --set full
    # capture of this workload (profiles/scan_traffic.json)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "scan_traffic.json")) as f:
            tr = json.load(f).get(cfg.name + ("_tscan" if tc else ""))
        if tr:
            traffic = tr["dram_read_bytes"] + tr["dram_write_bytes"]
    except (OSError, ValueError, KeyError):
        pass
    smem_peak = sms * 128 * f_sm / 1e9  # GB/s: 32 banks x 4 B per clock per SM
    # bytes per lookup the scan reads from shared memory: the fp16 pre-score
    # table (K2-F) or the exact fp32 eta table
    lut_bytes = 2 if plan["filter"] else 4
    smem_achieved = lut_rate * lut_bytes / 1e9
    Bp128 = (B + 127) // 128 * 128
    if tc:
        # the filter GEMM: 2*B*n*d algorithmic flops (queries x decoded points,
        # fp16 operands, fp32 accumulation) per launch / its event time
        tflops = 2.0 * B * idx.n_local * idx.d / (scan_max * 1e-3) / 1e12
        tpeak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 2250.0))
        roofline = {"bound": "tensor", "achieved": tflops, "peak": tpeak, "unit": "TFLOP/s",
                    "frac": tflops / tpeak, "traffic": traffic, "kernel": "tscan_kernel (K2-T filter GEMM)",
                    "plan": plan,
                    "note": ("achieved = 2*B*n*d per launch / event-timed filter kernel; peak = MEASURED_PEAKS "
                             "bf16_tflops_sustained (fp16 kind::f16 runs at the bf16 rate); every reported score "
                             "is re-computed exactly in fp32 by the finish kernel"),
                    # the filter's own limiter at small d: every fp32 accumulator is read out of
                    # TMEM once (tcgen05.ld, 64 B/clk/SM): B*n*4 bytes per launch
                    "tmem_view": {"bound": "tmem-read", "achieved": Bp128 * idx.n_local * 4 / (scan_max * 1e-3) / 1e9,
                                  "peak": sms * 64 * f_sm / 1e9, "unit": "GB/s",
                                  "frac": (Bp128 * idx.n_local * 4 / (scan_max * 1e-3)) / (sms * 64 * f_sm),
                                  "note": "accumulator bytes (queries padded to 128) / event-timed filter; peak = SMs x 64 B/clk "
                                          "x sm_mhz (TMEM read path, B300_MICROARCH.md); binds when 2*d*B*n / tensor peak "
                                          "< 4*B*n / TMEM peak, i.e. d < ~190"},
                    "smem_view": {"lookups_per_s": lut_rate, "exact_fp32_lut_ceiling": lut_peak},
                    "hbm_view": {"achieved": achieved, "peak": hbm_peak, "frac": achieved / hbm_peak,
                                 "alg_bytes_per_launch": alg_bytes, "peak_source": peak_src}}
    else:
        roofline = {"bound": "smem", "achieved": smem_achieved, "peak": smem_peak, "unit": "GB/s",
                    "frac": smem_achieved / smem_peak, "traffic": traffic,
                    "kernel": "scan_topk_kernel",
                    "plan": plan,
                    "note": (f"LUT bytes = B*n*m*{lut_bytes} per launch / event-timed scan"
                             + (" (K2-F: fp16 pre-score table; the few pairs that pass are re-scored exactly)"
                                if plan["filter"] else "") + "; peak = SMs x 128 B/clk x sm_mhz"),
                    "hbm_view": {"achieved": achieved, "peak": hbm_peak, "frac": achieved / hbm_peak,
                                 "alg_bytes_per_launch": alg_bytes, "peak_source": peak_src}}
    line = {
        "metric": "scored query x point pairs/s (LUT build + scan + top-k)",
        "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_of(cfg, n, B),
        "detail": {"parallelism": f"points sharded over {world} GPU(s)", "qps": B / (ms_per_step * 1e-3),
                   "index": (f"trained: build_pq_index({cfg.method}, 20 iterations) on the GPU in "
                             f"{getattr(args, 'train_s', 0.0):.1f} s" if args.index == "trained" else
                             "synth: datagen.synth_image"),
                   "stage_ms": ({"prep_and_seed": lut_ms, "filter": scan_ms, "rescore_topk": merge_ms} if tc else
                                {"lut": lut_ms, "scan": scan_ms, "merge": merge_ms})},
        # K2-T: the batch scan is a tensor-core GEMM filter (roofline: tensor);
        # the CUDA-core LUT scans (K2 / K2-F) are bound by shared-memory LUT reads
        # (SURVEY §8(d)); the HBM-bound regime (B = 1) is stream_mode_hbm.
        "roofline": roofline,
        "lut_roofline": {"bound": "smem-lut", "achieved": lut_rate, "peak": lut_peak, "unit": "lookups/s",
                         "frac": lut_rate / lut_peak,
                         "note": f"ceiling of an exact fp32-LUT scan: {sms} SMs x 32 fp32 LDS/clk x sm_mhz"
                                 + (" (K2-F reads 2-byte entries, so it can exceed it)" if plan["filter"] else "")},
        "stream_mode": stream_modes,
        "mid_batch": mid_batches,
        "stream_mode_hbm": {"config": args.stream_config, "peak_GBps": None, "runs": stream_c3},
        "cpu_baseline": cb,
        "e2e": {"value": e2e_value, "unit": "pairs/s", "h2d_bytes_per_step": B * idx.d * 4,
                "d2h_bytes_per_step": B * topn * 8, "ms_per_step": float(te[0])},
        "gpu_launches": launches * args.steps,
        "clocks": clocks,
    }
    line["stream_mode_hbm"]["peak_GBps"] = hbm_peak
    print(json.dumps(line), flush=True)


def run_c5(args):
    """BASELINE.json configs[4]: the anisotropic encode / train path.  One step =
    one build_pq_index(apcpq, m = 32, k = 16, s = 16, t_frac = 0.2, 10 iterations)
    of n = 1e7 x 128 points on the GPU (weights, assignment, ordered Lloyd
    statistics, scale quantizer; the reference's bytes at n = 1e6:
    tests/test_gpu_scale.py).  Host data in, index image out: the timed region is
    the public call."""
    import hashlib
    import paper_2112_02179_b200 as P
    from tests.golden.make_c5_ref import PARAMS, data as c5_data
    rank, world, local = dist_env()
    if rank != 0:
        return
    n = args.n or 10_000_000
    X = c5_data(n)
    devs = list(range(max(1, min(args.gpus, torch.cuda.device_count()))))
    cfg = P.PQConfig(method=PARAMS["method"], quantize_scalars=PARAMS["quantize"], m=PARAMS["m"], k=PARAMS["k"],
                     s=PARAMS["s"], t_frac=PARAMS["t_frac"], max_iters=PARAMS["max_iters"], seed=PARAMS["seed"])
    steps = max(1, min(args.steps, 3))
    walls, ph, img = [], None, b""
    with ClockSampler(0) as clk:
        for i in range(steps):
            t0 = time.perf_counter()
            img = P.build_pq_index(X, cfg, device=devs)
            walls.append(time.perf_counter() - t0)
            ph = P.train_phases()
    wall = statistics.mean(walls)
    line = {"metric": "encoded point-sections/s (apcpq build: assignment + Lloyd updates + scale quantizer)",
            "value": n * PARAMS["m"] / wall, "unit": "point-sections/s", "n_gpus": len(devs), "steps": steps,
            "warmup": 0, "ms_per_step": wall * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"c5: apcpq build n={n} d=128 m=32 k=16 s=16 t_frac=0.2 iters=10",
                       "global_batch": n},
            "detail": {"phases_s": ph, "weights_on_gpu": P.train_weights_on_gpu(), "image_bytes": len(img),
                       "sha256": hashlib.sha256(img).hexdigest(),
                       "parallelism": f"sections dealt to {len(devs)} GPU(s)",
                       "reference": "pcpq::build_pq_index, single-threaded: 2115 s at n = 1e6 "
                                    "(tests/golden/c5_1m_ref.json; same SHA-256 as the GPU build)"},
            "e2e": {"value": n * PARAMS["m"] / wall, "unit": "point-sections/s",
                    "h2d_bytes_per_step": n * 128 * 4, "d2h_bytes_per_step": len(img)},
            "clocks": clk.summary()}
    print(json.dumps(line), flush=True)


def self_launch(args) -> int:
    """`--gpus N` without a torchrun environment: launch N ranks (one per
    GPU, NCCL) on this node the way the driver does, and relay rank 0's line."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.config != "c5":
        if args.impl == "ours" and torch.cuda.device_count() < args.gpus:
            print(json.dumps({"error": f"--gpus {args.gpus} needs {args.gpus} GPUs, "
                                       f"{torch.cuda.device_count()} visible"}), flush=True)
            sys.exit(2)
        sys.exit(self_launch(args))
    if args.config == "c5":
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "config 5 reference build takes hours (2115 s at "
                              "n = 1e6, single-threaded); its image hash is committed in tests/golden/c5_1m_ref.json"}),
                  flush=True)
            return
        run_c5(args)
        return
    cfg = datagen.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)
    rank, world, _ = dist_env()
    if world > 1 and args.impl == "ours":
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
