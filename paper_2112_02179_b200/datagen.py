"""Seeded synthetic workloads for the BASELINE.json configs.

The configs' datasets are not in the reference (its generator only has
gaussian | unit_sphere | clustered, proj/core/src/datagen.cpp:55-89) and
Glove-100 / Last.fm are not in this container, so seeded Gaussian mixtures with
the configs' shapes stand in for them.

Index synthesis.  Training a 1e6-1e8 point index with the reference trainer
is infeasible inside a benchmark, and the scoring
path's cost and results do not depend on how the codes were trained — only on
the bytes of the PCPQIDX1 image, which both the GPU path and the CPU
reference read.  ``synth_index`` therefore builds a projective-clustering
index quickly and deterministically: per section, k unit directions from a few
projective Lloyd rounds on a subsample; full-data center codes by projective
assignment (argmax <x_s, c>^2, lowest index on ties), alpha = <x_s, c>; scale
codebooks by 1-D k-means over alpha (s levels, ascending) and nearest-level
codes, or raw alpha rounded to fp16-representable fp32 (config 3, SURVEY.md
Appendix C.1).  The small parity cases in tests/golden use the reference
trainer itself.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import pcpqidx


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    d: int
    components: int
    std: float
    zipf_s: float | None
    m: int
    k: int
    s: int           # 0 = raw alpha
    method: str
    raw_fp16: bool
    batch: int
    topn: int
    queries: str     # "gaussian" (unit) or "mixture"
    t_frac: float = 0.2


CONFIGS = {
    # BASELINE.json configs[0..3]; std of configs 3/4 is unspecified -> 0.3
    "c1": Config("c1", 100_000, 64, 64, 0.3, None, 16, 16, 16, "pcpq", False, 1000, 10, "gaussian"),
    "c2": Config("c2", 1_183_514, 100, 1000, 0.25, 1.1, 50, 16, 8, "apcpq", False, 10_000, 100, "mixture"),
    "c3": Config("c3", 10_000_000, 128, 4096, 0.3, None, 32, 16, 0, "pcpq", True, 1024, 100, "gaussian"),
    "c4": Config("c4", 100_000_000, 256, 16384, 0.3, None, 64, 256, 16, "pcpq", False, 4096, 100, "gaussian"),
}


def _gen(seed: int, device="cpu") -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def mixture_params(cfg: Config, seed: int, device="cpu"):
    g = _gen(seed * 1_000_003 + 17, device)
    centers = torch.randn(cfg.components, cfg.d, generator=g, device=device)
    if cfg.zipf_s is not None:
        w = 1.0 / torch.arange(1, cfg.components + 1, dtype=torch.float64, device=device) ** cfg.zipf_s
    else:
        w = torch.ones(cfg.components, dtype=torch.float64, device=device)
    return centers, w / w.sum()


def mixture_chunk(cfg: Config, centers, weights, start: int, count: int, seed: int, device="cpu"):
    """Points [start, start+count) of the seeded mixture, unit-normalised (fp32)."""
    g = _gen(seed * 7_919 + start, device)
    comp = torch.multinomial(weights, count, replacement=True, generator=g)
    x = centers[comp] + cfg.std * torch.randn(count, cfg.d, generator=g, device=device)
    return x / x.norm(dim=1, keepdim=True).clamp_min(1e-30)


def queries(cfg: Config, B: int, seed: int, device="cpu", mixture_seed=None) -> torch.Tensor:
    """The config's query batch.  "mixture" queries are fresh draws (stream
    `seed`) from the mixture whose parameters come from `mixture_seed` — pass the
    data set's seed to draw them from the SAME mixture as the points (config 2);
    None keeps the historical behaviour (parameters from `seed`)."""
    if cfg.queries == "mixture":
        centers, w = mixture_params(cfg, seed if mixture_seed is None else mixture_seed, device)
        return mixture_chunk(cfg, centers, w, 1 << 40, B, seed + 1, device)
    g = _gen(seed * 31 + 5, device)
    q = torch.randn(B, cfg.d, generator=g, device=device)
    return q / q.norm(dim=1, keepdim=True)


def _train_directions(xs: torch.Tensor, k: int, iters: int, g: torch.Generator) -> torch.Tensor:
    """Projective Lloyd on one section's subsample: unit directions (k, dbar)."""
    n, dbar = xs.shape
    idx = torch.randperm(n, generator=g, device=xs.device)[:k]
    c = xs[idx].clone()
    c = c / c.norm(dim=1, keepdim=True).clamp_min(1e-30)
    for _ in range(iters):
        a = (xs @ c.T).square().argmax(dim=1)
        gram = torch.zeros(k, dbar, dbar, dtype=torch.float64, device=xs.device)
        xd = xs.double()
        gram.index_add_(0, a, xd[:, :, None] * xd[:, None, :])
        evals, evecs = torch.linalg.eigh(gram + 1e-12 * torch.eye(dbar, dtype=torch.float64, device=xs.device))
        new = evecs[:, :, -1].float()
        cnt = torch.bincount(a, minlength=k)
        c = torch.where(cnt[:, None] > 0, new, c)
        c = c / c.norm(dim=1, keepdim=True).clamp_min(1e-30)
    return c


def _kmeans_1d(v: torch.Tensor, s: int, iters: int = 12) -> torch.Tensor:
    qs = torch.linspace(0.5 / s, 1 - 0.5 / s, s, dtype=torch.float64, device=v.device)
    lv = torch.quantile(v.double()[: 1 << 22], qs)
    for _ in range(iters):
        a = (v.double()[:, None] - lv[None, :]).abs().argmin(dim=1)
        sums = torch.zeros(s, dtype=torch.float64, device=v.device).index_add_(0, a, v.double())
        cnt = torch.bincount(a, minlength=s).double()
        lv = torch.where(cnt > 0, sums / cnt.clamp_min(1), lv)
    return torch.sort(lv).values.float()


def synth_image(cfg: Config, seed: int = 1, n: int | None = None, device="cpu", rows: tuple[int, int] | None = None,
                chunk: int = 1 << 20, train_sample: int = 65536, iters: int = 4) -> np.ndarray:
    """Deterministic PCPQIDX1 image of `cfg` as a uint8 array, written row chunk
    by row chunk (no n x m code arrays: config 4's 1e8-point image is 12.8 GB).
    rows=(b, e): a PART image — the header and codebooks of the n-point index
    followed only by rows [b, e) (pcpqg_index_load_part); its rows are the
    same bytes as in the full image."""
    n = cfg.n if n is None else n
    b0, e0 = rows if rows is not None else (0, n)
    m, k, d = cfg.m, cfg.k, cfg.d
    dbar = d // m
    centers, w = mixture_params(cfg, seed, device)
    sample = mixture_chunk(cfg, centers, w, 0, min(n, train_sample), seed, device)
    g = _gen(seed * 101 + 3, device)
    cbs = torch.stack([_train_directions(sample[:, j * dbar:(j + 1) * dbar].contiguous(), k, iters, g)
                       for j in range(m)])                                # (m, k, dbar)
    quant = cfg.s > 0
    if quant:
        # scale codebooks from the subsample's alphas
        lv = []
        for j in range(m):
            xs = sample[:, j * dbar:(j + 1) * dbar]
            ip = xs @ cbs[j].T
            a = ip.square().argmax(dim=1)
            lv.append(_kmeans_1d(ip.gather(1, a[:, None])[:, 0], cfg.s))
        scb = torch.stack(lv)                                              # (m, s)
    head = pcpqidx.header_bytes(pcpqidx.METHODS[cfg.method], n, d, d, m, k, cfg.s, cfg.t_frac,
                                cbs.cpu().numpy(), scb.cpu().numpy() if quant else np.zeros((m, 0), np.float32))
    rdt = pcpqidx.row_dtype(m, k, cfg.s)
    out = np.empty(len(head) + (e0 - b0) * rdt.itemsize, np.uint8)
    out[:len(head)] = np.frombuffer(head, np.uint8)
    body = out[len(head):].view(rdt)
    # the (chunk, m, k) inner-product tensor stays within ~4 GB; the chunk grid
    # is fixed by the config, so a part's rows equal the full image's
    chunk = max(4096, min(chunk, (1 << 30) // (m * k)))
    for start in range((b0 // chunk) * chunk, e0, chunk):
        cnt = min(chunk, n - start)
        x = mixture_chunk(cfg, centers, w, start, cnt, seed, device)
        lo, hi = max(start, b0), min(start + cnt, e0)
        x = x[lo - start:hi - start]
        xs = x.view(hi - lo, m, dbar)
        ip = torch.einsum("nja,jka->njk", xs, cbs)                         # (cnt, m, k)
        a = ip.square().argmax(dim=2)
        alpha = ip.gather(2, a[:, :, None])[:, :, 0]
        dst = body[lo - b0:hi - b0]
        dst["c"] = a.to(torch.int32).cpu().numpy()
        if quant:
            code = (alpha[:, :, None] - scb[None, :, :]).abs().argmin(dim=2)
            dst["s"] = code.to(torch.uint8).cpu().numpy()
        else:
            al = alpha.half().float() if cfg.raw_fp16 else alpha
            dst["a"] = al.cpu().numpy()
    return out


def synth_index(cfg: Config, seed: int = 1, n: int | None = None, device="cpu",
                chunk: int = 1 << 20, train_sample: int = 65536, iters: int = 4) -> bytes:
    """Deterministic PCPQIDX1 image for `cfg` (optionally with fewer points)."""
    return synth_image(cfg, seed, n, device, None, chunk, train_sample, iters).tobytes()


def _pq_image(x: torch.Tensor, m: int, k: int, s: int, raw_fp16: bool, method: str, g: torch.Generator,
              iters: int = 3) -> bytes:
    """PCPQIDX1 image of the rows of x (n, d) by the same fast projective
    encoding as synth_index (k lowered to n like build_ivf does)."""
    n, d = x.shape
    k = min(k, n)
    dbar = (d + m - 1) // m
    pd = dbar * m
    xp = torch.nn.functional.pad(x, (0, pd - d)) if pd != d else x
    xs = xp.view(n, m, dbar)
    cbs = torch.stack([_train_directions(xs[:, j].contiguous(), k, iters, g) for j in range(m)])
    ip = torch.einsum("nja,jka->njk", xs, cbs)
    a = ip.square().argmax(dim=2)
    alpha = ip.gather(2, a[:, :, None])[:, :, 0]
    if s > 0:
        scb = torch.stack([_kmeans_1d(alpha[:, j], s) for j in range(m)])
        code = (alpha[:, :, None] - scb[None, :, :]).abs().argmin(dim=2).to(torch.uint8)
        sc, ra, scbn = code.cpu().numpy(), None, scb.cpu().numpy()
    else:
        al = alpha.half().float() if raw_fp16 else alpha
        sc, ra, scbn = None, al.cpu().numpy(), np.zeros((m, 0), np.float32)
    ix = pcpqidx.IndexArrays(method=pcpqidx.METHODS[method], n=n, d=d, padded_d=pd, m=m, k=k, scales=s,
                             t=0.2, codebooks=cbs.cpu().numpy(), scalar_codebooks=scbn,
                             center_codes=a.to(torch.int64).cpu().numpy().astype(np.uint32),
                             scalar_codes=sc, raw_alphas=ra)
    return pcpqidx.serialize(ix)


def synth_ivf(n: int, d: int, kbar: int, m: int, k: int, s: int, seed: int = 1, raw_fp16: bool = False,
              method: str = "pcpq", zipf_s: float | None = 1.1, device="cpu") -> bytes:
    """Deterministic PCPQIVF1 container: a Gaussian mixture with kbar
    components (Zipf-weighted, so cell sizes are skewed and some cells end up
    with < 2 members and are stored raw, as build_ivf does), members = the
    generating component, coarse centers = the component means, per cell a
    PQ index over the residuals (the fast encoding of synth_index)."""
    from . import pcpqivf
    cfg = Config("ivf", n, d, kbar, 0.3, zipf_s, m, k, s, method, raw_fp16, 1, 10, "gaussian")
    centers, w = mixture_params(cfg, seed, device)
    g = _gen(seed * 7 + 1, device)
    lab = torch.multinomial(w, n, replacement=True, generator=g)
    x = centers[lab] + cfg.std * torch.randn(n, d, generator=g, device=device) / (d ** 0.5)
    x = x.float()
    order = torch.argsort(lab, stable=True)
    counts = torch.bincount(lab, minlength=kbar).cpu().numpy()
    offs = np.concatenate([[0], np.cumsum(counts)])
    ordc = order.cpu().numpy().astype(np.uint32)
    members, blobs = [], []
    cnp = centers.float()
    for r in range(kbar):
        ids = ordc[offs[r]:offs[r + 1]]
        members.append(ids)
        res = x[torch.as_tensor(ids.astype(np.int64), device=device)] - cnp[r][None, :]
        if len(ids) < 2:
            blobs.append(pcpqivf.raw_block(res.cpu().numpy()))
        else:
            blobs.append(_pq_image(res, m, k, s, raw_fp16, method, g))
    iv = pcpqivf.IVFArrays(n, d, kbar, cnp.cpu().numpy(), members, blobs)
    return pcpqivf.serialize(iv)
