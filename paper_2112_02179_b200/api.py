"""Host-side mirror of the reference's scoring API (namespace pcpq,
proj/core/include/pcpq/pq_index.hpp:36-108) over the C ABI of libpcpqg.so.

Same names, argument meaning and error behaviour as the reference:

    read_pq_index(path) / deserialize(bytes) -> DeviceIndex   (pq_index.cpp:409-505)
    build_lookup_table(index, q, counters=None) -> LookupTable (pq_index.cpp:170-210)
    score_all(index, lut, counters=None) -> float32[n]         (pq_index.cpp:212-244)
    score_query(index, q, counters=None) -> float32[n]         (pq_index.cpp:246-250)
    logical_payload_bits(n, m, k, scales)                      (pq_index.cpp:40-44)

plus the batched, fused entry points the GPU needs (the reference's flat
top-n lives inline in its CLI, proj/tools/main.cpp:229-243):

    search(index, Q, topn) -> (ids int32[B, topn], scores float32[B, topn])
    search_device(index, Q_cuda, topn) -> torch tensors, stream-ordered
    merge_device(keys[L, B, topn]) -> global top-n of per-shard lists

Errors raise PcpqError whose ``code`` is the reference errc (or CUDA /
UNSUPPORTED), like pcpq::error (proj/core/include/pcpq/types.hpp:14-34).
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field

import numpy as np

from . import _native as N


class errc(enum.IntEnum):
    usage = 0
    data = 1
    numeric = 2
    bad_magic = 3
    bad_version = 4
    truncated = 5
    code_out_of_range = 6
    size_mismatch = 7
    cuda = 99
    unsupported = 100


class PcpqError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status
        self.code = errc(status - 1) if 1 <= status <= 8 else (errc.cuda if status == 100 else errc.unsupported)


def _check(st: int):
    if st != 0:
        raise PcpqError(st, N.last_error().decode(errors="replace"))


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


@dataclass
class ScoreCounters:
    """pcpq::ScoreCounters (pq_index.hpp:49-55)."""
    table_madds: int = 0
    scalar_mults: int = 0
    point_mults: int = 0
    lookups: int = 0
    adds: int = 0

    def _arr(self):
        return np.array([self.table_madds, self.scalar_mults, self.point_mults, self.lookups, self.adds], np.uint64)

    def _set(self, a):
        self.table_madds, self.scalar_mults, self.point_mults, self.lookups, self.adds = (int(v) for v in a)


@dataclass
class LookupTable:
    """pcpq::LookupTable (pq_index.hpp:39-43); also keeps the query so the
    device scan can rebuild the identical tables next to the codes."""
    m: int
    k: int
    scales: int
    eta: np.ndarray
    eta_lambda: np.ndarray
    q: np.ndarray = field(repr=False, default=None)


class DeviceIndex:
    """A PCPQIDX1 index (or one shard of it) resident in one GPU's HBM."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        info = N.Info()
        _check(N.index_info(self._h, C.byref(info)))
        self.info = info
        self.n, self.d, self.m, self.k = info.n, info.d, info.m, info.k
        self.scales, self.padded_d, self.dbar, self.t = info.scales, info.padded_d, info.dbar, info.t
        self.method = info.method
        self.shard_begin, self.shard_end = info.shard_begin, info.shard_end
        self.device = info.device

    @property
    def n_local(self) -> int:
        return self.shard_end - self.shard_begin

    @property
    def code_bytes(self) -> int:
        return self.info.code_bytes

    @property
    def bytes_per_point(self) -> int:
        return 4 * self.info.words_per_point

    def close(self):
        if self._h:
            N.index_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _image_ptr(data):
    """(pointer, length, keepalive) of an image: bytes, bytearray, memoryview
    or a uint8 numpy array (no copy for bytes and arrays)."""
    if isinstance(data, np.ndarray):
        a = np.ascontiguousarray(data).view(np.uint8).reshape(-1)
        return (a.ctypes.data if a.size else None), a.size, a
    if isinstance(data, (bytearray, memoryview)):
        a = np.frombuffer(data, np.uint8)
        return (a.ctypes.data if a.size else None), a.size, a
    if len(data):
        buf = C.c_char_p(data)
        return C.cast(buf, C.c_void_p).value, len(data), buf
    return None, 0, None


def deserialize(data, device: int = 0, shard: tuple[int, int] | None = None,
                ingest: str = "host") -> DeviceIndex:
    """pcpq::deserialize onto `device`.  ingest="gpu" validates and repacks the
    code rows in HBM (pcpqg_index_load_gpu); the result is identical."""
    b, e = shard if shard is not None else (0, 0)
    h = C.c_void_p()
    ptr, n, _keep = _image_ptr(data)
    load = N.index_load_gpu if ingest == "gpu" else N.index_load
    _check(load(ptr, n, device, b, e or 0, C.byref(h)))
    return DeviceIndex(h)


def deserialize_part(data, row_begin: int, device: int = 0) -> DeviceIndex:
    """One shard from a PART image (header + codebooks of the whole index, then
    only the rows [row_begin, row_begin + count)): pcpqg_index_load_part.  The
    rows validate like pcpq::deserialize's; ids stay global."""
    h = C.c_void_p()
    ptr, n, _keep = _image_ptr(data)
    _check(N.index_load_part(ptr, n, row_begin, device, C.byref(h)))
    return DeviceIndex(h)


def read_pq_index(path: str | os.PathLike, device: int = 0, shard: tuple[int, int] | None = None,
                  ingest: str = "host") -> DeviceIndex:
    b, e = shard if shard is not None else (0, 0)
    h = C.c_void_p()
    load = N.index_load_file_gpu if ingest == "gpu" else N.index_load_file
    _check(load(os.fsencode(str(path)), device, b, e or 0, C.byref(h)))
    return DeviceIndex(h)


TRANSPORTS = {"auto": 0, "nccl": 1, "peer": 2}


class MultiIndex:
    """One index sharded over several GPUs of this process (pcpqg_multi_*):
    shard r = points [r*n/ndev, (r+1)*n/ndev) on devices[r]; searches gather
    the per-shard top-n key rows on devices[0] (NCCL AllGather or peer copies)
    and merge them, giving exactly the unsharded result."""

    def __init__(self, data, devices, transport: str = "auto"):
        ptr, n, _keep = _image_ptr(data)
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        _check(N.multi_load(ptr, n, devs, len(devices), TRANSPORTS[transport], C.byref(h)))
        self._h = h
        info = np.zeros(4, np.uint64)
        _check(N.multi_info(self._h, info.ctypes.data))
        self.n, self.ndev, self.d = int(info[0]), int(info[1]), int(info[3])
        self.transport = "nccl" if int(info[2]) == TRANSPORTS["nccl"] else "peer"
        self.devices = list(devices)

    def search(self, Q, topn: int):
        Q = _f32(Q)
        if Q.ndim == 1:
            Q = Q[None, :]
        B = Q.shape[0]
        ids = np.zeros((B, topn), np.int32)
        sc = np.zeros((B, topn), np.float32)
        _check(N.multi_search(self._h, Q.ctypes.data, B, Q.shape[1], topn, ids.ctypes.data, sc.ctypes.data))
        return ids, sc

    def close(self):
        if self._h:
            N.multi_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def deserialize_multi(data, devices, transport: str = "auto") -> MultiIndex:
    return MultiIndex(data, devices, transport)


def index_codes(index: DeviceIndex) -> np.ndarray:
    """The device code stream as uint32 words [n_blocks][W][32] (for tests)."""
    out = np.empty(index.code_bytes // 4, np.uint32)
    _check(N.index_codes(index._h, out.ctypes.data, out.nbytes))
    return out


def build_lookup_table(index: DeviceIndex, q, counters: ScoreCounters | None = None) -> LookupTable:
    q = _f32(q).reshape(-1)
    eta = np.zeros(index.m * index.k, np.float32)
    etal = np.zeros(index.m * index.k * index.scales, np.float32)
    cnt = counters._arr() if counters is not None else None
    _check(N.build_lut(index._h, q.ctypes.data, 1, q.size, eta.ctypes.data,
                       etal.ctypes.data if index.scales else None,
                       cnt.ctypes.data if cnt is not None else None))
    if counters is not None:
        counters._set(cnt)
    return LookupTable(index.m, index.k, index.scales, eta, etal, q.copy())


def score_all(index: DeviceIndex, lut: LookupTable, counters: ScoreCounters | None = None) -> np.ndarray:
    if lut.m != index.m or lut.k != index.k or lut.scales != index.scales:
        raise PcpqError(8, "score_all: table does not match index")  # pq_index.cpp:216-217
    out = score_all_batch(index, lut.q[None, :])
    if counters is not None:
        n, m = index.n_local, index.m
        if index.scales == 0:
            counters.point_mults += n * m
        counters.lookups += n * m
        counters.adds += n * (m - 1)
    return out[0]


def score_query(index: DeviceIndex, q, counters: ScoreCounters | None = None) -> np.ndarray:
    q = _f32(q).reshape(-1)
    out = np.zeros((1, index.n_local), np.float32)
    cnt = counters._arr() if counters is not None else None
    _check(N.score_all(index._h, q.ctypes.data, 1, q.size, out.ctypes.data, cnt.ctypes.data if cnt is not None else None))
    if counters is not None:
        counters._set(cnt)
    return out[0]


def score_all_batch(index: DeviceIndex, Q) -> np.ndarray:
    Q = _f32(Q)
    if Q.ndim != 2:
        raise PcpqError(8, "queries must be a (B, d) matrix")
    out = np.zeros((Q.shape[0], index.n_local), np.float32)
    _check(N.score_all(index._h, Q.ctypes.data, Q.shape[0], Q.shape[1], out.ctypes.data, None))
    return out


def search(index: DeviceIndex, Q, topn: int):
    """Batched flat top-n (score desc, id asc) over host arrays."""
    Q = _f32(Q)
    if Q.ndim == 1:
        Q = Q[None, :]
    B = Q.shape[0]
    ids = np.zeros((B, topn), np.int32)
    sc = np.zeros((B, topn), np.float32)
    _check(N.search(index._h, Q.ctypes.data, B, Q.shape[1], topn, ids.ctypes.data, sc.ctypes.data))
    return ids, sc


def search_device(index: DeviceIndex, Q, topn: int, stream=None, want_keys: bool = False, out=None):
    """Fused search on device-resident queries (torch CUDA tensor), ordered on
    `stream` (default: torch's current stream); returns torch tensors."""
    import torch
    Q = Q.contiguous()
    if Q.dtype != torch.float32 or not Q.is_cuda:
        raise PcpqError(2, "search_device expects a float32 CUDA tensor")
    B = Q.shape[0]
    if out is None:
        ids = torch.empty((B, topn), dtype=torch.int32, device=Q.device)
        sc = torch.empty((B, topn), dtype=torch.float32, device=Q.device)
        keys = torch.empty((B, topn), dtype=torch.int64, device=Q.device) if want_keys else None
    else:
        ids, sc, keys = out
    st = stream if stream is not None else torch.cuda.current_stream(Q.device)
    _check(N.search_device(index._h, Q.data_ptr(), B, Q.shape[1], topn,
                           ids.data_ptr() if ids is not None else None,
                           sc.data_ptr() if sc is not None else None,
                           keys.data_ptr() if keys is not None else None, st.cuda_stream))
    return ids, sc, keys


def merge_device(keys, topn: int | None = None, stream=None, want_keys: bool = False):
    """Merge per-shard top-n key lists [L, B, topn] (int64 view of the packed
    64-bit keys) into the global top-n (ids, scores[, keys])."""
    import torch
    keys = keys.contiguous()
    if keys.data_ptr() % 16:  # the TMA staging copies whole rows from 16-byte aligned addresses
        keys = keys.clone()
    L, B, K = keys.shape
    topn = K if topn is None else topn
    ids = torch.empty((B, topn), dtype=torch.int32, device=keys.device)
    sc = torch.empty((B, topn), dtype=torch.float32, device=keys.device)
    ko = torch.empty((B, topn), dtype=torch.int64, device=keys.device) if want_keys else None
    st = stream if stream is not None else torch.cuda.current_stream(keys.device)
    if topn != K:
        raise PcpqError(1, "merge_device: topn must equal the list width")
    _check(N.merge_device(keys.data_ptr(), L, B, topn, ids.data_ptr(), sc.data_ptr(),
                          ko.data_ptr() if ko is not None else None, keys.device.index or 0, st.cuda_stream))
    return ids, sc, ko


def counters_for(index: DeviceIndex, B: int) -> ScoreCounters:
    a = np.zeros(5, np.uint64)
    _check(N.counters(index._h, B, a.ctypes.data))
    c = ScoreCounters()
    c._set(a)
    return c


def logical_payload_bits(n: int, m: int, k: int, scales: int) -> int:
    return int(N.logical_payload_bits(n, m, k, scales))


def plan_info(index: DeviceIndex, B: int, topn: int) -> dict:
    """The scan plan pcpqg_search uses for B queries (pcpqg_plan_info)."""
    out = np.zeros(8, np.uint32)
    _check(N.plan_info(index._h, B, topn, out.ctypes.data))
    keys = ("nq", "threads", "ppt", "stages", "ctas_x", "groups", "filter", "table")
    return {k: int(v) for k, v in zip(keys, out)}


def set_option(name: str, value: int):
    """pcpqg_set_option: "lut_tensor_cores" (tcgen05 LUT, tolerance mode),
    "fused_merge", "scan_ws", "scan_filter" (K2-F fp16 pre-score, opt-in: default 0),
    "merge_wide", "gt_chunk", "scan_shape"."""
    _check(N.set_option(name.encode(), int(value)))


def set_profiling(enabled: bool):
    N.set_profiling(1 if enabled else 0)


def last_timings() -> tuple[float, float, float]:
    a = np.zeros(3, np.float32)
    N.last_timings(a.ctypes.data)
    return float(a[0]), float(a[1]), float(a[2])


# ------------------------------------------------------------- encode path
def assign_projective(x, centers, stream=None):
    """pcpq::assign_projective on the GPU (clustering.cpp:250-289): returns
    (assignment u32 as int64 tensor view, alpha f64, loss f64) torch tensors."""
    import torch
    x = x.contiguous().float()
    c = centers.contiguous().float()
    n, dbar = x.shape
    a = torch.empty(n, dtype=torch.int32, device=x.device)
    al = torch.empty(n, dtype=torch.float64, device=x.device)
    lo = torch.empty(n, dtype=torch.float64, device=x.device)
    st = stream if stream is not None else torch.cuda.current_stream(x.device)
    _check(N.assign_projective(x.data_ptr(), n, dbar, c.data_ptr(), c.shape[0], a.data_ptr(), al.data_ptr(),
                               lo.data_ptr(), x.device.index or 0, st.cuda_stream))
    return a, al, lo


def assign_anisotropic(x, centers, h_par, h_bot, stream=None, prev=None):
    """pcpq::assign_anisotropic(allow_scaling=true) on the GPU (clustering.cpp:298-368);
    with `prev`, the solver's keep-previous-center fallback (:339-349)."""
    import torch
    x = x.contiguous().float()
    c = centers.contiguous().float()
    hp = h_par.contiguous().double()
    hb = h_bot.contiguous().double()
    n, dbar = x.shape
    a = torch.empty(n, dtype=torch.int32, device=x.device)
    al = torch.empty(n, dtype=torch.float64, device=x.device)
    lo = torch.empty(n, dtype=torch.float64, device=x.device)
    st = stream if stream is not None else torch.cuda.current_stream(x.device)
    pv = prev.contiguous().int() if prev is not None else None
    _check(N.assign_anisotropic(x.data_ptr(), n, dbar, c.data_ptr(), c.shape[0], hp.data_ptr(), hb.data_ptr(),
                                pv.data_ptr() if pv is not None else None,
                                a.data_ptr(), al.data_ptr(), lo.data_ptr(), x.device.index or 0, st.cuda_stream))
    return a, al, lo


def center_stats(x, assign, alpha, h_par, h_bot, k, init=None, stream=None):
    """Sums of pcpq::center_anisotropic (clustering.cpp:382-402) for every
    (section, cluster): x (nsec, n, dbar) float32, assign (nsec, n),
    alpha/h_par/h_bot (nsec, n) float64.  Returns (nsec, k, S) float64 with
    S = dbar(dbar+1)/2 + dbar + 1; `init` seeds the running sums."""
    import torch
    x = x.contiguous().float()
    nsec, n, dbar = x.shape
    S = dbar * (dbar + 1) // 2 + dbar + 1
    a = assign.contiguous().int()
    al = alpha.contiguous().double()
    hp = h_par.contiguous().double()
    hb = h_bot.contiguous().double()
    out = torch.empty((nsec, k, S), dtype=torch.float64, device=x.device)
    ini = init.contiguous().double() if init is not None else None
    st = stream if stream is not None else torch.cuda.current_stream(x.device)
    _check(N.center_stats(x.data_ptr(), n, dbar, nsec, n * dbar, a.data_ptr(), al.data_ptr(), hp.data_ptr(),
                          hb.data_ptr(), k, ini.data_ptr() if ini is not None else None, out.data_ptr(),
                          x.device.index or 0, st.cuda_stream))
    return out


def aniso_alpha_codes(x, centers, assign, h_par, h_bot, values, stream=None):
    """Score-aware scale codes (scalar_quant.cpp:121-150) on the GPU."""
    import torch
    x = x.contiguous().float()
    c = centers.contiguous().float()
    a = assign.contiguous().int()
    hp = h_par.contiguous().double()
    hb = h_bot.contiguous().double()
    v = values.contiguous().float()
    n, dbar = x.shape
    codes = torch.empty(n, dtype=torch.uint8, device=x.device)
    st = stream if stream is not None else torch.cuda.current_stream(x.device)
    _check(N.aniso_alpha_codes(x.data_ptr(), n, dbar, c.data_ptr(), a.data_ptr(), hp.data_ptr(), hb.data_ptr(),
                               v.data_ptr(), v.numel(), codes.data_ptr(), x.device.index or 0, st.cuda_stream))
    return codes


# ---------------------------------------------------------------- IVF
# Mirror of proj/core/include/pcpq/ivf.hpp: deserialize_ivf / read_ivf_index
# (ivf.cpp:256-335) and query_ivf (ivf.cpp:89-153).

@dataclass
class QueryHit:
    """pcpq::QueryHit (ivf.hpp:33-36)."""
    id: int
    score: float


@dataclass
class IVFQueryOutput:
    """pcpq::IVFQueryOutput (ivf.hpp:37-44)."""
    top: list = field(default_factory=list)
    short_result: bool = False
    requested: list = field(default_factory=list)


class DeviceIVF:
    """A PCPQIVF1 container resident in one GPU's HBM."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        a = np.zeros(10, np.uint64)
        _check(N.ivf_info(self._h, a.ctypes.data))
        (self.n, self.d, self.kbar, self.m, self.k, self.scales, self.method, self.n_raw_cells,
         self.code_bytes, self.format) = (int(x) for x in a)

    def close(self):
        if self._h:
            N.ivf_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def deserialize_ivf(data: bytes, device: int = 0) -> DeviceIVF:
    buf = (C.c_uint8 * max(1, len(data))).from_buffer_copy(data) if data else (C.c_uint8 * 1)()
    h = C.c_void_p()
    _check(N.ivf_load(buf, len(data), device, C.byref(h)))
    return DeviceIVF(h)


def read_ivf_index(path: str | os.PathLike, device: int = 0) -> DeviceIVF:
    h = C.c_void_p()
    _check(N.ivf_load_file(os.fsencode(str(path)), device, C.byref(h)))
    return DeviceIVF(h)


def query_ivf_batch(index: DeviceIVF, Q, k_probe: int, topn: int, requested=None, want_probes=False):
    """Batched query_ivf on host queries Q [B, d] -> dict of arrays:
    ids int32[B, topn], scores float64[B, topn] (id -1 / NaN past counts[b]),
    counts uint32[B], short bool[B], requested float64[B, R], probes uint32[B, k_probe]."""
    Q = _f32(Q)
    if Q.ndim == 1:
        Q = Q.reshape(1, -1)
    B, d = Q.shape
    req = None if requested is None else np.ascontiguousarray(requested, np.uint32).reshape(B, -1)
    R = 0 if req is None else req.shape[1]
    ids = np.empty((B, max(topn, 0)), np.int32)
    sc = np.empty((B, max(topn, 0)), np.float64)
    cnt = np.empty(B, np.uint32)
    sh = np.empty(B, np.uint8)
    rs = np.empty((B, max(R, 1)), np.float64)
    pr = np.empty((B, max(k_probe, 1)), np.uint32) if want_probes else None
    _check(N.ivf_query(index._h, Q.ctypes.data, B, d, k_probe, topn,
                       req.ctypes.data if R else None, R, ids.ctypes.data, sc.ctypes.data, cnt.ctypes.data,
                       sh.ctypes.data, rs.ctypes.data if R else None, pr.ctypes.data if want_probes else None))
    out = {"ids": ids, "scores": sc, "counts": cnt, "short": sh.astype(bool), "requested": rs[:, :R]}
    if want_probes:
        out["probes"] = pr
    return out


def query_ivf(index: DeviceIVF, q, k_probe: int, topn: int, requested_ids=(),
              counters: ScoreCounters | None = None) -> IVFQueryOutput:
    """pcpq::query_ivf for one query (same arguments, errors and output)."""
    q = _f32(q).reshape(1, -1)
    req = np.asarray(requested_ids, np.uint32).reshape(1, -1) if len(requested_ids) else None
    r = query_ivf_batch(index, q, k_probe, topn, requested=req, want_probes=counters is not None)
    if counters is not None:
        ivf_counters(index, r["probes"], counters)
    k = int(r["counts"][0])
    return IVFQueryOutput(top=[QueryHit(int(i), float(s)) for i, s in zip(r["ids"][0, :k], r["scores"][0, :k])],
                          short_result=bool(r["short"][0]),
                          requested=[float(x) for x in r["requested"][0]] if req is not None else [])


def ivf_counters(index: DeviceIVF, probes, counters: ScoreCounters) -> ScoreCounters:
    """Accumulate the ScoreCounters query_ivf adds for these probes [B, k_probe]."""
    p = np.ascontiguousarray(probes, np.uint32)
    a = counters._arr()
    _check(N.ivf_counters(index._h, p.ctypes.data, p.shape[0], p.shape[1], a.ctypes.data))
    counters._set(a)
    return counters


def query_ivf_device(index: DeviceIVF, Q, k_probe: int, topn: int, requested=None, stream=None):
    """query_ivf on device-resident queries (float32 CUDA tensor [B, d]),
    ordered on `stream`; returns torch tensors (ids, scores f64, counts, short,
    requested scores)."""
    import torch
    Q = Q.contiguous()
    if Q.dtype != torch.float32 or not Q.is_cuda:
        raise PcpqError(2, "query_ivf_device expects a float32 CUDA tensor")
    B = Q.shape[0]
    dev = Q.device
    ids = torch.empty((B, topn), dtype=torch.int32, device=dev)
    sc = torch.empty((B, topn), dtype=torch.float64, device=dev)
    cnt = torch.empty(B, dtype=torch.int32, device=dev)
    sh = torch.empty(B, dtype=torch.uint8, device=dev)
    R = 0 if requested is None else requested.shape[1]
    rs = torch.empty((B, R), dtype=torch.float64, device=dev) if R else None
    req = requested.to(dev, torch.int32).contiguous() if R else None
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    _check(N.ivf_query_device(index._h, Q.data_ptr(), B, Q.shape[1], k_probe, topn,
                              req.data_ptr() if R else None, R, ids.data_ptr(), sc.data_ptr(),
                              cnt.data_ptr(), sh.data_ptr(), rs.data_ptr() if R else None, None,
                              st.cuda_stream))
    return ids, sc, cnt, sh.bool(), rs


# ---------------------------------------------------------------- eval
# Mirror of proj/core/include/pcpq/eval.hpp: brute_force_topn (eval.cpp:36-49)
# and recall1_single (eval.cpp:57-66), batched over queries.

@dataclass
class ScoredId:
    """pcpq::ScoredId (eval.hpp:15-18)."""
    id: int
    score: float


def brute_force_topn_batch(data, Q, topn: int, device: int = 0):
    """Exact top-n per query row of Q over the rows of data -> (ids int32[B, topn],
    scores float64[B, topn]), bit-identical to the reference."""
    X = _f32(data)
    Q = _f32(Q)
    if Q.ndim == 1:
        Q = Q.reshape(1, -1)
    if X.ndim != 2 or Q.shape[1] != X.shape[1]:
        raise PcpqError(2, "brute_force_topn: dimension mismatch")
    B = Q.shape[0]
    ids = np.empty((B, max(topn, 0)), np.int32)
    sc = np.empty((B, max(topn, 0)), np.float64)
    _check(N.brute_force_topn(X.ctypes.data, X.shape[0], X.shape[1], Q.ctypes.data, B, topn, ids.ctypes.data,
                              sc.ctypes.data, device))
    return ids, sc


def brute_force_topn(data, q, topn: int, device: int = 0) -> list:
    """pcpq::brute_force_topn for one query -> [ScoredId]."""
    ids, sc = brute_force_topn_batch(data, np.asarray(q).reshape(1, -1), topn, device)
    return [ScoredId(int(i), float(s)) for i, s in zip(ids[0], sc[0])]


def brute_force_topn_device(X, Q, topn: int, stream=None):
    """Device tensors X [n, d], Q [B, d] (float32 CUDA) -> (ids, scores f64) tensors."""
    import torch
    X = X.contiguous()
    Q = Q.contiguous()
    B = Q.shape[0]
    ids = torch.empty((B, topn), dtype=torch.int32, device=Q.device)
    sc = torch.empty((B, topn), dtype=torch.float64, device=Q.device)
    st = stream if stream is not None else torch.cuda.current_stream(Q.device)
    _check(N.brute_force_topn_device(X.data_ptr(), X.shape[0], X.shape[1], Q.data_ptr(), B, topn, ids.data_ptr(),
                                     sc.data_ptr(), Q.device.index or 0, st.cuda_stream))
    return ids, sc


def recall1_batch(data, Q, retrieved, exact_top1, device: int = 0) -> np.ndarray:
    """recall1_single per query -> int32[B] of 0/1."""
    X = _f32(data)
    Q = _f32(Q).reshape(-1, X.shape[1])
    ret = np.ascontiguousarray(retrieved, np.uint32).reshape(Q.shape[0], -1)
    e1 = np.ascontiguousarray(exact_top1, np.float64)
    hits = np.empty(Q.shape[0], np.int32)
    _check(N.recall1(X.ctypes.data, X.shape[0], X.shape[1], Q.ctypes.data, Q.shape[0], ret.ctypes.data,
                     ret.shape[1], e1.ctypes.data, hits.ctypes.data, device))
    return hits


def recall1_single(data, q, retrieved_ids, exact_top1_score: float, device: int = 0) -> int:
    """pcpq::recall1_single for one query."""
    return int(recall1_batch(data, np.asarray(q).reshape(1, -1), np.asarray(retrieved_ids).reshape(1, -1),
                             [exact_top1_score], device)[0])


# ---------------------------------------------------------------- training
def aniso_weights(x, t: float, device=None):
    """pcpq::aniso_weights (clustering.cpp:204-217) for every row of x [n][dbar]
    (norm = the row's L2 norm; zero rows get (0, 0)).  Returns (h_par, h_bot)
    float64 arrays; bit-identical to the reference.  device=None: host threads
    with the C library's sin; device=int: the CUDA kernel (raises unsupported
    when its restated sin does not reproduce this host's std::sin)."""
    X = _f32(x)
    if X.ndim != 2:
        raise PcpqError(errc.usage + 1, "aniso_weights: x must be a matrix")
    hp = np.empty(X.shape[0], np.float64)
    hb = np.empty(X.shape[0], np.float64)
    if device is None:
        _check(N.aniso_weights(X.ctypes.data if X.size else None, X.shape[0], X.shape[1], float(t),
                               hp.ctypes.data, hb.ctypes.data))
    else:
        _check(N.aniso_weights_gpu(X.ctypes.data if X.size else None, X.shape[0], X.shape[1], float(t),
                                   hp.ctypes.data, hb.ctypes.data, int(device)))
    return hp, hb


def sin_selfcheck(device: int = -1):
    """(mismatches, total) of the restated sin against this host's std::sin:
    evaluated on the host (device < 0) or by the kernel on `device`."""
    bad, tot = C.c_uint64(0), C.c_uint64(0)
    _check(N.sin_selfcheck(int(device), C.byref(bad), C.byref(tot)))
    return int(bad.value), int(tot.value)


def train_weights_on_gpu() -> bool:
    """Whether the last aniso / apcpq build on this thread computed its weights on the GPU."""
    out = C.c_int(0)
    _check(N.train_weights_on_gpu(C.byref(out)))
    return bool(out.value)



@dataclass
class PQConfig:
    """pcpq::PQConfig (proj/core/include/pcpq/types.hpp:74-84)."""
    method: str = "pcpq"
    quantize_scalars: bool = False
    m: int = 8
    k: int = 16
    s: int = 8
    t_frac: float = 0.2
    max_iters: int = 20
    tol: float = 1e-6
    seed: int = 1


def train_phases() -> dict:
    """Wall seconds of the last build_pq_index call on this thread, by phase."""
    out = np.zeros(4, np.float64)
    _check(N.train_phases(out.ctypes.data))
    return dict(zip(("prep", "lloyd", "scales", "serialize"), out.tolist()))


def build_pq_index(data, cfg: PQConfig, device=0) -> bytes:
    """pcpq::build_pq_index + serialize (pq_index.cpp:62-168, :372-407) with the
    Lloyd iterations on the GPU; returns the PCPQIDX1 image, byte-identical to
    the reference's.  Methods: "kmeans", "pcpq", "aniso" (alias "scann") and
    "apcpq".  For the score-aware methods `device` may be a list of devices:
    the sections are dealt round-robin to them (pcpqg_train_aniso_multi)."""
    if cfg.method not in ("kmeans", "pcpq", "aniso", "scann", "apcpq"):
        raise PcpqError(errc.usage + 1, f"build_pq_index: unknown method {cfg.method!r}")
    X = _f32(data)
    if X.ndim != 2:
        raise PcpqError(2, "build_pq_index: data must be a matrix")
    p = C.c_void_p()
    ln = C.c_uint64()
    ptr = X.ctypes.data if X.size else None
    if cfg.method in ("kmeans", "pcpq") and not isinstance(device, (int, np.integer)):
        raise PcpqError(errc.usage + 1, "build_pq_index: a device list is supported for aniso / apcpq only")
    if cfg.method == "kmeans":
        _check(N.train_kmeans(ptr, X.shape[0], X.shape[1], cfg.m, cfg.k, cfg.s, cfg.t_frac, cfg.max_iters,
                              cfg.tol, cfg.seed, device, C.byref(p), C.byref(ln)))
    elif cfg.method == "pcpq":
        _check(N.train_pcpq(ptr, X.shape[0], X.shape[1], cfg.m, cfg.k, cfg.s, int(cfg.quantize_scalars),
                            cfg.t_frac, cfg.max_iters, cfg.tol, cfg.seed, device, C.byref(p), C.byref(ln)))
    else:
        method = 3 if cfg.method == "apcpq" else 1
        devs = np.ascontiguousarray(np.atleast_1d(np.asarray(device, np.int32)))
        _check(N.train_aniso_multi(ptr, X.shape[0], X.shape[1], cfg.m, cfg.k, cfg.s, method,
                                   int(cfg.quantize_scalars), cfg.t_frac, cfg.max_iters, cfg.tol, cfg.seed,
                                   devs.ctypes.data, int(devs.size), C.byref(p), C.byref(ln)))
    try:
        return C.string_at(p, ln.value)
    finally:
        N.free(p)
