"""TEST INFRASTRUCTURE ONLY — ctypes bindings to the two CPU checkers.

* ``Port``  — oracle/_build/libpcpq_oracle.so, the plain-C restatement of the
  reference scoring path (oracle/pcpq_oracle.c).  Builds anywhere gcc exists,
  including the GPU box.
* ``Ref``   — oracle/_ref/libpcpq_ref.so, the *unmodified* reference library
  compiled from /root/reference/proj/core/src plus oracle/ref_shim.cpp.  Built
  only where /root/reference exists; the .so travels to the GPU box.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and the
``--impl reference`` arm) may import this module, and only as the checker or
the timed reference CPU arm.  The product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import struct

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libpcpq_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpcpq_ref.so")

_u8p = C.POINTER(C.c_uint8)
_fp = C.POINTER(C.c_float)
_dp = C.POINTER(C.c_double)
_u32p = C.POINTER(C.c_uint32)
_i32p = C.POINTER(C.c_int32)
_u64p = C.POINTER(C.c_uint64)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def build_port() -> str:
    if not os.path.exists(PORT_SO):
        subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)
    return PORT_SO


# --------------------------------------------------------------------- port
class PortIndex:
    def __init__(self, lib, handle):
        self._lib = lib
        self._h = handle
        x = handle.contents
        self.n, self.d, self.m, self.k = x.n, x.d, x.m, x.k
        self.scales, self.padded_d, self.dbar = x.scales, x.padded_d, x.dbar

    def __del__(self):
        try:
            self._lib.orc_free(self._h)
        except Exception:
            pass

    def build_lut(self, q):
        q = np.ascontiguousarray(q, np.float32)
        eta = np.zeros(self.m * self.k, np.float32)
        etal = np.zeros(max(1, self.m * self.k * self.scales), np.float32)
        cnt = np.zeros(5, np.uint64)
        st = self._lib.orc_build_lut(self._h, _ptr(q, _fp), q.size, _ptr(eta, _fp), _ptr(etal, _fp), _ptr(cnt, _u64p))
        if st:
            raise OracleError(st, "build_lut")
        return eta, (etal if self.scales else np.zeros(0, np.float32)), cnt

    def score_query(self, q):
        q = np.ascontiguousarray(q, np.float32)
        out = np.zeros(self.n, np.float32)
        cnt = np.zeros(5, np.uint64)
        st = self._lib.orc_score_query(self._h, _ptr(q, _fp), q.size, _ptr(out, _fp), _ptr(cnt, _u64p))
        if st:
            raise OracleError(st, "score_query")
        return out, cnt

    def search(self, Q, topn, threads=1):
        Q = np.ascontiguousarray(Q, np.float32)
        B = Q.shape[0]
        ids = np.zeros((B, topn), np.int32)
        sc = np.zeros((B, topn), np.float32)
        st = self._lib.orc_search(self._h, _ptr(Q, _fp), B, Q.shape[1], topn, threads, _ptr(ids, _i32p), _ptr(sc, _fp))
        if st:
            raise OracleError(st, "search")
        return ids, sc

    def serialize(self) -> bytes:
        p = _u8p()
        n = C.c_uint64()
        self._lib.orc_serialize(self._h, C.byref(p), C.byref(n))
        b = C.string_at(p, n.value)
        self._lib.orc_free_bytes(p)
        return b

    def arrays(self):
        """Decoded arrays (center codes n*m, scale codes or raw alphas)."""
        x = self._h.contents
        n, m = self.n, self.m
        cc = np.ctypeslib.as_array(x.center_codes, shape=(n * m,)).reshape(n, m).copy()
        if self.scales:
            sc = np.ctypeslib.as_array(x.scalar_codes, shape=(n * m,)).reshape(n, m).copy()
            return cc, sc, None
        ra = np.ctypeslib.as_array(x.raw_alphas, shape=(n * m,)).reshape(n, m).copy()
        return cc, None, ra


class _OrcIndex(C.Structure):
    _fields_ = [("method", C.c_uint32), ("n", C.c_uint32), ("d", C.c_uint32), ("padded_d", C.c_uint32),
                ("m", C.c_uint32), ("k", C.c_uint32), ("scales", C.c_uint32), ("dbar", C.c_uint32),
                ("t", C.c_double), ("codebooks", _fp), ("scalar_cb", _fp), ("center_codes", _u32p),
                ("scalar_codes", _u8p), ("raw_alphas", _fp)]


class PortIVF:
    """A parsed PCPQIVF1 container in the C restatement (orc_ivf)."""

    def __init__(self, lib, h, n, d, kbar):
        self.lib, self.h, self.n, self.d, self.kbar = lib, h, n, d, kbar

    def __del__(self):
        try:
            self.lib.orc_ivf_free(self.h)
        except Exception:
            pass

    def query(self, Q, k_probe, topn, requested=None):
        """Same outputs as Ref.ivf_query."""
        Q = np.ascontiguousarray(Q, np.float32)
        B, d = Q.shape
        req = np.zeros((B, 0), np.uint32) if requested is None else np.ascontiguousarray(requested, np.uint32)
        R = req.shape[1]
        ids = np.full((B, topn), -1, np.int32)
        sc = np.zeros((B, topn), np.float64)
        cnt = np.zeros(B, np.uint32)
        sh = np.zeros(B, np.uint8)
        rs = np.zeros((B, max(R, 1)), np.float64)
        c5 = np.zeros(5, np.uint64)
        for b in range(B):
            st = self.lib.orc_ivf_query(self.h, _ptr(Q[b], _fp), d, k_probe, topn,
                                        _ptr(req[b], _u32p) if R else None, R,
                                        _ptr(ids[b], _i32p), _ptr(sc[b], _dp),
                                        C.byref(C.c_uint32.from_buffer(cnt, 4 * b)),
                                        C.byref(C.c_uint8.from_buffer(sh, b)),
                                        _ptr(rs[b], _dp), _ptr(c5, _u64p))
            if st:
                raise OracleError(st, "ivf_query")
        return ids, sc, cnt, sh.astype(bool), rs[:, :R], c5


class Port:
    """The C restatement (oracle/pcpq_oracle.c)."""

    def __init__(self, path: str | None = None):
        self.lib = C.CDLL(path or build_port())
        L = self.lib
        L.orc_parse.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.POINTER(_OrcIndex)), C.c_char_p, C.c_size_t]
        L.orc_free.argtypes = [C.POINTER(_OrcIndex)]
        L.orc_serialize.argtypes = [C.POINTER(_OrcIndex), C.POINTER(_u8p), _u64p]
        L.orc_free_bytes.argtypes = [C.c_void_p]
        L.orc_build_lut.argtypes = [C.POINTER(_OrcIndex), _fp, C.c_uint32, _fp, _fp, _u64p]
        L.orc_score_query.argtypes = [C.POINTER(_OrcIndex), _fp, C.c_uint32, _fp, _u64p]
        L.orc_search.argtypes = [C.POINTER(_OrcIndex), _fp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_int, _i32p, _fp]
        L.orc_topn_of_scores.argtypes = [_fp, C.c_uint64, C.c_uint32, _i32p]
        L.orc_logical_payload_bits.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32]
        L.orc_logical_payload_bits.restype = C.c_uint64
        L.orc_assign_projective.argtypes = [_fp, C.c_uint64, C.c_uint32, _fp, C.c_uint32, _u32p, _dp, _dp]
        L.orc_assign_anisotropic.argtypes = [_fp, C.c_uint64, C.c_uint32, _fp, C.c_uint32, _dp, _dp, _u32p, _dp, _dp]
        L.orc_alpha_codes_aniso.argtypes = [_fp, C.c_uint64, C.c_uint32, _fp, _u32p, _dp, _dp, _fp, C.c_uint32, _u8p]
        L.orc_center_stats.argtypes = [_fp, _u32p, C.c_uint64, C.c_uint32, _dp, _dp, _dp, _dp]
        L.orc_center_from_stats.argtypes = [_dp, C.c_uint32, _dp]

    def center_stats(self, x, assign, alpha, h_par, h_bot, k, init=None):
        """Per-cluster member sums (members in increasing id order), seeded by `init`."""
        x = np.ascontiguousarray(x, np.float32)
        n, dbar = x.shape
        S = dbar * (dbar + 1) // 2 + dbar + 1
        out = np.zeros((k, S)) if init is None else np.array(init, np.float64).reshape(k, S).copy()
        a = np.asarray(assign)
        al = np.ascontiguousarray(alpha, np.float64)
        hp = np.ascontiguousarray(h_par, np.float64)
        hb = np.ascontiguousarray(h_bot, np.float64)
        for c in range(k):
            mem = np.ascontiguousarray(np.nonzero(a == c)[0].astype(np.uint32))
            row = np.ascontiguousarray(out[c])
            self.lib.orc_center_stats(_ptr(x, _fp), _ptr(mem, _u32p), mem.size, dbar, _ptr(al, _dp), _ptr(hp, _dp),
                                      _ptr(hb, _dp), _ptr(row, _dp))
            out[c] = row
        return out

    def center_from_stats(self, stats, dbar):
        s = np.ascontiguousarray(stats, np.float64)
        c = np.zeros(dbar)
        st = self.lib.orc_center_from_stats(_ptr(s, _dp), dbar, _ptr(c, _dp))
        if st:
            raise OracleError(st, "center_from_stats")
        return c

    def brute_force_topn(self, X, Q, topn):
        """brute_force_topn per query row -> (ids int32[B, topn], scores f64[B, topn])."""
        L = self.lib
        L.orc_brute_force_topn.argtypes = [_fp, C.c_uint64, C.c_uint32, _fp, C.c_uint32, _i32p, _dp]
        X = np.ascontiguousarray(X, np.float32)
        Q = np.ascontiguousarray(Q, np.float32)
        B = Q.shape[0]
        ids = np.zeros((B, topn), np.int32)
        sc = np.zeros((B, topn), np.float64)
        for b in range(B):
            st = L.orc_brute_force_topn(_ptr(X, _fp), X.shape[0], X.shape[1], _ptr(Q[b], _fp), topn,
                                        _ptr(ids[b], _i32p), _ptr(sc[b], _dp))
            if st:
                raise OracleError(st, "brute_force_topn")
        return ids, sc

    def recall1(self, X, Q, retrieved, exact_top1):
        L = self.lib
        L.orc_recall1.argtypes = [_fp, C.c_uint64, C.c_uint32, _fp, _u32p, C.c_uint32, C.c_double, _i32p]
        X = np.ascontiguousarray(X, np.float32)
        Q = np.ascontiguousarray(Q, np.float32)
        ret = np.ascontiguousarray(retrieved, np.uint32)
        hits = np.zeros(Q.shape[0], np.int32)
        for b in range(Q.shape[0]):
            st = L.orc_recall1(_ptr(X, _fp), X.shape[0], X.shape[1], _ptr(Q[b], _fp), _ptr(ret[b], _u32p),
                               ret.shape[1], float(exact_top1[b]), C.byref(C.c_int32.from_buffer(hits, 4 * b)))
            if st:
                raise OracleError(st, "recall1")
        return hits

    def ivf_parse(self, data: bytes) -> PortIVF:
        L = self.lib
        L.orc_ivf_parse.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]
        L.orc_ivf_free.argtypes = [C.c_void_p]
        L.orc_ivf_query.argtypes = [C.c_void_p, _fp, C.c_uint32, C.c_uint32, C.c_uint32, _u32p, C.c_uint32,
                                    _i32p, _dp, C.POINTER(C.c_uint32), C.POINTER(C.c_uint8), _dp, _u64p]
        h = C.c_void_p()
        err = C.create_string_buffer(256)
        buf = (C.c_uint8 * max(1, len(data))).from_buffer_copy(data if len(data) else b"\0")
        st = L.orc_ivf_parse(buf, len(data), C.byref(h), err, 256)
        if st:
            raise OracleError(st, err.value.decode())
        n, d, kbar = struct.unpack_from("<III", data, 12)
        return PortIVF(L, h, n, d, kbar)

    def parse(self, data: bytes) -> PortIndex:
        h = C.POINTER(_OrcIndex)()
        err = C.create_string_buffer(256)
        buf = (C.c_uint8 * max(1, len(data))).from_buffer_copy(data if len(data) else b"\0")
        st = self.lib.orc_parse(buf, len(data), C.byref(h), err, 256)
        if st:
            raise OracleError(st, err.value.decode())
        return PortIndex(self.lib, h)

    def topn_of_scores(self, scores, topn):
        s = np.ascontiguousarray(scores, np.float32)
        k = min(topn, s.size)
        ids = np.zeros(k, np.int32)
        self.lib.orc_topn_of_scores(_ptr(s, _fp), s.size, k, _ptr(ids, _i32p))
        return ids

    def logical_payload_bits(self, n, m, k, scales):
        return int(self.lib.orc_logical_payload_bits(n, m, k, scales))

    def assign_projective(self, x, centers):
        x = np.ascontiguousarray(x, np.float32)
        c = np.ascontiguousarray(centers, np.float32)
        n, dbar = x.shape
        a = np.zeros(n, np.uint32)
        al = np.zeros(n, np.float64)
        pl = np.zeros(n, np.float64)
        st = self.lib.orc_assign_projective(_ptr(x, _fp), n, dbar, _ptr(c, _fp), c.shape[0], _ptr(a, _u32p), _ptr(al, _dp), _ptr(pl, _dp))
        if st:
            raise OracleError(st, "assign_projective")
        return a, al, pl

    def assign_anisotropic(self, x, centers, h_par, h_bot):
        x = np.ascontiguousarray(x, np.float32)
        c = np.ascontiguousarray(centers, np.float32)
        hp = np.ascontiguousarray(h_par, np.float64)
        hb = np.ascontiguousarray(h_bot, np.float64)
        n, dbar = x.shape
        a = np.zeros(n, np.uint32)
        al = np.zeros(n, np.float64)
        pl = np.zeros(n, np.float64)
        st = self.lib.orc_assign_anisotropic(_ptr(x, _fp), n, dbar, _ptr(c, _fp), c.shape[0], _ptr(hp, _dp), _ptr(hb, _dp),
                                             _ptr(a, _u32p), _ptr(al, _dp), _ptr(pl, _dp))
        if st:
            raise OracleError(st, "assign_anisotropic")
        return a, al, pl

    def alpha_codes_aniso(self, x, centers, assign, h_par, h_bot, values):
        x = np.ascontiguousarray(x, np.float32)
        c = np.ascontiguousarray(centers, np.float32)
        a = np.ascontiguousarray(assign, np.uint32)
        hp = np.ascontiguousarray(h_par, np.float64)
        hb = np.ascontiguousarray(h_bot, np.float64)
        v = np.ascontiguousarray(values, np.float32)
        n, dbar = x.shape
        codes = np.zeros(n, np.uint8)
        self.lib.orc_alpha_codes_aniso(_ptr(x, _fp), n, dbar, _ptr(c, _fp), _ptr(a, _u32p), _ptr(hp, _dp), _ptr(hb, _dp),
                                       _ptr(v, _fp), v.size, _ptr(codes, _u8p))
        return codes


# ---------------------------------------------------------------- reference
class RefIndex:
    def __init__(self, lib, h):
        self._lib = lib
        self._h = h
        shape = np.zeros(6, np.uint64)
        lib.ref_index_shape(h, _ptr(shape, _u64p))
        self.n, self.d, self.m, self.k, self.scales, self.padded_d = (int(v) for v in shape)

    def __del__(self):
        try:
            self._lib.ref_index_close(self._h)
        except Exception:
            pass

    def _check(self, st, what):
        if st:
            raise OracleError(st, f"{what}: {self._lib.ref_last_error().decode()}")

    def build_lut(self, q):
        q = np.ascontiguousarray(q, np.float32)
        eta = np.zeros(self.m * self.k, np.float32)
        etal = np.zeros(max(1, self.m * self.k * self.scales), np.float32)
        cnt = np.zeros(5, np.uint64)
        self._check(self._lib.ref_build_lut(self._h, _ptr(q, _fp), q.size, _ptr(eta, _fp), _ptr(etal, _fp), _ptr(cnt, _u64p)), "build_lut")
        return eta, (etal if self.scales else np.zeros(0, np.float32)), cnt

    def score_query(self, q):
        q = np.ascontiguousarray(q, np.float32)
        out = np.zeros(self.n, np.float32)
        cnt = np.zeros(5, np.uint64)
        self._check(self._lib.ref_score_query(self._h, _ptr(q, _fp), q.size, _ptr(out, _fp), _ptr(cnt, _u64p)), "score_query")
        return out, cnt

    def search(self, Q, topn, threads=1):
        Q = np.ascontiguousarray(Q, np.float32)
        B = Q.shape[0]
        ids = np.zeros((B, topn), np.int32)
        sc = np.zeros((B, topn), np.float32)
        self._check(self._lib.ref_search(self._h, _ptr(Q, _fp), B, Q.shape[1], topn, threads, _ptr(ids, _i32p), _ptr(sc, _fp)), "search")
        return ids, sc

    def serialize(self) -> bytes:
        p = _u8p()
        n = C.c_uint64()
        self._check(self._lib.ref_serialize(self._h, C.byref(p), C.byref(n)), "serialize")
        b = C.string_at(p, n.value)
        self._lib.ref_free(p)
        return b


METHODS = {"kmeans": 0, "scann": 1, "aniso": 1, "pcpq": 2, "apcpq": 3}
DISTS = {"gaussian": 0, "unit_sphere": 1, "clustered": 2}


class Ref:
    """The unmodified reference library (oracle/_ref/libpcpq_ref.so)."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self, path: str | None = None):
        self.lib = C.CDLL(path or REF_SO)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_build_index.argtypes = [_fp, C.c_uint64, C.c_uint32, C.c_int, C.c_int, C.c_uint32, C.c_uint32, C.c_uint32,
                                      C.c_double, C.c_uint32, C.c_double, C.c_uint64, C.POINTER(_u8p), _u64p]
        L.ref_index_open.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_int)]
        L.ref_index_open.restype = C.c_void_p
        L.ref_index_close.argtypes = [C.c_void_p]
        L.ref_index_shape.argtypes = [C.c_void_p, _u64p]
        L.ref_serialize.argtypes = [C.c_void_p, C.POINTER(_u8p), _u64p]
        L.ref_build_lut.argtypes = [C.c_void_p, _fp, C.c_uint32, _fp, _fp, _u64p]
        L.ref_score_query.argtypes = [C.c_void_p, _fp, C.c_uint32, _fp, _u64p]
        L.ref_search.argtypes = [C.c_void_p, _fp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_int, _i32p, _fp]
        L.ref_logical_payload_bits.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32]
        L.ref_logical_payload_bits.restype = C.c_uint64
        L.ref_generate_dataset.argtypes = [C.c_int, C.c_uint64, C.c_uint32, C.c_uint64, _fp]
        L.ref_aniso_weights.argtypes = [C.c_double, C.c_double, C.c_int, _dp, _dp]
        L.ref_assign_projective.argtypes = [_fp, C.c_uint64, C.c_uint32, _fp, C.c_uint32, _u32p, _dp, _dp]
        L.ref_assign_anisotropic.argtypes = [_fp, C.c_uint64, C.c_uint32, _fp, C.c_uint32, _dp, _dp, C.c_int, _u32p, _dp, _dp]
        L.ref_quantize_anisotropic.argtypes = [_fp, C.c_uint64, C.c_uint32, _fp, C.c_uint32, _u32p, _dp, _dp, C.c_uint32,
                                               C.c_uint64, _fp, _u8p]

    def _check(self, st, what):
        if st:
            raise OracleError(st, f"{what}: {self.lib.ref_last_error().decode()}")

    def build_index(self, data, method="pcpq", quantize=True, m=8, k=16, s=8, t_frac=0.2,
                    max_iters=20, tol=1e-6, seed=1) -> bytes:
        x = np.ascontiguousarray(data, np.float32)
        p = _u8p()
        n = C.c_uint64()
        self._check(self.lib.ref_build_index(_ptr(x, _fp), x.shape[0], x.shape[1], METHODS[method], int(quantize),
                                             m, k, s, t_frac, max_iters, tol, seed, C.byref(p), C.byref(n)), "build_index")
        b = C.string_at(p, n.value)
        self.lib.ref_free(p)
        return b

    def open(self, data: bytes) -> RefIndex:
        st = C.c_int(0)
        buf = (C.c_uint8 * max(1, len(data))).from_buffer_copy(data if len(data) else b"\0")
        h = self.lib.ref_index_open(buf, len(data), C.byref(st))
        if st.value:
            raise OracleError(st.value, self.lib.ref_last_error().decode())
        return RefIndex(self.lib, h)

    # ---- IVF (proj/core/src/ivf.cpp)
    def build_ivf(self, data, kbar, method="pcpq", quantize=True, m=2, k=4, s=2, max_iters=20,
                  seed=1) -> bytes:
        """build_ivf + serialize: the PCPQIVF1 container bytes."""
        x = np.ascontiguousarray(data, np.float32)
        L = self.lib
        L.ref_build_ivf.argtypes = [_fp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_int, C.c_int, C.c_uint32,
                                    C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.POINTER(_u8p), _u64p]
        p = _u8p()
        n = C.c_uint64()
        self._check(L.ref_build_ivf(_ptr(x, _fp), x.shape[0], x.shape[1], kbar, METHODS[method], int(quantize),
                                    m, k, s, max_iters, seed, C.byref(p), C.byref(n)), "build_ivf")
        b = C.string_at(p, n.value)
        L.ref_free(p)
        return b

    def ivf_query(self, data: bytes, Q, k_probe, topn, requested=None):
        """query_ivf per row of Q -> (ids[B,topn], scores[B,topn] f64, counts[B],
        short[B] bool, requested_scores[B,R] f64, counters5)."""
        Q = np.ascontiguousarray(Q, np.float32)
        B, d = Q.shape
        req = np.zeros((B, 0), np.uint32) if requested is None else np.ascontiguousarray(requested, np.uint32)
        R = req.shape[1]
        L = self.lib
        L.ref_ivf_query.argtypes = [C.c_void_p, C.c_uint64, _fp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                    _u32p, C.c_uint32, _i32p, _dp, _u32p, _u8p, _dp, _u64p]
        ids = np.full((B, topn), -1, np.int32)
        sc = np.zeros((B, topn), np.float64)
        cnt = np.zeros(B, np.uint32)
        sh = np.zeros(B, np.uint8)
        rs = np.zeros((B, max(R, 1)), np.float64)
        c5 = np.zeros(5, np.uint64)
        buf = (C.c_uint8 * max(1, len(data))).from_buffer_copy(data if len(data) else b"\0")
        self._check(L.ref_ivf_query(buf, len(data), _ptr(Q, _fp), B, d, k_probe, topn,
                                    _ptr(req, _u32p) if R else None, R, _ptr(ids, _i32p), _ptr(sc, _dp),
                                    _ptr(cnt, _u32p), _ptr(sh, _u8p), _ptr(rs, _dp), _ptr(c5, _u64p)), "ivf_query")
        return ids, sc, cnt, sh.astype(bool), rs[:, :R], c5

    def ivf_open(self, data: bytes):
        """deserialize_ivf once -> handle for ivf_query_h (timing)."""
        L = self.lib
        L.ref_ivf_open.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_int)]
        L.ref_ivf_open.restype = C.c_void_p
        L.ref_ivf_close.argtypes = [C.c_void_p]
        L.ref_ivf_query_h.argtypes = [C.c_void_p, _fp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int,
                                      _i32p, _dp]
        st = C.c_int(0)
        buf = (C.c_uint8 * max(1, len(data))).from_buffer_copy(data if len(data) else b"\0")
        h = L.ref_ivf_open(buf, len(data), C.byref(st))
        if st.value:
            raise OracleError(st.value, L.ref_last_error().decode())
        return h

    def ivf_close(self, h):
        self.lib.ref_ivf_close(h)

    def ivf_query_h(self, h, Q, k_probe, topn, threads=1):
        Q = np.ascontiguousarray(Q, np.float32)
        B, d = Q.shape
        ids = np.full((B, topn), -1, np.int32)
        sc = np.zeros((B, topn), np.float64)
        self._check(self.lib.ref_ivf_query_h(h, _ptr(Q, _fp), B, d, k_probe, topn, threads, _ptr(ids, _i32p),
                                             _ptr(sc, _dp)), "ivf_query_h")
        return ids, sc

    def brute_force_topn(self, X, Q, topn, threads=1):
        L = self.lib
        L.ref_brute_force_topn.argtypes = [_fp, C.c_uint64, C.c_uint32, _fp, C.c_uint64, C.c_uint32, C.c_int,
                                           _i32p, _dp]
        X = np.ascontiguousarray(X, np.float32)
        Q = np.ascontiguousarray(Q, np.float32)
        B = Q.shape[0]
        ids = np.zeros((B, topn), np.int32)
        sc = np.zeros((B, topn), np.float64)
        self._check(L.ref_brute_force_topn(_ptr(X, _fp), X.shape[0], X.shape[1], _ptr(Q, _fp), B, topn, threads,
                                           _ptr(ids, _i32p), _ptr(sc, _dp)), "brute_force_topn")
        return ids, sc

    def recall1(self, X, Q, retrieved, exact_top1):
        L = self.lib
        L.ref_recall1.argtypes = [_fp, C.c_uint64, C.c_uint32, _fp, C.c_uint64, _u32p, C.c_uint32, _dp, _i32p]
        X = np.ascontiguousarray(X, np.float32)
        Q = np.ascontiguousarray(Q, np.float32)
        ret = np.ascontiguousarray(retrieved, np.uint32)
        e1 = np.ascontiguousarray(exact_top1, np.float64)
        hits = np.zeros(Q.shape[0], np.int32)
        self._check(L.ref_recall1(_ptr(X, _fp), X.shape[0], X.shape[1], _ptr(Q, _fp), Q.shape[0], _ptr(ret, _u32p),
                                  ret.shape[1], _ptr(e1, _dp), _ptr(hits, _i32p)), "recall1")
        return hits

    def ivf_validate(self, data: bytes) -> int:
        """deserialize_ivf status: 0 ok, errc + 1 on error."""
        self.lib.ref_ivf_validate.argtypes = [C.c_void_p, C.c_uint64]
        buf = (C.c_uint8 * max(1, len(data))).from_buffer_copy(data if len(data) else b"\0")
        return int(self.lib.ref_ivf_validate(buf, len(data)))

    def generate_dataset(self, dist, n, d, seed):
        out = np.zeros((n, d), np.float32)
        self._check(self.lib.ref_generate_dataset(DISTS[dist], n, d, seed, _ptr(out, _fp)), "generate_dataset")
        return out

    def logical_payload_bits(self, n, m, k, scales):
        return int(self.lib.ref_logical_payload_bits(n, m, k, scales))

    def aniso_weights(self, norm_x, t, dbar):
        hp, hb = C.c_double(), C.c_double()
        self._check(self.lib.ref_aniso_weights(norm_x, t, dbar, C.byref(hp), C.byref(hb)), "aniso_weights")
        return hp.value, hb.value

    def assign_projective(self, x, centers):
        x = np.ascontiguousarray(x, np.float32)
        c = np.ascontiguousarray(centers, np.float32)
        n, dbar = x.shape
        a = np.zeros(n, np.uint32)
        al = np.zeros(n, np.float64)
        pl = np.zeros(n, np.float64)
        self._check(self.lib.ref_assign_projective(_ptr(x, _fp), n, dbar, _ptr(c, _fp), c.shape[0], _ptr(a, _u32p),
                                                   _ptr(al, _dp), _ptr(pl, _dp)), "assign_projective")
        return a, al, pl

    def center_anisotropic(self, x, members, alpha, h_par, h_bot):
        x = np.ascontiguousarray(x, np.float32)
        mem = np.ascontiguousarray(members, np.uint32)
        out = np.zeros(x.shape[1])
        self.lib.ref_center_anisotropic.argtypes = [_fp, C.c_uint32, _u32p, C.c_uint64, _dp, _dp, _dp, _dp]
        self._check(self.lib.ref_center_anisotropic(_ptr(x, _fp), x.shape[1], _ptr(mem, _u32p), mem.size,
                                                    _ptr(np.ascontiguousarray(alpha, np.float64), _dp),
                                                    _ptr(np.ascontiguousarray(h_par, np.float64), _dp),
                                                    _ptr(np.ascontiguousarray(h_bot, np.float64), _dp),
                                                    _ptr(out, _dp)), "center_anisotropic")
        return out

    def quantize_anisotropic(self, x, centers, assign, h_par, h_bot, s, seed=1):
        x = np.ascontiguousarray(x, np.float32)
        c = np.ascontiguousarray(centers, np.float32)
        a = np.ascontiguousarray(assign, np.uint32)
        hp = np.ascontiguousarray(h_par, np.float64)
        hb = np.ascontiguousarray(h_bot, np.float64)
        n, dbar = x.shape
        values = np.zeros(s, np.float32)
        codes = np.zeros(n, np.uint8)
        self._check(self.lib.ref_quantize_anisotropic(_ptr(x, _fp), n, dbar, _ptr(c, _fp), c.shape[0], _ptr(a, _u32p),
                                                      _ptr(hp, _dp), _ptr(hb, _dp), s, seed, _ptr(values, _fp),
                                                      _ptr(codes, _u8p)), "quantize_anisotropic")
        return values, codes

    def assign_anisotropic(self, x, centers, h_par, h_bot, allow_scaling=True):
        x = np.ascontiguousarray(x, np.float32)
        c = np.ascontiguousarray(centers, np.float32)
        hp = np.ascontiguousarray(h_par, np.float64)
        hb = np.ascontiguousarray(h_bot, np.float64)
        n, dbar = x.shape
        a = np.zeros(n, np.uint32)
        al = np.zeros(n, np.float64)
        pl = np.zeros(n, np.float64)
        self._check(self.lib.ref_assign_anisotropic(_ptr(x, _fp), n, dbar, _ptr(c, _fp), c.shape[0], _ptr(hp, _dp), _ptr(hb, _dp),
                                                    int(allow_scaling), _ptr(a, _u32p), _ptr(al, _dp), _ptr(pl, _dp)), "assign_anisotropic")
        return a, al, pl
