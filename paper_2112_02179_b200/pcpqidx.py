"""PCPQIDX1 image writer / reader (numpy, vectorised).

The byte layout is the reference's serialization format
(proj/core/src/pq_index.cpp:372-407, documented at
proj/core/include/pcpq/pq_index.hpp:98-108):

    "PCPQIDX1" | u32 version=1, method, n, d, padded_d, m, k, scales | f64 t
    m x (k x dbar) f32 codebooks | m x scales f32 scale codebooks
    n rows: m center codes (u8 if k <= 256 else u16 LE), then m u8 scale codes
            (scales >= 1) or m f32 raw alphas (scales == 0)

Used to synthesise benchmark-scale indexes; the GPU side only ever consumes
the bytes through pcpqg_index_load (which validates them like
pcpq::deserialize).
"""
from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

METHODS = {"kmeans": 0, "scann": 1, "pcpq": 2, "apcpq": 3}
METHOD_NAMES = {v: k for k, v in METHODS.items()}


@dataclass
class IndexArrays:
    method: int
    n: int
    d: int
    padded_d: int
    m: int
    k: int
    scales: int
    t: float
    codebooks: np.ndarray            # (m, k, dbar) float32
    scalar_codebooks: np.ndarray     # (m, scales) float32
    center_codes: np.ndarray         # (n, m) uint32
    scalar_codes: np.ndarray | None  # (n, m) uint8 when scales >= 1
    raw_alphas: np.ndarray | None    # (n, m) float32 when scales == 0

    @property
    def dbar(self) -> int:
        return self.padded_d // self.m


def header_bytes(method: int, n: int, d: int, padded_d: int, m: int, k: int, scales: int, t: float,
                 codebooks: np.ndarray, scalar_codebooks: np.ndarray) -> bytes:
    """Header + codebooks + scale codebooks (everything before the code rows)."""
    head = b"PCPQIDX1" + struct.pack("<8I", 1, method, n, d, padded_d, m, k, scales)
    head += struct.pack("<d", t)
    cb = np.ascontiguousarray(codebooks, dtype="<f4").tobytes()
    scb = np.ascontiguousarray(scalar_codebooks, dtype="<f4").reshape(-1).tobytes() if scales else b""
    return head + cb + scb


def row_dtype(m: int, k: int, scales: int) -> np.dtype:
    """One code row: m center codes (u8, or u16 LE for k > 256), then m u8
    scale codes (scales >= 1) or m f32 raw alphas."""
    cdt = np.dtype("<u2") if k > 256 else np.dtype("u1")
    if scales >= 1:
        return np.dtype([("c", cdt, (m,)), ("s", "u1", (m,))])
    return np.dtype([("c", cdt, (m,)), ("a", "<f4", (m,))])


def serialize(ix: IndexArrays) -> bytes:
    m, k, n = ix.m, ix.k, ix.n
    head = header_bytes(ix.method, n, ix.d, ix.padded_d, m, k, ix.scales, ix.t, ix.codebooks,
                        ix.scalar_codebooks)
    cdt = np.dtype("<u2") if k > 256 else np.dtype("u1")
    row = row_dtype(m, k, ix.scales)
    rows = np.empty(n, dtype=row)
    rows["c"] = ix.center_codes.astype(cdt.base if hasattr(cdt, "base") else cdt)
    if ix.scales >= 1:
        rows["s"] = ix.scalar_codes
    else:
        rows["a"] = ix.raw_alphas
    return head + rows.tobytes()


def deserialize(data: bytes) -> IndexArrays:
    if data[:8] != b"PCPQIDX1":
        raise ValueError("bad magic")
    version, method, n, d, padded_d, m, k, scales = struct.unpack_from("<8I", data, 8)
    (t,) = struct.unpack_from("<d", data, 40)
    dbar = padded_d // m
    off = 48
    cb = np.frombuffer(data, "<f4", m * k * dbar, off).reshape(m, k, dbar).copy()
    off += 4 * m * k * dbar
    scb = np.frombuffer(data, "<f4", m * scales, off).reshape(m, scales).copy()
    off += 4 * m * scales
    cdt = np.dtype("<u2") if k > 256 else np.dtype("u1")
    row = np.dtype([("c", cdt, (m,)), ("s", "u1", (m,))]) if scales else np.dtype([("c", cdt, (m,)), ("a", "<f4", (m,))])
    rows = np.frombuffer(data, row, n, off)
    return IndexArrays(method, n, d, padded_d, m, k, scales, t, cb, scb,
                       rows["c"].astype(np.uint32), rows["s"].copy() if scales else None,
                       None if scales else rows["a"].astype(np.float32))


def row_bytes(m: int, k: int, scales: int) -> int:
    return m * (2 if k > 256 else 1) + (m if scales else 4 * m)
