"""PCPQIVF1 container writer / reader (numpy).

The byte layout is the reference's IVF container
(proj/core/src/ivf.cpp:229-255, documented at proj/core/include/pcpq/ivf.hpp:57-63):

    "PCPQIVF1" | u32 version=1, n, d, kbar
    kbar x d f32 coarse centers
    kbar member lists: u32 count, then count u32 ids
    kbar blobs: u64 length, then a PCPQIDX1 image (the cell's PQ index over the
                residuals x - c) or a raw block "PCPQRAW1" | u32 count | u32 d |
                count x d f32 residuals (cells with fewer than 2 members)

Host-side structure only (tests build corrupted containers with it, and the
synthetic IVF benchmark builds its cells with it); the GPU side consumes the
bytes through pcpqg_ivf_load, which validates them like pcpq::deserialize_ivf.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

IVF_MAGIC = b"PCPQIVF1"
RAW_MAGIC = b"PCPQRAW1"


@dataclass
class IVFArrays:
    n: int
    d: int
    kbar: int
    coarse: np.ndarray                       # (kbar, d) float32
    members: list = field(default_factory=list)  # kbar uint32 arrays
    blobs: list = field(default_factory=list)    # kbar bytes (PCPQIDX1 image or raw block)

    def is_raw(self, r: int) -> bool:
        return self.blobs[r][:8] == RAW_MAGIC


def raw_block(residuals: np.ndarray) -> bytes:
    res = np.ascontiguousarray(residuals, np.float32)
    return RAW_MAGIC + struct.pack("<II", res.shape[0], res.shape[1]) + res.tobytes()


def raw_residuals(blob: bytes) -> np.ndarray:
    count, d = struct.unpack_from("<II", blob, 8)
    return np.frombuffer(blob, np.float32, count * d, 16).reshape(count, d)


def serialize(x: IVFArrays) -> bytes:
    out = [IVF_MAGIC, struct.pack("<IIII", 1, x.n, x.d, x.kbar),
           np.ascontiguousarray(x.coarse, np.float32).tobytes()]
    for mem in x.members:
        mem = np.ascontiguousarray(mem, np.uint32)
        out += [struct.pack("<I", mem.size), mem.tobytes()]
    for blob in x.blobs:
        out += [struct.pack("<Q", len(blob)), blob]
    return b"".join(out)


def deserialize(data: bytes) -> IVFArrays:
    """Structural parse (no semantic validation; see pcpqg_ivf_load for that)."""
    if data[:8] != IVF_MAGIC:
        raise ValueError("not a PCPQIVF1 container")
    _, n, d, kbar = struct.unpack_from("<IIII", data, 8)
    pos = 24
    coarse = np.frombuffer(data, np.float32, kbar * d, pos).reshape(kbar, d).copy()
    pos += 4 * kbar * d
    members = []
    for _ in range(kbar):
        (cnt,) = struct.unpack_from("<I", data, pos)
        members.append(np.frombuffer(data, np.uint32, cnt, pos + 4).copy())
        pos += 4 + 4 * cnt
    blobs = []
    for _ in range(kbar):
        (ln,) = struct.unpack_from("<Q", data, pos)
        blobs.append(bytes(data[pos + 8:pos + 8 + ln]))
        pos += 8 + ln
    return IVFArrays(n, d, kbar, coarse, members, blobs)


def blob_offsets(data: bytes) -> list[int]:
    """Byte offset of each cell's blob (after its u64 length) in the container."""
    _, n, d, kbar = struct.unpack_from("<IIII", data, 8)
    pos = 24 + 4 * kbar * d
    for _ in range(kbar):
        (cnt,) = struct.unpack_from("<I", data, pos)
        pos += 4 + 4 * cnt
    offs = []
    for _ in range(kbar):
        (ln,) = struct.unpack_from("<Q", data, pos)
        offs.append(pos + 8)
        pos += 8 + ln
    return offs
