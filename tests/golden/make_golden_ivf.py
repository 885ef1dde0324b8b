"""Generate the IVF golden fixtures (tests/golden/ivf_*.ivf + .npz) from the
UNMODIFIED reference library (oracle/_ref/libpcpq_ref.so).  Run here, where
/root/reference exists:

    make -C oracle ref && python tests/golden/make_golden_ivf.py

Every case is a PCPQIVF1 container built by the reference's build_ivf
(proj/core/src/ivf.cpp:46-87) on a reference-generated dataset and serialized
by the reference (ivf.cpp:229-255), plus, for each probe count in `kprobes`
and each topn in `topns`, the outputs of the reference's query_ivf
(ivf.cpp:89-153) for 5 queries (the last one all zeros: every coarse and
residual score is +-0, so ranking is decided by the tie rules alone):
  ids_<kp>_<tn> / scores_<kp>_<tn> / counts_<kp>_<tn> / short_<kp>_<tn>
  req_<kp>_<tn>        scores of 12 requested ids per query (NaN = unprobed)
  counters_<kp>_<tn>   ScoreCounters summed over the 5 queries
and the error codes of deliberately corrupted containers (deserialize_ivf,
ivf.cpp:256-316), see corrupt_cases().
The cases cover raw (singleton) cells, all-raw containers (kbar = n), every
cell code layout the flat fixtures cover (JOINT8, PLANES with 4/8-bit
centers, raw fp16-exact/fp32 alphas), lowered k in small cells, and ties.
"""
import os
import struct
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Ref  # noqa: E402
from paper_2112_02179_b200 import pcpqivf  # noqa: E402

# name, dist, n, d, kbar, method, quantize, m, k, s, seed
CASES = [
    ("ivf_pcpq_q_k4", "clustered", 300, 8, 6, "pcpq", True, 2, 4, 2, 31),
    ("ivf_apcpq_q_k4_s4", "clustered", 240, 10, 5, "apcpq", True, 2, 4, 4, 32),
    ("ivf_pcpq_raw_cells", "gaussian", 40, 6, 20, "pcpq", True, 2, 2, 2, 33),
    ("ivf_kmeans_singletons", "gaussian", 24, 6, 24, "kmeans", False, 2, 2, 1, 34),
    ("ivf_apcpq_rawalpha", "clustered", 400, 12, 8, "apcpq", False, 3, 4, 4, 35),
    ("ivf_aniso_k16_s8", "clustered", 500, 16, 10, "aniso", True, 4, 16, 8, 36),
    ("ivf_pcpq_k16_rawalpha", "clustered", 600, 32, 12, "pcpq", False, 8, 16, 8, 37),
    ("ivf_kmeans_k64", "clustered", 800, 16, 4, "kmeans", False, 4, 64, 1, 38),
]


def corrupt_cases(data: bytes):
    """(label, bytes) of corrupted containers; the reference's error code is
    recorded for each (0 = accepted)."""
    iv = pcpqivf.deserialize(data)
    out = [("bad_magic", b"PCPQIVFX" + data[8:]),
           ("bad_version", data[:8] + struct.pack("<I", 2) + data[12:]),
           ("kbar_zero", data[:20] + struct.pack("<I", 0) + data[24:]),
           ("kbar_gt_n", data[:20] + struct.pack("<I", iv.n + 1) + data[24:]),
           ("trailing", data + b"\0"),
           ("empty", b"")]
    for cut in (4, 10, 23, 24 + 4 * iv.d, len(data) // 2, len(data) - 1):
        out.append((f"cut_{cut}", data[:cut]))
    # member count above n
    pos = 24 + 4 * iv.kbar * iv.d
    out.append(("count_gt_n", data[:pos] + struct.pack("<I", iv.n + 1) + data[pos + 4:]))
    # duplicated id (cell 0's first member copied over cell 1's first member): partition error
    a = pcpqivf.deserialize(data)
    if len(a.members[0]) and len(a.members[1]):
        a.members[1] = a.members[1].copy()
        a.members[1][0] = a.members[0][0]
        out.append(("dup_member", pcpqivf.serialize(a)))
    a = pcpqivf.deserialize(data)
    a.members[0] = a.members[0].copy()
    if len(a.members[0]):
        a.members[0][0] = iv.n  # id out of range
        out.append(("id_out_of_range", pcpqivf.serialize(a)))
    # a PQ cell whose blob n does not match its member list / whose d differs
    for r in range(iv.kbar):
        if not iv.is_raw(r):
            a = pcpqivf.deserialize(data)
            blob = bytearray(a.blobs[r])
            struct.pack_into("<I", blob, 20, struct.unpack_from("<I", blob, 20)[0] + 1)  # d
            a.blobs[r] = bytes(blob)
            out.append(("sub_d_mismatch", pcpqivf.serialize(a)))
            a = pcpqivf.deserialize(data)
            a.blobs[r] = a.blobs[r][:-1]
            out.append(("sub_truncated", pcpqivf.serialize(a)))
            a = pcpqivf.deserialize(data)
            blob = bytearray(a.blobs[r])
            blob[0] ^= 0x40
            a.blobs[r] = bytes(blob)
            out.append(("sub_bad_magic", pcpqivf.serialize(a)))
            break
    for r in range(iv.kbar):
        if iv.is_raw(r):
            a = pcpqivf.deserialize(data)
            blob = bytearray(a.blobs[r])
            struct.pack_into("<I", blob, 12, iv.d + 1)
            a.blobs[r] = bytes(blob)
            out.append(("raw_dim_mismatch", pcpqivf.serialize(a)))
            a = pcpqivf.deserialize(data)
            blob = bytearray(a.blobs[r])
            struct.pack_into("<I", blob, 8, struct.unpack_from("<I", blob, 8)[0] + 1)
            a.blobs[r] = bytes(blob)
            out.append(("raw_count_mismatch", pcpqivf.serialize(a)))
            a = pcpqivf.deserialize(data)
            a.blobs[r] = a.blobs[r] + b"\0\0\0\0"
            out.append(("raw_trailing", pcpqivf.serialize(a)))
            break
    return out


def kprobes_of(kbar):
    return sorted({1, 2, max(1, kbar // 2), kbar})


def main():
    R = Ref()
    rng = np.random.default_rng(2024)
    for name, dist, n, d, kbar, method, quant, m, k, s, seed in CASES:
        X = R.generate_dataset(dist, n, d, seed)
        data = R.build_ivf(X, kbar, method=method, quantize=quant, m=m, k=k, s=s, seed=seed)
        Q = rng.standard_normal((5, d)).astype(np.float32)
        Q[4] = 0.0
        req = rng.integers(0, n, (5, 12)).astype(np.uint32)
        arrays = {"queries": Q, "requested": req, "kprobes": np.array(kprobes_of(kbar), np.uint32),
                  "topns": np.array([10, n + 3], np.uint32)}
        for kp in kprobes_of(kbar):
            for tn in (10, n + 3):
                ids, sc, cnt, sh, rs, c5 = R.ivf_query(data, Q, kp, tn, requested=req)
                arrays[f"ids_{kp}_{tn}"] = ids
                arrays[f"scores_{kp}_{tn}"] = sc
                arrays[f"counts_{kp}_{tn}"] = cnt
                arrays[f"short_{kp}_{tn}"] = sh
                arrays[f"req_{kp}_{tn}"] = rs
                arrays[f"counters_{kp}_{tn}"] = c5
        labels, codes = [], []
        for label, bad in corrupt_cases(data):
            labels.append(label)
            codes.append(R.ivf_validate(bad))
        arrays["error_labels"] = np.array(labels)
        arrays["error_codes"] = np.array(codes, np.int32)
        with open(os.path.join(HERE, name + ".ivf"), "wb") as f:
            f.write(data)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrays)
        print(name, len(data), "bytes; errors", dict(zip(labels, codes)))


if __name__ == "__main__":
    main()
