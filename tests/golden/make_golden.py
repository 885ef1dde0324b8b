"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference
library (oracle/_ref/libpcpq_ref.so, built from /root/reference/proj/core/src
by oracle/Makefile).  Run here, where /root/reference exists:

    make -C oracle ref && python tests/golden/make_golden.py

Every case is an index trained by the reference's own build_pq_index
(proj/core/src/pq_index.cpp:62-168) on a reference-generated dataset
(proj/core/src/datagen.cpp), serialized by the reference, plus:
  queries        6 seeded Gaussian queries (the last one all zeros: every
                 score is +-0, so the whole top-n is decided by the id tie rule)
  scores         score_query for every query (pq_index.cpp:246-250)
  ids / top      the flat query loop of proj/tools/main.cpp:229-243 at topn=10
                 and at topn = n + 3 (clamped, padded with -1)
  eta / etal     build_lookup_table of query 0 (pq_index.cpp:170-210)
  counters       ScoreCounters of score_query(query 0)
  errors         error codes of deliberately corrupted images (deserialize,
                 pq_index.cpp:409-488)
The cases cover every device code layout (JOINT8 and PLANES with 4/8/16-bit
centers and 0/4/8-bit scale codes, fp16-exact and fp32 raw alphas), padding
(d % m != 0), m % 8 != 0, wide k (two-byte codes), ties and -0.0 scores.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Ref  # noqa: E402
from paper_2112_02179_b200 import pcpqidx  # noqa: E402

# name, dist, n, d, method, quantize, m, k, s, seed, post
CASES = [
    ("kmeans_m3_k8", "clustered", 300, 24, "kmeans", False, 3, 8, 1, 11, None),
    ("scann_m2_k16", "gaussian", 300, 24, "scann", False, 2, 16, 1, 12, None),
    ("pcpq_q_m8_k16_s16", "clustered", 400, 64, "pcpq", True, 8, 16, 16, 13, None),
    ("pcpq_raw_m4_k16", "clustered", 300, 32, "pcpq", False, 4, 16, 8, 14, None),
    ("pcpq_raw16_m4_k16", "clustered", 300, 32, "pcpq", False, 4, 16, 8, 14, "fp16"),
    ("apcpq_q_m10_k16_s8", "clustered", 300, 20, "apcpq", True, 10, 16, 8, 15, None),
    ("apcpq_raw_m3_k8", "clustered", 250, 24, "apcpq", False, 3, 8, 8, 16, None),
    ("pcpq_q_k32_s8", "clustered", 400, 16, "pcpq", True, 2, 32, 8, 17, None),
    ("pcpq_q_k64_s16", "clustered", 500, 16, "pcpq", True, 4, 64, 16, 18, None),
    ("pcpq_q_k256_s16", "clustered", 600, 16, "pcpq", True, 4, 256, 16, 19, None),
    ("kmeans_k300_wide", "gaussian", 400, 4, "kmeans", False, 1, 300, 1, 20, None),
    ("pcpq_q_s32", "clustered", 300, 24, "pcpq", True, 3, 16, 32, 21, None),
    ("pcpq_q_pad_d5_m2", "gaussian", 40, 5, "pcpq", True, 2, 4, 4, 22, None),
    ("kmeans_m1_k2", "gaussian", 50, 8, "kmeans", False, 1, 2, 1, 23, None),
    ("pcpq_q_m13_odd", "clustered", 200, 26, "pcpq", True, 13, 8, 4, 24, None),
    ("pcpq_raw_m16_k16", "clustered", 200, 64, "pcpq", False, 16, 16, 8, 25, None),
    ("pcpq_q_ties", "clustered", 300, 24, "pcpq", True, 3, 8, 4, 26, "ties"),
    ("pcpq_raw_zero_rows", "clustered", 200, 16, "pcpq", False, 4, 8, 8, 27, "zeros"),
]


def make_data(R, dist, n, d, seed, post):
    if post == "ties":  # 50 distinct rows repeated: identical codes -> identical scores
        base = R.generate_dataset(dist, 50, d, seed)
        return np.tile(base, (n // 50 + 1, 1))[:n].copy()
    x = R.generate_dataset(dist, n, d, seed)
    if post == "zeros":  # zero sections -> alpha 0 -> +-0 score terms
        x[::7] = 0.0
        x[3::5, : d // 2] = 0.0
    return x


def corrupt_cases(data: bytes, ix: pcpqidx.IndexArrays):
    out = {}
    b = bytearray(data)
    b[0] ^= 0xFF
    out["bad_magic"] = bytes(b)
    b = bytearray(data)
    b[8] = 0x7F
    out["bad_version"] = bytes(b)
    b = bytearray(data)
    b[12] = 9
    out["bad_method"] = bytes(b)
    out["truncated_half"] = data[: len(data) // 2]
    out["truncated_header"] = data[:30]
    out["truncated_last"] = data[:-1]
    out["trailing"] = data + b"\0"
    row = pcpqidx.row_bytes(ix.m, ix.k, ix.scales)
    body = len(data) - ix.n * row
    b = bytearray(data)
    b[body + 3 * row] = 0xFF if ix.k <= 255 else b[body + 3 * row]
    if ix.k <= 255:
        out["center_code_range"] = bytes(b)
    if 0 < ix.scales < 256:
        b = bytearray(data)
        b[body + 5 * row + (2 if ix.k > 256 else 1) * ix.m] = 0xFF
        out["scale_code_range"] = bytes(b)
        # bad code *before* the truncation point wins over truncation
        out["range_then_truncated"] = bytes(b[: body + 7 * row + 1])
    b = bytearray(data)
    b[24:28] = (ix.padded_d + 1).to_bytes(4, "little")  # padded_d % m != 0 (m > 1) / < d
    out["bad_padded_d"] = bytes(b)
    return out


def main():
    R = Ref()
    for (name, dist, n, d, method, quant, m, k, s, seed, post) in CASES:
        x = make_data(R, dist, n, d, seed, post)
        data = R.build_index(x, method, quant, m=m, k=k, s=s, max_iters=8, seed=seed)
        if post == "fp16":  # round raw alphas to fp16-representable fp32
            ix = pcpqidx.deserialize(data)
            ix.raw_alphas = ix.raw_alphas.astype(np.float16).astype(np.float32)
            data = pcpqidx.serialize(ix)
        ix = pcpqidx.deserialize(data)
        ri = R.open(data)
        assert ri.serialize() == data
        rng = np.random.default_rng(seed)
        Q = rng.standard_normal((6, d)).astype(np.float32)
        Q[5] = 0.0
        scores = np.stack([ri.score_query(q)[0] for q in Q])
        ids10, top10 = ri.search(Q, 10, threads=1)
        idsx, topx = ri.search(Q, n + 3, threads=1)
        eta, etal, _ = ri.build_lut(Q[0])
        _, cnt = ri.score_query(Q[0])
        errs = {}
        for ename, bad in corrupt_cases(data, ix).items():
            try:
                R.open(bad)
                errs[ename] = 0
            except Exception as e:  # OracleError carries the status (errc + 1)
                errs[ename] = int(getattr(e, "code"))
        with open(os.path.join(HERE, name + ".idx"), "wb") as f:
            f.write(data)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), queries=Q, scores=scores, ids10=ids10,
                            top10=top10, idsx=idsx, topx=topx, eta=eta, etal=etal, counters=cnt,
                            err_names=np.array(list(errs.keys())), err_codes=np.array(list(errs.values())),
                            shape=np.array([ix.n, ix.d, ix.m, ix.k, ix.scales, ix.padded_d]))
        print(f"{name}: n={n} d={d} m={m} k={k} scales={ix.scales} bytes={len(data)} errs={errs}")
    # logical payload bits (pq_index.cpp:40-44) on a grid
    grid = [(n, m, k, sc) for n in (1, 10, 100000) for m in (1, 2, 8, 25) for k in (2, 3, 16, 17, 256, 300)
            for sc in (0, 1, 2, 5, 8, 16)]
    bits = [R.logical_payload_bits(*g) for g in grid]
    np.savez_compressed(os.path.join(HERE, "payload_bits.npz"), grid=np.array(grid), bits=np.array(bits, np.uint64))


if __name__ == "__main__":
    main()
