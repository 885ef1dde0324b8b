"""Golden vectors for GPU training (tests/golden/train_*.npz) from the
UNMODIFIED reference (oracle/_ref): the PCPQIDX1 image of build_pq_index +
serialize (proj/core/src/pq_index.cpp:62-168, :372-407) for small seeded
datasets.  Run here: python tests/golden/make_golden_train.py
Cases: methods kmeans, pcpq, apcpq (quantized and raw scales) and aniso with clustered / gaussian / unit-sphere data, d % m != 0 (padding),
k > 256 (two-byte codes), duplicated rows (empty clusters -> reseeding), a
max_iters = 1 run and a loose tol (early convergence)."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import Ref  # noqa: E402

# name, dist, n, d, m, k, max_iters, tol, seed, post
CASES = [
    ("train_kmeans_clustered", "clustered", 1500, 16, 4, 16, 20, 1e-6, 5, None),
    ("train_kmeans_pad", "gaussian", 900, 10, 3, 8, 20, 1e-6, 6, None),
    ("train_kmeans_wide", "gaussian", 700, 4, 1, 300, 10, 1e-6, 7, None),
    ("train_kmeans_dups", "clustered", 800, 8, 2, 32, 20, 1e-6, 8, "dups"),
    ("train_kmeans_iter1", "clustered", 600, 12, 6, 4, 1, 1e-6, 9, None),
    ("train_kmeans_tol", "clustered", 1200, 8, 2, 8, 50, 1e-2, 10, None),
]
# method pcpq: name, dist, n, d, m, k, s, quantize, max_iters, tol, seed, post
PCPQ_CASES = [
    ("train_pcpq_q_s8", "clustered", 1500, 16, 4, 16, 8, True, 20, 1e-6, 21, None),
    ("train_pcpq_raw", "clustered", 1000, 12, 3, 8, 8, False, 20, 1e-6, 22, None),
    ("train_pcpq_pad_s4", "gaussian", 900, 10, 3, 8, 4, True, 20, 1e-6, 23, None),
    ("train_pcpq_dups", "clustered", 800, 8, 2, 32, 8, True, 20, 1e-6, 24, "dups"),
    ("train_pcpq_zero_rows", "clustered", 700, 8, 4, 8, 16, True, 15, 1e-6, 25, "zeros"),
    ("train_pcpq_s2_tol", "unit_sphere", 1200, 12, 6, 4, 2, True, 50, 1e-3, 26, None),
]

# methods aniso (ScaNN baseline) / apcpq: name, method, dist, n, d, m, k, s, quantize, t_frac, max_iters, tol,
# seed, post
ANISO_CASES = [
    ("train_apcpq_q_s8", "apcpq", "clustered", 1500, 16, 4, 16, 8, True, 0.2, 20, 1e-6, 31, None),
    ("train_apcpq_raw", "apcpq", "clustered", 1000, 12, 3, 8, 8, False, 0.2, 20, 1e-6, 32, None),
    ("train_apcpq_pad_s4", "apcpq", "gaussian", 900, 10, 3, 8, 4, True, 0.3, 20, 1e-6, 33, None),
    ("train_apcpq_dups", "apcpq", "clustered", 800, 8, 2, 32, 8, True, 0.2, 20, 1e-6, 34, "dups"),
    ("train_apcpq_zero_rows", "apcpq", "clustered", 700, 8, 4, 8, 16, True, 0.2, 15, 1e-6, 35, "zeros"),
    ("train_apcpq_d2_tol", "apcpq", "unit_sphere", 1200, 12, 6, 4, 2, True, 0.2, 50, 1e-3, 36, None),
    ("train_apcpq_t0", "apcpq", "clustered", 600, 8, 2, 8, 4, True, 0.0, 10, 1e-6, 37, None),
    ("train_aniso_k16", "aniso", "clustered", 1500, 16, 4, 16, 1, False, 0.2, 20, 1e-6, 38, None),
    ("train_aniso_pad", "aniso", "gaussian", 900, 10, 3, 8, 1, False, 0.5, 20, 1e-6, 39, None),
    ("train_aniso_dups", "aniso", "clustered", 800, 8, 2, 32, 1, False, 0.2, 20, 1e-6, 40, "dups"),
]


def main():
    R = Ref()
    for name, dist, n, d, m, k, iters, tol, seed, post in CASES:
        X = R.generate_dataset(dist, n, d, seed)
        if post == "dups":
            X = np.concatenate([X[:20]] * (n // 20))  # 20 distinct rows, k = 32
        img = R.build_index(X, method="kmeans", quantize=False, m=m, k=k, s=1, t_frac=0.2,
                            max_iters=iters, tol=tol, seed=seed)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), data=X,
                            cfg=np.array([m, k, 1, iters, seed], np.int64), tol=np.float64(tol),
                            t_frac=np.float64(0.2), image=np.frombuffer(img, np.uint8))
        print(name, X.shape, len(img))
    for name, dist, n, d, m, k, sc, quant, iters, tol, seed, post in PCPQ_CASES:
        X = R.generate_dataset(dist, n, d, seed)
        if post == "dups":
            X = np.concatenate([X[:20]] * (n // 20))
        if post == "zeros":
            X[::7] = 0.0  # zero points: alpha 0, excluded from the seeding candidates
        img = R.build_index(X, method="pcpq", quantize=quant, m=m, k=k, s=sc, t_frac=0.2,
                            max_iters=iters, tol=tol, seed=seed)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), data=X,
                            cfg=np.array([m, k, sc, iters, seed], np.int64), tol=np.float64(tol),
                            t_frac=np.float64(0.2), quantize=np.bool_(quant), method=np.array("pcpq"),
                            image=np.frombuffer(img, np.uint8))
        print(name, X.shape, len(img))

    for name, method, dist, n, d, m, k, sc, quant, t_frac, iters, tol, seed, post in ANISO_CASES:
        X = R.generate_dataset(dist, n, d, seed)
        if post == "dups":
            X = np.concatenate([X[:20]] * (n // 20))
        if post == "zeros":
            X[::7] = 0.0
        img = R.build_index(X, method=method, quantize=quant, m=m, k=k, s=sc, t_frac=t_frac,
                            max_iters=iters, tol=tol, seed=seed)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), data=X,
                            cfg=np.array([m, k, sc, iters, seed], np.int64), tol=np.float64(tol),
                            t_frac=np.float64(t_frac), quantize=np.bool_(quant), method=np.array(method),
                            image=np.frombuffer(img, np.uint8))
        print(name, X.shape, len(img))


if __name__ == "__main__":
    main()
