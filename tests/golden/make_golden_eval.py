"""Golden vectors for exact ground truth / recall (tests/golden/eval_*.npz)
from the UNMODIFIED reference (oracle/_ref): brute_force_topn
(proj/core/src/eval.cpp:36-49) and recall1_single (eval.cpp:57-66) on
reference-generated datasets.  Run here: python tests/golden/make_golden_eval.py
Cases: clustered / gaussian / unit_sphere data, odd d, duplicated rows (exact
ties decided by id), an all-zero query (every score +-0), topN 1 / 10 / 257 (n for the tie case)."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import Ref  # noqa: E402

CASES = [("eval_clustered_d24", "clustered", 5000, 24, 41, None),
         ("eval_gaussian_d7", "gaussian", 3000, 7, 42, None),
         ("eval_sphere_d33", "unit_sphere", 4000, 33, 43, None),
         ("eval_ties_d16", "clustered", 2000, 16, 44, "ties")]


def main():
    R = Ref()
    rng = np.random.default_rng(7)
    for name, dist, n, d, seed, post in CASES:
        X = R.generate_dataset(dist, n, d, seed)
        if post == "ties":
            X = np.concatenate([X[: n // 4]] * 4)  # every row 4 times
        Q = rng.standard_normal((6, d)).astype(np.float32)
        Q[5] = 0.0
        out = {"data": X, "queries": Q}
        # topN = n (the maximum) only for the small tie case, to keep fixtures small
        for tn in (1, 10, X.shape[0] if post == "ties" else 257):
            ids, sc = R.brute_force_topn(X, Q, tn, threads=8)
            out[f"ids_{tn}"], out[f"scores_{tn}"] = ids, sc
        ret = rng.integers(0, X.shape[0], (6, 12)).astype(np.uint32)
        ret[:3, 5] = out["ids_1"][:3, 0]  # half the queries retrieve their exact top-1
        out["retrieved"] = ret
        out["hits"] = R.recall1(X, Q, ret, out["scores_1"][:, 0])
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
        print(name, X.shape, out["hits"])


if __name__ == "__main__":
    main()
