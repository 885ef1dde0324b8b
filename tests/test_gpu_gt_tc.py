"""GT-T: brute_force_topn (proj/core/src/eval.cpp:36-49) with the tcgen05 fp16
pre-score filter in front of the exact fp64 re-score (csrc/pcpqg_tscan.cu,
csrc/pcpqg_eval.cu).  The result must be the reference's ids and double score
bits — compared with the C oracle (orc_brute_force_topn, pinned to the
reference's golden vectors by tests/test_eval.py) — with the filter on, off
(the exact kernel alone) and over several point chunks; on clustered data,
duplicated points (ties -> lower id), zero / huge / tiny / lopsided queries and
rescaled data sets.  Tolerance: none."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _data(n, d, seed, clusters=64):
    rng = np.random.default_rng(seed)
    c = rng.standard_normal((clusters, d)).astype(np.float32)
    x = c[rng.integers(0, clusters, n)] + 0.25 * rng.standard_normal((n, d)).astype(np.float32)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    return np.ascontiguousarray(x.astype(np.float32))


def _check(port, X, Q, topn):
    import paper_2112_02179_b200 as P
    ids, sc = P.brute_force_topn_batch(X, Q, topn)
    ri, rs = port.brute_force_topn(X, Q, topn)
    bad = np.argwhere(ids != ri)
    assert bad.size == 0, bad[:5]
    assert np.array_equal(sc.view(np.uint64), rs.view(np.uint64))
    return ids, sc


@pytest.mark.parametrize("n,d,B,topn", [(20000, 33, 7, 10), (50000, 100, 130, 100), (30000, 128, 64, 1),
                                         (8192, 16, 300, 256), (12345, 7, 5, 50), (40000, 200, 33, 100)])
def test_gt_tc_matches_oracle(port, n, d, B, topn):
    X = _data(n, d, n + d)
    Q = _data(B, d, 7 * n + 1, clusters=16)
    _check(port, X, Q, topn)


def test_gt_tc_filter_on_off_and_chunked(port):
    import paper_2112_02179_b200 as P
    X = _data(60000, 97, 3)
    Q = _data(40, 97, 4)
    a = _check(port, X, Q, 100)
    try:
        P.set_option("gt_tc", 0)  # the exact kernel alone
        b = P.brute_force_topn_batch(X, Q, 100)
        P.set_option("gt_tc", 1)
        P.set_option("gt_chunk", 16384)  # 4 chunks, the last one short (exact)
        c = P.brute_force_topn_batch(X, Q, 100)
        P.set_option("gt_chunk", 59904)  # a 96-point tail chunk
        e = P.brute_force_topn_batch(X, Q, 100)
    finally:
        P.set_option("gt_tc", 1)
        P.set_option("gt_chunk", 0)
    for r in (b, c, e):
        assert np.array_equal(a[0], r[0])
        assert np.array_equal(a[1].view(np.uint64), r[1].view(np.uint64))


def test_gt_tc_ties_and_degenerate_queries(port):
    X = _data(30000, 48, 9)
    X[10000:20000] = X[:10000]          # every point twice: ties resolve to the lower id
    X[25000:25050] = 0.0                 # zero rows
    rng = np.random.default_rng(2)
    Q = _data(12, 48, 10)
    Q[1] = 0.0                           # all-zero query: every score ties at 0 -> ids 0..topn-1
    Q[2] *= 1e20
    Q[3] *= 1e-25
    Q[4] = 0.0
    Q[4, 5] = 1.0                        # one-hot
    Q[5] = X[123]                        # a data point
    Q[6, ::2] *= 1e6                     # lopsided coordinates
    Q[7] = -X[77]
    Q[8] = rng.standard_normal(48).astype(np.float32) * 1e-3
    ids, sc = _check(port, X, Q, 100)
    assert np.array_equal(ids[1], np.arange(100))


@pytest.mark.parametrize("scale", [1e-18, 3e12, 1e-30])
def test_gt_tc_rescaled_data(port, scale):
    X = (_data(20000, 64, 21) * np.float32(scale)).astype(np.float32)
    Q = _data(20, 64, 22)
    _check(port, X, Q, 20)


def test_gt_tc_near_duplicates_overflow_to_exact(port):
    """More than a candidate list of points within 2*eps of each other: the
    filter cannot prune, the flagged queries are scored exactly."""
    rng = np.random.default_rng(5)
    base = _data(1, 32, 1)[0]
    X = (base[None, :] + 1e-5 * rng.standard_normal((30000, 32))).astype(np.float32)
    Q = np.stack([base, -base, rng.standard_normal(32).astype(np.float32)]).astype(np.float32)
    Q = np.concatenate([Q, _data(5, 32, 3)]).astype(np.float32)
    _check(port, X, Q, 10)


def test_gt_tc_device_entry_and_config2_shape(port):
    import torch
    import paper_2112_02179_b200 as P
    from paper_2112_02179_b200 import datagen
    cfg = datagen.CONFIGS["c2"]
    X = datagen.mixture_chunk(cfg, *datagen.mixture_params(cfg, 3), 0, 300000, 3).numpy()
    Q = datagen.queries(cfg, 64, seed=6).numpy()
    ri, rs = port.brute_force_topn(X, Q, 100)
    di, ds = P.brute_force_topn_device(torch.from_numpy(X).cuda(), torch.from_numpy(Q).cuda(), 100)
    assert np.array_equal(di.cpu().numpy(), ri)
    assert np.array_equal(ds.cpu().numpy().view(np.uint64), rs.view(np.uint64))
