"""Tensor-core (tcgen05, 4-way tf32 split) LUT build — tolerance mode.

Scores are not bit-identical to the reference's sequential fp32 LUT, so the
north-star tolerance applies: every returned score agrees with the exact one
within 1e-5 x max|score| of its query, and the top-n differs from the exact
top-n only across ties within that tolerance."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.mark.parametrize("cfg_name,n,B", [("c4", 20000, 384), ("c2", 30000, 256), ("c3", 30000, 200)])
def test_tc_lut_search_within_tolerance(port, cfg_name, n, B):
    import paper_2112_02179_b200 as P
    from paper_2112_02179_b200 import datagen
    cfg = datagen.CONFIGS[cfg_name]
    data = datagen.synth_index(cfg, seed=11, n=n)
    Q = datagen.queries(cfg, B, seed=12).numpy()
    idx = P.deserialize(data, device=0)
    K = cfg.topn
    P.set_option("lut_tensor_cores", 1)
    try:
        ids, sc = P.search(idx, Q, K)
    finally:
        P.set_option("lut_tensor_cores", 0)
    pi = port.parse(data)
    worst = 0.0
    for b in range(0, B, max(1, B // 24)):
        exact, _ = pi.score_query(Q[b])
        scale = float(np.abs(exact).max())
        err = np.abs(sc[b].astype(np.float64) - exact[ids[b]].astype(np.float64)).max()
        worst = max(worst, err / scale)
        kth = np.sort(exact)[::-1][K - 1]
        # every returned point is within tolerance of the exact K-th score ...
        assert (exact[ids[b]] >= kth - 2 * TOL * scale).all()
        # ... and every point clearly above it is returned
        must = np.nonzero(exact > kth + 2 * TOL * scale)[0]
        assert np.isin(must, ids[b]).all()
    assert worst <= TOL, worst


def test_tc_lut_is_off_by_default_and_exact(port):
    import paper_2112_02179_b200 as P
    from paper_2112_02179_b200 import datagen
    cfg = datagen.CONFIGS["c4"]
    data = datagen.synth_index(cfg, seed=13, n=8000)
    Q = datagen.queries(cfg, 160, seed=14).numpy()
    ids, sc = P.search(P.deserialize(data, device=0), Q, 10)
    rids, rsc = port.parse(data).search(Q, 10, threads=8)
    assert np.array_equal(ids, rids) and sc.tobytes() == rsc.tobytes()
