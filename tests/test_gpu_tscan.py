"""K2-T, the tensor-core pre-score filter of the batch scan (csrc/pcpqg_tscan.cu,
DESIGN.md §4): a tcgen05 fp16 GEMM of the queries against the decoded points
decides which pairs can reach the top-K; those are re-scored with the
reference's exact fp32 chain (proj/core/src/pq_index.cpp:212-244) and ordered
by (score desc, id asc) (proj/tools/main.cpp:233-237).  Results must be
identical — ids, bit-exact scores, tie order — with K2-T on, with it off (the
CUDA-core scans), and to the CPU oracle, on every layout it takes (JOINT8
dbar 1/2/4/8, PLANES raw fp16 alpha, PLANES 8-bit centers / 4-bit scales) and
on adversarial indexes: duplicate points (ties, list overflow -> exact
fallback), scales from 1e-30 to 1e30, zero sections, zero / lopsided /
1e-20 queries (the scaling-range guard)."""
import contextlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@contextlib.contextmanager
def _opts(**kw):
    import paper_2112_02179_b200 as P
    try:
        for k, v in kw.items():
            P.set_option(k, v)
        yield
    finally:
        P.set_option("scan_tc", 1)
        P.set_option("scan_tc_min_batch", 8)
        P.set_option("scan_tc_min_work", 8000000)
        P.set_option("scan_filter", 0)


def _check(port, data, Q, topn, expect_tc=True):
    import paper_2112_02179_b200 as P
    idx = P.deserialize(data, device=0)
    with _opts(scan_tc=1, scan_tc_min_batch=1, scan_tc_min_work=0):
        plan = P.plan_info(idx, Q.shape[0], topn)
        ids, sc = P.search(idx, Q, topn)
    if expect_tc:
        assert plan["filter"] == 2, plan
    with _opts(scan_tc=0):
        ids0, sc0 = P.search(idx, Q, topn)
    rids, rsc = port.parse(data).search(Q, topn, threads=8)
    assert np.array_equal(ids0, rids) and sc0.tobytes() == rsc.tobytes()
    bad = np.argwhere(ids != rids)
    assert bad.size == 0, (bad[:5], ids[bad[0][0]][:8], rids[bad[0][0]][:8])
    assert sc.tobytes() == rsc.tobytes()
    return idx


@pytest.mark.parametrize("cfg_name,n,B,topn", [("c1", 40000, 300, 10), ("c2", 60000, 300, 100),
                                               ("c2", 30000, 20, 7), ("c2", 50000, 129, 256),
                                               ("c3", 200000, 256, 100), ("c3", 50000, 19, 10),
                                               ("c4", 300000, 256, 100), ("c4", 100000, 7, 20)])
def test_tscan_synthetic(port, cfg_name, n, B, topn):
    from paper_2112_02179_b200 import datagen
    cfg = datagen.CONFIGS[cfg_name]
    data = datagen.synth_index(cfg, seed=21, n=n)
    Q = datagen.queries(cfg, B, seed=22).numpy()
    _check(port, data, Q, topn)


def _index(n, m, dbar, k, s, lam, seed, dups=0, same=False, raw=None):
    from paper_2112_02179_b200 import pcpqidx
    rng = np.random.default_rng(seed)
    cb = rng.standard_normal((m, k, dbar)).astype(np.float32)
    cc = rng.integers(0, k, (n, m)).astype(np.uint32)
    sc = rng.integers(0, max(s, 1), (n, m)).astype(np.uint8) if s else None
    if same:
        cc[:] = cc[0]
        if sc is not None:
            sc[:] = sc[0]
    if dups:
        cc[dups:2 * dups] = cc[:dups]
        if sc is not None:
            sc[dups:2 * dups] = sc[:dups]
    ix = pcpqidx.IndexArrays(method=2, n=n, d=m * dbar, padded_d=m * dbar, m=m, k=k, scales=s, t=0.2,
                             codebooks=cb,
                             scalar_codebooks=(lam.astype(np.float32) if s else np.zeros((m, 0), np.float32)),
                             center_codes=cc, scalar_codes=sc, raw_alphas=raw)
    return pcpqidx.serialize(ix), rng


@pytest.mark.parametrize("dbar", [1, 2, 4, 8])
@pytest.mark.parametrize("case", ["plain", "ties", "tiny", "huge", "mixed", "zero_sections", "near_overflow"])
def test_tscan_adversarial_joint8(port, dbar, case):
    m, s, n, k = 24 if dbar <= 2 else 12, 8, 20000, 16
    rng = np.random.default_rng(7)
    lam = np.tile(np.linspace(-1.0, 1.5, s), (m, 1))
    if case == "tiny":
        lam = lam * 1e-30
    elif case == "huge":
        lam = lam * 1e18
    elif case == "mixed":
        lam = lam * (10.0 ** rng.integers(-12, 12, (m, 1)))
    elif case == "zero_sections":
        lam[::3] = 0.0
    elif case == "near_overflow":
        lam = lam * 1e30
    data, rng = _index(n, m, dbar, k, s, lam, 3, dups=5000 if case == "ties" else 0)
    Q = rng.standard_normal((300, m * dbar)).astype(np.float32)
    Q[5] = 0.0                      # all scores +-0: ties broken by id (exact fallback)
    Q[7, :dbar] *= 1e6              # one dominant section
    Q[9] *= 1e-20                   # with 'tiny' scales: products below fp32's range
    Q[11] *= 1e-3
    if case == "near_overflow":
        Q[13] *= 1e7
    _check(port, data, Q, 50)


@pytest.mark.parametrize("k,s,dbar", [(256, 16, 4), (256, 16, 2), (300, 4, 4), (16, 0, 4), (16, 0, 2), (64, 1, 4)])
def test_tscan_planes(port, k, s, dbar):
    """PLANES layouts: 8/16-bit centers with 4-bit scale codes, raw alpha, one-level scales."""
    m, n = 16, 30000
    rng = np.random.default_rng(k + s + dbar)
    lam = rng.standard_normal((m, max(s, 1))) * 0.7
    raw = None
    if s == 0:
        raw = (rng.standard_normal((n, m)) * 10.0 ** rng.integers(-4, 3, (1, m))).astype(np.float16).astype(np.float32)
    data, rng = _index(n, m, dbar, k, s, lam, 5, raw=raw)
    Q = rng.standard_normal((260, m * dbar)).astype(np.float32)
    _check(port, data, Q, 100)


def test_tscan_overflow_fallback(port):
    """every point identical: no list can be pruned below capacity, every
    query falls back to the exact full scan in the finish kernel."""
    m, dbar, s, n = 8, 2, 4, 6000
    lam = np.tile(np.linspace(0.5, 1.0, s), (m, 1))
    data, rng = _index(n, m, dbar, 16, s, lam, 9, same=True)
    Q = rng.standard_normal((130, m * dbar)).astype(np.float32)
    _check(port, data, Q, 10)


def test_tscan_small_n_large_k(port):
    """K (256) > what a short shard holds per range; n barely above the
    eligibility floor."""
    m, dbar, s, n = 8, 4, 8, 2100
    lam = np.tile(np.linspace(-1.0, 1.0, s), (m, 1))
    data, rng = _index(n, m, dbar, 16, s, lam, 11)
    Q = rng.standard_normal((140, m * dbar)).astype(np.float32)
    _check(port, data, Q, 256)


def test_tscan_not_taken():
    """K > 256, small batches and unsupported dbar keep the CUDA-core scans."""
    import paper_2112_02179_b200 as P
    from paper_2112_02179_b200 import datagen
    data = datagen.synth_index(datagen.CONFIGS["c2"], seed=2, n=20000)
    idx = P.deserialize(data, device=0)
    assert P.plan_info(idx, 1000, 100)["filter"] == 2
    assert P.plan_info(idx, 1000, 300)["filter"] != 2
    # mid batches take K2-T from n * B >= 8e6 pairs, at least 8 queries (the measured crossover,
    # tools/ab_midbatch.py)
    assert P.plan_info(idx, 200, 100)["filter"] != 2
    assert P.plan_info(idx, 256, 100)["filter"] == 2
    assert P.plan_info(idx, 400, 100)["filter"] == 2
    with _opts(scan_tc_min_work=8 * 20000):
        assert P.plan_info(idx, 8, 100)["filter"] == 2
        assert P.plan_info(idx, 7, 100)["filter"] != 2
    with _opts(scan_tc=0):
        assert P.plan_info(idx, 1000, 100)["filter"] != 2


def test_tscan_sharded_ids(port):
    """a shard's K2-T rows carry global ids: the shard top-n of [b, e) equals
    the oracle's top-n over those points."""
    import paper_2112_02179_b200 as P
    from paper_2112_02179_b200 import datagen
    cfg = datagen.CONFIGS["c2"]
    data = datagen.synth_index(cfg, seed=4, n=40000)
    Q = datagen.queries(cfg, 260, seed=5).numpy()
    b, e = 13000, 31000
    idx = P.deserialize(data, device=0, shard=(b, e))
    with _opts(scan_tc=1, scan_tc_min_batch=1, scan_tc_min_work=0):
        assert P.plan_info(idx, 260, 50)["filter"] == 2
        ids, sc = P.search(idx, Q, 50)
    pi = port.parse(data)
    for qi in range(0, 260, 37):
        s, _ = pi.score_query(Q[qi])
        part = s[b:e]
        order = np.lexsort((np.arange(b, e), -part))[:50]
        assert np.array_equal(ids[qi], order + b)
        assert sc[qi].tobytes() == part[order].tobytes()
