"""K2-F, the fp16 pre-score filter of the batch scan (JOINT8 layouts with
k = 16 and raw fp16 alpha (config 3) in query groups of 16; PLANES with 8-bit centers and 4-bit scales
(config 4, k = 256) in groups of 4): it only decides which points get
the exact score, so the results must be identical — ids, bit-exact scores,
tie order — with the filter on, with it off, and to the CPU oracle, also on
adversarial indexes (duplicate points -> ties, tiny / huge / negative scale
values, sections without scale, zero and lopsided queries)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _cuda_core_paths():
    """This module tests the CUDA-core filter K2-F: keep the tensor-core filter
    (K2-T, the default from 16 queries up) out of the way."""
    import paper_2112_02179_b200 as P
    P.set_option("scan_tc", 0)
    P.set_option("scan_filter", 1)  # (opt-in by default)
    try:
        yield
    finally:
        P.set_option("scan_tc", 1)
        P.set_option("scan_filter", 0)


def _search_both(data, Q, topn):
    import paper_2112_02179_b200 as P
    idx = P.deserialize(data, device=0)
    try:
        P.set_option("scan_filter", 1)
        on = P.search(idx, Q, topn)
        P.set_option("scan_filter", 0)
        off = P.search(idx, Q, topn)
    finally:
        P.set_option("scan_filter", 1)
    return on, off


def _check(port, data, Q, topn):
    (ids, sc), (ids0, sc0) = _search_both(data, Q, topn)
    rids, rsc = port.parse(data).search(Q, topn, threads=8)
    assert np.array_equal(ids0, rids) and sc0.tobytes() == rsc.tobytes()
    assert np.array_equal(ids, rids), np.argwhere(ids != rids)[:5]
    assert sc.tobytes() == rsc.tobytes()


@pytest.mark.parametrize("cfg_name,n,B,topn", [("c1", 40000, 48, 10), ("c2", 60000, 32, 100),
                                               ("c2", 30000, 20, 7), ("c4", 300000, 12, 100),
                                               ("c4", 100000, 7, 20), ("c3", 200000, 32, 100),
                                               ("c3", 50000, 19, 10)])
def test_filter_synthetic(port, cfg_name, n, B, topn):
    from paper_2112_02179_b200 import datagen
    cfg = datagen.CONFIGS[cfg_name]
    data = datagen.synth_index(cfg, seed=11, n=n)
    Q = datagen.queries(cfg, B, seed=12).numpy()
    _check(port, data, Q, topn)


def _adversarial(n, m, dbar, s, lam, seed, dups=0):
    from paper_2112_02179_b200 import pcpqidx
    rng = np.random.default_rng(seed)
    k = 16
    cb = rng.standard_normal((m, k, dbar)).astype(np.float32)
    cc = rng.integers(0, k, (n, m)).astype(np.uint32)
    sc = rng.integers(0, s, (n, m)).astype(np.uint8)
    if dups:
        cc[dups:2 * dups] = cc[:dups]
        sc[dups:2 * dups] = sc[:dups]
    ix = pcpqidx.IndexArrays(method=2, n=n, d=m * dbar, padded_d=m * dbar, m=m, k=k, scales=s, t=0.2,
                             codebooks=cb, scalar_codebooks=lam.astype(np.float32), center_codes=cc,
                             scalar_codes=sc, raw_alphas=None)
    return pcpqidx.serialize(ix), rng


@pytest.mark.parametrize("case", ["ties", "tiny", "huge", "mixed", "zero_sections", "near_overflow"])
def test_filter_adversarial(port, case):
    m, dbar, s, n = 13, 3, 8, 20000
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
    elif case == "near_overflow":  # products near fp32's top: sigma out of range, the exact path decides
        lam = lam * 1e30
    data, rng = _adversarial(n, m, dbar, s, lam, 3, dups=5000 if case == "ties" else 0)
    Q = rng.standard_normal((48, m * dbar)).astype(np.float32)
    Q[5] = 0.0                                   # all scores +-0: ties broken by id
    Q[7, :dbar] *= 1e6                           # one dominant section
    Q[9] *= 1e-20  # with the 'tiny' scales: products below fp32's range, no filter for this query
    if case == "near_overflow":
        Q[11] *= 1e7
    _check(port, data, Q, 50)


def test_filter_plan_c4(port):
    """config 4's layout takes the filter in groups of 4 (the exact fp32 table of k = 256 admits 2)."""
    import paper_2112_02179_b200 as P
    from paper_2112_02179_b200 import datagen
    data = datagen.synth_index(datagen.CONFIGS["c4"], seed=2, n=20000)
    idx = P.deserialize(data, device=0)
    pl = P.plan_info(idx, 64, 100)
    assert pl["filter"] == 1 and pl["nq"] == 4
    P.set_option("scan_filter", 0)
    try:
        assert P.plan_info(idx, 64, 100)["filter"] == 0
    finally:
        P.set_option("scan_filter", 1)


def test_filter_plan_c3_raw_alpha(port):
    """config 3 (raw fp16 alpha) takes the filter in groups of 16; alphas far
    outside [1/16, 16] keep the exact scan (fp16 eta_hat range)."""
    import paper_2112_02179_b200 as P
    from paper_2112_02179_b200 import datagen, pcpqidx
    data = datagen.synth_index(datagen.CONFIGS["c3"], seed=2, n=20000)
    idx = P.deserialize(data, device=0)
    assert P.plan_info(idx, 64, 100)["filter"] == 1
    rng = np.random.default_rng(4)
    n, m, dbar = 5000, 8, 4
    ra = (rng.standard_normal((n, m)) * 1e-3).astype(np.float16).astype(np.float32)
    ix = pcpqidx.IndexArrays(method=2, n=n, d=m * dbar, padded_d=m * dbar, m=m, k=16, scales=0, t=0.2,
                             codebooks=rng.standard_normal((m, 16, dbar)).astype(np.float32),
                             scalar_codebooks=np.zeros((m, 0), np.float32),
                             center_codes=rng.integers(0, 16, (n, m)).astype(np.uint32), scalar_codes=None,
                             raw_alphas=ra)
    data2 = pcpqidx.serialize(ix)
    idx2 = P.deserialize(data2, device=0)
    assert P.plan_info(idx2, 64, 10)["filter"] == 0
    Q = rng.standard_normal((20, m * dbar)).astype(np.float32)
    _check(port, data2, Q, 10)


@pytest.mark.parametrize("cfg_name,n,B,topn", [("c2", 90000, 32, 100), ("c4", 120000, 8, 50)])
def test_filter_sharded_merge(port, cfg_name, n, B, topn):
    """Shards keep global ids through the carried top-K (own-range test uses
    the shard's id base): 3 shards + the device merge equal the unsharded oracle."""
    import torch
    import paper_2112_02179_b200 as P
    from paper_2112_02179_b200 import datagen
    from paper_2112_02179_b200.sharded import shard_range
    cfg = datagen.CONFIGS[cfg_name]
    data = datagen.synth_index(cfg, seed=21, n=n)
    Qn = datagen.queries(cfg, B, seed=22).numpy()
    Q = torch.from_numpy(Qn).cuda()
    keys = []
    for r in range(3):
        b, e = shard_range(n, r, 3)
        ix = P.deserialize(data, device=0, shard=(b, e))
        assert P.plan_info(ix, B, topn)["filter"] == 1
        _, _, k = P.search_device(ix, Q, topn, want_keys=True)
        keys.append(k)
    ids, top, _ = P.merge_device(torch.stack(keys), topn)
    torch.cuda.synchronize()
    rids, rsc = port.parse(data).search(Qn, topn, threads=8)
    assert np.array_equal(ids.cpu().numpy(), rids)
    assert top.cpu().numpy().tobytes() == rsc.tobytes()


@pytest.mark.parametrize("case", ["zero_sections", "negative", "subnormal"])
def test_filter_raw_alpha_adversarial(port, case):
    """Raw fp16 alpha (config 3's layout) under the filter: sections whose alphas
    are all zero, negative alphas, fp16-subnormal alphas next to normal ones."""
    import paper_2112_02179_b200 as P
    from paper_2112_02179_b200 import pcpqidx
    rng = np.random.default_rng(11)
    n, m, dbar = 30000, 16, 4
    ra = rng.uniform(0.1, 1.5, (n, m))
    if case == "zero_sections":
        ra[:, ::4] = 0.0
    elif case == "negative":
        ra *= np.where(rng.random((n, m)) < 0.5, -1.0, 1.0)
    else:
        ra[::3, 1] = 3e-6  # fp16 subnormal
        ra[::5, 2] = -6e-8
    ra = ra.astype(np.float16).astype(np.float32)
    cc = rng.integers(0, 16, (n, m)).astype(np.uint32)
    cc[5000:10000] = cc[:5000]
    ra[5000:10000] = ra[:5000]
    ix = pcpqidx.IndexArrays(method=2, n=n, d=m * dbar, padded_d=m * dbar, m=m, k=16, scales=0, t=0.2,
                             codebooks=rng.standard_normal((m, 16, dbar)).astype(np.float32),
                             scalar_codebooks=np.zeros((m, 0), np.float32), center_codes=cc, scalar_codes=None,
                             raw_alphas=ra)
    data = pcpqidx.serialize(ix)
    idx = P.deserialize(data, device=0)
    assert P.plan_info(idx, 48, 30)["filter"] == 1
    Q = rng.standard_normal((48, m * dbar)).astype(np.float32)
    Q[3] = 0.0
    Q[4, :dbar] *= 1e5
    _check(port, data, Q, 30)
