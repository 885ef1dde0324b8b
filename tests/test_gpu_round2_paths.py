"""Round-2 code paths that the default plans choose by shape, exercised on and
off against the CPU oracle (score_query + partial_sort,
proj/core/src/pq_index.cpp:212-250, proj/tools/main.cpp:229-243) — ids and
score bits must not depend on any of them:

* small batches: programmatic dependent launch (LUT -> scan -> merge) and the
  one-shot sorted merge;
* K2-T: one / two query tiles per CTA, the query operand in shared memory / in
  TMEM, the Cauchy-Schwarz bound, and the parallel exact fallback for queries
  whose candidates cannot be pruned (near-duplicate points) or that lie
  outside the scaling range;
* an index trained by the GPU apcpq trainer (large scale levels)."""
import contextlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DEFAULTS = dict(pdl=1, merge_oneshot=1, scan_lut_fused=1, scan_tc=1, scan_tc_min_batch=8, scan_tc_min_work=8000000, scan_tc_qt=2, scan_tc_at=1, scan_tc_cs=1,
                scan_tc_qh=0, scan_filter=0)


@contextlib.contextmanager
def _opts(**kw):
    import paper_2112_02179_b200 as P
    try:
        for k, v in kw.items():
            P.set_option(k, v)
        yield
    finally:
        for k, v in DEFAULTS.items():
            P.set_option(k, v)


def _same(a, b):
    assert np.array_equal(a[0], b[0])
    assert a[1].tobytes() == b[1].tobytes()


@pytest.mark.parametrize("cfg_name,n,B,topn", [("c3", 300000, 1, 100), ("c3", 300000, 3, 100), ("c2", 200000, 4, 10),
                                               ("c1", 50000, 2, 10), ("c4", 150000, 1, 100)])
def test_small_batch_pdl_and_oneshot_merge(port, cfg_name, n, B, topn):
    import paper_2112_02179_b200 as P
    from paper_2112_02179_b200 import datagen
    cfg = datagen.CONFIGS[cfg_name]
    data = datagen.synth_index(cfg, seed=31, n=n)
    Q = datagen.queries(cfg, B, seed=32).numpy()
    idx = P.deserialize(data, device=0)
    ref = port.parse(data).search(Q, topn, threads=4)
    for pdl in (0, 1):
        for one in (0, 1):
            for lf in (0, 1):  # LUT kernel before the scan / tables built inside the scan
                with _opts(pdl=pdl, merge_oneshot=one, scan_lut_fused=lf):
                    for _ in range(2):  # back-to-back searches on one stream
                        _same(P.search(idx, Q, topn), ref)


@pytest.mark.parametrize("cfg_name,n,B,topn", [("c3", 200000, 512, 100), ("c3", 120000, 700, 50),
                                               ("c4", 200000, 300, 100), ("c2", 100000, 1024, 100)])
def test_tscan_kernel_variants_agree(port, cfg_name, n, B, topn):
    import paper_2112_02179_b200 as P
    from paper_2112_02179_b200 import datagen
    cfg = datagen.CONFIGS[cfg_name]
    data = datagen.synth_index(cfg, seed=41, n=n)
    Q = datagen.queries(cfg, B, seed=42, mixture_seed=41).numpy()
    idx = P.deserialize(data, device=0)
    assert P.plan_info(idx, B, topn)["filter"] == 2
    ref = port.parse(data).search(Q, topn, threads=8)
    for qt in (1, 2):
        for at in (0, 1):
            for cs in (0, 1):
                with _opts(scan_tc_qt=qt, scan_tc_at=at, scan_tc_cs=cs):
                    _same(P.search(idx, Q, topn), ref)
    with _opts(scan_tc_qh=1):  # hi/lo query operand (taken for kpad <= 112: the c2 case)
        _same(P.search(idx, Q, topn), ref)


def test_tscan_parallel_fallback(port):
    """Near-duplicate points (more than a candidate list within 2 eps of the
    K-th best) and queries outside the scaling range: the flagged queries are
    scored by the parallel exact fallback kernels."""
    import paper_2112_02179_b200 as P
    from paper_2112_02179_b200 import datagen, pcpqidx
    cfg = datagen.CONFIGS["c2"]
    data = datagen.synth_index(cfg, seed=51, n=60000)
    ix = pcpqidx.deserialize(bytes(data) if not isinstance(data, bytes) else data)
    # 40,000 copies of one point's codes: every query sees 40,000 tied scores
    ix.center_codes[10000:50000] = ix.center_codes[7]
    ix.scalar_codes[10000:50000] = ix.scalar_codes[7]
    data2 = pcpqidx.serialize(ix)
    Q = datagen.queries(cfg, 300, seed=52, mixture_seed=51).numpy()
    Q[5] = 0.0
    Q[9] *= 1e-30
    Q[11] *= 1e25
    idx = P.deserialize(data2, device=0)
    with _opts(scan_tc_min_batch=1, scan_tc_min_work=0):
        assert P.plan_info(idx, Q.shape[0], 100)["filter"] == 2
        got = P.search(idx, Q, 100)
    ref = port.parse(data2).search(Q, 100, threads=8)
    _same(got, ref)


def test_tscan_on_gpu_trained_apcpq_index(port):
    """The configured kind of index (anisotropic, quantized scales with a few
    large levels) built by the GPU trainer: K2-T, K2-F and the exact scan
    against the oracle on the same image."""
    import paper_2112_02179_b200 as P
    from paper_2112_02179_b200 import datagen
    cfg = datagen.CONFIGS["c2"]
    centers, w = datagen.mixture_params(cfg, 61)
    X = datagen.mixture_chunk(cfg, centers, w, 0, 40000, 61).numpy()
    img = P.build_pq_index(X, P.PQConfig(method="apcpq", quantize_scalars=True, m=cfg.m, k=cfg.k, s=cfg.s,
                                         t_frac=cfg.t_frac, max_iters=8, seed=3))
    Q = datagen.queries(cfg, 400, seed=62, mixture_seed=61).numpy()
    idx = P.deserialize(img, device=0)
    ref = port.parse(img).search(Q, 100, threads=8)
    assert P.plan_info(idx, 400, 100)["filter"] == 2
    _same(P.search(idx, Q, 100), ref)
    with _opts(scan_tc=0):
        _same(P.search(idx, Q, 100), ref)
    with _opts(scan_tc=0, scan_filter=0):
        _same(P.search(idx, Q, 100), ref)


def test_tscan_two_tiles_with_a_padded_tile(port):
    """5 query tiles: the two-tile kernel pads a sixth, empty tile."""
    import paper_2112_02179_b200 as P
    from paper_2112_02179_b200 import datagen
    cfg = datagen.CONFIGS["c3"]
    data = datagen.synth_index(cfg, seed=71, n=150000)
    Q = datagen.queries(cfg, 600, seed=72).numpy()
    idx = P.deserialize(data, device=0)
    assert P.plan_info(idx, 600, 100)["filter"] == 2
    _same(P.search(idx, Q, 100), port.parse(data).search(Q, 100, threads=8))


@pytest.mark.parametrize("d,B", [(130, 300), (160, 700), (200, 64), (300, 40)])
def test_gt_tc_other_kernel_variants(port, d, B):
    """Ground truth at dimensions that pick the two-tile kernel (113..172), the
    128-column tiles (173..) and the TMEM query operand (>= 177 -> kpad >= 192)."""
    import paper_2112_02179_b200 as P
    rng = np.random.default_rng(d)
    c = rng.standard_normal((32, d)).astype(np.float32)
    X = c[rng.integers(0, 32, 30000)] + 0.3 * rng.standard_normal((30000, d)).astype(np.float32)
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    Q = X[rng.integers(0, 30000, B)] + 0.1 * rng.standard_normal((B, d)).astype(np.float32)
    X, Q = np.ascontiguousarray(X, np.float32), np.ascontiguousarray(Q, np.float32)
    ids, sc = P.brute_force_topn_batch(X, Q, 50)
    ri, rs = port.brute_force_topn(X, Q, 50)
    assert np.array_equal(ids, ri)
    assert np.array_equal(sc.view(np.uint64), rs.view(np.uint64))
