"""GPU training: build_pq_index(method = kmeans / pcpq / apcpq / aniso) with
the Lloyd iterations on the GPU must serialize to the reference's image byte
for byte (golden: tests/golden/train_*.npz from make_golden_train.py; live:
the reference library where oracle/_ref is built)."""
import glob
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "train_*.npz")))

pytestmark = pytest.mark.gpu


def test_train_fixtures_present():
    assert len(NAMES) >= 22


@pytest.mark.parametrize("name", NAMES)
def test_gpu_build_matches_reference_bytes(name):
    import paper_2112_02179_b200 as P
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    m, k, s, iters, seed = (int(v) for v in z["cfg"])
    method = str(z["method"]) if "method" in z.files else "kmeans"
    quant = bool(z["quantize"]) if "quantize" in z.files else False
    cfg = P.PQConfig(method=method, quantize_scalars=quant, m=m, k=k, s=s, t_frac=float(z["t_frac"]),
                     max_iters=iters, tol=float(z["tol"]), seed=seed)
    img = P.build_pq_index(z["data"], cfg)
    ref = z["image"].tobytes()
    assert len(img) == len(ref)
    assert img == ref


def test_gpu_kmeans_build_larger_vs_reference_live():
    from oracle.oracle import Ref
    if not Ref.available():
        pytest.skip("oracle/_ref not built")
    import paper_2112_02179_b200 as P
    R = Ref()
    X = R.generate_dataset("clustered", 30000, 24, 11)
    for method, quant, m, k, s in (("kmeans", False, 8, 16, 1), ("kmeans", False, 3, 64, 1),
                                   ("pcpq", True, 8, 16, 8), ("pcpq", False, 6, 16, 8),
                                   ("apcpq", True, 8, 16, 8), ("apcpq", False, 6, 16, 8), ("aniso", False, 8, 16, 1)):
        img = P.build_pq_index(X, P.PQConfig(method=method, quantize_scalars=quant, m=m, k=k, s=s, max_iters=15,
                                             seed=3))
        ref = R.build_index(X, method=method, quantize=quant, m=m, k=k, s=s, t_frac=0.2, max_iters=15,
                            tol=1e-6, seed=3)
        assert img == ref, (method, quant, m, k)


def test_gpu_kmeans_build_errors():
    import paper_2112_02179_b200 as P
    X = np.random.default_rng(0).standard_normal((50, 6)).astype(np.float32)
    for cfg in (P.PQConfig(method="kmeans", m=7, k=4), P.PQConfig(method="kmeans", m=2, k=1),
                P.PQConfig(method="kmeans", m=2, k=51), P.PQConfig(method="kmeans", m=2, k=4, max_iters=0),
                P.PQConfig(method="kmeans", m=2, k=4, tol=0.0)):
        with pytest.raises(P.PcpqError) as e:
            P.build_pq_index(X, cfg)
        assert e.value.code == P.errc.data
    bad = X.copy()
    bad[3, 2] = np.nan
    with pytest.raises(P.PcpqError) as e:
        P.build_pq_index(bad, P.PQConfig(method="kmeans", m=2, k=4))
    assert e.value.code == P.errc.data


def test_gpu_aniso_build_errors():
    import paper_2112_02179_b200 as P
    X = np.random.default_rng(1).standard_normal((60, 6)).astype(np.float32)
    with pytest.raises(P.PcpqError) as e:  # section width 1: score-aware solvers need >= 2
        P.build_pq_index(X, P.PQConfig(method="apcpq", m=6, k=4))
    assert e.value.code == P.errc.data
    with pytest.raises(P.PcpqError) as e:
        P.build_pq_index(X, P.PQConfig(method="apcpq", quantize_scalars=True, m=3, k=4, s=300))
    assert e.value.code == P.errc.data


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0], [0] * 40])
def test_gpu_multi_device_build_is_byte_identical(devices):
    """pcpqg_train_aniso_multi: the sections dealt round-robin to a device list
    (one host thread per entry; here the same GPU several times — the pool has
    one) must give the reference's bytes for every list, because each section
    is an independent problem (its own seeds Rng::mix(seed, 2j+1 / 2j+2),
    proj/core/src/pq_index.cpp:86-139).  40 entries > m: surplus devices idle."""
    import paper_2112_02179_b200 as P
    hit = 0
    for name in NAMES:
        z = np.load(os.path.join(GOLDEN, name + ".npz"))
        method = str(z["method"]) if "method" in z.files else "kmeans"
        if method not in ("aniso", "apcpq"):
            continue
        m, k, s, iters, seed = (int(v) for v in z["cfg"])
        quant = bool(z["quantize"]) if "quantize" in z.files else False
        cfg = P.PQConfig(method=method, quantize_scalars=quant, m=m, k=k, s=s, t_frac=float(z["t_frac"]),
                         max_iters=iters, tol=float(z["tol"]), seed=seed)
        assert P.build_pq_index(z["data"], cfg, device=devices) == z["image"].tobytes(), name
        hit += 1
    assert hit >= 4


def test_gpu_multi_device_build_errors():
    import paper_2112_02179_b200 as P
    X = np.random.default_rng(1).standard_normal((60, 6)).astype(np.float32)
    with pytest.raises(P.PcpqError) as e:
        P.build_pq_index(X, P.PQConfig(method="apcpq", m=3, k=4), device=[])
    assert e.value.code == P.errc.usage
    with pytest.raises(P.PcpqError) as e:
        P.build_pq_index(X, P.PQConfig(method="kmeans", m=3, k=4), device=[0, 0])
    assert e.value.code == P.errc.usage
    with pytest.raises(P.PcpqError):  # a device that does not exist
        P.build_pq_index(X, P.PQConfig(method="apcpq", m=3, k=4), device=[0, 99])


def test_gpu_scale_quantizer_level_sort_on_and_off():
    """The scale quantizer's per-level ordered sums (numerics.cpp:328-383) have
    two device paths: a stable counting sort by level + one run per level
    (train_level_sort, default, s <= 16) and one warp per level walking the
    whole assignment.  Both must give the reference's bytes, including
    sections whose quad count is not a multiple of 16 or of the 4096 chunk."""
    import paper_2112_02179_b200 as P
    hit = 0
    try:
        for flag in (0, 1):
            P.set_option("train_level_sort", flag)
            for name in NAMES:
                z = np.load(os.path.join(GOLDEN, name + ".npz"))
                method = str(z["method"]) if "method" in z.files else "kmeans"
                quant = bool(z["quantize"]) if "quantize" in z.files else False
                if method not in ("aniso", "apcpq") or not quant:
                    continue
                m, k, s, iters, seed = (int(v) for v in z["cfg"])
                cfg = P.PQConfig(method=method, quantize_scalars=True, m=m, k=k, s=s, t_frac=float(z["t_frac"]),
                                 max_iters=iters, tol=float(z["tol"]), seed=seed)
                assert P.build_pq_index(z["data"], cfg) == z["image"].tobytes(), (name, flag)
                hit += 1
            rng = np.random.default_rng(5)
            X = (rng.standard_normal((9001, 12)) * rng.gamma(2.0, 1.0, (9001, 1))).astype(np.float32)
            cfg = P.PQConfig(method="apcpq", quantize_scalars=True, m=3, k=8, s=16, max_iters=6, seed=9)
            img = P.build_pq_index(X, cfg)
            if flag == 0:
                first = img
            else:
                assert img == first
    finally:
        P.set_option("train_level_sort", 1)
    assert hit >= 2
