"""GPU anisotropic weights (csrc/pcpqg_weights.cu) against the
reference's aniso_weights (proj/core/src/clustering.cpp:204-217 ->
sin_power_integral, proj/core/src/numerics.cpp:174-186): bit for bit, through
the C ABI (pcpqg_aniso_weights_gpu)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_gpu_sin_matches_host_libm():
    import paper_2112_02179_b200 as P
    bad, total = P.sin_selfcheck(0)
    assert total > 300000
    assert bad == 0


def _rows(rng, n, dbar):
    x = rng.standard_normal((n, dbar)).astype(np.float32) * rng.uniform(0.01, 3.0, (n, 1)).astype(np.float32)
    x[::17] = 0.0
    return x


@pytest.mark.parametrize("dbar,t", [(2, 0.2), (4, 0.2), (4, 0.05), (3, 1.7), (8, 0.3), (4, 0.0), (5, 1e-9), (2, 40.0)])
def test_gpu_weights_match_reference_bits(dbar, t):
    from oracle.oracle import Ref
    if not Ref.available():
        pytest.skip("oracle/_ref not built")
    import paper_2112_02179_b200 as P
    R = Ref()
    rng = np.random.default_rng(11 + dbar)
    x = _rows(rng, 400, dbar)
    hp, hb = P.aniso_weights(x, t, device=0)
    for i in range(x.shape[0]):
        acc = 0.0
        for v in x[i].astype(np.float64):  # dotf's sequential order
            acc += v * v
        nrm = float(np.sqrt(acc))
        if nrm == 0.0:
            assert hp[i] == 0.0 and hb[i] == 0.0
            continue
        rp, rb = R.aniso_weights(nrm, t, dbar)
        assert hp[i].tobytes() == np.float64(rp).tobytes() and hb[i].tobytes() == np.float64(rb).tobytes(), (dbar, t, i)


@pytest.mark.parametrize("n,dbar,t", [(200_000, 4, 0.2), (100_000, 2, 0.2), (50_000, 8, 0.037)])
def test_gpu_weights_equal_host_path(n, dbar, t):
    """Large row sets (unit-norm data cut into sections, like the configs'):
    the GPU kernel against the host-thread path, which tests/test_weights.py
    pins to the reference."""
    import paper_2112_02179_b200 as P
    rng = np.random.default_rng(n)
    x = rng.standard_normal((n, dbar)).astype(np.float32)
    x *= (rng.uniform(0.05, 0.4, (n, 1)) / np.linalg.norm(x, axis=1, keepdims=True)).astype(np.float32)
    x[5] = 0.0
    g = P.aniso_weights(x, t, device=0)
    h = P.aniso_weights(x, t)
    assert g[0].tobytes() == h[0].tobytes()
    assert g[1].tobytes() == h[1].tobytes()


def test_gpu_weights_errors():
    import paper_2112_02179_b200 as P
    x = np.ones((3, 4), np.float32)
    for t, xx in ((-1.0, x), (float("inf"), x), (0.2, np.ones((3, 1), np.float32))):
        with pytest.raises(P.PcpqError) as e:
            P.aniso_weights(xx, t, device=0)
        assert e.value.code == P.errc.data
    hp, hb = P.aniso_weights(np.zeros((0, 4), np.float32), 0.2, device=0)
    assert hp.size == 0 and hb.size == 0


def test_trainer_uses_gpu_weights():
    """An apcpq build computes its weights on the GPU (and the golden training
    tests pin the resulting images to the reference's bytes)."""
    import paper_2112_02179_b200 as P
    rng = np.random.default_rng(3)
    x = rng.standard_normal((3000, 16)).astype(np.float32)
    cfg = P.PQConfig(method="apcpq", quantize_scalars=True, m=4, k=8, s=4, max_iters=3, seed=2)
    img = P.build_pq_index(x, cfg, device=0)
    assert P.train_weights_on_gpu()
    try:
        P.set_option("weights_gpu", 0)
        img_host = P.build_pq_index(x, cfg, device=0)
        assert not P.train_weights_on_gpu()
    finally:
        P.set_option("weights_gpu", 1)
    assert img == img_host
