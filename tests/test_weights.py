"""pcpqg_aniso_weights (host, C ABI) against the reference's aniso_weights
(proj/core/src/clustering.cpp:204-217) bit for bit: the weights feed every
score-aware kernel, so they must be identical."""
import numpy as np
import pytest


def test_weights_match_reference_bits():
    from oracle.oracle import Ref
    if not Ref.available():
        pytest.skip("oracle/_ref not built")
    import paper_2112_02179_b200 as P
    R = Ref()
    rng = np.random.default_rng(5)
    for dbar, t in ((2, 0.2), (4, 0.2), (4, 0.05), (3, 1.7), (8, 0.3), (4, 0.0)):
        x = rng.standard_normal((300, dbar)).astype(np.float32) * rng.uniform(0.01, 3.0, (300, 1)).astype(np.float32)
        x[::17] = 0.0
        hp, hb = P.aniso_weights(x, t)
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


def test_weights_frozen_values():
    """Frozen quadrature values of test_clustering.cpp:59-62 (t = 0.2, |x| = 1, dbar = 4)."""
    import paper_2112_02179_b200 as P
    x = np.array([[1.0, 0.0, 0.0, 0.0]], np.float32)
    hp, hb = P.aniso_weights(x, 0.2)
    assert hp[0] == pytest.approx(0.00774786647816975, rel=1e-9)  # doctest::Approx(...).epsilon(1e-9)
    assert hb[0] == pytest.approx(6.279226344747205e-05, rel=1e-9)


def test_weights_errors():
    import paper_2112_02179_b200 as P
    x = np.ones((3, 4), np.float32)
    for t, xx in ((-1.0, x), (float("inf"), x), (0.2, np.ones((3, 1), np.float32))):
        with pytest.raises(P.PcpqError) as e:
            P.aniso_weights(xx, t)
        assert e.value.code == P.errc.data


def test_restated_sin_matches_host_libm():
    """The sin the GPU weights kernel evaluates (csrc/pcpqg_hostsin.cuh) against
    this host's std::sin — the one the reference's sin_power_integral calls
    (proj/core/src/numerics.cpp:174-186) — on the library's self-check arguments,
    evaluated on the host (no GPU needed)."""
    import paper_2112_02179_b200 as P
    bad, total = P.sin_selfcheck(-1)
    assert total > 300000
    assert bad == 0


def test_committed_sincos_table_is_the_host_libms():
    """csrc/pcpqg_sincostab.inc was read from a libm binary (tools/gen_sincostab.py);
    it must equal the table of the C library on this machine."""
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "tools"))
    import gen_sincostab as G
    path = G.find_libm()
    if path is None:
        pytest.skip("libm.so.6 not found")
    try:
        tab = G.extract(path)
    except RuntimeError as e:
        pytest.skip(str(e))
    inc = os.path.join(root, "paper_2112_02179_b200", "csrc", "pcpqg_sincostab.inc")
    vals = []
    with open(inc) as f:
        for line in f:
            if line.startswith("//"):
                continue
            vals += [float.fromhex(v) for v in line.replace(",", " ").split()]
    assert len(vals) == 4 * G.ENTRIES
    assert np.array(vals).tobytes() == np.array(tab).tobytes()
