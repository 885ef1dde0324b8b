"""Pin the CPU oracle (oracle/pcpq_oracle.c) to the reference: golden vectors
made by the unmodified reference library, and — where oracle/_ref is built —
the reference itself on fresh seeded cases."""
import numpy as np
import pytest

from tests import _golden

CASES = _golden.names()


@pytest.mark.parametrize("name", CASES)
def test_port_matches_golden(port, name):
    data, g = _golden.load(name)
    ix = port.parse(data)
    assert ix.serialize() == data  # bytewise-stable round trip (test_pq_index.cpp:179-193)
    Q = g["queries"]
    for b in range(Q.shape[0]):
        s, _ = ix.score_query(Q[b])
        assert s.tobytes() == g["scores"][b].tobytes()
    ids, top = ix.search(Q, 10, threads=2)
    assert np.array_equal(ids, g["ids10"])
    assert top.tobytes() == g["top10"].tobytes()
    ids, top = ix.search(Q, ix.n + 3, threads=1)
    assert np.array_equal(ids, g["idsx"])
    assert top.tobytes() == g["topx"].tobytes()
    eta, etal, _ = ix.build_lut(Q[0])
    assert eta.tobytes() == g["eta"].tobytes()
    assert etal.tobytes() == g["etal"].tobytes()
    _, cnt = ix.score_query(Q[0])
    assert np.array_equal(cnt, g["counters"])


@pytest.mark.parametrize("name", CASES)
def test_port_error_taxonomy(port, name):
    from oracle.oracle import OracleError
    data, g = _golden.load(name)
    bad = _golden.corruptions(name, data)
    for ename, code in zip(g["err_names"], g["err_codes"]):
        with pytest.raises(OracleError) as e:
            port.parse(bad[str(ename)])
        assert e.value.code == int(code), ename


def test_tie_rule_and_negative_zero(port):
    """The all-zero query scores every point +-0: the top-n is ids 0..n-1."""
    data, g = _golden.load("pcpq_q_ties")
    assert np.array_equal(g["ids10"][5], np.arange(10))
    ix = port.parse(data)
    ids, _ = ix.search(g["queries"][5:6], 10)
    assert np.array_equal(ids[0], np.arange(10))


def test_payload_bits(port):
    import os
    z = np.load(os.path.join(_golden.GOLDEN, "payload_bits.npz"))
    for (n, m, k, s), b in zip(z["grid"], z["bits"]):
        assert port.logical_payload_bits(int(n), int(m), int(k), int(s)) == int(b)


def test_dense_oracle_tolerance(port):
    """Reference acceptance check 1 (proj/tests/acceptance.cpp:126-187): table
    scores agree with a dense double reconstruction within 1e-5 * max|score|."""
    for name in CASES:
        data, g = _golden.load(name)
        from paper_2112_02179_b200 import pcpqidx
        ix = pcpqidx.deserialize(data)
        dbar = ix.dbar
        lam = (ix.scalar_codebooks[np.arange(ix.m)[None, :], ix.scalar_codes] if ix.scales
               else ix.raw_alphas).astype(np.float64)
        rec = ix.codebooks[np.arange(ix.m)[None, :], ix.center_codes].astype(np.float64) * lam[:, :, None]
        rec = rec.reshape(ix.n, ix.m * dbar)
        for b in range(5):
            q = np.zeros(ix.padded_d)
            q[: ix.d] = g["queries"][b]
            dense = rec @ q
            scale = max(np.abs(dense).max(), 1e-12)
            assert np.abs(g["scores"][b].astype(np.float64) - dense).max() <= 1e-5 * scale


ref_only = pytest.mark.skipif(not __import__("oracle.oracle", fromlist=["Ref"]).Ref.available(),
                              reason="oracle/_ref (reference library) not built")


@ref_only
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_port_matches_reference_live(port, seed):
    from oracle.oracle import Ref
    R = Ref()
    rng = np.random.default_rng(seed)
    for method, quant in [("pcpq", True), ("pcpq", False), ("apcpq", True), ("kmeans", False), ("scann", False)]:
        m = int(rng.integers(1, 6))
        d = m * int(rng.integers(2, 5)) - int(rng.integers(0, 2))
        k = int(rng.choice([2, 5, 16, 33]))
        s = int(rng.choice([1, 3, 8, 16]))
        x = R.generate_dataset("clustered", 200, d, seed * 7 + m)
        data = R.build_index(x, method, quant, m=m, k=k, s=s, max_iters=5, seed=seed)
        ri, pi = R.open(data), port.parse(data)
        Q = rng.standard_normal((4, d)).astype(np.float32)
        for q in Q:
            assert ri.score_query(q)[0].tobytes() == pi.score_query(q)[0].tobytes()
        a, b = ri.search(Q, 7), pi.search(Q, 7, threads=3)
        assert np.array_equal(a[0], b[0]) and a[1].tobytes() == b[1].tobytes()


@ref_only
def test_encode_restatement_matches_reference(port):
    from oracle.oracle import Ref
    R = Ref()
    rng = np.random.default_rng(5)
    for dbar in (2, 4):
        x = rng.standard_normal((500, dbar)).astype(np.float32)
        x[::17] = 0.0
        c = rng.standard_normal((16, dbar)).astype(np.float32)
        a1, al1, l1 = R.assign_projective(x, c)
        a2, al2, l2 = port.assign_projective(x, c)
        assert np.array_equal(a1, a2) and al1.tobytes() == al2.tobytes() and l1.tobytes() == l2.tobytes()
        hp = np.zeros(500)
        hb = np.zeros(500)
        for i in range(500):
            nrm = float(np.sqrt(np.dot(x[i].astype(np.float64), x[i].astype(np.float64))))
            if nrm > 0:
                hp[i], hb[i] = R.aniso_weights(nrm, 0.2, dbar)
        a1, al1, l1 = R.assign_anisotropic(x, c, hp, hb)
        a2, al2, l2 = port.assign_anisotropic(x, c, hp, hb)
        assert np.array_equal(a1, a2) and al1.tobytes() == al2.tobytes() and l1.tobytes() == l2.tobytes()


@ref_only
def test_alpha_code_restatement_matches_reference(port):
    """The score-aware alpha-code argmin (scalar_quant.cpp:121-150) given the
    reference's fitted codebook reproduces quantize_anisotropic's codes."""
    from oracle.oracle import Ref
    R = Ref()
    rng = np.random.default_rng(11)
    for dbar in (2, 4):
        x = (rng.standard_normal((3000, dbar)) * 0.4).astype(np.float32)
        x[::31] = 0.0
        c = rng.standard_normal((16, dbar)).astype(np.float32)
        hp = np.zeros(3000)
        hb = np.zeros(3000)
        for i in range(3000):
            nrm = float(np.sqrt(np.dot(x[i].astype(np.float64), x[i].astype(np.float64))))
            if nrm > 0:
                hp[i], hb[i] = R.aniso_weights(nrm, 0.2, dbar)
        a, _, _ = R.assign_anisotropic(x, c, hp, hb)
        values, codes = R.quantize_anisotropic(x, c, a, hp, hb, 8, seed=3)
        assert np.array_equal(port.alpha_codes_aniso(x, c, a, hp, hb, values), codes)


@ref_only
def test_center_stats_restatement_matches_reference(port):
    """Sequential member sums + solve_spd restated == pcpq::center_anisotropic."""
    from oracle.oracle import Ref
    R = Ref()
    rng = np.random.default_rng(21)
    for dbar in (2, 4):
        x = (rng.standard_normal((4000, dbar)) * 0.5).astype(np.float32)
        x[::41] = 0.0
        assign = rng.integers(0, 8, 4000)
        alpha = rng.standard_normal(4000)
        hp = rng.uniform(0.01, 0.2, 4000)
        hb = hp * rng.uniform(0.01, 0.9, 4000)
        stats = port.center_stats(x, assign, alpha, hp, hb, 8)
        for c in range(8):
            mem = np.nonzero(assign == c)[0]
            want = R.center_anisotropic(x, mem, alpha, hp, hb)
            got = port.center_from_stats(stats[c], dbar)
            assert got.tobytes() == want.tobytes()
        # the chain property the multi-GPU path relies on
        half = port.center_stats(x[:2000], assign[:2000], alpha, hp, hb, 8)
        full = port.center_stats(x, assign, alpha, hp, hb, 8)
        xb = x.copy()
        xb[:2000] = 0.0  # rows below the split contribute nothing on the second leg
        chained = port.center_stats(xb, assign, alpha, hp, hb, 8, init=half)
        assert chained.tobytes() == full.tobytes()
