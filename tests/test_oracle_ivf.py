"""The IVF restatement in oracle/ (orc_ivf_parse / orc_ivf_query) pinned
against the reference's golden vectors (tests/golden/ivf_*, made by
tests/golden/make_golden_ivf.py from the unmodified reference) and, where
oracle/_ref is built, against the reference live on fresh seeded cases.
Reference: proj/core/src/ivf.cpp:89-153 (query_ivf), :256-316 (container)."""
import glob
import os

import numpy as np
import pytest

from oracle.oracle import OracleError, Ref

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "ivf_*.ivf")))


def load_ivf(name):
    with open(os.path.join(GOLDEN, name + ".ivf"), "rb") as f:
        data = f.read()
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return data, {k: z[k] for k in z.files}


def corruptions(data):
    import sys
    sys.path.insert(0, GOLDEN)
    from make_golden_ivf import corrupt_cases  # noqa: E402
    return corrupt_cases(data)


def test_ivf_fixtures_present():
    assert len(NAMES) >= 8


@pytest.mark.parametrize("name", NAMES)
def test_port_ivf_query_matches_golden(port, name):
    data, g = load_ivf(name)
    iv = port.ivf_parse(data)
    for kp in g["kprobes"]:
        for tn in g["topns"]:
            ids, sc, cnt, sh, rs, c5 = iv.query(g["queries"], int(kp), int(tn), requested=g["requested"])
            key = f"{kp}_{tn}"
            assert np.array_equal(ids, g["ids_" + key]), key
            # bit-identical doubles (NaN padding past the returned length)
            assert np.array_equal(np.nan_to_num(sc, nan=7.0).view(np.uint64),
                                  np.nan_to_num(g["scores_" + key], nan=7.0).view(np.uint64)), key
            assert np.array_equal(cnt, g["counts_" + key])
            assert np.array_equal(sh, g["short_" + key])
            assert np.array_equal(np.nan_to_num(rs, nan=7.0).view(np.uint64),
                                  np.nan_to_num(g["req_" + key], nan=7.0).view(np.uint64)), key
            assert np.array_equal(c5, g["counters_" + key])


@pytest.mark.parametrize("name", NAMES)
def test_port_ivf_container_errors_match_golden(port, name):
    data, g = load_ivf(name)
    cases = corruptions(data)
    assert [c[0] for c in cases] == list(g["error_labels"])
    for (label, bad), code in zip(cases, g["error_codes"]):
        try:
            port.ivf_parse(bad)
            st = 0
        except OracleError as e:
            st = e.code
        assert st == code, label


def test_port_ivf_usage_errors(port):
    data, g = load_ivf(NAMES[0])
    iv = port.ivf_parse(data)
    Q = g["queries"]
    with pytest.raises(OracleError):
        iv.query(Q, 0, 5)              # k_probe < 1
    with pytest.raises(OracleError):
        iv.query(Q, iv.kbar + 1, 5)    # k_probe > kbar
    with pytest.raises(OracleError):
        iv.query(Q, 1, 0)              # topN < 1
    with pytest.raises(OracleError):
        iv.query(Q[:, :-1], 1, 5)      # dimension mismatch
    with pytest.raises(OracleError):
        iv.query(Q, 1, 5, requested=np.full((Q.shape[0], 1), iv.n, np.uint32))


@pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_port_ivf_matches_reference_live(port, seed):
    R = Ref()
    rng = np.random.default_rng(seed)
    n, d = int(rng.integers(60, 400)), int(rng.integers(4, 20))
    kbar = int(rng.integers(2, max(3, n // 8)))
    method = ["kmeans", "pcpq", "apcpq", "aniso"][seed % 4]
    X = R.generate_dataset("clustered", n, d, seed)
    data = R.build_ivf(X, kbar, method=method, quantize=bool(seed % 2), m=2, k=8, s=4, seed=seed)
    Q = rng.standard_normal((6, d)).astype(np.float32)
    req = rng.integers(0, n, (6, 9)).astype(np.uint32)
    iv = port.ivf_parse(data)
    for kp in (1, kbar):
        a = R.ivf_query(data, Q, kp, 15, requested=req)
        b = iv.query(Q, kp, 15, requested=req)
        for x, y in zip(a, b):
            if x.dtype.kind == "f":
                assert np.array_equal(np.nan_to_num(x, nan=7.0), np.nan_to_num(y, nan=7.0))
            else:
                assert np.array_equal(x, y)
