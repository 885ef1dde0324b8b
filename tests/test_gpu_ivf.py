"""GPU parity of the IVF query path (pcpqg_ivf_query, the batched
pcpq::query_ivf of proj/core/src/ivf.cpp:89-153) through the C ABI:

* golden: every fixture of tests/golden/ivf_* (reference outputs) at every
  recorded (k_probe, topN): ids, double scores bit-for-bit, counts, short
  flags, requested-id scores (NaN where unprobed) and ScoreCounters;
* synthetic containers far larger than the fixtures against the C
  restatement (oracle/, pinned to the reference by tests/test_oracle_ivf.py):
  skewed cell sizes with raw singleton cells, every cell code layout;
* the device-pointer entry point against the host one, and query_ivf's
  argument errors.
Tolerance: none — bit-identical (fp32 cell scores in the reference order,
double coarse + combination)."""
import numpy as np
import pytest
import torch

import paper_2112_02179_b200 as P
from paper_2112_02179_b200 import datagen
from tests.test_oracle_ivf import NAMES, load_ivf

pytestmark = pytest.mark.gpu


def bits(a):
    return np.nan_to_num(np.asarray(a, np.float64), nan=7.25).view(np.uint64)


@pytest.mark.parametrize("name", NAMES)
def test_ivf_golden(name):
    data, g = load_ivf(name)
    iv = P.deserialize_ivf(data)
    for kp in g["kprobes"]:
        for tn in g["topns"]:
            key = f"{kp}_{tn}"
            r = P.query_ivf_batch(iv, g["queries"], int(kp), int(tn), requested=g["requested"], want_probes=True)
            assert np.array_equal(r["ids"], g["ids_" + key]), key
            assert np.array_equal(bits(r["scores"]), bits(g["scores_" + key])), key
            assert np.array_equal(r["counts"], g["counts_" + key]), key
            assert np.array_equal(r["short"], g["short_" + key]), key
            assert np.array_equal(bits(r["requested"]), bits(g["req_" + key])), key
            c = P.ScoreCounters()
            P.ivf_counters(iv, r["probes"], c)
            assert np.array_equal(c._arr(), g["counters_" + key]), key


def test_ivf_single_query_api_matches_golden():
    data, g = load_ivf(NAMES[0])
    iv = P.deserialize_ivf(data)
    kp, tn = int(g["kprobes"][1]), int(g["topns"][0])
    for b in range(g["queries"].shape[0]):
        c = P.ScoreCounters()
        out = P.query_ivf(iv, g["queries"][b], kp, tn, requested_ids=g["requested"][b], counters=c)
        k = int(g[f"counts_{kp}_{tn}"][b])
        assert [h.id for h in out.top] == g[f"ids_{kp}_{tn}"][b, :k].tolist()
        assert np.array_equal(bits([h.score for h in out.top]), bits(g[f"scores_{kp}_{tn}"][b, :k]))
        assert out.short_result == bool(g[f"short_{kp}_{tn}"][b])
        assert np.array_equal(bits(out.requested), bits(g[f"req_{kp}_{tn}"][b]))


SYNTH = [
    # n, d, kbar, m, k, s, raw_fp16, method, seed
    (20000, 32, 64, 8, 16, 8, False, "apcpq", 3),      # JOINT8 (4+3 bits)
    (20000, 32, 64, 8, 16, 0, True, "pcpq", 4),        # PLANES 4-bit + fp16 alpha
    (12000, 24, 300, 6, 16, 0, False, "pcpq", 5),      # many tiny / raw cells, fp32 alpha
    (15000, 40, 32, 5, 64, 16, False, "pcpq", 6),      # PLANES 8-bit centers + 4-bit scale codes, m % 8 != 0
    (8000, 30, 16, 4, 256, 32, False, "kmeans", 7),    # 8-bit centers + 8-bit scales, padded d
    (6000, 8, 5000, 2, 4, 2, False, "pcpq", 8),        # kbar > 4096: the CUB probe-order path
]


@pytest.fixture(scope="module")
def synth_cases(port):
    out = []
    for (n, d, kbar, m, k, s, f16, meth, seed) in SYNTH:
        data = datagen.synth_ivf(n, d, kbar, m, k, s, seed=seed, raw_fp16=f16, method=meth)
        out.append((data, port.ivf_parse(data)))
    return out


@pytest.mark.parametrize("case", range(len(SYNTH)))
def test_ivf_synthetic_matches_oracle(synth_cases, case):
    data, ref = synth_cases[case]
    iv = P.deserialize_ivf(data)
    rng = np.random.default_rng(case)
    B = 12
    Q = rng.standard_normal((B, iv.d)).astype(np.float32)
    Q[-1] = 0.0
    req = rng.integers(0, iv.n, (B, 20)).astype(np.uint32)
    for kp in sorted({1, 3, iv.kbar // 4 or 1, iv.kbar}):
        for tn in (10, 257):
            a = ref.query(Q, kp, tn, requested=req)
            r = P.query_ivf_batch(iv, Q, kp, tn, requested=req, want_probes=True)
            assert np.array_equal(r["ids"], a[0]), (kp, tn)
            assert np.array_equal(bits(r["scores"]), bits(a[1])), (kp, tn)
            assert np.array_equal(r["counts"], a[2]) and np.array_equal(r["short"], a[3])
            assert np.array_equal(bits(r["requested"]), bits(a[4])), (kp, tn)
            c = P.ScoreCounters()
            P.ivf_counters(iv, r["probes"], c)
            assert np.array_equal(c._arr(), a[5]), (kp, tn)


def test_ivf_device_api_matches_host(synth_cases):
    data, _ = synth_cases[0]
    iv = P.deserialize_ivf(data)
    rng = np.random.default_rng(11)
    Q = rng.standard_normal((33, iv.d)).astype(np.float32)
    req = rng.integers(0, iv.n, (33, 5)).astype(np.uint32)
    h = P.query_ivf_batch(iv, Q, 7, 50, requested=req)
    ids, sc, cnt, sh, rs = P.query_ivf_device(iv, torch.from_numpy(Q).cuda(), 7, 50,
                                              requested=torch.from_numpy(req.astype(np.int32)))
    torch.cuda.synchronize()
    assert np.array_equal(ids.cpu().numpy(), h["ids"])
    assert np.array_equal(bits(sc.cpu().numpy()), bits(h["scores"]))
    assert np.array_equal(cnt.cpu().numpy().astype(np.uint32), h["counts"])
    assert np.array_equal(sh.cpu().numpy(), h["short"])
    assert np.array_equal(bits(rs.cpu().numpy()), bits(h["requested"]))


def test_ivf_query_errors():
    data, g = load_ivf(NAMES[0])
    iv = P.deserialize_ivf(data)
    Q = g["queries"]
    cases = [((Q, 0, 5), P.errc.data), ((Q, iv.kbar + 1, 5), P.errc.data), ((Q, 1, 0), P.errc.data),
             ((Q[:, :-1], 1, 5), P.errc.size_mismatch)]
    for args, code in cases:
        with pytest.raises(P.PcpqError) as e:
            P.query_ivf_batch(iv, *args)
        assert e.value.code == code
    with pytest.raises(P.PcpqError) as e:
        P.query_ivf_batch(iv, Q, 1, 5, requested=np.full((Q.shape[0], 1), iv.n, np.uint32))
    assert e.value.code == P.errc.data
    with pytest.raises(P.PcpqError) as e:
        P.query_ivf_device(iv, torch.from_numpy(Q).cuda(), 1, 5,
                           requested=torch.full((Q.shape[0], 1), iv.n, dtype=torch.int32))
    assert e.value.code == P.errc.data


@pytest.mark.parametrize("case", [0, 1, 3, 4])
def test_ivf_grouped_scan_matches_oracle(synth_cases, case):
    """The batched multi-cell scan (cells inverted to their probing queries,
    scored 16 queries at a time) against the per-(query, cell) kernel and the
    oracle: many queries per cell, ties from duplicate queries, a zero query."""
    data, ref = synth_cases[case]
    iv = P.deserialize_ivf(data)
    rng = np.random.default_rng(100 + case)
    B = 150
    Q = rng.standard_normal((B, iv.d)).astype(np.float32)
    Q[40:60] = Q[:20]
    Q[-1] = 0.0
    req = rng.integers(0, iv.n, (B, 4)).astype(np.uint32)
    for kp, tn in ((max(1, iv.kbar // 2), 10), (iv.kbar, 100)):
        try:
            P.set_option("ivf_grouped", 1)
            r = P.query_ivf_batch(iv, Q, kp, tn, requested=req)
            P.set_option("ivf_grouped", 0)
            r0 = P.query_ivf_batch(iv, Q, kp, tn, requested=req)
        finally:
            P.set_option("ivf_grouped", 1)
        for k in ("ids", "counts", "short"):
            assert np.array_equal(r[k], r0[k]), (kp, tn, k)
        assert np.array_equal(bits(r["scores"]), bits(r0["scores"])), (kp, tn)
        a = ref.query(Q[:30], kp, tn, requested=req[:30])
        assert np.array_equal(r["ids"][:30], a[0]), (kp, tn)
        assert np.array_equal(bits(r["scores"][:30]), bits(a[1])), (kp, tn)
