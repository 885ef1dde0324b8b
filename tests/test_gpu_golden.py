"""GPU parity against the golden vectors made by the unmodified reference
library: bit-identical scores, LUTs and top-n (incl. ties and -0.0), the
counters, the loader's error taxonomy, and sharded search + device merge."""
import numpy as np
import pytest

from tests import _golden

pytestmark = pytest.mark.gpu
CASES = _golden.names()


@pytest.mark.parametrize("name", CASES)
def test_scores_lut_topn_bit_exact(name):
    import paper_2112_02179_b200 as P
    data, g = _golden.load(name)
    idx = P.deserialize(data, device=0)
    Q = g["queries"]
    got = P.score_all_batch(idx, Q)
    for b in range(Q.shape[0]):
        assert got[b].tobytes() == g["scores"][b].tobytes(), f"query {b}"
        assert P.score_query(idx, Q[b]).tobytes() == g["scores"][b].tobytes()
    ids, top = P.search(idx, Q, 10)
    assert np.array_equal(ids, g["ids10"])
    assert top.tobytes() == g["top10"].tobytes()
    ids, top = P.search(idx, Q, idx.n + 3)  # topn > n: clamped, padded with -1 / -inf
    assert np.array_equal(ids, g["idsx"])
    assert top.tobytes() == g["topx"].tobytes()
    c = P.ScoreCounters()
    lut = P.build_lookup_table(idx, Q[0], c)
    assert lut.eta.tobytes() == g["eta"].tobytes()
    assert lut.eta_lambda.tobytes() == g["etal"].tobytes()
    s = P.score_all(idx, lut, c)
    assert s.tobytes() == g["scores"][0].tobytes()
    assert [c.table_madds, c.scalar_mults, c.point_mults, c.lookups, c.adds] == [int(v) for v in g["counters"]]


@pytest.mark.parametrize("name", CASES)
def test_search_every_batch_size(name):
    """Every query-group width (NQ = 1, 2, 4, 8, 16) gives the same lists."""
    import paper_2112_02179_b200 as P
    data, g = _golden.load(name)
    idx = P.deserialize(data, device=0)
    Qbig = np.tile(g["queries"], (6, 1))  # 36 queries -> groups of 16 + tail
    for B in (1, 2, 3, 5, 8, 36):
        QB = Qbig[:B]
        ids, top = P.search(idx, QB, 10)
        for b in range(B):
            assert np.array_equal(ids[b], g["ids10"][b % 6]), (B, b)
            assert top[b].tobytes() == g["top10"][b % 6].tobytes()


@pytest.mark.parametrize("name", ["pcpq_q_m8_k16_s16", "pcpq_raw16_m4_k16", "pcpq_q_ties", "kmeans_k300_wide",
                                  "pcpq_q_k256_s16"])
@pytest.mark.parametrize("shards", [2, 3])
def test_sharded_search_and_device_merge(name, shards):
    import torch
    import paper_2112_02179_b200 as P
    from paper_2112_02179_b200.sharded import shard_range
    data, g = _golden.load(name)
    n = int(g["shape"][0])
    Q = torch.from_numpy(g["queries"]).cuda()
    keys = []
    for r in range(shards):
        b, e = shard_range(n, r, shards)
        ix = P.deserialize(data, device=0, shard=(b, e))
        _, _, k = P.search_device(ix, Q, 10, want_keys=True)
        keys.append(k)
    ids, top, _ = P.merge_device(torch.stack(keys), 10)
    torch.cuda.synchronize()
    assert np.array_equal(ids.cpu().numpy(), g["ids10"])
    assert top.cpu().numpy().tobytes() == g["top10"].tobytes()


@pytest.mark.parametrize("name", CASES)
def test_loader_error_taxonomy(name):
    import paper_2112_02179_b200 as P
    data, g = _golden.load(name)
    bad = _golden.corruptions(name, data)
    for ename, code in zip(g["err_names"], g["err_codes"]):
        with pytest.raises(P.PcpqError) as e:
            P.deserialize(bad[str(ename)], device=0)
        assert e.value.status == int(code), ename


def test_query_width_mismatch_is_size_mismatch():
    import paper_2112_02179_b200 as P
    data, g = _golden.load("pcpq_q_pad_d5_m2")
    idx = P.deserialize(data, device=0)
    with pytest.raises(P.PcpqError) as e:
        P.score_query(idx, np.zeros(6, np.float32))  # pq_index.cpp:174-175
    assert e.value.code == P.errc.size_mismatch
    with pytest.raises(P.PcpqError) as e:
        P.search(idx, np.full((1, 5), np.nan, np.float32), 3)
    assert e.value.code == P.errc.data
