"""GPU parity on synthetic config-shaped indexes (reduced n), against the
oracle C restatement (itself pinned to the reference by test_oracle.py)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(port, cfg_name, n, B, topn, seed=1):
    import paper_2112_02179_b200 as P
    from paper_2112_02179_b200 import datagen
    cfg = datagen.CONFIGS[cfg_name]
    data = datagen.synth_index(cfg, seed=seed, n=n)
    Q = datagen.queries(cfg, B, seed=seed + 1).numpy()
    idx = P.deserialize(data, device=0)
    ids, sc = P.search(idx, Q, topn)
    pi = port.parse(data)
    rids, rsc = pi.search(Q, topn, threads=8)
    assert np.array_equal(ids, rids)
    assert sc.tobytes() == rsc.tobytes()
    # score_all parity for a couple of queries (bit-exact)
    for qi in range(min(2, B)):
        got = P.score_query(idx, Q[qi])
        want, _ = pi.score_query(Q[qi])
        assert got.tobytes() == want.tobytes()
    return idx


@pytest.mark.parametrize("B", [1, 2, 3, 5, 16, 40])
def test_c1_shape(port, B):
    _run(port, "c1", 20000, B, 10)


@pytest.mark.parametrize("B", [1, 17])
def test_c2_shape(port, B):
    _run(port, "c2", 30000, B, 100)


@pytest.mark.parametrize("B", [1, 4, 33])
def test_c3_shape_raw_fp16(port, B):
    idx = _run(port, "c3", 20000, B, 100)
    assert idx.info.scale_bits == 16


@pytest.mark.parametrize("B", [1, 3])
def test_c4_shape_k256(port, B):
    _run(port, "c4", 5000, B, 100)
