"""Exact ground truth / recall.

CPU: the C restatement (orc_brute_force_topn / orc_recall1) against the
reference's golden vectors (tests/golden/eval_*.npz, make_golden_eval.py).
GPU (-m gpu): pcpqg_brute_force_topn / pcpqg_recall1 against the same vectors
bit-for-bit (ids and double scores), with the approximate-pass chunk forced
small so the candidate union over many chunks is exercised, and against the
oracle on larger data.  Tolerance: none (exact re-rank in the reference order)."""
import glob
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "eval_*.npz")))


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return {k: z[k] for k in z.files}


def topns(g):
    return sorted(int(k[4:]) for k in g if k.startswith("ids_"))


def test_eval_fixtures_present():
    assert len(NAMES) >= 4


@pytest.mark.parametrize("name", NAMES)
def test_port_brute_force_matches_golden(port, name):
    g = load(name)
    for tn in topns(g):
        ids, sc = port.brute_force_topn(g["data"], g["queries"], tn)
        assert np.array_equal(ids, g[f"ids_{tn}"])
        assert np.array_equal(sc.view(np.uint64), g[f"scores_{tn}"].view(np.uint64))
    assert np.array_equal(port.recall1(g["data"], g["queries"], g["retrieved"], g["scores_1"][:, 0]), g["hits"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("chunk", [0, 4096])
def test_gpu_brute_force_matches_golden(name, chunk):
    import paper_2112_02179_b200 as P
    g = load(name)
    P.set_option("gt_chunk", chunk)
    try:
        for tn in topns(g):
            ids, sc = P.brute_force_topn_batch(g["data"], g["queries"], tn)
            assert np.array_equal(ids, g[f"ids_{tn}"]), tn
            assert np.array_equal(sc.view(np.uint64), g[f"scores_{tn}"].view(np.uint64)), tn
    finally:
        P.set_option("gt_chunk", 0)
    hits = P.recall1_batch(g["data"], g["queries"], g["retrieved"], g["scores_1"][:, 0])
    assert np.array_equal(hits, g["hits"])


@pytest.mark.gpu
def test_gpu_brute_force_large_vs_oracle(port):
    import torch
    import paper_2112_02179_b200 as P
    from paper_2112_02179_b200 import datagen
    cfg = datagen.CONFIGS["c2"]
    X = datagen.mixture_chunk(cfg, *datagen.mixture_params(cfg, 3), 0, 60000, 3).numpy()
    X = np.ascontiguousarray(X[:, :97])  # odd d
    Q = np.random.default_rng(5).standard_normal((9, 97)).astype(np.float32)
    P.set_option("gt_chunk", 8192)
    try:
        ids, sc = P.brute_force_topn_batch(X, Q, 100)
    finally:
        P.set_option("gt_chunk", 0)
    ri, rs = port.brute_force_topn(X, Q, 100)
    assert np.array_equal(ids, ri)
    assert np.array_equal(sc.view(np.uint64), rs.view(np.uint64))
    # device-pointer entry point
    di, ds = P.brute_force_topn_device(torch.from_numpy(X).cuda(), torch.from_numpy(Q).cuda(), 100)
    assert np.array_equal(di.cpu().numpy(), ri)
    assert np.array_equal(ds.cpu().numpy().view(np.uint64), rs.view(np.uint64))


@pytest.mark.gpu
def test_gpu_eval_errors():
    import paper_2112_02179_b200 as P
    g = load(NAMES[0])
    for tn in (0, g["data"].shape[0] + 1):
        with pytest.raises(P.PcpqError) as e:
            P.brute_force_topn_batch(g["data"], g["queries"], tn)
        assert e.value.code == P.errc.data
    bad = g["retrieved"].copy()
    bad[0, 0] = g["data"].shape[0]
    with pytest.raises(P.PcpqError) as e:
        P.recall1_batch(g["data"], g["queries"], bad, g["scores_1"][:, 0])
    assert e.value.code == P.errc.data
