"""GPU merge of sorted per-list top-n keys (`merge_device` -> merge_sorted_kernel),
against the host merge (sort every key descending, keep topn).  Covers both
kernel paths: the block-parallel one (few queries; rank placement of the head
threshold and the output rows) and the warp tournament (many queries or many
lists), with empty and ragged lists, a single list, and scores tied within and
across lists (ids break them; keys are unique, as every producer's are)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _lists(rng, L, B, K, dup, full=False):
    from paper_2112_02179_b200.sharded import make_keys
    keys = np.zeros((L, B, K), np.uint64)
    pool_scores = rng.standard_normal(64).astype(np.float32)
    for l in range(L):
        for b in range(B):
            c = K if full else int(rng.integers(0, K + 1))
            if c == 0:
                continue
            if dup:  # few distinct scores: ties within and across lists, broken by id
                sc = rng.choice(pool_scores, c)
                ids = rng.choice(max(32, K), c, replace=False) + max(32, K) * l
            else:
                sc = rng.standard_normal(c).astype(np.float32)
                ids = rng.choice(1 << 30, c, replace=False)
            k = np.unique(make_keys(sc, ids.astype(np.int64)))[::-1]
            keys[l, b, :k.size] = k
    return keys


@pytest.mark.parametrize("L,B,K", [(1, 1, 10), (3, 2, 100), (100, 1, 100), (148, 1, 100), (148, 4, 100),
                                   (256, 3, 10), (256, 1, 100), (37, 200, 10), (148, 160, 100)])
@pytest.mark.parametrize("dup", [False, True])
def test_merge_device_equals_host_merge(L, B, K, dup):
    import torch
    import paper_2112_02179_b200 as P
    from paper_2112_02179_b200.sharded import merge_keys_host
    rng = np.random.default_rng(L * 1000 + B * 10 + K + dup)
    keys = _lists(rng, L, B, K, dup)
    want_ids, want_sc = merge_keys_host(keys, K)
    dk = torch.from_numpy(keys.view(np.int64)).cuda()
    ids, sc, ko = P.merge_device(dk, K, want_keys=True)
    torch.cuda.synchronize()
    flat = np.sort(keys.transpose(1, 0, 2).reshape(B, L * K), axis=1)[:, ::-1][:, :K]
    assert np.array_equal(ko.cpu().numpy().view(np.uint64), flat)
    assert np.array_equal(ids.cpu().numpy(), want_ids)
    assert sc.cpu().numpy().tobytes() == want_sc.tobytes()


# Every list full: L x (K + 1) keys exceed the sorted merge's 24576-key staging
# buffer at (256, 100) and (8, 4096), so the merge must take the select-over-
# global path instead of dropping lists.  (100, 100) and
# (148, 100) stay under it: the block-parallel head-threshold path with L >= K.
@pytest.mark.parametrize("L,B,K", [(256, 1, 100), (256, 200, 100), (8, 1, 4096), (8, 3, 4096), (100, 1, 100),
                                   (148, 2, 100), (240, 2, 100)])
@pytest.mark.parametrize("dup", [False, True])
def test_merge_device_full_lists(L, B, K, dup):
    import torch
    import paper_2112_02179_b200 as P
    rng = np.random.default_rng(L * 7 + B * 3 + K + dup)
    keys = _lists(rng, L, B, K, dup, full=True)
    flat = np.sort(keys.transpose(1, 0, 2).reshape(B, L * K), axis=1)[:, ::-1][:, :K]
    dk = torch.from_numpy(keys.view(np.int64)).cuda()
    ids, sc, ko = P.merge_device(dk, K, want_keys=True)
    torch.cuda.synchronize()
    assert np.array_equal(ko.cpu().numpy().view(np.uint64), flat)
