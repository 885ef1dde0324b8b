"""Multi-rank orchestration on CPU (gloo, world_size 2): points sharded by
rank, per-shard top-n as packed keys with global ids, all-gather, merge.  The
per-shard search is the oracle here (no GPU); the result must equal the
unsharded flat top-n, tie rule included."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests import _golden


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _local_fn_factory(data):
    from oracle.oracle import Port
    from paper_2112_02179_b200.sharded import make_keys
    pi = Port().parse(data)

    def local(Q, topn, begin, end):
        out = np.zeros((Q.shape[0], topn), np.uint64)
        for b in range(Q.shape[0]):
            s, _ = pi.score_query(Q[b])
            s = s[begin:end]
            ids = pi_topn(s, topn) + begin
            valid = ids >= begin
            keys = make_keys(np.where(valid, s[np.clip(ids - begin, 0, None)], 0), np.where(valid, ids, -1))
            out[b] = keys
        return out

    from oracle.oracle import Port as _P
    _port = _P()

    def pi_topn(s, topn):
        ids = _port.topn_of_scores(s, topn).astype(np.int64)
        return np.concatenate([ids, np.full(topn - ids.size, -10**9, np.int64)])

    return local


def _worker(rank, world, port, name, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2112_02179_b200.sharded import ShardedSearcher
    data, g = _golden.load(name)
    sh = ShardedSearcher(data, rank, world, local_fn=_local_fn_factory(data))
    ids, scores = sh.search_host(torch.from_numpy(g["queries"]), 10)
    ret[rank] = (ids, scores)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["pcpq_q_m8_k16_s16", "pcpq_q_ties", "pcpq_raw_zero_rows", "kmeans_m1_k2"])
def test_gloo_two_ranks_equal_unsharded(name):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    ret = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, ret)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    _, g = _golden.load(name)
    for r in range(2):
        ids, scores = ret[r]
        assert np.array_equal(ids, g["ids10"])
        assert scores.tobytes() == g["top10"].tobytes()


def test_key_packing_round_trip_and_order():
    from paper_2112_02179_b200.sharded import decode_keys, make_keys
    s = np.array([1.5, -0.0, 0.0, -2.0, np.inf, -np.inf, 1.5, 3e-41], np.float32)
    ids = np.array([7, 3, 2, 9, 1, 0, 4, 5], np.int32)
    k = make_keys(s, ids)
    di, ds = decode_keys(k)
    assert np.array_equal(di, ids) and ds.tobytes() == s.tobytes()
    # key order == (score desc, id asc) with -0 == +0
    order = np.argsort(-k.astype(np.float64), kind="stable")
    order = sorted(range(len(s)), key=lambda i: -int(k[i]))
    ref = sorted(range(len(s)), key=lambda i: (-float(s[i]), int(ids[i])))
    assert order == ref


def _chain_worker(rank, world, port_, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Port
    from paper_2112_02179_b200.sharded import ordered_center_stats, shard_range
    rng = np.random.default_rng(7)
    n, dbar, k = 9000, 4, 8
    x = (rng.standard_normal((n, dbar)) * 0.5).astype(np.float32)
    assign = rng.integers(0, k, n)
    alpha, hp = rng.standard_normal(n), rng.uniform(0.01, 0.2, n)
    hb = hp * 0.5
    b, e = shard_range(n, rank, world)
    mine = np.zeros_like(x)
    mine[b:e] = x[b:e]  # rows of other ranks contribute nothing

    def local(init):
        st = Port().center_stats(mine, assign, alpha, hp, hb, k, init=None if init is None else init.numpy())
        return torch.from_numpy(st)

    out = ordered_center_stats(local, rank, world, (k, dbar * (dbar + 1) // 2 + dbar + 1))
    ret[rank] = (out.numpy(), Port().center_stats(x, assign, alpha, hp, hb, k))
    dist.destroy_process_group()


def test_gloo_ordered_center_stats_chain_is_bit_exact():
    ctx = mp.get_context("spawn")
    ret = ctx.Manager().dict()
    port_ = _free_port()
    procs = [ctx.Process(target=_chain_worker, args=(r, 3, port_, ret)) for r in range(3)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for r in range(3):
        got, want = ret[r]
        assert got.tobytes() == want.tobytes()
