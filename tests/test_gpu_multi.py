"""Multi-GPU sharding with the real kernels (VERDICT r01,
next 3).  The pool has one GPU per call, so:

* pcpqg_multi_* (one process driving several devices) runs with repeated
  devices [0, 0(, 0)] — the peer-copy transport, which is also what serves
  distinct devices without libnccl — and with NCCL over the one device
  (ncclCommInitAll / grouped AllGather with one rank).  Results must equal the
  unsharded search and the reference's golden top-10 (proj/tools/main.cpp:
  229-243 over score_query, proj/core/src/pq_index.cpp:246-250).
* Two processes share GPU 0 through ShardedSearcher with a gloo group: each
  runs the fused search on its own shard (global-id keys), gloo gathers the
  CPU copies, merge_device merges on the GPU.  No kernel waits on another
  rank, so sharing the device is sound.
* Part images (pcpqg_index_load_part): a rank that holds only its rows loads
  the same shard as the full image's [b, e), with the reference's validation.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests import _golden

pytestmark = pytest.mark.gpu
NAMES = ["pcpq_q_m8_k16_s16", "apcpq_q_m10_k16_s8", "kmeans_k300_wide", "pcpq_raw_m16_k16", "pcpq_q_ties"]


def _names():
    have = set(_golden.names())
    return [n for n in NAMES if n in have] or _golden.names()[:3]


@pytest.mark.parametrize("name", _names())
@pytest.mark.parametrize("devices,transport", [([0, 0], "peer"), ([0, 0, 0], "peer"), ([0], "nccl"), ([0], "auto")])
def test_multi_index_equals_golden(name, devices, transport):
    import paper_2112_02179_b200 as P
    data, g = _golden.load(name)
    Q = g["queries"]
    mi = P.deserialize_multi(data, devices, transport)
    assert mi.ndev == len(devices)
    if transport == "nccl":
        assert mi.transport == "nccl"
    ids, sc = mi.search(Q, 10)
    assert np.array_equal(ids, g["ids10"])
    one = P.deserialize(data, device=0)
    ids1, sc1 = P.search(one, Q, 10)
    assert np.array_equal(ids, ids1) and sc.tobytes() == sc1.tobytes()


@pytest.mark.parametrize("cfg_name,n,B,topn", [("c2", 60000, 300, 100), ("c3", 100000, 40, 100), ("c1", 30000, 1000, 10)])
def test_multi_index_batch_configs(port, cfg_name, n, B, topn):
    """three shards on the peer transport, the batch paths (K2-T for B >= 256)
    inside each shard: equal to the oracle"""
    import paper_2112_02179_b200 as P
    from paper_2112_02179_b200 import datagen
    cfg = datagen.CONFIGS[cfg_name]
    img = datagen.synth_image(cfg, seed=8, n=n)
    Q = datagen.queries(cfg, B, seed=9).numpy()
    mi = P.deserialize_multi(img, [0, 0, 0], "peer")
    ids, sc = mi.search(Q, topn)
    rids, rsc = port.parse(img).search(Q, topn, threads=8)
    assert np.array_equal(ids, rids) and sc.tobytes() == rsc.tobytes()


def test_multi_nccl_rejects_repeated_devices():
    import paper_2112_02179_b200 as P
    data, _ = _golden.load(_names()[0])
    with pytest.raises(P.PcpqError) as e:
        P.deserialize_multi(data, [0, 0], "nccl")
    assert e.value.code == P.errc.unsupported


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, part, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2112_02179_b200 as P
    from paper_2112_02179_b200 import pcpqidx
    from paper_2112_02179_b200.sharded import ShardedSearcher, shard_range
    torch.cuda.set_device(0)
    data, g = _golden.load(name)
    if part:  # this rank holds only its own rows
        ix = pcpqidx.deserialize(data)
        rdt = pcpqidx.row_dtype(ix.m, ix.k, ix.scales)
        head = len(data) - ix.n * rdt.itemsize
        b, e = shard_range(ix.n, rank, world)
        img = data[:head] + data[head + b * rdt.itemsize: head + e * rdt.itemsize]
        sh = ShardedSearcher.from_index(P.deserialize_part(img, b, device=0), ix.n, rank, world)
    else:
        sh = ShardedSearcher(data, rank, world, device=0)
    ids, sc = sh.search_device(torch.from_numpy(g["queries"]).cuda(), 10)
    ret[rank] = (ids.cpu().numpy(), sc.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,part", [(2, False), (2, True), (3, True)])
def test_two_processes_real_kernels_gloo(world, part):
    name = _names()[0]
    _, g = _golden.load(name)
    ctx = mp.get_context("spawn")
    with ctx.Manager() as m:
        ret = m.dict()
        mp.start_processes(_worker, args=(world, _free_port(), name, part, ret), nprocs=world, join=True,
                           start_method="spawn")
        for r in range(world):
            ids, sc = ret[r]
            assert np.array_equal(ids, g["ids10"]), r


def test_part_image_equals_shard_and_validates():
    import paper_2112_02179_b200 as P
    from paper_2112_02179_b200 import datagen, pcpqidx
    cfg = datagen.CONFIGS["c2"]
    n = 20000
    full = datagen.synth_image(cfg, seed=4, n=n)
    b, e = 7001, 13999
    part = datagen.synth_image(cfg, seed=4, n=n, rows=(b, e))
    Q = datagen.queries(cfg, 32, seed=5).numpy()
    a = P.deserialize(full, device=0, shard=(b, e))
    p = P.deserialize_part(part, b, device=0)
    assert p.shard_begin == b and p.n_local == e - b and p.n == n
    assert np.array_equal(P.index_codes(a), P.index_codes(p))
    ia, sa = P.search(a, Q, 50)
    ip, sp = P.search(p, Q, 50)
    assert np.array_equal(ia, ip) and sa.tobytes() == sp.tobytes()
    rdt = pcpqidx.row_dtype(cfg.m, cfg.k, cfg.s)
    # the reference's checks on the part's rows
    bad = part.copy()
    bad[-rdt.itemsize + 3] = 200  # a center code >= k in the last row
    with pytest.raises(P.PcpqError) as ex:
        P.deserialize_part(bad, b, device=0)
    assert ex.value.code == P.errc.code_out_of_range
    with pytest.raises(P.PcpqError) as ex:
        P.deserialize_part(part[:-5], b, device=0)  # a partial last row: bytes past the whole rows
    assert ex.value.code == P.errc.size_mismatch
    with pytest.raises(P.PcpqError) as ex:
        P.deserialize_part(part, n - 10, device=0)  # rows beyond the index
    assert ex.value.code == P.errc.usage
