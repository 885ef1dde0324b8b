"""Database sharding across the GPUs of one box.

Rank r keeps the contiguous id range [r*n/W, (r+1)*n/W) resident in its HBM
(the code stream of that shard only; codebooks are replicated).  A query
batch is scored by every rank against its own shard with the fused kernel,
which emits per-query top-n lists of packed 64-bit keys carrying *global*
ids; the lists are all-gathered over NCCL (NVLink/NVSwitch) and merged on the
GPU by the same merge kernel that merges the per-CTA lists.  Because keys
order by (score desc, id asc), the merged list equals the unsharded
partial_sort of proj/tools/main.cpp:233-237 exactly.

The collective is the only exchange: B x topn x 8 bytes per rank per batch
(C4: 4096 x 100 x 8 = 3.3 MB), latency-bound on NVLink 5.

`local_fn` / `merge_fn` are injectable so the orchestration (sharding,
gather, merge) is testable on CPU with gloo (tests/test_sharded.py).
"""
from __future__ import annotations

import struct

import numpy as np
import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    return n * rank // world, n * (rank + 1) // world


def index_n(data: bytes) -> int:
    return struct.unpack_from("<I", data, 16)[0]


# ---- host-side key packing (identical to the device's make_key/key_id) ----
def make_keys(scores: np.ndarray, ids: np.ndarray) -> np.ndarray:
    s = np.ascontiguousarray(scores, np.float32)
    b = s.view(np.uint32).astype(np.uint64)
    negz = (b == 0x80000000).astype(np.uint64)
    b = np.where((b << np.uint64(1)) & np.uint64(0xFFFFFFFF) == 0, np.uint64(0), b)
    ordv = np.where(b & np.uint64(0x80000000), (~b) & np.uint64(0xFFFFFFFF), b | np.uint64(0x80000000))
    key = (ordv << np.uint64(32)) | ((np.uint64(0x7FFFFFFF) - ids.astype(np.uint64)) << np.uint64(1)) | negz
    return np.where(ids < 0, np.uint64(0), key)


def decode_keys(keys: np.ndarray):
    k = keys.astype(np.uint64)
    o = (k >> np.uint64(32)) & np.uint64(0xFFFFFFFF)
    bits = np.where(o & np.uint64(0x80000000), o & np.uint64(0x7FFFFFFF), (~o) & np.uint64(0xFFFFFFFF))
    bits = np.where(k & np.uint64(1), np.uint64(0x80000000), bits).astype(np.uint32)
    scores = bits.view(np.float32).copy()
    ids = (np.uint64(0x7FFFFFFF) - ((k >> np.uint64(1)) & np.uint64(0x7FFFFFFF))).astype(np.int64).astype(np.int32)
    empty = k == 0
    ids[empty] = -1
    scores[empty] = -np.inf
    return ids, scores


def merge_keys_host(all_keys: np.ndarray, topn: int):
    """[L, B, K] keys -> global top-n (ids, scores); host reference merge."""
    L, B, K = all_keys.shape
    flat = np.sort(all_keys.transpose(1, 0, 2).reshape(B, L * K), axis=1)[:, ::-1][:, :topn]
    return decode_keys(np.ascontiguousarray(flat))


class ShardedSearcher:
    """One rank's view of a sharded index."""

    def __init__(self, data: bytes, rank: int, world: int, device: int | None = None,
                 group=None, local_fn=None, merge_fn=None):
        self.rank, self.world, self.group = rank, world, group
        self.n = index_n(data)
        self.begin, self.end = shard_range(self.n, rank, world)
        self.local_fn = local_fn
        self.merge_fn = merge_fn
        self.index = None
        if local_fn is None:
            from . import api
            if device is None:
                import torch
                device = torch.cuda.current_device()
            self.index = api.deserialize(data, device=device, shard=(self.begin, self.end))

    @classmethod
    def from_index(cls, index, n: int, rank: int, world: int, group=None):
        """Wrap an already loaded shard (e.g. api.deserialize_part of a part
        image holding only this rank's rows)."""
        self = cls.__new__(cls)
        self.rank, self.world, self.group = rank, world, group
        self.n = n
        self.begin, self.end = shard_range(n, rank, world)
        self.local_fn = self.merge_fn = None
        self.index = index
        return self

    def search_device(self, dQ: torch.Tensor, topn: int, stream=None):
        """dQ: (B, d) float32 on this rank's GPU -> (ids, scores) of the global top-n."""
        from . import api
        if self.world == 1:
            ids, sc, _ = api.search_device(self.index, dQ, topn, stream=stream)
            return ids, sc
        B = dQ.shape[0]
        # one stream for scan, collective and merge: NCCL orders against torch's
        # current stream, so make `stream` current for the whole exchange
        with torch.cuda.stream(stream if stream is not None else torch.cuda.current_stream(dQ.device)):
            _, _, keys = api.search_device(self.index, dQ, topn, want_keys=True,
                                           out=(None, None, torch.empty((B, topn), dtype=torch.int64,
                                                                        device=dQ.device)))
            if dist.get_backend(self.group) == "nccl":
                gathered = torch.empty((self.world, B, topn), dtype=torch.int64, device=dQ.device)
                dist.all_gather_into_tensor(gathered, keys, group=self.group)
            else:  # gloo (CPU tensors): e.g. several ranks sharing one GPU in tests
                hk = keys.cpu()
                parts = [torch.empty_like(hk) for _ in range(self.world)]
                dist.all_gather(parts, hk, group=self.group)
                gathered = torch.stack(parts).to(dQ.device)
            ids, sc, _ = api.merge_device(gathered, topn)
        return ids, sc

    def search_host(self, Q: torch.Tensor, topn: int):
        """CPU/gloo path with injected local search + merge (used by tests)."""
        keys = torch.from_numpy(self.local_fn(Q.numpy(), topn, self.begin, self.end).view(np.int64))
        gathered = [torch.empty_like(keys) for _ in range(self.world)]
        dist.all_gather(gathered, keys, group=self.group)
        all_keys = torch.stack(gathered).numpy().view(np.uint64)
        merge = self.merge_fn or merge_keys_host
        return merge(all_keys, topn)


def ordered_center_stats(local_fn, rank: int, world: int, shape, group=None, device=None):
    """Lloyd center statistics over id-sharded ranks, bit-identical to one
    process: the reference sums each cluster's members in
    increasing id order, so rank r continues the running sums of ranks < r
    (point-to-point chain 0 -> 1 -> ... -> W-1, ~86 KB at config 5), then the
    last rank broadcasts the result.  local_fn(init) -> stats folds this
    rank's members onto `init` (None on rank 0), e.g. api.center_stats."""
    init = None
    if rank > 0:
        init = torch.empty(shape, dtype=torch.float64, device=device)
        dist.recv(init, src=rank - 1, group=group)
    stats = local_fn(init)
    if rank < world - 1:
        dist.send(stats.contiguous(), dst=rank + 1, group=group)
    out = stats if rank == world - 1 else torch.empty(shape, dtype=torch.float64, device=device)
    dist.broadcast(out, src=world - 1, group=group)
    return out
