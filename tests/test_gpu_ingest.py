"""GPU ingest: pcpqg_index_load_gpu / _file_gpu must
produce the same device code stream, layout and errors as the host loader
(pcpqg_index_load, itself pinned to pcpq::deserialize by the golden
corruption fixtures): every golden index, every corruption, shards, and
config-shaped images."""
import os

import numpy as np
import pytest

import paper_2112_02179_b200 as P
from paper_2112_02179_b200 import datagen
from tests import _golden

pytestmark = pytest.mark.gpu


def same_index(a, b):
    assert (a.info.format, a.info.center_bits, a.info.scale_bits, a.info.words_per_point) == \
        (b.info.format, b.info.center_bits, b.info.scale_bits, b.info.words_per_point)
    assert (a.n_local, a.m, a.k, a.scales) == (b.n_local, b.m, b.k, b.scales)
    assert np.array_equal(P.index_codes(a), P.index_codes(b))


@pytest.mark.parametrize("name", _golden.names())
def test_gpu_ingest_matches_host(name, tmp_path):
    data, g = _golden.load(name)
    host = P.deserialize(data)
    gpu = P.deserialize(data, ingest="gpu")
    same_index(host, gpu)
    f = tmp_path / "x.idx"
    f.write_bytes(data)
    same_index(host, P.read_pq_index(f, ingest="gpu"))
    n = host.n
    if n >= 8:
        sh = (n // 3, n - 1)
        same_index(P.deserialize(data, shard=sh), P.deserialize(data, shard=sh, ingest="gpu"))
    Q = g["queries"]
    a = P.search(host, Q, 10)
    b = P.search(gpu, Q, 10)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("name", _golden.names())
def test_gpu_ingest_error_classes(name, tmp_path):
    data, g = _golden.load(name)
    corrupted = _golden.corruptions(name, data)
    for label, code in zip(g["err_names"], g["err_codes"]):
        bad = corrupted[str(label)]
        for mode in ("bytes", "file"):
            try:
                if mode == "bytes":
                    P.deserialize(bad, ingest="gpu")
                else:
                    f = tmp_path / "bad.idx"
                    f.write_bytes(bad)
                    P.read_pq_index(f, ingest="gpu")
                st = 0
            except P.PcpqError as e:
                st = e.status
            assert st == int(code), (label, mode)


@pytest.mark.parametrize("cfg,n", [("c2", 200_000), ("c3", 300_000), ("c4", 100_000)])
def test_gpu_ingest_config_shapes(cfg, n):
    data = datagen.synth_index(datagen.CONFIGS[cfg], seed=3, n=n)
    same_index(P.deserialize(data), P.deserialize(data, ingest="gpu"))
