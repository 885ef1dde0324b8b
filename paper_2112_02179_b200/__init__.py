"""B200-native PCPQ query-time scoring path (arXiv 2112.02179).

The product is libpcpqg.so (CUDA sm_100a kernels behind the C ABI in
include/pcpqg.h); this package is its host-side mirror of the reference
``pcpq`` scoring API.  Touching any API name without the built extension
fails loudly.

The API is imported lazily (PEP 562): ``import paper_2112_02179_b200.datagen``
or ``.pcpqidx`` (pure numpy / torch data tools) does not map libpcpqg.so, so
the benchmark's reference arm can build its workload without loading the
product.
"""
_API = (
    "DeviceIndex", "LookupTable", "PcpqError", "ScoreCounters", "aniso_alpha_codes", "assign_anisotropic",
    "assign_projective", "build_lookup_table", "center_stats", "counters_for", "deserialize", "errc",
    "last_timings", "logical_payload_bits", "merge_device", "read_pq_index", "score_all", "score_all_batch",
    "score_query", "search", "search_device", "set_option", "set_profiling", "plan_info",
    "DeviceIVF", "IVFQueryOutput", "QueryHit", "deserialize_ivf", "ivf_counters", "query_ivf", "query_ivf_batch",
    "query_ivf_device", "read_ivf_index",
    "ScoredId", "brute_force_topn", "brute_force_topn_batch", "brute_force_topn_device", "recall1_batch",
    "recall1_single", "index_codes", "deserialize_part", "MultiIndex", "deserialize_multi", "PQConfig", "build_pq_index", "aniso_weights", "train_phases", "sin_selfcheck", "train_weights_on_gpu",
)

__all__ = list(_API)


def __getattr__(name):
    if name in _API:
        from . import api
        v = getattr(api, name)
        globals()[name] = v
        return v
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")


def __dir__():
    return sorted(list(globals()) + list(_API))
