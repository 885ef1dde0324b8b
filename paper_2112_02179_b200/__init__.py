"""B200-native PCPQ query-time scoring path (arXiv 2112.02179).

The product is libpcpqg.so (CUDA sm_100a kernels behind the C ABI in
include/pcpqg.h); this package is its host-side mirror of the reference
``pcpq`` scoring API.  Importing it without the built extension fails loudly.
"""
from .api import (  # noqa: F401
    DeviceIndex, LookupTable, PcpqError, ScoreCounters, aniso_alpha_codes, assign_anisotropic,
    assign_projective, build_lookup_table, center_stats, counters_for, deserialize, errc, last_timings,
    logical_payload_bits, merge_device, read_pq_index, score_all, score_all_batch, score_query, search,
    search_device, set_option, set_profiling, plan_info,
    DeviceIVF, IVFQueryOutput, QueryHit, deserialize_ivf, ivf_counters, query_ivf, query_ivf_batch,
    query_ivf_device, read_ivf_index,
    ScoredId, brute_force_topn, brute_force_topn_batch, brute_force_topn_device, recall1_batch, recall1_single,
    index_codes, PQConfig, build_pq_index, aniso_weights, train_phases,
)
