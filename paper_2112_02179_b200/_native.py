"""ctypes binding of libpcpqg.so (the C ABI in include/pcpqg.h).

The library is built in-tree (paper_2112_02179_b200/lib/libpcpqg.so) by
``make -C paper_2112_02179_b200/csrc`` / ``__graft_entry__.build()``.  There is
no fallback: if the shared object is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PCPQG_LIB") or os.path.join(HERE, "lib", "libpcpqg.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA extension first "
        "(python -c 'import __graft_entry__ as g; g.build()')")

lib = C.CDLL(LIB_PATH)

_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_i32p = C.POINTER(C.c_int32)
_fp = C.POINTER(C.c_float)
_dp = C.POINTER(C.c_double)
_vp = C.c_void_p


class Info(C.Structure):
    _fields_ = [("method", C.c_uint32), ("n", C.c_uint32), ("d", C.c_uint32), ("padded_d", C.c_uint32),
                ("m", C.c_uint32), ("k", C.c_uint32), ("scales", C.c_uint32), ("dbar", C.c_uint32),
                ("t", C.c_double), ("shard_begin", C.c_uint64), ("shard_end", C.c_uint64),
                ("format", C.c_uint32), ("center_bits", C.c_uint32), ("scale_bits", C.c_uint32),
                ("words_per_point", C.c_uint32), ("code_bytes", C.c_uint64), ("device", C.c_int)]


def _sig(name, restype, *argtypes):
    try:
        f = getattr(lib, name)
    except AttributeError:
        if "PCPQG_LIB" in os.environ:  # an older build selected for an A/B run
            return None
        raise
    f.restype = restype
    f.argtypes = list(argtypes)
    return f


last_error = _sig("pcpqg_last_error", C.c_char_p)
index_load = _sig("pcpqg_index_load", C.c_int, _vp, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, C.POINTER(_vp))
index_load_part = _sig("pcpqg_index_load_part", C.c_int, _vp, C.c_uint64, C.c_uint64, C.c_int, C.POINTER(_vp))
multi_load = _sig("pcpqg_multi_load", C.c_int, _vp, C.c_uint64, _vp, C.c_int, C.c_int, C.POINTER(_vp))
multi_free = _sig("pcpqg_multi_free", None, _vp)
multi_info = _sig("pcpqg_multi_info", C.c_int, _vp, _vp)
multi_search = _sig("pcpqg_multi_search", C.c_int, _vp, _vp, C.c_uint32, C.c_uint32, C.c_uint32, _vp, _vp)
index_load_file = _sig("pcpqg_index_load_file", C.c_int, C.c_char_p, C.c_int, C.c_uint64, C.c_uint64, C.POINTER(_vp))
index_free = _sig("pcpqg_index_free", None, _vp)
index_load_gpu = _sig("pcpqg_index_load_gpu", C.c_int, _vp, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64,
                      C.POINTER(_vp))
index_load_file_gpu = _sig("pcpqg_index_load_file_gpu", C.c_int, C.c_char_p, C.c_int, C.c_uint64, C.c_uint64,
                           C.POINTER(_vp))
index_codes = _sig("pcpqg_index_codes", C.c_int, _vp, _vp, C.c_uint64)
index_info = _sig("pcpqg_index_info", C.c_int, _vp, C.POINTER(Info))
build_lut = _sig("pcpqg_build_lut", C.c_int, _vp, _vp, C.c_uint32, C.c_uint32, _vp, _vp, _vp)
score_all = _sig("pcpqg_score_all", C.c_int, _vp, _vp, C.c_uint32, C.c_uint32, _vp, _vp)
search = _sig("pcpqg_search", C.c_int, _vp, _vp, C.c_uint32, C.c_uint32, C.c_uint32, _vp, _vp)
search_device = _sig("pcpqg_search_device", C.c_int, _vp, _vp, C.c_uint32, C.c_uint32, C.c_uint32,
                     _vp, _vp, _vp, _vp)
merge_device = _sig("pcpqg_merge_device", C.c_int, _vp, C.c_uint32, C.c_uint32, C.c_uint32, _vp, _vp,
                    _vp, C.c_int, _vp)
counters = _sig("pcpqg_counters", C.c_int, _vp, C.c_uint32, _vp)
plan_info = _sig("pcpqg_plan_info", C.c_int, _vp, C.c_uint32, C.c_uint32, _vp)
logical_payload_bits = _sig("pcpqg_logical_payload_bits", C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32,
                            C.c_uint32)
set_profiling = _sig("pcpqg_set_profiling", C.c_int, C.c_int)
set_option = _sig("pcpqg_set_option", C.c_int, C.c_char_p, C.c_int64)
last_timings = _sig("pcpqg_last_timings", C.c_int, _vp)
assign_projective = _sig("pcpqg_assign_projective", C.c_int, _vp, C.c_uint64, C.c_uint32, _vp, C.c_uint32,
                         _vp, _vp, _vp, C.c_int, _vp)
assign_anisotropic = _sig("pcpqg_assign_anisotropic", C.c_int, _vp, C.c_uint64, C.c_uint32, _vp, C.c_uint32,
                          _vp, _vp, _vp, _vp, _vp, _vp, C.c_int, _vp)
center_stats = _sig("pcpqg_center_stats", C.c_int, _vp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, _vp, _vp,
                    _vp, _vp, C.c_uint32, _vp, _vp, C.c_int, _vp)
ivf_load = _sig("pcpqg_ivf_load", C.c_int, _vp, C.c_uint64, C.c_int, C.POINTER(_vp))
ivf_load_file = _sig("pcpqg_ivf_load_file", C.c_int, C.c_char_p, C.c_int, C.POINTER(_vp))
ivf_free = _sig("pcpqg_ivf_free", None, _vp)
ivf_info = _sig("pcpqg_ivf_info", C.c_int, _vp, _vp)
ivf_query = _sig("pcpqg_ivf_query", C.c_int, _vp, _vp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, _vp,
                 C.c_uint32, _vp, _vp, _vp, _vp, _vp, _vp)
ivf_query_device = _sig("pcpqg_ivf_query_device", C.c_int, _vp, _vp, C.c_uint32, C.c_uint32, C.c_uint32,
                        C.c_uint32, _vp, C.c_uint32, _vp, _vp, _vp, _vp, _vp, _vp, _vp)
ivf_counters = _sig("pcpqg_ivf_counters", C.c_int, _vp, _vp, C.c_uint32, C.c_uint32, _vp)
brute_force_topn = _sig("pcpqg_brute_force_topn", C.c_int, _vp, C.c_uint64, C.c_uint32, _vp, C.c_uint32,
                        C.c_uint32, _vp, _vp, C.c_int)
brute_force_topn_device = _sig("pcpqg_brute_force_topn_device", C.c_int, _vp, C.c_uint64, C.c_uint32, _vp,
                               C.c_uint32, C.c_uint32, _vp, _vp, C.c_int, _vp)
recall1 = _sig("pcpqg_recall1", C.c_int, _vp, C.c_uint64, C.c_uint32, _vp, C.c_uint32, _vp, C.c_uint32, _vp,
               _vp, C.c_int)
train_kmeans = _sig("pcpqg_train_kmeans", C.c_int, _vp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                    C.c_uint32, C.c_double, C.c_uint32, C.c_double, C.c_uint64, C.c_int, C.POINTER(_vp),
                    C.POINTER(C.c_uint64))
train_pcpq = _sig("pcpqg_train_pcpq", C.c_int, _vp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                  C.c_uint32, C.c_int, C.c_double, C.c_uint32, C.c_double, C.c_uint64, C.c_int, C.POINTER(_vp),
                  C.POINTER(C.c_uint64))
train_aniso = _sig("pcpqg_train_aniso", C.c_int, _vp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                   C.c_uint32, C.c_int, C.c_int, C.c_double, C.c_uint32, C.c_double, C.c_uint64, C.c_int,
                   C.POINTER(_vp), C.POINTER(C.c_uint64))
train_aniso_multi = _sig("pcpqg_train_aniso_multi", C.c_int, _vp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                         C.c_uint32, C.c_int, C.c_int, C.c_double, C.c_uint32, C.c_double, C.c_uint64, _vp, C.c_int,
                         C.POINTER(_vp), C.POINTER(C.c_uint64))
aniso_weights = _sig("pcpqg_aniso_weights", C.c_int, _vp, C.c_uint64, C.c_uint32, C.c_double, _vp, _vp)
aniso_weights_gpu = _sig("pcpqg_aniso_weights_gpu", C.c_int, _vp, C.c_uint64, C.c_uint32, C.c_double, _vp, _vp,
                         C.c_int)
sin_selfcheck = _sig("pcpqg_sin_selfcheck", C.c_int, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64))
train_weights_on_gpu = _sig("pcpqg_train_weights_on_gpu", C.c_int, C.POINTER(C.c_int))
train_phases = _sig("pcpqg_train_phases", C.c_int, _vp)
free = _sig("pcpqg_free", None, _vp)
aniso_alpha_codes = _sig("pcpqg_aniso_alpha_codes", C.c_int, _vp, C.c_uint64, C.c_uint32, _vp, _vp, _vp,
                         _vp, _vp, C.c_uint32, _vp, C.c_int, _vp)

EXPORTED = [
    "pcpqg_last_error", "pcpqg_index_load", "pcpqg_index_load_part", "pcpqg_index_load_file", "pcpqg_index_free", "pcpqg_index_info",
    "pcpqg_build_lut", "pcpqg_score_all", "pcpqg_search", "pcpqg_search_device", "pcpqg_merge_device",
    "pcpqg_counters", "pcpqg_plan_info", "pcpqg_logical_payload_bits", "pcpqg_set_profiling", "pcpqg_set_option", "pcpqg_last_timings",
    "pcpqg_assign_projective", "pcpqg_assign_anisotropic", "pcpqg_aniso_alpha_codes", "pcpqg_center_stats",
    "pcpqg_ivf_load", "pcpqg_ivf_load_file", "pcpqg_ivf_free", "pcpqg_ivf_info", "pcpqg_ivf_query",
    "pcpqg_ivf_query_device", "pcpqg_ivf_counters", "pcpqg_brute_force_topn", "pcpqg_brute_force_topn_device",
    "pcpqg_recall1", "pcpqg_index_load_gpu", "pcpqg_index_load_file_gpu", "pcpqg_index_codes",
    "pcpqg_train_kmeans", "pcpqg_train_pcpq", "pcpqg_train_aniso", "pcpqg_train_aniso_multi", "pcpqg_aniso_weights", "pcpqg_aniso_weights_gpu", "pcpqg_sin_selfcheck", "pcpqg_train_weights_on_gpu", "pcpqg_train_phases", "pcpqg_free",
    "pcpqg_multi_load", "pcpqg_multi_free", "pcpqg_multi_info", "pcpqg_multi_search",
]
