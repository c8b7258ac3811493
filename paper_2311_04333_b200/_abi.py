"""ctypes binding of the C ABI in include/dg_b200.h (libdg_b200.so).

No fallback: if the shared object is missing this raises at import time, and
every computing call returns DG_E_CUDA when no B200 is visible.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libdg_b200.so")

u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)
u8p = C.POINTER(C.c_uint8)


class DgOutcome(C.Structure):
    _fields_ = [("rho_edges", C.c_uint64), ("rho_verts", C.c_uint64),
                ("best_prefix", C.c_uint64), ("width", C.c_uint64)]


class DgRunConfig(C.Structure):
    _fields_ = [("algorithm", C.c_int), ("pruning", C.c_int), ("iterations", C.c_uint64),
                ("epsilon", C.c_double), ("iteration_cap", C.c_uint64), ("c_num", C.c_uint64),
                ("c_den", C.c_uint64), ("reset_loads", C.c_int), ("slack_samples", C.c_uint64)]


class DgIterRecord(C.Structure):
    _fields_ = [("iter", C.c_uint64), ("rho_edges", C.c_uint64), ("rho_verts", C.c_uint64),
                ("n", C.c_uint64), ("m", C.c_uint64), ("width", C.c_uint64), ("ms", C.c_double),
                ("order_ms", C.c_double), ("update_ms", C.c_double), ("batches", C.c_uint64)]


class DgRunResult(C.Structure):
    _fields_ = [("best_edges", C.c_uint64), ("best_verts", C.c_uint64),
                ("witness_size", C.c_uint64), ("witness_edges", C.c_uint64),
                ("iterations", C.c_uint64), ("max_width", C.c_uint64),
                ("slack_violations", C.c_uint64), ("kmax_known", C.c_int),
                ("kmax_exact", C.c_int), ("kmax", C.c_uint32), ("threshold", C.c_uint32),
                ("pruned_n", C.c_uint64), ("pruned_m", C.c_uint64), ("final_n", C.c_uint64),
                ("peel_rounds", C.c_uint32), ("reprunes", C.c_uint32),
                ("coreness_ms", C.c_double), ("coreness_kernel_ms", C.c_double),
                ("init_ms", C.c_double), ("total_ms", C.c_double), ("reprune_ms", C.c_double),
                ("device_ms", C.c_double)]


GP = C.c_void_p  # dg_graph*
GPP = C.POINTER(C.c_void_p)

# name -> (restype, argtypes); kept in the order of include/dg_b200.h
PROTOTYPES = {
    "dg_last_error": (C.c_char_p, []),
    "dg_version": (C.c_char_p, []),
    "dg_graph_build": (C.c_int, [u64p, u64p, C.c_uint64, C.c_int, GPP]),
    "dg_graph_generate": (C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_double,
                                    C.c_uint64, GPP]),
    "dg_parse_edge_list": (C.c_int, [C.c_char_p, C.c_uint64, C.c_char, C.c_int, GPP, u64p]),
    "dg_graph_from_csr": (C.c_int, [C.c_uint64, u64p, u32p, u64p, C.c_int, GPP]),
    "dg_graph_info": (C.c_int, [GP, u64p, u64p, u64p]),
    "dg_graph_download": (C.c_int, [GP, u64p, u32p, u64p]),
    "dg_graph_device_ptrs": (C.c_int, [GP, C.POINTER(u64p), C.POINTER(u32p), C.POINTER(u64p)]),
    "dg_graph_free": (None, [GP]),
    "dg_induced": (C.c_int, [GP, u8p, GPP, u32p]),
    "dg_get_core": (C.c_int, [GP, u32p, C.c_uint32, GPP, u32p]),
    "dg_coreness": (C.c_int, [GP, C.c_int, C.c_uint64, C.c_uint64, u32p, u32p, u32p]),
    "dg_peel_order": (C.c_int, [GP, u64p, C.c_int, u32p]),
    "dg_sort_order": (C.c_int, [C.c_uint64, u64p, u32p]),
    "dg_density_load_update": (C.c_int, [GP, u32p, u64p, C.POINTER(DgOutcome), u64p]),
    "dg_charikar_peel": (C.c_int, [GP, C.POINTER(DgOutcome)]),
    "dg_slack_violations": (C.c_int, [C.c_uint64, u32p, u64p, C.c_uint64, C.c_uint64,
                                      C.c_uint64, u64p]),
    "dg_default_iterations": (C.c_int, [C.c_uint64, C.c_double, C.c_uint64, C.c_double,
                                        C.c_uint64, u64p]),
    "dg_run": (C.c_int, [GP, C.POINTER(DgRunConfig), C.POINTER(DgRunResult),
                         C.POINTER(DgIterRecord), C.c_uint64, u64p, C.c_uint64, u64p,
                         C.c_uint64]),
    "dg_run_pruned": (C.c_int, [GP, u32p, C.c_uint32, C.c_uint32, C.POINTER(DgRunConfig),
                                C.POINTER(DgRunResult), C.POINTER(DgIterRecord), C.c_uint64,
                                u64p, C.c_uint64, u64p, C.c_uint64]),
    "dg_shard_create": (C.c_int, [GP, u64p, C.c_uint32, C.c_uint32, GPP]),
    "dg_shard_create_rows": (C.c_int, [C.c_uint64, u64p, C.c_uint32, C.c_uint32, u64p, u32p,
                                       C.c_int, GPP]),
    "dg_shard_free": (None, [GP]),
    "dg_shard_min_alive": (C.c_int, [GP, u32p]),
    "dg_shard_collect": (C.c_int, [GP, C.c_uint32, C.c_uint32, u64p]),
    "dg_shard_count_remote": (C.c_int, [GP, u64p]),
    "dg_shard_expand": (C.c_int, [GP, C.c_uint32, C.c_uint32, u64p, C.c_void_p]),
    "dg_shard_apply": (C.c_int, [GP, C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, u64p]),
    "dg_shard_labels": (C.c_int, [GP, u32p]),
    "dg_shard_ipc_handle": (C.c_int, [GP, C.c_void_p]),
    "dg_shard_peer_open": (C.c_int, [GP, C.c_uint32, C.c_void_p]),
    "dg_shard_peer_link": (C.c_int, [GP, C.c_uint32, GP]),
    "dg_shard_expand_peer": (C.c_int, [GP, C.c_uint32, C.c_uint32, u64p]),
    "dg_shard_finish_round": (C.c_int, [GP, u64p]),
    "dg_shard_xctrl_reset": (C.c_int, [GP]),
    "dg_dist_max_id": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, u64p]),
    "dg_dist_endpoint_hist": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32,
                                        C.c_uint32, u64p]),
    "dg_dist_route": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, u64p, C.c_uint32,
                                C.c_void_p, u64p]),
    "dg_dist_rows": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
                               u64p, u64p]),
    "dg_dist_unique": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, u64p]),
    "dg_dist_lookup": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_uint64,
                                 C.c_void_p]),
    "dg_dist_bucket_counts": (C.c_int, [C.c_void_p, C.c_uint64, u64p, C.c_uint32, u64p]),
    "dg_dist_take": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint32,
                               C.c_void_p]),
    "dg_dist_relabel": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    "dg_dist_keep_map": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint64, C.c_void_p,
                                   u64p]),
    "dg_dist_core_rows": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p, u64p, u64p]),
    "dg_shard_coreness_persistent": (C.c_int, [C.POINTER(C.c_void_p), C.c_uint32, C.c_int,
                                               C.c_uint64, C.c_uint64, C.POINTER(C.c_uint32),
                                               C.POINTER(C.c_uint32), C.POINTER(C.c_float)]),
    "dg_gen_rmat": (C.c_int, [C.c_uint32, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p,
                              C.c_int]),
    "dg_gen_rmat_range": (C.c_int, [C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p,
                                    C.c_void_p, C.c_int]),
    "dg_gen_chung_lu": (C.c_int, [C.c_uint64, C.c_uint64, C.c_double, C.c_uint64, C.c_void_p,
                                  C.c_void_p, C.c_int]),
    "dg_brute_force_densest": (C.c_int, [GP, C.c_uint32, u64p, u64p, u64p, u64p]),
    "dg_device_alloc": (C.c_int, [C.c_uint64, C.POINTER(C.c_void_p)]),
    "dg_device_free": (C.c_int, [C.c_void_p]),
    "dg_memcpy": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int]),
    "dg_synchronize": (C.c_int, []),
    "dg_set_device": (C.c_int, [C.c_int]),
    "dg_launch_count": (C.c_uint64, []),
    "dg_flush_l2": (C.c_int, []),
    "dg_trim_memory": (C.c_int, []),
    "dg_set_peel_mode": (C.c_int, [C.c_int]),
}


DIAG_PATH = os.path.join(PKG, "libdg_b200_diag.so")
DIAG_PROTOTYPES = {
    "dg_microbench": (C.c_int, [C.c_int, C.c_uint64, C.POINTER(C.c_double)]),
    "dg_peel_profile": (C.c_int, [u64p]),
    "dg_peel_trace_arm": (C.c_int, [C.c_uint32]),
    "dg_peel_trace_read": (C.c_int, [u64p]),
    "dg_kcore_profile": (C.c_int, [u64p]),
}


def load_diag(path: str = "") -> C.CDLL:
    """The diagnostics library (include/dg_b200_diag.h) built against the
    loaded product library (DG_B200_LIB selects a tuning build): tools only."""
    path = path or os.environ.get("DG_B200_LIB", LIB_PATH)[:-3] + "_diag.so"
    lib = C.CDLL(path)
    for name, (res, args) in DIAG_PROTOTYPES.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    return lib


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()'). "
            "There is no CPU fallback for the densegraph B200 path.")
    lib = C.CDLL(path)
    for name, (res, args) in PROTOTYPES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


LIB = load(os.environ.get("DG_B200_LIB", LIB_PATH))
