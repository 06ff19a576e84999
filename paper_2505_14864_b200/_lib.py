"""ctypes loader for libdynmo.so (the C-ABI of include/dynmo.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
sm_100a).  There is no fallback: if it is missing, importing the binding
raises, so no product call can silently run anywhere but the CUDA path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# DYNMO_DEBUG=1 loads the bounds-checked build (csrc: make debug) instead
# (DYNMO_LIB=<path> loads another build of the same ABI, for A/B measurements)
LIB_PATH = os.environ.get("DYNMO_LIB") or os.path.join(
    _HERE, "libdynmo_dbg.so" if os.environ.get("DYNMO_DEBUG") == "1" else "libdynmo.so")

OK, E_INVALID, E_INFEASIBLE, E_OVERFLOW, E_CUDA, E_NCCL, E_NOMEM = 0, -1, -2, -3, -4, -5, -6
W_NOT_CONVERGED, W_BOUND_UNMET = 1, 2

SRC_MASK_BITS, SRC_MASK_U8, SRC_NZ_BF16, SRC_NZ_F32 = 0, 1, 2, 3
SRC_TOKMASK_BITS, SRC_EXIT_U8, SRC_EXPERT_I64, SRC_EXPERT_I32, SRC_TIME_NS = 4, 5, 6, 7, 8
REPACK_BOUND, REPACK_ALG2 = 0, 1
PHASES = ["profile", "epilogue", "exchange", "partition", "diffuse", "repack", "migrate"]
MAX_LAYERS = 1023


class Segment(C.Structure):
    _fields_ = [("d_ptr", C.c_void_p), ("n_elem", C.c_int64), ("layer", C.c_int32),
                ("src_kind", C.c_int32), ("n_experts", C.c_int32), ("top_k", C.c_int32)]


class Buf(C.Structure):
    _fields_ = [("d_ptr", C.c_void_p), ("bytes", C.c_int64)]


W_F32, W_BF16 = 0, 1


class PruneSegment(C.Structure):
    _fields_ = [("d_w", C.c_void_p), ("d_mask", C.c_void_p), ("n", C.c_int64), ("dtype", C.c_int32),
                ("pad", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    p, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    sigs = {
        "dynmo_strerror": (C.c_char_p, [i32]),
        "dynmo_last_error": (C.c_char_p, []),
        "dynmo_version": (C.c_char_p, []),
        "dynmo_get_unique_id": (i32, [p]),
        "dynmo_ctx_create": (i32, [i32, i32, i32, p, C.POINTER(p)]),
        "dynmo_ctx_destroy": (None, [p]),
        "dynmo_ctx_nranks": (i32, [p]),
        "dynmo_ctx_rank": (i32, [p]),
        "dynmo_ctx_set_timing": (i32, [p, i32]),
        "dynmo_ctx_timing_read": (i32, [p, i32, p, p]),
        "dynmo_ctx_timing_poll": (i32, [p]),
        "dynmo_profile_plan_create": (i32, [p, p, i32, i32, i32, i32, i32, C.POINTER(p)]),
        "dynmo_profile_plan_destroy": (None, [p]),
        "dynmo_plan_num_tiles": (i64, [p]),
        "dynmo_plan_bytes": (i64, [p]),
        "dynmo_plan_max_experts": (i32, [p]),
        "dynmo_profile_layers": (i32, [p, p, p, p, p, p, p, p, p, p, p]),
        "dynmo_timestamp": (i32, [p, p, p]),
        "dynmo_publish": (i32, [p, p, p, i64, p]),
        "dynmo_diag_step_stamps": (i32, [p, i32]),
        "dynmo_ctx_split": (i32, [p, i32, i32, p]),
        "dynmo_ctx_timing_detach": (i32, [p]),
        "dynmo_ctx_barrier": (i32, [p, p]),
        "dynmo_map_stages": (i32, [p, i32, i32, p, p, i32, p, p, i32, C.c_uint32, p, p, p, p, p]),
        "dynmo_partition_stages": (i32, [p, i32, i32, p, p, p, p, p, p, p, p, p, p, p]),
        "dynmo_diffuse_balance": (i32, [p, i32, i32, p, p, p, p, p, p, p, p, p, i32,
                                        p, p, p, p, p, p, p, p, p, p]),
        "dynmo_repack_workers": (i32, [p, i32, i32, p, p, p, p, p, p, p, p, p, i32,
                                       p, p, p, p, p]),
        "dynmo_migrate_layers": (i32, [p, i32, i32, p, p, i32, p, p, p, p, i32, p, p, p]),
        "dynmo_migration_plan": (i32, [i32, i32, p, p, i32, p, p, p]),
        "dynmo_prune_plan_create": (i32, [p, p, i32, p]),
        "dynmo_prune_plan_destroy": (None, [p]),
        "dynmo_global_prune": (i32, [p, p, i64, p, p, p]),
        "dynmo_migrate_plan_create": (i32, [p, i32, i32, p, p, C.POINTER(p)]),
        "dynmo_migrate_plan_destroy": (None, [p]),
        "dynmo_migrate_layers_p2p": (i32, [p, p, i32, p, p, i32, p, p, p, p, p]),
        "dynmo_ctx_p2p_error": (i32, [p, p]),
        "dynmo_migrate_layers_dev": (i32, [p, p, i32, p, p, i32, p, p, p, p, p]),
        "dynmo_migrate_plan_set_ctas": (i32, [p, i32]),
        "dynmo_migrate_bwd_begin": (i32, [p, p, p]),
        "dynmo_migrate_layer_ready": (i32, [p, p, i32, p]),
        "dynmo_migrate_layers_bwd": (i32, [p, p, i32, p, p, i32, p, p, p, p]),
        "dynmo_migrate_bwd_end": (i32, [p, p, i32, p, p, i32, p, p, p, p]),
        "dynmo_ctx_profile_span": (i32, [p, p, p]),
        "dynmo_ctx_window_snapshot": (i32, [p, i32, p, C.c_int64]),
        "dynmo_migrate_bwd_abort": (i32, [p, p]),
        "dynmo_ctx_p2p_error_clear": (i32, [p]),
    }
    for name, (res, args) in sigs.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


EXPORTED = ["dynmo_strerror", "dynmo_last_error", "dynmo_version", "dynmo_get_unique_id",
            "dynmo_ctx_create", "dynmo_ctx_destroy", "dynmo_ctx_nranks", "dynmo_ctx_rank",
            "dynmo_ctx_set_timing", "dynmo_ctx_timing_read", "dynmo_ctx_timing_poll",
            "dynmo_profile_plan_create", "dynmo_profile_plan_destroy", "dynmo_plan_num_tiles",
            "dynmo_plan_bytes", "dynmo_plan_max_experts", "dynmo_profile_layers", "dynmo_timestamp", "dynmo_publish", "dynmo_diag_step_stamps", "dynmo_ctx_split", "dynmo_map_stages", "dynmo_ctx_timing_detach",
            "dynmo_ctx_barrier",
            "dynmo_partition_stages", "dynmo_diffuse_balance", "dynmo_repack_workers",
            "dynmo_migrate_layers", "dynmo_migration_plan", "dynmo_migrate_plan_create",
            "dynmo_prune_plan_create", "dynmo_prune_plan_destroy", "dynmo_global_prune",
            "dynmo_migrate_plan_destroy", "dynmo_migrate_layers_p2p", "dynmo_ctx_p2p_error",
            "dynmo_migrate_layers_dev", "dynmo_migrate_plan_set_ctas",
            "dynmo_migrate_bwd_begin", "dynmo_migrate_layer_ready", "dynmo_migrate_layers_bwd",
            "dynmo_migrate_bwd_end", "dynmo_ctx_profile_span",
            "dynmo_ctx_window_snapshot", "dynmo_migrate_bwd_abort",
            "dynmo_ctx_p2p_error_clear"]
