"""ctypes binding of the native library ``_sfgpu.so`` (C ABI: include/sfgpu.h).

There is no fallback: if the shared library is missing the import fails
loudly with instructions to build it.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_sfgpu.so")

c_i64p = C.POINTER(C.c_int64)
c_i32p = C.POINTER(C.c_int32)


class sfg_config(C.Structure):
    _fields_ = [
        ("deterministic", C.c_int),
        ("debug_checksum", C.c_int),
        ("force_remote", C.c_int),
        ("dense_discovery_threshold", C.c_int),
        ("seed", C.c_uint64),
        ("timeout_s", C.c_double),
    ]


class sfg_sf_info(C.Structure):
    _fields_ = [
        ("state", C.c_int),
        ("self_first", C.c_int),
        ("contiguous_leaves", C.c_int),
        ("n_root_groups", C.c_int),
        ("n_leaf_groups", C.c_int),
        ("nroots", C.c_int64),
        ("nleaves", C.c_int64),
        ("leaf_index_bound", C.c_int64),
    ]


class sfg_pattern(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("has_duplicates", C.c_int),
        ("count", C.c_int64),
        ("start", C.c_int64),
        ("dx", C.c_int64),
        ("dy", C.c_int64),
        ("dz", C.c_int64),
        ("s1", C.c_int64),
        ("s2", C.c_int64),
        ("bound", C.c_int64),
    ]


class sfg_counters(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "pack_copies", "pack_elided", "unpack_copies", "unpack_elided",
        "replace_dup_collisions", "kernel_launches", "bytes_sent", "bytes_recv",
        "transport_calls")]


ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)
ALLTOALLV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.c_void_p,
                           C.POINTER(C.c_int64))
BARRIER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p)


class sfg_ctrl_ops(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("allgather", ALLGATHER_FN), ("alltoallv", ALLTOALLV_FN),
                ("barrier", BARRIER_FN)]


# name -> (restype, argtypes); every function returns an int status
_V = C.c_void_p
_SIGS = {
    "sfg_last_error": (C.c_char_p, []),
    "sfg_version": (C.c_int, []),
    "sfg_config_default": (None, [C.POINTER(sfg_config)]),
    "sfg_world_create": (C.c_int, [C.c_int, C.c_double, C.POINTER(_V)]),
    "sfg_world_abort": (C.c_int, [_V]),
    "sfg_world_destroy": (C.c_int, [_V]),
    "sfg_nccl_unique_id": (C.c_int, [_V, C.c_size_t]),
    "sfg_comm_create": (C.c_int, [_V, C.c_int, C.c_int, C.c_int, C.c_char_p, _V,
                                  C.POINTER(sfg_config), C.POINTER(_V)]),
    "sfg_comm_create_ext": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_char_p, _V,
                                      C.POINTER(sfg_config), C.POINTER(sfg_ctrl_ops),
                                      C.POINTER(_V)]),
    "sfg_comm_destroy": (C.c_int, [_V]),
    "sfg_comm_rank": (C.c_int, [_V, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "sfg_comm_allgather": (C.c_int, [_V, _V, C.c_size_t, _V]),
    "sfg_sf_create": (C.c_int, [_V, C.POINTER(_V)]),
    "sfg_sf_destroy": (C.c_int, [_V]),
    "sfg_sf_set_graph": (C.c_int, [_V, C.c_int64, C.c_int64, _V, _V, _V]),
    "sfg_sf_set_graph_device": (C.c_int, [_V, C.c_int64, C.c_int64, _V, _V, _V]),
    "sfg_sf_setup": (C.c_int, [_V, C.c_int]),
    "sfg_sf_prepare": (C.c_int, [_V, C.c_int, C.c_int64]),
    "sfg_sf_get_info": (C.c_int, [_V, C.POINTER(sfg_sf_info)]),
    "sfg_sf_group": (C.c_int, [_V, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int64),
                               C.POINTER(sfg_pattern)]),
    "sfg_sf_group_items": (C.c_int, [_V, C.c_int, C.c_int, _V]),
    "sfg_sf_compute_degrees": (C.c_int, [_V, _V]),
    "sfg_sf_multi_sf": (C.c_int, [_V, C.POINTER(_V)]),
    "sfg_sf_graph": (C.c_int, [_V, _V, _V, _V]),
    "sfg_bcast": (C.c_int, [_V, C.c_int, C.c_int64, _V, _V, C.c_int, _V]),
    "sfg_reduce": (C.c_int, [_V, C.c_int, C.c_int64, _V, _V, C.c_int, _V]),
    "sfg_fetch_and_op": (C.c_int, [_V, C.c_int, C.c_int64, _V, _V, _V, C.c_int, _V]),
    "sfg_gather": (C.c_int, [_V, C.c_int, C.c_int64, _V, _V, _V]),
    "sfg_scatter": (C.c_int, [_V, C.c_int, C.c_int64, _V, _V, _V]),
    "sfg_bcast_begin": (C.c_int, [_V, C.c_int, C.c_int64, _V, _V, C.c_int, _V, C.POINTER(_V)]),
    "sfg_bcast_end": (C.c_int, [_V]),
    "sfg_reduce_begin": (C.c_int, [_V, C.c_int, C.c_int64, _V, _V, C.c_int, _V, C.POINTER(_V)]),
    "sfg_reduce_end": (C.c_int, [_V]),
    "sfg_fetch_and_op_begin": (C.c_int, [_V, C.c_int, C.c_int64, _V, _V, _V, C.c_int, _V,
                                         C.POINTER(_V)]),
    "sfg_fetch_and_op_end": (C.c_int, [_V]),
    "sfg_gather_begin": (C.c_int, [_V, C.c_int, C.c_int64, _V, _V, _V, C.POINTER(_V)]),
    "sfg_gather_end": (C.c_int, [_V]),
    "sfg_scatter_begin": (C.c_int, [_V, C.c_int, C.c_int64, _V, _V, _V, C.POINTER(_V)]),
    "sfg_scatter_end": (C.c_int, [_V]),
    "sfg_sf_compose": (C.c_int, [_V, _V, C.c_int, C.POINTER(_V)]),
    "sfg_sf_embed": (C.c_int, [_V, C.c_int, _V, C.c_int64, C.POINTER(_V)]),
    "sfg_sf_identity": (C.c_int, [_V, C.c_int64, C.POINTER(_V)]),
    "sfg_mat_create": (C.c_int, [_V, C.c_int64, C.c_int64, _V, _V, _V, C.c_int, C.POINTER(_V)]),
    "sfg_mat_destroy": (C.c_int, [_V]),
    "sfg_spmv": (C.c_int, [_V, _V, _V, _V, _V, _V, _V]),
    "sfg_spmv_transpose": (C.c_int, [_V, _V, _V, _V, _V, _V, _V]),
    "sfg_handle_info": (C.c_int, [_V, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "sfg_handle_free": (C.c_int, [_V]),
    "sfg_pattern_analyze": (C.c_int, [_V, C.c_int64, C.c_int, C.c_int64, C.c_int64,
                                      C.POINTER(sfg_pattern)]),
    "sfg_counters_get": (C.c_int, [C.POINTER(sfg_counters)]),
    "sfg_counters_reset": (C.c_int, []),
    "sfg_timing_enable": (C.c_int, [C.c_int]),
    "sfg_trace_dump": (C.c_int, [C.c_char_p]),
    "sfg_timing_collect": (C.c_int, [_V, C.c_int, C.POINTER(C.c_int)]),
}


class sfg_timing(C.Structure):
    _fields_ = [("tag", C.c_char * 32), ("launches", C.c_uint64), ("total_ms", C.c_double),
                ("bytes", C.c_double), ("link_bytes", C.c_double)]

EXPORTED = tuple(_SIGS)

_lib = None


def load() -> C.CDLL:
    """Load (once) and return the native library; raise if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"native library {LIB_PATH} is missing; build it with "
            "`python -m paper_2102_13018_b200.build` (there is no CPU fallback)")
    # torch first, so its NCCL/cudart are the ones resolved by soname
    try:
        import torch  # noqa: F401
    except Exception:
        pass
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().sfg_last_error()
    return msg.decode() if msg else ""
