"""ctypes binding of the C-ABI in ``include/sfcnl_cu.h`` (``libsfcnl_b200.so``).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2602_19873_b200``). There is no fallback: if the library is
missing, importing the GPU API raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# SFCNL_LIB: an alternative build of the same library (A/B runs of compile-time variants)
LIB_PATH = os.environ.get("SFCNL_LIB") or os.path.join(HERE, "libsfcnl_b200.so")

# status codes (sfcnl_cu.h)
OK, INPUT_ERROR, BUILD_ERROR, DECODE_ERROR, CUDA_ERROR = 0, 1, 2, 3, 4


class InputError(ValueError):
    """sfcnl::InputError (core.hpp:18)."""


class BuildError(RuntimeError):
    """sfcnl::BuildError (core.hpp:23)."""


class DecodeError(RuntimeError):
    """sfcnl::DecodeError (core.hpp:28); carries ``byte_offset``."""

    def __init__(self, msg, byte_offset=0):
        super().__init__(msg)
        self.byte_offset = byte_offset


class CudaError(RuntimeError):
    pass


def raise_for(code: int, msg: str, offset: int = 0):
    if code == OK:
        return
    if code == INPUT_ERROR:
        raise InputError(msg)
    if code == BUILD_ERROR:
        raise BuildError(msg)
    if code == DECODE_ERROR:
        raise DecodeError(msg, offset)
    raise CudaError(msg)


class Box(C.Structure):
    _fields_ = [("lo", C.c_double * 3), ("hi", C.c_double * 3), ("periodic", C.c_int32 * 3)]


class Node(C.Structure):
    _fields_ = [("key_first", C.c_uint64), ("key_last", C.c_uint64), ("particle_begin", C.c_uint32),
                ("particle_end", C.c_uint32), ("first_child", C.c_int32), ("depth", C.c_uint8),
                ("pad_", C.c_uint8 * 3)]


class BuildParamsC(C.Structure):
    _fields_ = [("ci", C.c_uint32), ("cj", C.c_uint32), ("w", C.c_int32), ("mode", C.c_int32),
                ("compress", C.c_int32), ("build_radius_scale", C.c_double)]


class PassParamsC(C.Structure):
    _fields_ = [("kernel", C.c_int32), ("precision", C.c_int32), ("query_scale", C.c_double),
                ("epsilon", C.c_double), ("sigma", C.c_double), ("coulomb_k", C.c_double)]


# every symbol the header declares (checked by tests/test_abi.py)
EXPORTS = [
    "sfcnl_cu_ctx_create", "sfcnl_cu_ctx_destroy", "sfcnl_cu_last_error", "sfcnl_cu_stream",
    "sfcnl_cu_synchronize", "sfcnl_cu_launch_count", "sfcnl_cu_set_timing", "sfcnl_cu_stage_times",
    "sfcnl_cu_set_particles", "sfcnl_cu_set_field", "sfcnl_cu_set_sorted_particles",
    "sfcnl_cu_set_sorted_field", "sfcnl_cu_sort_by_sfc", "sfcnl_cu_get_order", "sfcnl_cu_set_order",
    "sfcnl_cu_apply_order", "sfcnl_cu_get_sorted", "sfcnl_cu_build_octree", "sfcnl_cu_get_octree",
    "sfcnl_cu_set_octree", "sfcnl_cu_node_geometry", "sfcnl_cu_build_store", "sfcnl_cu_get_store",
    "sfcnl_cu_set_store", "sfcnl_cu_reduce", "sfcnl_cu_get_device_view", "sfcnl_cu_sorted_field_ptr",
    "sfcnl_codec_encode", "sfcnl_codec_decode_into",
    "sfcnl_hilbert_encode", "sfcnl_hilbert_decode", "sfcnl_last_host_error", "sfcnl_make_uniform",
    "sfcnl_make_evrard", "sfcnl_cu_build_store_range", "sfcnl_cu_alloc_sorted", "sfcnl_cu_write_sorted",
    "sfcnl_cu_read_sorted", "sfcnl_cu_read_order", "sfcnl_cu_set_keys", "sfcnl_cu_apply_order_into",
    "sfcnl_cu_node_geometry_range", "sfcnl_cu_halo_mark", "sfcnl_cu_device_array",
    "sfcnl_cu_set_particle_records", "sfcnl_cu_build_full_list", "sfcnl_cu_get_full_list",
    "sfcnl_cu_set_full_list", "sfcnl_cu_reduce_full", "sfcnl_cu_cluster_slots", "sfcnl_cu_sym_range_entries",
    "sfcnl_cu_sym_range_final", "sfcnl_cu_key_hist", "sfcnl_cu_merge_runs", "sfcnl_cu_build_octree_dist",
    "sfcnl_cu_leaf_boxes", "sfcnl_cu_domain_boxes", "sfcnl_cu_halo_select", "sfcnl_cu_pack_clusters",
    "sfcnl_cu_dd_place", "sfcnl_cu_dd_localize", "sfcnl_cu_dd_lc2g", "sfcnl_cu_dd_clear", "sfcnl_cu_memory_bytes",
]

# int (*)(void* user, uint32_t* device_data, uint64_t count): in-place SUM over ranks
ALLREDUCE_U32 = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64)

_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build() or make -C paper_2602_19873_b200")
    L = C.CDLL(LIB_PATH)
    P = C.c_void_p
    pd = C.POINTER(C.c_double)
    u64, u32, i32 = C.c_uint64, C.c_uint32, C.c_int32
    sig = {
        "sfcnl_cu_ctx_create": (C.c_int, [C.c_int, C.POINTER(P)]),
        "sfcnl_cu_ctx_destroy": (None, [P]),
        "sfcnl_cu_last_error": (C.c_char_p, [P, C.POINTER(u64)]),
        "sfcnl_cu_stream": (P, [P]),
        "sfcnl_cu_synchronize": (C.c_int, [P]),
        "sfcnl_cu_launch_count": (u64, [P]),
        "sfcnl_cu_set_timing": (C.c_int, [P, C.c_int]),
        "sfcnl_cu_stage_times": (C.c_int, [P, pd, C.c_int]),
        "sfcnl_cu_set_particles": (C.c_int, [P, u64, P, P, P, P, C.POINTER(Box)]),
        "sfcnl_cu_set_field": (C.c_int, [P, C.c_char_p, P]),
        "sfcnl_cu_set_sorted_particles": (C.c_int, [P, u64, P, P, P, P, C.POINTER(Box)]),
        "sfcnl_cu_set_sorted_field": (C.c_int, [P, C.c_char_p, P]),
        "sfcnl_cu_sort_by_sfc": (C.c_int, [P, C.c_int]),
        "sfcnl_cu_get_order": (C.c_int, [P, P, P]),
        "sfcnl_cu_set_order": (C.c_int, [P, u64, P, P, C.c_int]),
        "sfcnl_cu_apply_order": (C.c_int, [P]),
        "sfcnl_cu_get_sorted": (C.c_int, [P, C.c_char_p, P]),
        "sfcnl_cu_build_octree": (C.c_int, [P, u32, C.POINTER(u64)]),
        "sfcnl_cu_get_octree": (C.c_int, [P, P]),
        "sfcnl_cu_set_octree": (C.c_int, [P, u64, P, C.c_int, u64]),
        "sfcnl_cu_node_geometry": (C.c_int, [P, P, P, P]),
        "sfcnl_cu_build_store": (C.c_int, [P, C.POINTER(BuildParamsC), C.POINTER(u64), C.POINTER(u64)]),
        "sfcnl_cu_get_store": (C.c_int, [P, P, P, P]),
        "sfcnl_cu_set_store": (C.c_int, [P, C.POINTER(BuildParamsC), u64, u64, P, P, P, u64]),
        "sfcnl_cu_reduce": (C.c_int, [P, C.POINTER(PassParamsC), C.POINTER(P), P]),
        "sfcnl_codec_encode": (C.c_int, [P, u64, C.c_int, P, u64, C.POINTER(u64)]),
        "sfcnl_codec_decode_into": (C.c_int, [P, u64, u32, C.c_int, P, C.POINTER(u64)]),
        "sfcnl_hilbert_encode": (C.c_int, [u32, u32, u32, C.c_int, C.POINTER(u64)]),
        "sfcnl_hilbert_decode": (C.c_int, [u64, C.c_int, C.POINTER(u32)]),
        "sfcnl_last_host_error": (C.c_char_p, [C.POINTER(u64)]),
        "sfcnl_make_uniform": (C.c_int, [u64, C.c_double, C.c_double, C.POINTER(i32), C.c_double, u64,
                                         P, P, P, P, P, P, P]),
        "sfcnl_make_evrard": (C.c_int, [u64, C.c_double, i32, C.POINTER(i32), u64, P, P, P, P, P, P, P]),
        "sfcnl_cu_build_store_range": (C.c_int, [P, C.POINTER(BuildParamsC), u64, u64, C.c_double,
                                                 C.POINTER(u64), C.POINTER(u64)]),
        "sfcnl_cu_alloc_sorted": (C.c_int, [P, u64, C.POINTER(Box), C.POINTER(C.c_char_p), C.c_int]),
        "sfcnl_cu_write_sorted": (C.c_int, [P, C.c_char_p, u64, u64, P, C.c_int]),
        "sfcnl_cu_read_sorted": (C.c_int, [P, C.c_char_p, u64, u64, P, C.c_int]),
        "sfcnl_cu_read_order": (C.c_int, [P, u64, u64, P, P, C.c_int]),
        "sfcnl_cu_set_keys": (C.c_int, [P, u64, P, C.c_int, C.c_int]),
        "sfcnl_cu_apply_order_into": (C.c_int, [P, u64]),
        "sfcnl_cu_node_geometry_range": (C.c_int, [P, u64, u64]),
        "sfcnl_cu_halo_mark": (C.c_int, [P, C.POINTER(BuildParamsC), u64, u64, C.POINTER(u64)]),
        "sfcnl_cu_device_array": (C.c_int, [P, C.c_char_p, C.POINTER(P), C.POINTER(u64)]),
        "sfcnl_cu_set_particle_records": (C.c_int, [P, u64, P, C.c_int, C.POINTER(C.c_char_p), C.POINTER(Box)]),
        "sfcnl_cu_build_full_list": (C.c_int, [P, C.c_double, C.POINTER(u64)]),
        "sfcnl_cu_get_full_list": (C.c_int, [P, P, P]),
        "sfcnl_cu_set_full_list": (C.c_int, [P, u64, C.c_int, C.c_double, P, P, u64]),
        "sfcnl_cu_reduce_full": (C.c_int, [P, C.POINTER(PassParamsC), C.POINTER(P), P]),
        "sfcnl_cu_cluster_slots": (C.c_int, [P, C.POINTER(u64)]),
        "sfcnl_cu_sym_range_entries": (C.c_int, [P, C.POINTER(PassParamsC), C.POINTER(u64)]),
        "sfcnl_cu_sym_range_final": (C.c_int, [P, C.POINTER(PassParamsC), u64, P, P, P, P, C.POINTER(P), P]),
        "sfcnl_cu_key_hist": (C.c_int, [P, u32, P, C.c_int, P]),
        "sfcnl_cu_merge_runs": (C.c_int, [P, u64, u32, C.POINTER(P), P, u32, C.POINTER(u64), C.POINTER(P)]),
        "sfcnl_cu_build_octree_dist": (C.c_int, [P, u32, u64, ALLREDUCE_U32, P, C.POINTER(u64)]),
        "sfcnl_cu_leaf_boxes": (C.c_int, [P, u64, u64, P, P, P, P]),
        "sfcnl_cu_domain_boxes": (C.c_int, [P, u64, P, P, P, u32, P]),
        "sfcnl_cu_halo_select": (C.c_int, [P, u64, u64, u32, P, u32, u32, u32, P, C.c_double, P]),
        "sfcnl_cu_pack_clusters": (C.c_int, [P, u64, u64, u32, P, u64, u32, C.POINTER(P), P]),
        "sfcnl_cu_dd_place": (C.c_int, [P, u64, u64, u64, u32, P, u64, u32, C.POINTER(P), P, u64, P, P]),
        "sfcnl_cu_dd_localize": (C.c_int, [P, u32, P, P, u64, P]),
        "sfcnl_cu_dd_lc2g": (C.c_int, [P, u64, P, P, P, u64]),
        "sfcnl_cu_dd_clear": (C.c_int, [P]),
        "sfcnl_cu_memory_bytes": (C.c_int, [P, C.POINTER(u64)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def host_check(rc):
    if rc:
        off = C.c_uint64(0)
        msg = lib().sfcnl_last_host_error(C.byref(off)).decode()
        raise_for(rc, msg, off.value)
