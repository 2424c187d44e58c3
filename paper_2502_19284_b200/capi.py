"""ctypes binding of the C ABI declared in include/spmvlab_cuda.h.

The shared library is built in-tree (paper_2502_19284_b200/build.py) for sm_100a.  There is no
fallback: if the library is missing, importing the product API raises.
"""
from __future__ import annotations

import ctypes as C
import os

from .build import LIB

_lib = None

ABI_VERSION = 3  # SPMVLAB_CUDA_ABI_VERSION of include/spmvlab_cuda.h

# Every symbol include/spmvlab_cuda.h declares (checked by tests/test_capi_cpu.py).
EXPORTS = [
    "spmvlab_cuda_abi_version", "spmvlab_cuda_last_error", "spmvlab_cuda_release_pool", "spmvlab_cuda_build_format",
    "spmvlab_cuda_run_spmv", "spmvlab_cuda_run_spmv_host", "spmvlab_cuda_storage_report",
    "spmvlab_cuda_get_format_info", "spmvlab_cuda_format_array", "spmvlab_cuda_download_array",
    "spmvlab_cuda_free_format", "spmvlab_cuda_validate", "spmvlab_cuda_select_block_size",
    "spmvlab_cuda_partition_rows_by_nnz", "spmvlab_cuda_merge_path_search",
    "spmvlab_cuda_curve_keys", "spmvlab_cuda_sort_pairs", "spmvlab_cuda_exclusive_scan",
    "spmvlab_cuda_launch_count", "spmvlab_cuda_kernel_timing", "spmvlab_cuda_kernel_time",
    "spmvlab_cuda_cache_read", "spmvlab_cuda_cache_write", "spmvlab_cuda_free_coo", "spmvlab_cuda_cache_info",
    "spmvlab_cuda_iterate", "spmvlab_cuda_read_matrix_market", "spmvlab_cuda_read_matrix_market_host",
    "spmvlab_cuda_free_host_coo", "spmvlab_cuda_load_matrix", "spmvlab_cuda_crs_to_icrs",
    "spmvlab_cuda_triplet_to_bicrs", "spmvlab_cuda_bicrs_spmv", "spmvlab_cuda_bicrs_to_triplet",
    "spmvlab_cuda_free_bicrs", "spmvlab_cuda_exchange_alloc", "spmvlab_cuda_exchange_open",
    "spmvlab_cuda_exchange_close", "spmvlab_cuda_run_spmv_scatter", "spmvlab_cuda_csb_work_items",
    "spmvlab_cuda_format_to_triplet", "spmvlab_cuda_build_format_beta", "spmvlab_cuda_row_prefix",
]


class Bicrs(C.Structure):
    _fields_ = [("m", C.c_uint32), ("n", C.c_uint32), ("nnz", C.c_uint64), ("kind", C.c_int),
                ("col_inc", C.c_void_p), ("row_jump", C.c_void_p), ("n_row_jump", C.c_uint64),
                ("data", C.c_void_p)]


class MmHeader(C.Structure):
    _fields_ = [("field", C.c_int), ("symmetry", C.c_int), ("m", C.c_uint32), ("n", C.c_uint32),
                ("declared_nnz", C.c_uint64)]


class HostCoo(C.Structure):
    _fields_ = [("m", C.c_uint32), ("n", C.c_uint32), ("nnz", C.c_uint64), ("row_ind", C.POINTER(C.c_uint32)),
                ("col_ind", C.POINTER(C.c_uint32)), ("data", C.POINTER(C.c_double))]


class Coo(C.Structure):
    _fields_ = [("m", C.c_uint32), ("n", C.c_uint32), ("nnz", C.c_uint64), ("row_ind", C.c_void_p),
                ("col_ind", C.c_void_p), ("data", C.c_void_p)]


class Options(C.Structure):
    _fields_ = [("l2_bytes", C.c_uint64), ("split_threshold", C.c_uint64), ("build_threads", C.c_uint32),
                ("deterministic", C.c_uint32)]


class StorageArray(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("bytes", C.c_uint64)]


class FormatInfo(C.Structure):
    _fields_ = [("alg", C.c_int), ("m", C.c_uint32), ("n", C.c_uint32), ("nnz", C.c_uint64),
                ("log2_beta", C.c_uint32), ("block_rows", C.c_uint32), ("block_cols", C.c_uint32),
                ("element_level", C.c_uint32), ("block_level", C.c_uint32), ("bands", C.c_uint32),
                ("merge_tiles", C.c_uint32), ("work_items", C.c_uint32),
                ("merge_ipt", C.c_uint32), ("merge_panels", C.c_uint32), ("merge_panel_row_visits", C.c_uint64),
                ("merge_hot_slots", C.c_uint32), ("merge_hot_share", C.c_double)]


def lib_path() -> str:
    return LIB


def load() -> C.CDLL:
    """Loads libspmvlab_cuda.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB):
        raise RuntimeError(f"CUDA library not built: {LIB} (run __graft_entry__.build())")
    L = C.CDLL(LIB)
    vp, u32, u64, i = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
    L.spmvlab_cuda_abi_version.restype = i
    L.spmvlab_cuda_last_error.restype = C.c_char_p
    L.spmvlab_cuda_build_format.argtypes = [i, C.POINTER(Coo), C.c_uint, C.POINTER(Options), C.POINTER(vp), vp]
    L.spmvlab_cuda_run_spmv.argtypes = [i, vp, vp, u64, vp, u64, C.c_uint, C.POINTER(Options), vp]
    L.spmvlab_cuda_iterate.argtypes = [i, vp, vp, vp, u32, C.c_uint, i, vp, vp]
    L.spmvlab_cuda_read_matrix_market.argtypes = [C.c_char_p, C.POINTER(Coo), C.POINTER(MmHeader), vp]
    L.spmvlab_cuda_read_matrix_market_host.argtypes = [C.c_char_p, C.POINTER(HostCoo), C.POINTER(MmHeader)]
    L.spmvlab_cuda_free_host_coo.argtypes = [C.POINTER(HostCoo)]
    L.spmvlab_cuda_free_host_coo.restype = None
    L.spmvlab_cuda_load_matrix.argtypes = [C.c_char_p, C.POINTER(Coo), vp]
    L.spmvlab_cuda_crs_to_icrs.argtypes = [vp, C.POINTER(Bicrs), vp]
    L.spmvlab_cuda_triplet_to_bicrs.argtypes = [C.POINTER(Coo), vp, C.POINTER(Bicrs), vp]
    L.spmvlab_cuda_bicrs_spmv.argtypes = [C.POINTER(Bicrs), vp, u64, vp, u64, vp, vp]
    L.spmvlab_cuda_bicrs_to_triplet.argtypes = [C.POINTER(Bicrs), vp, vp, vp]
    L.spmvlab_cuda_free_bicrs.argtypes = [C.POINTER(Bicrs)]
    L.spmvlab_cuda_free_bicrs.restype = None
    L.spmvlab_cuda_csb_work_items.argtypes = [vp, u64, vp, u64, C.POINTER(u64), vp]
    L.spmvlab_cuda_format_to_triplet.argtypes = [vp, vp, vp, vp, vp]
    L.spmvlab_cuda_row_prefix.argtypes = [C.POINTER(Coo), vp, vp]
    L.spmvlab_cuda_build_format_beta.argtypes = [i, C.POINTER(Coo), C.c_uint, C.c_uint, C.POINTER(vp), vp]
    L.spmvlab_cuda_exchange_alloc.argtypes = [u64, C.POINTER(vp), C.POINTER(C.c_ubyte)]
    L.spmvlab_cuda_exchange_open.argtypes = [C.POINTER(C.c_ubyte), C.POINTER(vp)]
    L.spmvlab_cuda_exchange_close.argtypes = [vp, i]
    L.spmvlab_cuda_run_spmv_scatter.argtypes = [vp, vp, u64, vp, u64, C.POINTER(vp), C.c_uint, u64, u64, vp]
    L.spmvlab_cuda_run_spmv_host.argtypes = [i, vp, vp, u64, vp, u64, C.c_uint, C.POINTER(Options), vp, vp, vp]
    L.spmvlab_cuda_storage_report.argtypes = [vp, C.POINTER(StorageArray), C.c_size_t, C.POINTER(C.c_size_t)]
    L.spmvlab_cuda_get_format_info.argtypes = [vp, C.POINTER(FormatInfo)]
    L.spmvlab_cuda_format_array.argtypes = [vp, C.c_char_p, C.POINTER(vp), C.POINTER(u64)]
    L.spmvlab_cuda_download_array.argtypes = [vp, C.c_char_p, vp, u64, C.POINTER(u64)]
    L.spmvlab_cuda_free_format.argtypes = [vp]
    L.spmvlab_cuda_free_format.restype = None
    L.spmvlab_cuda_validate.argtypes = [C.POINTER(Coo), vp]
    L.spmvlab_cuda_select_block_size.restype = C.c_uint
    L.spmvlab_cuda_select_block_size.argtypes = [u64, C.c_uint, u64]
    L.spmvlab_cuda_partition_rows_by_nnz.argtypes = [vp, u32, C.c_uint, C.c_uint, vp]
    L.spmvlab_cuda_merge_path_search.argtypes = [vp, u64, vp, u64, vp, u64, vp, vp]
    L.spmvlab_cuda_curve_keys.argtypes = [i, vp, vp, u64, C.c_uint, vp, vp]
    L.spmvlab_cuda_sort_pairs.argtypes = [vp, vp, u64, i, i, vp]
    L.spmvlab_cuda_exclusive_scan.argtypes = [vp, vp, u64, vp]
    L.spmvlab_cuda_launch_count.restype = u64
    L.spmvlab_cuda_launch_count.argtypes = []
    L.spmvlab_cuda_kernel_timing.restype = None
    L.spmvlab_cuda_kernel_timing.argtypes = [i]
    L.spmvlab_cuda_kernel_time.argtypes = [C.POINTER(C.c_double), C.POINTER(u64), C.c_char_p, C.c_size_t]
    L.spmvlab_cuda_cache_read.argtypes = [C.c_char_p, C.POINTER(Coo), vp]
    L.spmvlab_cuda_cache_write.argtypes = [C.c_char_p, C.POINTER(Coo), vp]
    L.spmvlab_cuda_free_coo.argtypes = [C.POINTER(Coo)]
    L.spmvlab_cuda_free_coo.restype = None
    L.spmvlab_cuda_cache_info.argtypes = [C.c_char_p, C.POINTER(u32), C.POINTER(u32), C.POINTER(u64)]
    if L.spmvlab_cuda_abi_version() != ABI_VERSION:
        raise RuntimeError(f"{LIB} has ABI {L.spmvlab_cuda_abi_version()}, this package needs {ABI_VERSION} "
                           "(stale build: run __graft_entry__.build())")
    _lib = L
    return L
