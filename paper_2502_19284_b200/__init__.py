"""spmvlab-b200: B200-native (sm_100a) SpMV hot path of arXiv 2502.19284.

The product is libspmvlab_cuda.so (C ABI: include/spmvlab_cuda.h); this package is its Python
host mirror of the reference's algorithm interface (inc/engine.hpp).
"""
from .engine import (  # noqa: F401
    Algorithm, BuiltFormat, EngineOptions, Error, ErrorKind, StorageBreakdown, TripletMatrix,
    algorithm_from_name, algorithm_name, all_algorithms, build_format, build_format_beta, row_prefix, cache_read, cache_write, curve_keys,
    MatrixHeader, load_matrix, read_matrix_market, read_matrix_market_host,
    IncrementalRowStorage, bicrs_from_arrays, crs_to_icrs, triplet_to_bicrs,
    CSB_ITEM_DTYPE, csb_items_numpy, csb_work_items,
    format_to_triplet, crs_to_triplet, csb_to_triplet, bcoh_to_triplet, mergeb_to_triplet,
    engine_block_size, exclusive_scan, iterate, merge_path_search, partition_rows_by_nnz, release_cached_memory, run_spmv,
    run_spmv_host, select_block_size, sort_pairs, storage_report, validate,
)
