"""ctypes front end for the CPU checkers (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs import
this module, and only to CHECK or to time the reference's CPU path.  The product
(paper_2502_19284_b200) never imports it.

Two checkers share one interface:
  * ``Oracle``    -- oracle/liboracle.so, the plain-C restatement (spmv_oracle.c), always present;
  * ``Reference`` -- oracle/_ref/libspmvref.so, the unmodified reference headers behind a C shim
                     (ref_shim.cpp); built in the dev container, travels to the GPU box prebuilt.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspmvref.so")

ALGORITHMS = ["crs", "parcrs", "merge", "csb", "csbh", "bcoh", "bcohc", "bcohch", "bcohchp",
              "mergeb", "mergebh"]

_DT = {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}
# CsbWorkItem (inc/spmv_parallel.hpp:167-174) as orc_csb_item / spmvlab_cuda_csb_item
CSB_ITEM_DTYPE = np.dtype([("block_row", np.uint32), ("cell_begin", np.uint32), ("cell_end", np.uint32),
                           ("temp_slot", np.int32), ("elem_begin", np.uint64), ("elem_end", np.uint64)])
_SIGNED = {"row_jump_block": np.int16, "col_jump_block": np.int16, "data": np.float64}


class OrcArray(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("data", C.c_void_p), ("bytes", C.c_uint64),
                ("elem_size", C.c_uint32)]


class OrcFormat(C.Structure):
    _fields_ = [("alg", C.c_int), ("m", C.c_uint32), ("n", C.c_uint32), ("nnz", C.c_uint32),
                ("log2_beta", C.c_uint32), ("block_rows", C.c_uint32), ("block_cols", C.c_uint32),
                ("element_level", C.c_uint32), ("block_level", C.c_uint32), ("bands", C.c_uint32),
                ("nstorage", C.c_int), ("narrays", C.c_int), ("arrays", OrcArray * 24)]


META = ("alg", "m", "n", "nnz", "log2_beta", "block_rows", "block_cols", "element_level",
        "block_level", "bands")


class CheckerError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"checker error {code}: {msg}")
        self.code = code


@dataclass
class Built:
    """A CPU-built format: named numpy arrays (copies) plus geometry."""
    meta: dict
    arrays: dict = field(default_factory=dict)
    storage: list = field(default_factory=list)  # [(name, bytes)] in storage_report order
    handle: object = None  # checker-side object used by spmv()

    def storage_total(self) -> int:
        return sum(b for _, b in self.storage)


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _export(fp) -> tuple[dict, dict, list]:
    f = fp.contents
    meta = {k: int(getattr(f, k)) for k in META}
    arrays, storage = {}, []
    for i in range(f.narrays):
        a = f.arrays[i]
        name = a.name.decode()
        dt = _SIGNED.get(name, _DT[a.elem_size])
        cnt = a.bytes // a.elem_size
        buf = (C.c_char * a.bytes).from_address(a.data) if a.bytes else b""
        arrays[name] = np.frombuffer(bytes(buf), dtype=dt, count=cnt).copy() if a.bytes else \
            np.zeros(0, dtype=dt)
        if i < f.nstorage:
            storage.append((name, int(a.bytes)))
    return meta, arrays, storage


def _coo_args(rows, cols, vals):
    rows = np.ascontiguousarray(rows, dtype=np.uint32)
    cols = np.ascontiguousarray(cols, dtype=np.uint32)
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    return rows, cols, vals


class Oracle:
    """The C restatement (spmv_oracle.c)."""

    kind = "port"

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle)")
        L = self.lib = C.CDLL(path)
        L.orc_build_format.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64,
                                       C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                       C.POINTER(C.c_double), C.c_uint, C.c_uint64,
                                       C.POINTER(C.POINTER(OrcFormat))]
        L.orc_free_format.argtypes = [C.POINTER(OrcFormat)]
        L.orc_run_spmv.argtypes = [C.c_int, C.POINTER(OrcFormat), C.POINTER(C.c_double), C.c_uint64,
                                   C.POINTER(C.c_double), C.c_uint64, C.c_uint, C.c_uint64]
        L.orc_spmv_triplet.argtypes = [C.c_uint32, C.c_uint64, C.POINTER(C.c_uint32),
                                       C.POINTER(C.c_uint32), C.POINTER(C.c_double),
                                       C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.orc_abs_spmv.argtypes = L.orc_spmv_triplet.argtypes
        L.orc_select_block_size.restype = C.c_uint
        L.orc_select_block_size.argtypes = [C.c_uint64, C.c_uint, C.c_uint64]
        L.orc_engine_log2_beta.restype = C.c_uint
        L.orc_engine_log2_beta.argtypes = [C.c_int, C.c_uint32, C.c_uint64]
        L.orc_partition_rows_by_nnz.argtypes = [C.POINTER(C.c_uint32), C.c_uint32, C.c_uint, C.c_uint,
                                                C.POINTER(C.c_uint32)]
        for fn in ("orc_morton_encode", "orc_hilbert_encode"):
            getattr(L, fn).restype = C.c_uint64
            getattr(L, fn).argtypes = [C.c_uint32, C.c_uint32, C.c_uint]
        for fn in ("orc_morton_decode", "orc_hilbert_decode"):
            getattr(L, fn).argtypes = [C.c_uint64, C.c_uint, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.orc_covering_level.restype = C.c_uint
        L.orc_covering_level.argtypes = [C.c_uint32, C.c_uint32]
        L.orc_diagonal_search.argtypes = [C.POINTER(C.c_uint32), C.c_uint64, C.c_uint64, C.c_uint64,
                                          C.c_int, C.POINTER(C.c_uint32), C.POINTER(C.c_uint64),
                                          C.POINTER(C.c_uint64)]
        L.orc_row_prefix.argtypes = [C.c_uint32, C.c_uint64, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.orc_validate.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.POINTER(C.c_uint32),
                                   C.POINTER(C.c_uint32)]
        L.orc_verification_input.argtypes = [C.c_uint32, C.c_uint64, C.POINTER(C.c_double)]
        L.orc_cache_read.argtypes = [C.c_char_p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                     C.POINTER(C.c_uint64), C.POINTER(C.POINTER(C.c_uint32)),
                                     C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.POINTER(C.c_double))]
        L.orc_cache_write.argtypes = [C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint64, C.POINTER(C.c_uint32),
                                      C.POINTER(C.c_uint32), C.POINTER(C.c_double)]
        L.orc_free.argtypes = [C.c_void_p]
        L.orc_build_format_beta.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, C.POINTER(C.c_uint32),
                                            C.POINTER(C.c_uint32), C.POINTER(C.c_double), C.c_uint, C.c_uint,
                                            C.POINTER(C.POINTER(OrcFormat))]
        L.orc_format_to_triplet.argtypes = [C.POINTER(OrcFormat), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                            C.POINTER(C.c_double)]
        L.orc_csb_work_items.argtypes = [C.POINTER(OrcFormat), C.c_uint64, C.c_void_p, C.c_uint64,
                                         C.POINTER(C.c_uint64)]

    # -- formats ----------------------------------------------------------------------------
    def build(self, alg: int, m: int, n: int, rows, cols, vals, threads: int = 1,
              l2_bytes: int = 512 * 1024) -> Built:
        rows, cols, vals = _coo_args(rows, cols, vals)
        fp = C.POINTER(OrcFormat)()
        rc = self.lib.orc_build_format(alg, m, n, len(vals), _p(rows, C.c_uint32), _p(cols, C.c_uint32),
                                       _p(vals, C.c_double), threads, l2_bytes, C.byref(fp))
        if rc:
            raise CheckerError(rc, "orc_build_format")
        try:
            meta, arrays, storage = _export(fp)
        finally:
            self.lib.orc_free_format(fp)
        return Built(meta, arrays, storage, handle=None)

    def build_beta(self, alg: int, m: int, n: int, rows, cols, vals, log2_beta: int, threads: int = 1) -> Built:
        """build_csb / build_mergeb / build_bcoh with an explicit block size."""
        rows, cols, vals = _coo_args(rows, cols, vals)
        fp = C.POINTER(OrcFormat)()
        rc = self.lib.orc_build_format_beta(alg, m, n, len(vals), _p(rows, C.c_uint32), _p(cols, C.c_uint32),
                                            _p(vals, C.c_double), log2_beta, threads, C.byref(fp))
        if rc:
            raise CheckerError(rc, "orc_build_format_beta")
        try:
            meta, arrays, storage = _export(fp)
        finally:
            self.lib.orc_free_format(fp)
        return Built(meta, arrays, storage, handle=None)

    @staticmethod
    def _struct(built: Built):
        """The C struct over the numpy arrays (returned with the arrays it points into)."""
        f = OrcFormat()
        for k, v in built.meta.items():
            setattr(f, k, v)
        keep = []
        names = list(built.arrays)
        f.narrays = len(names)
        f.nstorage = len(built.storage)
        for i, name in enumerate(names):
            a = np.ascontiguousarray(built.arrays[name])
            keep.append(a)
            f.arrays[i].name = name.encode()
            f.arrays[i].data = a.ctypes.data if a.size else None
            f.arrays[i].bytes = a.nbytes
            f.arrays[i].elem_size = a.itemsize
        return f, keep

    def spmv(self, built: Built, alg: int, x, p: int = 1, split_threshold: int = 0):
        """Rebuilds the C struct from the numpy arrays and replays the reference kernel."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(built.meta["m"], dtype=np.float64)
        f, keep = self._struct(built)
        rc = self.lib.orc_run_spmv(alg, C.byref(f), _p(x, C.c_double), len(x), _p(y, C.c_double),
                                   len(y), p, split_threshold)
        if rc:
            raise CheckerError(rc, "orc_run_spmv")
        return y

    def to_triplet(self, built: Built):
        """orc_format_to_triplet: (rows, cols, vals) in storage order."""
        f, keep = self._struct(built)
        nnz = built.meta["nnz"]
        r, c, v = np.zeros(nnz, np.uint32), np.zeros(nnz, np.uint32), np.zeros(nnz)
        rc = self.lib.orc_format_to_triplet(C.byref(f), _p(r, C.c_uint32), _p(c, C.c_uint32), _p(v, C.c_double))
        if rc:
            raise CheckerError(rc, "orc_format_to_triplet")
        return r, c, v

    def csb_work_items(self, built: Built, split_threshold: int = 0) -> np.ndarray:
        """spmv_csb's work-item list (structured array, CSB_ITEM_DTYPE)."""
        f, keep = self._struct(built)
        cnt = C.c_uint64()
        rc = self.lib.orc_csb_work_items(C.byref(f), split_threshold, None, 0, C.byref(cnt))
        if rc:
            raise CheckerError(rc, "orc_csb_work_items")
        out = np.zeros(cnt.value, dtype=CSB_ITEM_DTYPE)
        rc = self.lib.orc_csb_work_items(C.byref(f), split_threshold, out.ctypes.data_as(C.c_void_p),
                                         len(out), C.byref(cnt))
        if rc:
            raise CheckerError(rc, "orc_csb_work_items")
        return out

    # -- primitives -------------------------------------------------------------------------
    def spmv_triplet(self, m, rows, cols, vals, x):
        rows, cols, vals = _coo_args(rows, cols, vals)
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(m, dtype=np.float64)
        self.lib.orc_spmv_triplet(m, len(vals), _p(rows, C.c_uint32), _p(cols, C.c_uint32),
                                  _p(vals, C.c_double), _p(x, C.c_double), _p(y, C.c_double))
        return y

    def abs_spmv(self, m, rows, cols, vals, x):
        rows, cols, vals = _coo_args(rows, cols, vals)
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(m, dtype=np.float64)
        self.lib.orc_abs_spmv(m, len(vals), _p(rows, C.c_uint32), _p(cols, C.c_uint32),
                              _p(vals, C.c_double), _p(x, C.c_double), _p(y, C.c_double))
        return y

    def select_block_size(self, n, cap, l2=512 * 1024):
        return int(self.lib.orc_select_block_size(n, cap, l2))

    def engine_log2_beta(self, alg, n, l2=512 * 1024):
        return int(self.lib.orc_engine_log2_beta(alg, n, l2))

    def partition_rows_by_nnz(self, prefix, p, log2_beta):
        prefix = np.ascontiguousarray(prefix, dtype=np.uint32)
        out = np.zeros(p + 1, dtype=np.uint32)
        rc = self.lib.orc_partition_rows_by_nnz(_p(prefix, C.c_uint32), len(prefix) - 1, p, log2_beta,
                                                _p(out, C.c_uint32))
        if rc:
            raise CheckerError(rc, "partition")
        return out

    def morton(self, r, c, level):
        return int(self.lib.orc_morton_encode(r, c, level))

    def hilbert(self, r, c, level):
        return int(self.lib.orc_hilbert_encode(r, c, level))

    def hilbert_decode(self, d, level):
        r, c = C.c_uint32(), C.c_uint32()
        self.lib.orc_hilbert_decode(d, level, C.byref(r), C.byref(c))
        return r.value, c.value

    def morton_decode(self, d, level):
        r, c = C.c_uint32(), C.c_uint32()
        self.lib.orc_morton_decode(d, level, C.byref(r), C.byref(c))
        return r.value, c.value

    def covering_level(self, rows, cols):
        return int(self.lib.orc_covering_level(rows, cols))

    def diagonal_search(self, a, b, diag):
        """Merge path crossing of diagonal ``diag`` for explicit lists a, b."""
        a = np.ascontiguousarray(a, dtype=np.uint32)
        b = np.ascontiguousarray(b, dtype=np.uint32)
        i, j = C.c_uint64(), C.c_uint64()
        rc = self.lib.orc_diagonal_search(_p(a, C.c_uint32), len(a), len(b), diag, 0, _p(b, C.c_uint32),
                                          C.byref(i), C.byref(j))
        if rc:
            raise CheckerError(rc, "diagonal_search")
        return i.value, j.value

    def row_prefix(self, m, rows):
        rows = np.ascontiguousarray(rows, dtype=np.uint32)
        out = np.zeros(m + 1, dtype=np.uint32)
        self.lib.orc_row_prefix(m, len(rows), _p(rows, C.c_uint32), _p(out, C.c_uint32))
        return out

    def validate(self, m, n, rows, cols):
        rows = np.ascontiguousarray(rows, dtype=np.uint32)
        cols = np.ascontiguousarray(cols, dtype=np.uint32)
        return int(self.lib.orc_validate(m, n, len(rows), _p(rows, C.c_uint32), _p(cols, C.c_uint32)))

    def verification_input(self, n, seed=1):
        x = np.zeros(n, dtype=np.float64)
        self.lib.orc_verification_input(n, seed, _p(x, C.c_double))
        return x

    def cache_read(self, path):
        """(m, n, rows, cols, vals) or CheckerError (inc/cache_io.hpp:69-91)."""
        return _cache_read(self.lib.orc_cache_read, self.lib.orc_free, path)

    def cache_write(self, path, m, n, rows, cols, vals):
        rows, cols, vals = _coo_args(rows, cols, vals)
        rc = self.lib.orc_cache_write(path.encode(), m, n, len(vals), _p(rows, C.c_uint32),
                                      _p(cols, C.c_uint32), _p(vals, C.c_double))
        if rc:
            raise CheckerError(rc, "orc_cache_write")


def _cache_read(fn, free, path):
    m, n, nnz = C.c_uint32(), C.c_uint32(), C.c_uint64()
    r, c, v = C.POINTER(C.c_uint32)(), C.POINTER(C.c_uint32)(), C.POINTER(C.c_double)()
    rc = fn(path.encode(), C.byref(m), C.byref(n), C.byref(nnz), C.byref(r), C.byref(c), C.byref(v))
    if rc:
        raise CheckerError(rc, f"cache_read {path}")
    k = nnz.value
    out = (m.value, n.value, np.ctypeslib.as_array(r, (k,)).copy() if k else np.zeros(0, np.uint32),
           np.ctypeslib.as_array(c, (k,)).copy() if k else np.zeros(0, np.uint32),
           np.ctypeslib.as_array(v, (k,)).copy() if k else np.zeros(0))
    for p in (r, c, v):
        free(C.cast(p, C.c_void_p))
    return out


class RefBenchRecord(C.Structure):
    _fields_ = [("alg", C.c_int), ("threads", C.c_uint), ("min_time", C.c_double), ("speedup", C.c_double),
                ("convert_time", C.c_double), ("convert_ratio", C.c_double), ("density", C.c_double),
                ("status", C.c_char * 128)]


class Reference:
    """The unmodified reference (oracle/_ref/libspmvref.so)."""

    kind = "reference"

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle ref, needs /root/reference)")
        L = self.lib = C.CDLL(path)
        L.ref_build.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, C.POINTER(C.c_uint32),
                                C.POINTER(C.c_uint32), C.POINTER(C.c_double), C.c_uint, C.c_uint64,
                                C.c_uint, C.POINTER(C.c_void_p)]
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_run.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_double), C.c_uint64,
                              C.POINTER(C.c_double), C.c_uint64, C.c_uint, C.c_uint64]
        L.ref_time_spmv.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_double), C.c_uint64, C.c_uint64,
                                    C.c_uint, C.c_uint, C.c_uint, C.POINTER(C.c_double),
                                    C.POINTER(C.c_double)]
        L.ref_export.argtypes = [C.c_void_p, C.POINTER(C.POINTER(OrcFormat))]
        L.ref_free_export.argtypes = [C.POINTER(OrcFormat)]
        L.ref_storage_total.restype = C.c_uint64
        L.ref_storage_total.argtypes = [C.c_void_p]
        L.ref_last_error.restype = C.c_char_p
        L.ref_select_block_size.restype = C.c_uint
        L.ref_select_block_size.argtypes = [C.c_uint64, C.c_uint, C.c_uint64]
        for fn in ("ref_morton", "ref_hilbert"):
            getattr(L, fn).restype = C.c_uint64
            getattr(L, fn).argtypes = [C.c_uint32, C.c_uint32, C.c_uint]
        L.ref_diagonal_search.argtypes = [C.POINTER(C.c_uint32), C.c_uint64, C.POINTER(C.c_uint32),
                                          C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64),
                                          C.POINTER(C.c_uint64)]
        L.ref_partition_rows_by_nnz.argtypes = [C.POINTER(C.c_uint32), C.c_uint32, C.c_uint, C.c_uint,
                                                C.POINTER(C.c_uint32)]
        L.ref_verification_input.argtypes = [C.c_uint32, C.c_uint64, C.POINTER(C.c_double)]
        L.ref_hardware_threads.restype = C.c_uint
        L.ref_cache_read.argtypes = [C.c_char_p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                     C.POINTER(C.c_uint64), C.POINTER(C.POINTER(C.c_uint32)),
                                     C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.POINTER(C.c_double))]
        L.ref_cache_write.argtypes = [C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint64, C.POINTER(C.c_uint32),
                                      C.POINTER(C.c_uint32), C.POINTER(C.c_double)]
        L.ref_free_buf.argtypes = [C.c_void_p]
        L.ref_build_beta.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, C.POINTER(C.c_uint32),
                                     C.POINTER(C.c_uint32), C.POINTER(C.c_double), C.c_uint, C.c_uint,
                                     C.POINTER(C.c_void_p)]
        L.ref_to_triplet.argtypes = [C.c_void_p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                     C.POINTER(C.c_double)]
        L.ref_bench.restype = C.c_int64
        L.ref_bench.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, C.POINTER(C.c_uint32),
                                C.POINTER(C.c_uint32), C.POINTER(C.c_double), C.POINTER(C.c_int), C.c_uint,
                                C.POINTER(C.c_uint), C.c_uint, C.c_uint, C.c_uint, C.c_uint,
                                C.POINTER(RefBenchRecord), C.c_uint64]
        L.ref_csb_leaves.restype = C.c_int64
        L.ref_csb_leaves.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64), C.c_uint64]

    def cache_read(self, path):
        return _cache_read(self.lib.ref_cache_read, self.lib.ref_free_buf, path)

    def cache_write(self, path, m, n, rows, cols, vals):
        rows, cols, vals = _coo_args(rows, cols, vals)
        rc = self.lib.ref_cache_write(path.encode(), m, n, len(vals), _p(rows, C.c_uint32),
                                      _p(cols, C.c_uint32), _p(vals, C.c_double))
        if rc:
            self._err(rc, "ref_cache_write")

    def _err(self, rc, what):
        raise CheckerError(rc, f"{what}: {self.lib.ref_last_error().decode()}")

    def build(self, alg: int, m: int, n: int, rows, cols, vals, threads: int = 1,
              l2_bytes: int = 512 * 1024, build_threads: int = 1, export: bool = True) -> Built:
        rows, cols, vals = _coo_args(rows, cols, vals)
        h = C.c_void_p()
        rc = self.lib.ref_build(alg, m, n, len(vals), _p(rows, C.c_uint32), _p(cols, C.c_uint32),
                                _p(vals, C.c_double), threads, l2_bytes, build_threads, C.byref(h))
        if rc:
            self._err(rc, "ref_build")
        built = Built({"alg": alg, "m": m, "n": n, "nnz": len(vals)}, handle=_RefHandle(self.lib, h))
        if export:
            fp = C.POINTER(OrcFormat)()
            self.lib.ref_export(h, C.byref(fp))
            try:
                built.meta, built.arrays, built.storage = _export(fp)
            finally:
                self.lib.ref_free_export(fp)
        return built

    def build_beta(self, alg: int, m: int, n: int, rows, cols, vals, log2_beta: int, threads: int = 1) -> Built:
        rows, cols, vals = _coo_args(rows, cols, vals)
        h = C.c_void_p()
        rc = self.lib.ref_build_beta(alg, m, n, len(vals), _p(rows, C.c_uint32), _p(cols, C.c_uint32),
                                     _p(vals, C.c_double), log2_beta, threads, C.byref(h))
        if rc:
            self._err(rc, "ref_build_beta")
        built = Built({"alg": alg, "m": m, "n": n, "nnz": len(vals)}, handle=_RefHandle(self.lib, h))
        fp = C.POINTER(OrcFormat)()
        self.lib.ref_export(h, C.byref(fp))
        try:
            built.meta, built.arrays, built.storage = _export(fp)
        finally:
            self.lib.ref_free_export(fp)
        return built

    def spmv(self, built: Built, alg: int, x, p: int = 1, split_threshold: int = 0):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(built.meta["m"], dtype=np.float64)
        rc = self.lib.ref_run(built.handle.h, alg, _p(x, C.c_double), len(x), _p(y, C.c_double), len(y),
                              p, split_threshold)
        if rc:
            self._err(rc, "ref_run")
        return y

    def time_spmv(self, built: Built, alg: int, x, p: int, reps: int, warmup: int):
        x = np.ascontiguousarray(x, dtype=np.float64)
        mn, tot = C.c_double(), C.c_double()
        rc = self.lib.ref_time_spmv(built.handle.h, alg, _p(x, C.c_double), len(x), built.meta["m"], p,
                                    reps, warmup, C.byref(mn), C.byref(tot))
        if rc:
            self._err(rc, "ref_time_spmv")
        return mn.value, tot.value

    def storage_total(self, built: Built) -> int:
        return int(self.lib.ref_storage_total(built.handle.h))

    def bench(self, kind: int, m: int, n: int, rows, cols, vals, algs, threads, spmv_reps: int = 550,
              convert_reps: int = 25, warmup: int = 5) -> list:
        """The reference's bench_spmv (kind 0) / bench_convert (kind 1), inc/bench.hpp:239-329, run
        unmodified on this host: one dict per (algorithm, threads)."""
        rows, cols, vals = _coo_args(rows, cols, vals)
        a = (C.c_int * len(algs))(*algs)
        t = (C.c_uint * len(threads))(*threads)
        cap = len(algs) * len(threads)
        out = (RefBenchRecord * cap)()
        k = self.lib.ref_bench(kind, m, n, len(vals), _p(rows, C.c_uint32), _p(cols, C.c_uint32),
                               _p(vals, C.c_double), a, len(algs), t, len(threads), spmv_reps, convert_reps,
                               warmup, out, cap)
        if k < 0:
            raise CheckerError(int(-k), f"ref_bench: {self.lib.ref_last_error().decode()}")
        recs = []
        for r in out[:k]:
            recs.append({"alg": r.alg, "threads": r.threads, "min_time_s": r.min_time, "speedup": r.speedup,
                         "convert_time_s": None if r.convert_time < 0 else r.convert_time,
                         "convert_ratio": None if r.convert_ratio < 0 else r.convert_ratio,
                         "density": r.density, "status": r.status.decode()})
        return recs

    def to_triplet(self, built: Built):
        """crs_/csb_/mergeb_/bcoh_to_triplet: (rows, cols, vals) in the reference's order."""
        nnz = built.meta["nnz"]
        r, c, v = np.zeros(nnz, np.uint32), np.zeros(nnz, np.uint32), np.zeros(nnz)
        rc = self.lib.ref_to_triplet(built.handle.h, _p(r, C.c_uint32), _p(c, C.c_uint32), _p(v, C.c_double))
        if rc:
            self._err(rc, "ref_to_triplet")
        return r, c, v

    def csb_leaves(self, built: Built, threshold: int) -> np.ndarray:
        """detail::split_block_range's leaves of every cell above `threshold`: rows (cell, lo, hi)."""
        cap = max(16, built.meta["nnz"] + 1)
        out = np.zeros(3 * cap, dtype=np.uint64)
        k = self.lib.ref_csb_leaves(built.handle.h, threshold, _p(out, C.c_uint64), cap)
        if k < 0:
            raise CheckerError(2, f"ref_csb_leaves: {k}")
        return out[: 3 * k].reshape(k, 3)

    def select_block_size(self, n, cap, l2=512 * 1024):
        return int(self.lib.ref_select_block_size(n, cap, l2))

    def morton(self, r, c, level):
        return int(self.lib.ref_morton(r, c, level))

    def hilbert(self, r, c, level):
        return int(self.lib.ref_hilbert(r, c, level))

    def diagonal_search(self, a, b, diag):
        a = np.ascontiguousarray(a, dtype=np.uint32)
        b = np.ascontiguousarray(b, dtype=np.uint32)
        i, j = C.c_uint64(), C.c_uint64()
        self.lib.ref_diagonal_search(_p(a, C.c_uint32), len(a), _p(b, C.c_uint32), len(b), diag,
                                     C.byref(i), C.byref(j))
        return i.value, j.value

    def partition_rows_by_nnz(self, prefix, p, log2_beta):
        prefix = np.ascontiguousarray(prefix, dtype=np.uint32)
        out = np.zeros(p + 1, dtype=np.uint32)
        rc = self.lib.ref_partition_rows_by_nnz(_p(prefix, C.c_uint32), len(prefix) - 1, p, log2_beta,
                                                _p(out, C.c_uint32))
        if rc:
            self._err(rc, "partition")
        return out

    def verification_input(self, n, seed=1):
        x = np.zeros(n, dtype=np.float64)
        self.lib.ref_verification_input(n, seed, _p(x, C.c_double))
        return x

    def hardware_threads(self):
        return int(self.lib.ref_hardware_threads())


class _RefHandle:
    def __init__(self, lib, h):
        self.lib, self.h = lib, h

    def __del__(self):
        try:
            self.lib.ref_free(self.h)
        except Exception:
            pass


def reference_available() -> bool:
    return os.path.exists(REF_SO)
