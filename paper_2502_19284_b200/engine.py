"""Python mirror of the reference's algorithm interface (inc/engine.hpp) over the CUDA C ABI.

Same names, argument meaning and error behaviour as the reference:

  * ``Algorithm`` / ``all_algorithms`` / ``algorithm_name`` / ``algorithm_from_name``
    (inc/engine.hpp:30-72)
  * ``EngineOptions`` (inc/engine.hpp:75-79)
  * ``build_format(alg, a, threads, opt)`` (inc/engine.hpp:96-122) -> ``BuiltFormat``
  * ``run_spmv(alg, format, x, y, p, opt)`` (inc/engine.hpp:126-156); y fully overwritten
  * ``storage_report(format)`` (inc/engine.hpp:158-160, inc/storage.hpp:38-123)
  * ``validate(a)`` (inc/triplet.hpp:42-59)
  * ``Error`` carrying an ``ErrorKind`` (inc/types.hpp:47-104)

Matrices and vectors live in device memory as torch tensors (torch is only the allocator and
stream provider here); every computation runs in libspmvlab_cuda.so.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np
import torch

from . import capi


class Algorithm(enum.IntEnum):
    SeqCrs = 0
    ParCrs = 1
    Merge = 2
    Csb = 3
    Csbh = 4
    Bcoh = 5
    Bcohc = 6
    Bcohch = 7
    Bcohchp = 8
    MergeB = 9
    MergeBH = 10


all_algorithms = tuple(Algorithm)
_NAMES = ["crs", "parcrs", "merge", "csb", "csbh", "bcoh", "bcohc", "bcohch", "bcohchp", "mergeb",
          "mergebh"]


def algorithm_name(alg) -> str:
    return _NAMES[int(alg)]


def algorithm_from_name(name: str) -> Algorithm:
    if name in _NAMES:
        return Algorithm(_NAMES.index(name))
    raise Error(ErrorKind.InvalidArgument, f"unknown algorithm '{name}'")


class ErrorKind(enum.IntEnum):
    DimensionMismatch = 0
    InvalidArgument = 1
    CorruptFormat = 2
    Overflow = 3
    BadHeader = 4
    UnsupportedFormat = 5
    UnsupportedField = 6
    UnsupportedSymmetry = 7
    IndexOutOfRange = 8
    DuplicateEntry = 9
    ParseError = 10
    Truncated = 11
    BadMagic = 12
    IoError = 13


class Error(RuntimeError):
    """spmvlab::Error (inc/types.hpp:86-96)."""

    def __init__(self, kind: ErrorKind, message: str):
        super().__init__(f"{kind.name}: {message}")
        self.kind = kind


class CudaError(RuntimeError):
    pass


def _check(rc: int):
    if rc == 0:
        return
    msg = capi.load().spmvlab_cuda_last_error().decode(errors="replace")
    if rc < 100:
        raise Error(ErrorKind(rc - 1), msg)
    raise CudaError(f"CUDA failure {rc}: {msg}")


DEFAULT_L2_BYTES = 512 * 1024  # inc/block_size.hpp:39


@dataclass
class EngineOptions:
    l2_bytes: int = DEFAULT_L2_BYTES
    split_threshold: int = 0
    build_threads: int = 1
    # build option for the blocked formats: bitwise-reproducible y (exclusive block-row owners,
    # fixed add order) instead of the faster atomics; the CRS engines always are deterministic
    deterministic: bool = False

    def _c(self) -> capi.Options:
        return capi.Options(self.l2_bytes, self.split_threshold, self.build_threads, int(self.deterministic))


@dataclass
class TripletMatrix:
    """Device-resident COO (inc/triplet.hpp:30-38): int32-typed u32 indices, float64 data."""
    m: int
    n: int
    row_ind: torch.Tensor
    col_ind: torch.Tensor
    data: torch.Tensor

    def nnz(self) -> int:
        return int(self.data.numel())

    @staticmethod
    def from_host(m, n, rows, cols, vals, device="cuda") -> "TripletMatrix":
        r = torch.from_numpy(np.ascontiguousarray(rows, dtype=np.uint32).view(np.int32)).to(device)
        c = torch.from_numpy(np.ascontiguousarray(cols, dtype=np.uint32).view(np.int32)).to(device)
        v = torch.from_numpy(np.ascontiguousarray(vals, dtype=np.float64)).to(device)
        return TripletMatrix(int(m), int(n), r, c, v)

    def _c(self) -> capi.Coo:
        for t in (self.row_ind, self.col_ind, self.data):
            if self.nnz() and (not t.is_cuda or not t.is_contiguous()):
                raise Error(ErrorKind.InvalidArgument, "triplet arrays must be contiguous CUDA tensors")
        if not (self.row_ind.numel() == self.col_ind.numel() == self.data.numel()):
            raise Error(ErrorKind.InvalidArgument, "triplet arrays must have equal length")
        if self.data.dtype != torch.float64:
            raise Error(ErrorKind.InvalidArgument, "triplet data must be float64")
        return capi.Coo(self.m, self.n, self.nnz(), self.row_ind.data_ptr(), self.col_ind.data_ptr(),
                        self.data.data_ptr())


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


@dataclass
class StorageArray:
    name: str
    bytes: int


@dataclass
class StorageBreakdown:
    """inc/storage.hpp:38-55."""
    format: str
    arrays: list = field(default_factory=list)

    def bytes(self, name: str) -> int:
        return sum(a.bytes for a in self.arrays if a.name == name)

    def total(self) -> int:
        return sum(a.bytes for a in self.arrays)

    def index_bytes(self) -> int:
        return self.total() - self.bytes("data")


_DT = {"data": np.float64, "row_jump_block": np.int16, "col_jump_block": np.int16,
       "col_inc": np.uint16, "row_jump": np.uint16, "merge_carry_val": np.float64,
       "merge_panel_data": np.float64}
_U64 = {"off_elem", "off_block", "off_row_jump_block", "off_blk_ptr", "off_row_jump"}


class BuiltFormat:
    """A device-resident format (the BuiltFormat variant, inc/engine.hpp:82)."""

    def __init__(self, handle: int, alg: Algorithm):
        self._h = C.c_void_p(handle)
        self.alg = Algorithm(alg)
        info = capi.FormatInfo()
        _check(capi.load().spmvlab_cuda_get_format_info(self._h, C.byref(info)))
        self.info = {k: getattr(info, k) for k, _ in capi.FormatInfo._fields_}
        self.m, self.n, self.nnz_ = info.m, info.n, info.nnz

    def nnz(self) -> int:
        return int(self.nnz_)

    @property
    def handle(self):
        return self._h

    def array(self, name: str) -> np.ndarray:
        """Synchronous host copy of one named array (parity downloads)."""
        L = capi.load()
        nbytes = C.c_uint64()
        _check(L.spmvlab_cuda_download_array(self._h, name.encode(), None, 0, C.byref(nbytes)))
        dt = np.uint64 if name in _U64 else _DT.get(name, np.uint32)
        out = np.zeros(nbytes.value // np.dtype(dt).itemsize, dtype=dt)
        if out.size:
            _check(L.spmvlab_cuda_download_array(self._h, name.encode(), out.ctypes.data, out.nbytes,
                                                 C.byref(nbytes)))
        return out

    def array_device(self, name: str) -> torch.Tensor:
        """Device copy of one named array as a torch tensor (full-size parity checks without a host
        round trip): float64 for values, int64 for every integer array (unsigned values kept)."""
        L = capi.load()
        ptr, nbytes = C.c_void_p(), C.c_uint64()
        _check(L.spmvlab_cuda_format_array(self._h, name.encode(), C.byref(ptr), C.byref(nbytes)))
        dt = np.dtype(np.uint64 if name in _U64 else _DT.get(name, np.uint32))
        count = nbytes.value // dt.itemsize
        dev = torch.device("cuda", torch.cuda.current_device())
        torch.cuda.synchronize()
        if dt == np.float64:
            return _view_copy(ptr.value, count, "<f8", torch.float64, dev)
        signed = {1: ("<i1", torch.int8), 2: ("<i2", torch.int16), 4: ("<i4", torch.int32),
                  8: ("<i8", torch.int64)}[dt.itemsize]
        t = _view_copy(ptr.value, count, signed[0], signed[1], dev).to(torch.int64)
        if dt.kind == "u" and dt.itemsize < 8:
            t &= (1 << (8 * dt.itemsize)) - 1
        return t

    def close(self):
        if self._h:
            try:
                capi.load().spmvlab_cuda_free_format(self._h)
            except Exception:
                pass
            self._h = C.c_void_p(0)

    def __del__(self):
        self.close()


def build_format(alg, a: TripletMatrix, threads: int = 1, opt: EngineOptions | None = None,
                 stream=None) -> BuiltFormat:
    """inc/engine.hpp:96-122 (COO -> format on the device)."""
    opt = opt or EngineOptions()
    h = C.c_void_p()
    coo = a._c()
    _check(capi.load().spmvlab_cuda_build_format(int(alg), C.byref(coo), int(threads), C.byref(opt._c()),
                                                 C.byref(h), _stream(stream)))
    return BuiltFormat(h.value, alg)


def row_prefix(a: TripletMatrix, stream=None) -> torch.Tensor:
    """row_counts + row_prefix (inc/triplet.hpp:75-87) on the device: m + 1 exclusive prefix sums
    (int32-typed u32)."""
    out = torch.empty(a.m + 1, dtype=torch.int32, device="cuda")
    coo = a._c()
    _check(capi.load().spmvlab_cuda_row_prefix(C.byref(coo), out.data_ptr(), _stream(stream)))
    return out


def build_format_beta(alg, a: TripletMatrix, log2_beta: int, threads: int = 1, stream=None) -> BuiltFormat:
    """The per-format builders with an explicit block size 2^log2_beta: build_csb (inc/csb.hpp:51),
    build_mergeb (inc/mergeb.hpp:50), build_bcoh with p = threads bands (inc/bcoh.hpp:194)."""
    h = C.c_void_p()
    coo = a._c()
    _check(capi.load().spmvlab_cuda_build_format_beta(int(alg), C.byref(coo), int(log2_beta), int(threads),
                                                      C.byref(h), _stream(stream)))
    return BuiltFormat(h.value, alg)


def run_spmv(alg, fmt: BuiltFormat, x: torch.Tensor, y: torch.Tensor | None = None, p: int = 1,
             opt: EngineOptions | None = None, stream=None) -> torch.Tensor:
    """inc/engine.hpp:126-156: y = A x on the device (stream-ordered; y fully overwritten)."""
    if y is None:
        y = torch.empty(fmt.m, dtype=torch.float64, device=x.device)
    if x.dtype != torch.float64 or y.dtype != torch.float64:
        raise Error(ErrorKind.InvalidArgument, "x and y must be float64")
    c_opt = (opt or EngineOptions())._c()
    _check(capi.load().spmvlab_cuda_run_spmv(int(alg), fmt.handle, x.data_ptr(), x.numel(), y.data_ptr(),
                                             y.numel(), int(p), C.byref(c_opt), _stream(stream)))
    return y


def run_spmv_host(alg, fmt: BuiltFormat, x_host: torch.Tensor, y_host: torch.Tensor, p: int,
                  x_dev: torch.Tensor, y_dev: torch.Tensor, opt: EngineOptions | None = None,
                  stream=None) -> torch.Tensor:
    """Host-buffer multiply through the C ABI: H2D x, multiply, D2H y on one stream."""
    c_opt = (opt or EngineOptions())._c()
    _check(capi.load().spmvlab_cuda_run_spmv_host(int(alg), fmt.handle, x_host.data_ptr(), x_host.numel(),
                                                  y_host.data_ptr(), y_host.numel(), int(p), C.byref(c_opt),
                                                  x_dev.data_ptr(), y_dev.data_ptr(), _stream(stream)))
    return y_host


ITER_NORMALIZE = 1
ITER_GRAPH = 2


def iterate(alg, fmt: BuiltFormat, x: torch.Tensor, iters: int, p: int = 1, normalize: bool = False,
            graph: bool = False, norms: bool = True, work: torch.Tensor | None = None, stream=None):
    """x <- A x, `iters` times, in place on the device (the cfg5 application loop around
    inc/engine.hpp:126-148).  Returns (x, norms) with norms a (iters, 2) device tensor of
    (||A x_k - x_k||_1, mass of A x_k) per iteration, or None (one pass per iteration after the
    multiply; the rescale is a deferred scalar).  graph=True runs the loop as one
    CUDA graph on `stream` (a torch.cuda.Stream; the current stream if None)."""
    if x.dtype != torch.float64:
        raise Error(ErrorKind.InvalidArgument, "x must be float64")
    if work is None:
        work = torch.empty_like(x)
    nb = torch.empty((iters, 2), dtype=torch.float64, device=x.device) if norms else None
    flags = (ITER_NORMALIZE if normalize else 0) | (ITER_GRAPH if graph else 0)
    cur = torch.cuda.current_stream(x.device)
    st = stream if stream is not None else cur
    side = None
    if graph and _stream(st) == 0:  # graphs cannot be captured on the legacy default stream
        side = torch.cuda.Stream(x.device)
        side.wait_stream(st)
        st = side
    _check(capi.load().spmvlab_cuda_iterate(int(alg), fmt.handle, x.data_ptr(), work.data_ptr(), int(iters), int(p),
                                            flags, nb.data_ptr() if nb is not None else None, _stream(st)))
    if side is not None:
        cur.wait_stream(side)
    return x, nb


_FORMAT_NAMES = {0: "crs", 1: "crs", 2: "crs", 3: "csb", 4: "csbh", 5: "bcoh", 6: "bcohc", 7: "bcohch",
                 8: "bcohchp", 9: "mergeb", 10: "mergebh"}


def storage_report(fmt: BuiltFormat) -> StorageBreakdown:
    """inc/engine.hpp:158-160."""
    L = capi.load()
    rows = (capi.StorageArray * 16)()
    cnt = C.c_size_t()
    _check(L.spmvlab_cuda_storage_report(fmt.handle, rows, 16, C.byref(cnt)))
    return StorageBreakdown(_FORMAT_NAMES[int(fmt.alg)],
                            [StorageArray(rows[i].name.decode(), int(rows[i].bytes)) for i in range(cnt.value)])


def validate(a: TripletMatrix, stream=None) -> None:
    """inc/triplet.hpp:42-59."""
    coo = a._c()
    _check(capi.load().spmvlab_cuda_validate(C.byref(coo), _stream(stream)))


def cache_read(path: str, stream=None) -> TripletMatrix:
    """SPMVLAB1 triplet cache -> device triplet (inc/cache_io.hpp:69-91, validated)."""
    L = capi.load()
    m, n, nnz = C.c_uint32(), C.c_uint32(), C.c_uint64()
    _check(L.spmvlab_cuda_cache_info(str(path).encode(), C.byref(m), C.byref(n), C.byref(nnz)))
    dev = torch.device("cuda", torch.cuda.current_device())
    k = int(nnz.value)
    rows = torch.empty(max(k, 1), dtype=torch.int32, device=dev)
    cols = torch.empty(max(k, 1), dtype=torch.int32, device=dev)
    vals = torch.empty(max(k, 1), dtype=torch.float64, device=dev)
    coo = capi.Coo(m.value, n.value, k, rows.data_ptr(), cols.data_ptr(), vals.data_ptr())
    _check(L.spmvlab_cuda_cache_read(str(path).encode(), C.byref(coo), _stream(stream)))
    return TripletMatrix(int(coo.m), int(coo.n), rows[:k], cols[:k], vals[:k])


@dataclass
class MatrixHeader:
    """MatrixHeader (inc/matrix_market.hpp:35-41)."""
    field: str      # "real" | "integer" | "pattern"
    symmetry: str   # "general" | "symmetric"
    m: int
    n: int
    declared_nnz: int


def _mm_header(h) -> MatrixHeader:
    return MatrixHeader(("real", "integer", "pattern")[h.field], ("general", "symmetric")[h.symmetry], int(h.m),
                        int(h.n), int(h.declared_nnz))


def _device_coo_to_triplet(coo) -> TripletMatrix:
    """Copies a library-allocated device triplet into torch tensors and releases it."""
    L = capi.load()
    k = int(coo.nnz)
    dev = torch.device("cuda", torch.cuda.current_device())
    rows = torch.empty(k, dtype=torch.int32, device=dev)
    cols = torch.empty(k, dtype=torch.int32, device=dev)
    vals = torch.empty(k, dtype=torch.float64, device=dev)
    class _View:  # __cuda_array_interface__ view of library memory, copied before it is released
        def __init__(self, ptr, typestr):
            self.__cuda_array_interface__ = {"shape": (k,), "typestr": typestr, "data": (ptr, False), "version": 3,
                                             "strides": None}

    try:
        if k:
            rows.copy_(torch.as_tensor(_View(coo.row_ind, "<i4"), device=dev))
            cols.copy_(torch.as_tensor(_View(coo.col_ind, "<i4"), device=dev))
            vals.copy_(torch.as_tensor(_View(coo.data, "<f8"), device=dev))
            torch.cuda.synchronize()
    finally:
        L.spmvlab_cuda_free_coo(C.byref(coo))
    return TripletMatrix(int(coo.m), int(coo.n), rows, cols, vals)


def read_matrix_market(path: str, stream=None, with_header: bool = False):
    """read_matrix_market (inc/matrix_market.hpp:94-190) into a device triplet (validated on the
    device).  Returns the TripletMatrix, or (TripletMatrix, MatrixHeader) with with_header."""
    L = capi.load()
    coo = capi.Coo(0, 0, 0, None, None, None)
    h = capi.MmHeader()
    _check(L.spmvlab_cuda_read_matrix_market(str(path).encode(), C.byref(coo), C.byref(h), _stream(stream)))
    torch.cuda.synchronize()
    m, n = int(coo.m), int(coo.n)
    a = _device_coo_to_triplet(coo)
    a.m, a.n = m, n
    return (a, _mm_header(h)) if with_header else a


def read_matrix_market_host(path: str):
    """The same parse + validate on the host: (m, n, rows u32, cols u32, vals f64, MatrixHeader)."""
    L = capi.load()
    out = capi.HostCoo()
    h = capi.MmHeader()
    _check(L.spmvlab_cuda_read_matrix_market_host(str(path).encode(), C.byref(out), C.byref(h)))
    try:
        k = int(out.nnz)
        rows = np.ctypeslib.as_array(out.row_ind, shape=(k,)).copy() if k else np.zeros(0, np.uint32)
        cols = np.ctypeslib.as_array(out.col_ind, shape=(k,)).copy() if k else np.zeros(0, np.uint32)
        vals = np.ctypeslib.as_array(out.data, shape=(k,)).copy() if k else np.zeros(0, np.float64)
        return int(out.m), int(out.n), rows, cols, vals, _mm_header(h)
    finally:
        L.spmvlab_cuda_free_host_coo(C.byref(out))


def load_matrix(path: str, stream=None) -> TripletMatrix:
    """load_matrix (inc/io.hpp:29-40): SPMVLAB1 cache or Matrix Market text, sniffed by magic."""
    L = capi.load()
    coo = capi.Coo(0, 0, 0, None, None, None)
    _check(L.spmvlab_cuda_load_matrix(str(path).encode(), C.byref(coo), _stream(stream)))
    torch.cuda.synchronize()
    m, n = int(coo.m), int(coo.n)
    a = _device_coo_to_triplet(coo)
    a.m, a.n = m, n
    return a


def _view_copy(ptr, count: int, typestr: str, dtype, dev) -> torch.Tensor:
    """Copy of `count` elements of library device memory into a torch tensor."""
    out = torch.empty(count, dtype=dtype, device=dev)
    if count:
        class _V:
            def __init__(self):
                self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr, "data": (ptr, False),
                                                 "version": 3, "strides": None}
        out.copy_(torch.as_tensor(_V(), device=dev))
    return out


class IncrementalRowStorage:
    """IncrementalRowStorage (inc/bicrs.hpp:33-45) on the device: ICRS (kind 0, u32 increments)
    or BICRS (kind 1, i64 increments).  Owns the library arrays."""

    def __init__(self, c: "capi.Bicrs", keep=None):
        self._c = c
        self._keep = keep  # torch tensors backing the arrays (then the library does not own them)

    kind = property(lambda self: int(self._c.kind))
    m = property(lambda self: int(self._c.m))
    n = property(lambda self: int(self._c.n))

    def nnz(self) -> int:
        return int(self._c.nnz)

    def arrays(self) -> dict:
        """Host copies: col_inc (nnz + 1), row_jump, data (numpy)."""
        dev = torch.device("cuda", torch.cuda.current_device())
        ts, dt = ("<u4", torch.int32) if self.kind == 0 else ("<i8", torch.int64)
        ci = _view_copy(self._c.col_inc, self.nnz() + 1, ts, dt, dev).cpu().numpy()
        rj = _view_copy(self._c.row_jump, int(self._c.n_row_jump), ts, dt, dev).cpu().numpy()
        if self.kind == 0:
            ci, rj = ci.view(np.uint32), rj.view(np.uint32)
        data = _view_copy(self._c.data, self.nnz(), "<f8", torch.float64, dev).cpu().numpy()
        return {"col_inc": ci, "row_jump": rj, "data": data}

    def spmv(self, x: torch.Tensor, y: torch.Tensor | None = None, stream=None):
        """spmv_bicrs_seq (inc/bicrs.hpp:98-109) -> (y, (overflow_events, row_jumps_consumed))."""
        if y is None:
            y = torch.empty(self.m, dtype=torch.float64, device=x.device)
        stats = (C.c_uint64 * 2)()
        _check(capi.load().spmvlab_cuda_bicrs_spmv(C.byref(self._c), x.data_ptr(), x.numel(), y.data_ptr(),
                                                   y.numel(), stats, _stream(stream)))
        return y, (int(stats[0]), int(stats[1]))

    def to_triplet(self, stream=None):
        """bicrs_to_triplet (inc/bicrs.hpp:111-118) -> device (rows, cols) in element order."""
        dev = torch.device("cuda", torch.cuda.current_device())
        k = self.nnz()
        rows = torch.empty(max(k, 1), dtype=torch.int32, device=dev)
        cols = torch.empty(max(k, 1), dtype=torch.int32, device=dev)
        _check(capi.load().spmvlab_cuda_bicrs_to_triplet(C.byref(self._c), rows.data_ptr(), cols.data_ptr(),
                                                         _stream(stream)))
        return rows[:k], cols[:k]

    def close(self):
        if self._c is not None and self._keep is None:
            capi.load().spmvlab_cuda_free_bicrs(C.byref(self._c))
        self._c = None
        self._keep = None

    __del__ = close


def crs_to_icrs(fmt: BuiltFormat, stream=None) -> IncrementalRowStorage:
    """crs_to_icrs (inc/bicrs.hpp:120-150) from a CRS-family format."""
    c = capi.Bicrs()
    _check(capi.load().spmvlab_cuda_crs_to_icrs(fmt.handle, C.byref(c), _stream(stream)))
    return IncrementalRowStorage(c)


def format_to_triplet(fmt: BuiltFormat, stream=None) -> TripletMatrix:
    """crs_/csb_/mergeb_/bcoh_to_triplet (crs.hpp:94-105, csb.hpp:103-120, mergeb.hpp:110-127,
    bcoh.hpp:379-392): the elements of any built format in the reference's output order (storage
    order, BCOH band by band), decoded on the device."""
    nnz = fmt.nnz()
    r = torch.empty(nnz, dtype=torch.int32, device="cuda")
    c = torch.empty(nnz, dtype=torch.int32, device="cuda")
    v = torch.empty(nnz, dtype=torch.float64, device="cuda")
    ptr = (lambda t: t.data_ptr() if nnz else None)
    _check(capi.load().spmvlab_cuda_format_to_triplet(fmt.handle, ptr(r), ptr(c), ptr(v), _stream(stream)))
    return TripletMatrix(fmt.m, fmt.n, r, c, v)


def _family_to_triplet(algs, what):
    def fn(fmt: BuiltFormat, stream=None) -> TripletMatrix:
        if int(fmt.alg) not in algs:
            raise Error(ErrorKind.InvalidArgument, f"{what} needs a {what.split('_')[0].upper()} format")
        return format_to_triplet(fmt, stream)
    fn.__name__ = what
    fn.__doc__ = f"{what}: format_to_triplet restricted to its format family."
    return fn


crs_to_triplet = _family_to_triplet((0, 1, 2), "crs_to_triplet")
csb_to_triplet = _family_to_triplet((3, 4), "csb_to_triplet")
bcoh_to_triplet = _family_to_triplet((5, 6, 7, 8), "bcoh_to_triplet")
mergeb_to_triplet = _family_to_triplet((9, 10), "mergeb_to_triplet")


CSB_ITEM_DTYPE = np.dtype([("block_row", np.uint32), ("cell_begin", np.uint32), ("cell_end", np.uint32),
                           ("temp_slot", np.int32), ("elem_begin", np.uint64), ("elem_end", np.uint64)])


def csb_work_items(fmt: BuiltFormat, split_threshold: int = 0, stream=None) -> torch.Tensor:
    """spmv_csb's work-item list (inc/spmv_parallel.hpp:202-264: CsbWorkItem per block row, cell
    chunk or quadrant leaf of split_block_range :178-193), built on the device from a CSB / CSBH
    format; split_threshold 0 = 2 * beta.  Returns a device uint8 tensor of shape (count, 32) in
    the spmvlab_cuda_csb_item layout; csb_items_numpy() views a host copy as CSB_ITEM_DTYPE."""
    L = capi.load()
    cnt = C.c_uint64()
    _check(L.spmvlab_cuda_csb_work_items(fmt.handle, split_threshold, None, 0, C.byref(cnt), _stream(stream)))
    out = torch.empty((cnt.value, CSB_ITEM_DTYPE.itemsize), dtype=torch.uint8, device="cuda")
    _check(L.spmvlab_cuda_csb_work_items(fmt.handle, split_threshold, out.data_ptr() if cnt.value else None,
                                         cnt.value, C.byref(cnt), _stream(stream)))
    return out


def csb_items_numpy(items: torch.Tensor) -> np.ndarray:
    return items.cpu().numpy().reshape(-1).view(CSB_ITEM_DTYPE)


def triplet_to_bicrs(a: TripletMatrix, order: torch.Tensor, stream=None) -> IncrementalRowStorage:
    """triplet_to_bicrs (inc/bicrs.hpp:154-200) with the elements in `order` (device int32)."""
    c = capi.Bicrs()
    coo = a._c()
    _check(capi.load().spmvlab_cuda_triplet_to_bicrs(C.byref(coo), order.data_ptr() if order.numel() else None,
                                                     C.byref(c), _stream(stream)))
    return IncrementalRowStorage(c)


def bicrs_from_arrays(m: int, n: int, col_inc, row_jump, data, kind: int = 1) -> IncrementalRowStorage:
    """Wraps host arrays (e.g. a stream from elsewhere) as a device ICRS / BICRS for the multiply
    and the replay checks (device copies held by torch)."""
    dt = np.uint32 if kind == 0 else np.int64
    ci = np.ascontiguousarray(col_inc, dtype=dt)
    rj = np.ascontiguousarray(row_jump, dtype=dt)
    dv = np.ascontiguousarray(data, dtype=np.float64)
    if len(ci) != len(dv) + 1:  # replay_bicrs, inc/bicrs.hpp:58-59
        raise Error(ErrorKind.CorruptFormat, "col_inc must hold nnz + 1 entries")
    to = lambda a: torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).cuda()
    tci, trj, tdv = to(ci), to(rj), to(dv)
    ptr = lambda t: t.data_ptr() if t.numel() else None
    c = capi.Bicrs(m, n, len(dv), kind, ptr(tci), ptr(trj), len(rj), ptr(tdv))
    return IncrementalRowStorage(c, keep=(tci, trj, tdv))


def cache_write(path: str, a: TripletMatrix, stream=None) -> None:
    """Device triplet -> SPMVLAB1 cache, byte-identical to the reference's cache_write."""
    coo = a._c()
    _check(capi.load().spmvlab_cuda_cache_write(str(path).encode(), C.byref(coo), _stream(stream)))


def release_cached_memory() -> None:
    """Returns cached free device memory of both allocators in the process -- the library's stream-
    ordered pool (conversion scratch kept between builds) and torch's caching allocator -- to the
    driver, before a phase that needs tens of GB from the other one."""
    if torch.cuda.is_available():
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
    _check(capi.load().spmvlab_cuda_release_pool())


def select_block_size(n: int, index_bits_cap: int, l2_bytes: int = DEFAULT_L2_BYTES) -> int:
    """inc/block_size.hpp:47-61 -> log2(beta)."""
    return int(capi.load().spmvlab_cuda_select_block_size(n, index_bits_cap, l2_bytes))


def engine_block_size(alg, n: int, opt: EngineOptions | None = None) -> int:
    """inc/engine.hpp:84-91 -> log2(beta)."""
    opt = opt or EngineOptions()
    cap = 15 if Algorithm(alg) in (Algorithm.Bcoh, Algorithm.Bcohc, Algorithm.Bcohch, Algorithm.Bcohchp) else 16
    return select_block_size(max(n, 1), cap, opt.l2_bytes)


def partition_rows_by_nnz(prefix, p: int, log2_beta: int) -> np.ndarray:
    """inc/block_size.hpp:73-102 (host)."""
    prefix = np.ascontiguousarray(prefix, dtype=np.uint32)
    out = np.zeros(p + 1, dtype=np.uint32)
    _check(capi.load().spmvlab_cuda_partition_rows_by_nnz(prefix.ctypes.data, len(prefix) - 1, p, log2_beta,
                                                          out.ctypes.data))
    return out


def merge_path_search(a: torch.Tensor, b, diags: torch.Tensor, stream=None) -> torch.Tensor:
    """diagonal_search (inc/spmv_parallel.hpp:47-69) for many diagonals.  ``b`` is either a device
    tensor (list B) or an int b_len meaning B[j] = j (the CRS merge path)."""
    out = torch.empty(diags.numel(), dtype=torch.int64, device=a.device)
    if isinstance(b, int):
        bp, blen = None, b
    else:
        bp, blen = b.data_ptr(), b.numel()
    _check(capi.load().spmvlab_cuda_merge_path_search(a.data_ptr(), a.numel(), bp, blen, diags.data_ptr(),
                                                      diags.numel(), out.data_ptr(), _stream(stream)))
    return out


def curve_keys(kind: int, rows: torch.Tensor, cols: torch.Tensor, level: int, stream=None) -> torch.Tensor:
    """Morton (kind 0) / Hilbert (kind 1) ranks on the device (inc/curves.hpp:107-143)."""
    out = torch.empty(rows.numel(), dtype=torch.int64, device=rows.device)
    _check(capi.load().spmvlab_cuda_curve_keys(kind, rows.data_ptr(), cols.data_ptr(), rows.numel(), level,
                                               out.data_ptr(), _stream(stream)))
    return out


def sort_pairs(keys: torch.Tensor, values: torch.Tensor, begin_bit: int, end_bit: int, stream=None):
    """In-place stable LSD radix sort of (u64 key, u32 value) pairs."""
    _check(capi.load().spmvlab_cuda_sort_pairs(keys.data_ptr(), values.data_ptr(), keys.numel(), begin_bit,
                                               end_bit, _stream(stream)))
    return keys, values


def exclusive_scan(counts: torch.Tensor, stream=None) -> torch.Tensor:
    out = torch.empty(counts.numel() + 1, dtype=torch.int32, device=counts.device)
    _check(capi.load().spmvlab_cuda_exclusive_scan(counts.data_ptr(), out.data_ptr(), counts.numel(),
                                                   _stream(stream)))
    return out
