"""GPU benchmark harness and reports: the reference's BenchRecord / bench_spmv / bench_convert /
emit_csv / parse_csv / emit_markdown (inc/bench.hpp:59-71, 239-329, 367-554) for the device
engines, extended as SURVEY.md §8f item 3 asks with effective GB/s, the fraction of the measured
HBM roofline and the break-even multiply count of each conversion.

The plain CSV and markdown are byte-identical to the reference's emitters for the same records
(tests/test_report_cpu.py pins them against the reference's own output); the extended CSV appends
the GPU columns after the reference's nine.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from decimal import Decimal
from typing import Iterable, Optional

import torch

from . import engine as E

CSV_HEADER = "matrix,algorithm,threads,min_time_s,speedup,convert_time_s,convert_ratio,density,status"
CSV_EXT_HEADER = CSV_HEADER + ",gbs,roofline_frac,break_even"
DENSITY_CLASS_THRESHOLD = 1e-6  # inc/bench.hpp:54


@dataclass
class BenchRecord:
    """inc/bench.hpp:58-70, plus the GPU columns (None when not measured)."""
    matrix: str
    algorithm: int
    threads: int = 1
    min_time: float = 0.0
    speedup: float = 0.0
    convert_time: Optional[float] = None
    convert_ratio: Optional[float] = None
    density: float = 0.0
    status: str = "ok"
    gbs: Optional[float] = None            # algorithmic bytes / min_time
    roofline_frac: Optional[float] = None  # gbs / measured HBM peak
    break_even: Optional[float] = None     # convert_time / (t_merge - min_time), when faster than merge


# ------------------------------------------------------------------------------ formatting
def format_double(v: float) -> str:
    """std::to_chars(double) shortest round-trip form (detail::format_double, inc/bench.hpp:334-339):
    the shortest digit string that round-trips, printed in fixed or scientific notation,
    whichever is shorter (fixed on a tie)."""
    v = float(v)
    if math.isnan(v):
        return "nan"
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    if v == 0.0:
        return "-0" if math.copysign(1.0, v) < 0 else "0"
    sign = "-" if v < 0 else ""
    d = Decimal(repr(abs(v)))
    tup = d.as_tuple()
    digits = "".join(map(str, tup.digits)).rstrip("0") or "0"
    exp10 = tup.exponent + len(tup.digits) - 1  # scientific exponent of the leading digit
    # scientific: d[.ddd]e+XX (at least two exponent digits)
    mant = digits[0] + ("." + digits[1:] if len(digits) > 1 else "")
    sci = f"{mant}e{'-' if exp10 < 0 else '+'}{abs(exp10):02d}"
    # fixed
    nd = len(digits)
    if exp10 >= nd - 1:
        fixed = digits + "0" * (exp10 - nd + 1)
    elif exp10 >= 0:
        fixed = digits[:exp10 + 1] + "." + digits[exp10 + 1:]
    else:
        fixed = "0." + "0" * (-exp10 - 1) + digits
    return sign + (fixed if len(fixed) <= len(sci) else sci)


def parse_double(token: str) -> float:
    """detail::parse_double (inc/bench.hpp:341-347): the whole token must be a number."""
    try:
        return float(token)
    except ValueError:
        raise E.Error(E.ErrorKind.ParseError, f"bad numeric field '{token}'") from None


def _sanitize(s: str) -> str:
    return s.replace(",", ";").replace("\n", ";")


def _fixed(v: float, digits: int) -> str:
    return f"{v:.{digits}f}"


# ------------------------------------------------------------------------------ CSV
def emit_csv(records: Iterable[BenchRecord], extended: bool = False) -> str:
    """emit_csv (inc/bench.hpp:367-394); extended=True appends gbs, roofline_frac, break_even."""
    out = [CSV_EXT_HEADER if extended else CSV_HEADER]
    for r in records:
        f = [_sanitize(r.matrix), E.algorithm_name(r.algorithm), str(int(r.threads)), format_double(r.min_time),
             format_double(r.speedup), format_double(r.convert_time) if r.convert_time is not None else "",
             format_double(r.convert_ratio) if r.convert_ratio is not None else "", format_double(r.density),
             _sanitize(r.status)]
        if extended:
            f += [format_double(x) if x is not None else "" for x in (r.gbs, r.roofline_frac, r.break_even)]
        out.append(",".join(f))
    return "\n".join(out) + "\n"


def parse_csv(text: str) -> list[BenchRecord]:
    """parse_csv (inc/bench.hpp:398-429), accepting the extended header too."""
    lines = text.split("\n")
    if not lines or not lines[0]:
        raise E.Error(E.ErrorKind.ParseError, "empty CSV")
    ext = lines[0] == CSV_EXT_HEADER
    if lines[0] != CSV_HEADER and not ext:
        raise E.Error(E.ErrorKind.ParseError, "unexpected CSV header")
    want = 12 if ext else 9
    recs = []
    for line in lines[1:]:
        if not line:
            continue
        f = line.split(",")
        if len(f) != want:
            raise E.Error(E.ErrorKind.ParseError, f"expected {want} CSV fields, got {len(f)}")
        r = BenchRecord(matrix=f[0], algorithm=int(E.algorithm_from_name(f[1])), threads=int(f[2]),
                        min_time=parse_double(f[3]), speedup=parse_double(f[4]),
                        convert_time=parse_double(f[5]) if f[5] else None,
                        convert_ratio=parse_double(f[6]) if f[6] else None, density=parse_double(f[7]),
                        status=f[8])
        if ext:
            r.gbs, r.roofline_frac, r.break_even = (parse_double(x) if x else None for x in f[9:12])
        recs.append(r)
    return recs


# ------------------------------------------------------------------------------ markdown
def emit_markdown(records: list[BenchRecord], gpu_columns: bool = False) -> str:
    """emit_markdown (inc/bench.hpp:435-546): per density class, algorithms down the rows and
    matrices across, best speedup per column in bold with its thread count, then the conversion
    grid.  gpu_columns=True adds, per class, grids of effective GB/s (with the fraction of the HBM
    roofline) and break-even multiply counts."""
    low, high, algs = [], [], []
    best: dict = {}
    ratio: dict = {}
    gbs: dict = {}
    beven: dict = {}
    for r in records:
        cols = low if r.density < DENSITY_CLASS_THRESHOLD else high
        if r.matrix not in cols:
            cols.append(r.matrix)
        if r.algorithm not in algs:
            algs.append(r.algorithm)
        if r.status == "ok" and r.min_time > 0.0:
            b = best.setdefault(r.matrix, {}).get(r.algorithm)
            if b is None or r.speedup > b[0]:
                best[r.matrix][r.algorithm] = (r.speedup, r.threads)
            if r.gbs is not None:
                g = gbs.setdefault(r.matrix, {}).get(r.algorithm)
                if g is None or r.gbs > g[0]:
                    gbs[r.matrix][r.algorithm] = (r.gbs, r.roofline_frac)
        if r.convert_ratio is not None:
            d = ratio.setdefault(r.matrix, {})
            d[r.algorithm] = min(d.get(r.algorithm, r.convert_ratio), r.convert_ratio)
        if r.break_even is not None:
            d = beven.setdefault(r.matrix, {})
            d[r.algorithm] = min(d.get(r.algorithm, r.break_even), r.break_even)
    out = ["# SpMV benchmark report\n\n",
           "Minimum-of-runs protocol; speedups relative to sequential CRS. Threads are not pinned to cores.\n"]

    def grid(title, cols, table, cell):
        out.append(f"\n{title}\n\n" if title else "")
        out.append("| Method |" + "".join(f" {m} |" for m in cols) + "\n|---|" + "---|" * len(cols) + "\n")
        for a in algs:
            out.append(f"| {E.algorithm_name(a)} |")
            for m in cols:
                col = table.get(m)
                out.append(f" {cell(col, a)} |" if col is not None and a in col else " - |")
            out.append("\n")

    def speed_cell(col, a):
        s, th = col[a]
        bold = s == max(v[0] for v in col.values())
        txt = _fixed(s, 2)
        return (f"**{txt}**" if bold else txt) + f" ({th})"

    def emit_class(title, cols):
        if not cols:
            return
        out.append(f"\n## {title}\n\n")
        if any(best.get(m) for m in cols):
            grid(None, cols, best, speed_cell)
        if any(m in ratio for m in cols):
            grid("Conversion cost (ParCRS multiplications):", cols, ratio, lambda col, a: _fixed(col[a], 1))
        if gpu_columns and any(m in gbs for m in cols):
            grid("Effective bandwidth (GB/s of algorithmic bytes; fraction of the measured HBM peak):", cols, gbs,
                 lambda col, a: f"{_fixed(col[a][0], 0)} ({_fixed(col[a][1], 2)})" if col[a][1] is not None
                 else _fixed(col[a][0], 0))
        if gpu_columns and any(m in beven for m in cols):
            grid("Break-even multiplies against merge-CSR (conversion time / time saved per multiply):", cols,
                 beven, lambda col, a: _fixed(col[a], 1))

    emit_class("Low density (< 1e-6)", low)
    emit_class("Higher density (>= 1e-6)", high)
    return "".join(out)


def emit_report(records: list[BenchRecord], fmt: str = "csv", extended: bool = False) -> str:
    """emit_report (inc/bench.hpp:548-552)."""
    if not records:
        raise E.Error(E.ErrorKind.InvalidArgument, "no records to report")
    return emit_csv(records, extended) if fmt == "csv" else emit_markdown(records, extended)


# ------------------------------------------------------------------------------ measurement
@dataclass
class BenchConfig:
    """BenchConfig (inc/bench.hpp:38-52) for the device engines."""
    algorithms: list = field(default_factory=lambda: list(E.all_algorithms))
    threads: list = field(default_factory=lambda: [8])
    spmv_reps: int = 50
    convert_reps: int = 3
    warmup: int = 3
    l2_bytes: int = 512 * 1024
    seed: int = 5
    peak_gbs: Optional[float] = None  # measured HBM peak for roofline_frac


def _min_time(fn, reps, warmup, stream):
    for _ in range(warmup):
        fn()
    best = float("inf")
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    return best


def _density(a: E.TripletMatrix) -> float:
    return a.nnz() / (float(a.m) * float(a.n)) if a.m and a.n else 0.0


def bench_all(a: E.TripletMatrix, matrix_name: str, cfg: BenchConfig | None = None) -> list[BenchRecord]:
    """bench_spmv + bench_convert (inc/bench.hpp:239-329) merged into one row per (algorithm,
    threads): min multiply time over spmv_reps (each y checked against an independent device
    scatter-add within 1e-12 * sum|a_ij x_j|), speedup over the device SeqCrs, min conversion time
    over convert_reps, ratio to the fastest ParCRS multiply, GB/s, roofline fraction and the
    break-even count against merge-CSR at the same thread count."""
    cfg = cfg or BenchConfig()
    stream = torch.cuda.current_stream()
    dev = a.row_ind.device
    g = torch.Generator(device=dev).manual_seed(cfg.seed)
    x = torch.rand(a.n, dtype=torch.float64, device=dev, generator=g) + 0.5  # strictly positive, like
    y_ref = torch.zeros(a.m, dtype=torch.float64, device=dev)             # verification_input
    rows = a.row_ind.long()
    prod = a.data * x[a.col_ind.long()]
    y_ref.index_add_(0, rows, prod)
    bound = torch.zeros(a.m, dtype=torch.float64, device=dev).index_add_(0, rows, prod.abs())
    del prod
    opt = E.EngineOptions(l2_bytes=cfg.l2_bytes)
    density = _density(a)
    crs = E.build_format(E.Algorithm.Merge, a, 1, opt)
    y = torch.empty(a.m, dtype=torch.float64, device=dev)
    t_seq = _min_time(lambda: E.run_spmv(E.Algorithm.SeqCrs, crs, x, y, 1), max(3, cfg.spmv_reps // 10), cfg.warmup,
                      stream)
    parcrs_best = min(_min_time(lambda: E.run_spmv(E.Algorithm.ParCrs, crs, x, y, p), cfg.spmv_reps, cfg.warmup,
                                stream) for p in cfg.threads)
    del crs
    recs = []
    for alg in cfg.algorithms:
        for p in cfg.threads:
            r = BenchRecord(matrix_name, int(alg), p, density=density)
            try:
                best_c = float("inf")
                f = None
                for _ in range(max(1, cfg.convert_reps)):
                    f = None
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    f = E.build_format(alg, a, p, opt)
                    e1.record(stream)
                    e1.synchronize()
                    best_c = min(best_c, e0.elapsed_time(e1) / 1e3)
                r.convert_time = best_c
                r.convert_ratio = best_c / parcrs_best
                E.run_spmv(alg, f, x, y, p)
                err = (y - y_ref).abs() - 1e-12 * bound
                if bool((err > 0).any()):
                    r.status = f"verify failed at element {int(torch.nonzero(err > 0)[0, 0])}"
                else:
                    reps = max(3, cfg.spmv_reps // 10) if alg == E.Algorithm.SeqCrs else cfg.spmv_reps
                    r.min_time = _min_time(lambda: E.run_spmv(alg, f, x, y, p), reps, cfg.warmup, stream)
                    r.speedup = t_seq / r.min_time if r.min_time > 0 else math.inf
                    byts = E.storage_report(f).total() + 8 * a.n + 8 * a.m
                    r.gbs = byts / r.min_time / 1e9
                    if cfg.peak_gbs:
                        r.roofline_frac = r.gbs / cfg.peak_gbs
                del f
            except E.Error as ex:
                r.status = str(ex)
            recs.append(r)
    merge_t = {r.threads: r.min_time for r in recs if r.algorithm == int(E.Algorithm.Merge) and r.min_time > 0}
    for r in recs:
        tm = merge_t.get(r.threads)
        if tm and r.min_time > 0 and r.min_time < tm and r.convert_time is not None:
            r.break_even = r.convert_time / (tm - r.min_time)
    recs.sort(key=lambda r: (r.matrix, r.algorithm, r.threads))  # detail::sort_records
    return recs
