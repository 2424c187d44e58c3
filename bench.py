#!/usr/bin/env python
"""Benchmark of the SpMV hot path (BASELINE.json metric: SpMV GFLOP/s & HBM GB/s per format;
conversion ms).

Default (N = 1): BASELINE.json configs[1] -- R-MAT scale 22, edge factor 16, (.57,.19,.19,.05),
duplicates summed, values U(0,1] -- generated on the device from a fixed seed.  One "step" is one
merge-CSR multiply y = A x (the north-star engine, spmv_merge) through the C ABI with A, x and y
resident in HBM; `value` = 2 nnz K / t  (GFLOP/s).  Inputs (866 MB of algorithmic bytes) are
larger than the 126 MB L2, so no flush is needed between steps.

N > 1 (torchrun, one process per GPU): BASELINE configs[4] by default -- R-MAT scale 26, column-
normalised, the iterated x <- A x of north_star's multi-GPU row (--config overrides).  The matrix
is row-sharded by nonzeros across ranks (partition_rows_by_nnz with beta = 1,
inc/block_size.hpp:73-102); a step is one iteration x_next = A x on every rank: the local multiply
whose warp tiles copy their finished rows into every rank's next x (CUDA IPC peer stores over
NVLink, --exchange fused, default) or the local multiply followed by an NCCL all-gatherv of the y_r
slices (--exchange nccl), then a stream-ordered rendezvous; time is the max over ranks; scaling
"strong".  "multi_gpu" reports, on the same matrix: the 1-GPU step (rank 0 multiplies the whole
matrix before sharding), the shard multiply alone, and step / exchange time of BOTH exchanges
(SURVEY §8e).

Extra keys: e2e (host buffers through the C ABI, copies timed), roofline (dominant kernel,
event-timed in the library), cpu_baseline (the reference's own engine on the host cores),
clocks, gpu_launches, formats (every engine: conversion ms, SpMV us, GFLOP/s, GB/s, fraction of
the measured HBM peak, break-even count).

--impl reference: the reference's own CPU implementation (oracle/_ref, the unmodified headers)
timed on the host cores on the same matrix (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
UNIT = "GFLOP/s"
CPU_MAX_NNZ = 70_000_000  # bound on the CPU-baseline sample (cfg5 has ~1.04G entries)
CONFIG_DESC = {
    1: "cfg1: Erdos-Renyi n=65,536, Binomial(n,16/n) rows, U[-1,1]",
    2: "cfg2: R-MAT scale 22, edge factor 16, (.57,.19,.19,.05), duplicates summed, U(0,1]",
    3: "cfg3: Zipf degrees (k^-2.1 on [1,2^20]), n=2^24, U[-1,1]",
    4: "cfg4: 5-point Laplacian 4096^2, seeded symmetric permutation",
    5: "cfg5: R-MAT scale 26, column-normalised",
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------------------ clocks
CLOCK_FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")


class Clocks:
    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={CLOCK_FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.gpu)], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.25)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            p = [s.strip() for s in line.split(",")]
            if len(p) >= 9:
                rows.append(p)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------------------ helpers
def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_traffic(cfg: int, kernel: str):
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    e = d.get(f"cfg{cfg}:{kernel}")
    return e.get("dram_bytes_per_launch") if e else None


def l2_roofline(cfg: int, kernel: str, kernel_ms: float):
    """The roofline that binds the gather kernels: whole 32-byte L2 sectors per random 8-byte x
    gather, L2 -> SM bytes (ncu, per launch) over the kernel time, against the same rate of the
    pure x-gather probe (tools/microbench.py gather_x; no merge logic)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    e, probe = d.get(f"cfg{cfg}:{kernel}"), d.get("probe:gather_x")
    if not e or "l2_to_sm_bytes_per_launch" not in e or not probe:
        return None
    achieved = e["l2_to_sm_bytes_per_launch"] / (kernel_ms / 1e3) / 1e9
    peak = probe["l2_to_sm_bytes_per_launch"] / (probe["us"] / 1e6) / 1e9
    out = {"bytes_per_launch": e["l2_to_sm_bytes_per_launch"], "achieved": achieved, "peak": peak,
           "unit": "GB/s", "frac": achieved / peak, "peak_kind": "probe (x-gather only kernel)"}
    if "l1tex_lsu_wavefront_pct_of_peak" in e:  # the L1TEX data pipe (one wavefront per gathered line)
        out["l1tex_data_pipe_pct_of_peak_ncu"] = e["l1tex_lsu_wavefront_pct_of_peak"]
    return out


def ev_time(fn, reps: int, warmup: int, stream, flush=None) -> list:
    """Per-call device times; `flush` (a tensor larger than the L2) is overwritten before every call."""
    for _ in range(warmup):
        fn()
    out = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        if flush is not None:
            flush.fill_(0.0)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        out.append(a.elapsed_time(b))
    return out


def make_matrix(cfg: int, device):
    from paper_2502_19284_b200 import gen
    name, fn = gen.CONFIGS[cfg]
    m, n, r, c, v = fn(device)
    return name, m, n, r, c, v


# ------------------------------------------------------------------------------ reference arm
def cpu_reference(m, n, r, c, v, reps: int, warmup: int):
    """The reference's merge engine (spmv_merge, inc/spmv_parallel.hpp:130-160) and its CRS
    conversion, unmodified, through oracle/_ref on all host threads."""
    from oracle.oracle import Oracle, Reference, reference_available
    sample_note = "full matrix"
    if v.numel() > CPU_MAX_NNZ:  # bound the CPU sample: the leading rows holding <= CPU_MAX_NNZ entries
        counts = torch.bincount(r.long(), minlength=m)
        prefix = torch.cumsum(counts, 0)
        m = int(torch.searchsorted(prefix, torch.tensor([CPU_MAX_NNZ], device=prefix.device)).item())
        sel = r < m
        r, c, v = r[sel], c[sel], v[sel]
        sample_note = f"leading {m} rows"
    rows = r.cpu().numpy().view(np.uint32)
    cols = c.cpu().numpy().view(np.uint32)
    vals = v.cpu().numpy()
    x = np.random.default_rng(7).uniform(0.0, 1.0, n)
    if reference_available():
        lib = Reference()
        threads = lib.hardware_threads()
        t0 = time.perf_counter()
        built = lib.build(2, m, n, rows, cols, vals, threads=threads, build_threads=threads, export=False)
        conv_s = time.perf_counter() - t0
        mn, tot = lib.time_spmv(built, 2, x, threads, reps, warmup)
        kind = "reference"
    else:  # the C restatement (single thread)
        lib = Oracle()
        threads = 1
        t0 = time.perf_counter()
        built = lib.build(2, m, n, rows, cols, vals)
        conv_s = time.perf_counter() - t0
        lib.spmv(built, 2, x, p=1)
        t1 = time.perf_counter()
        for _ in range(reps):
            lib.spmv(built, 2, x, p=1)
        tot = time.perf_counter() - t1
        mn = tot / reps
        kind = "port"
    nnz = len(vals)
    # value from the minimum multiply time, the reference protocol's statistic (inc/bench.hpp:98-110)
    return {"value": 2 * nnz / mn / 1e9, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{sample_note} ({nnz} nnz), merge engine p={threads}, min of {reps} multiplies after "
                      f"{warmup} warm-up (mean {tot / reps * 1e3:.2f} ms); triplet_to_crs conversion {conv_s:.2f} s",
            "min_ms": mn * 1e3, "mean_ms": tot / reps * 1e3, "conversion_s": conv_s}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    dev = torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")
    name, m, n, r, c, v = make_matrix(args.config, dev)
    nnz = v.numel()
    steps = max(1, args.steps if args.steps <= 200 else 50)
    cb = cpu_reference(m, n, r, c, v, steps, max(1, min(args.warmup, 3)))
    line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": steps, "warmup": max(1, min(args.warmup, 3)), "ms_per_step": cb["min_ms"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": CONFIG_DESC[args.config], "matrix": name, "n": n,
                                             "nnz": nnz, "engine": "merge (spmv_merge)"},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ our arm
def all_formats(sp, a, m, n, nnz, x, stream, peak, merge_us, threads=8):
    out = {}
    parcrs_us = None
    for alg in sp.all_algorithms:
        name = sp.algorithm_name(alg)
        p = threads
        # conversion time = min of 3 builds (the reference protocol takes the min of its
        # conversion repetitions, inc/bench.hpp:315-318); the first build also warms the pools
        conv_ms = float("inf")
        f = None
        for _ in range(3):
            f = None  # release the previous build outside the timed region
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            f = sp.build_format(alg, a, p)
            e1.record(stream)
            e1.synchronize()
            conv_ms = min(conv_ms, e0.elapsed_time(e1))
        y = torch.empty(m, dtype=torch.float64, device=x.device)
        reps = 5 if alg == sp.Algorithm.SeqCrs else 20
        byts = sp.storage_report(f).total() + 8 * n + 8 * m
        # a working set that fits the L2 is flushed before every multiply
        flush = torch.empty(32 << 20, dtype=torch.float64, device=x.device) if byts < (256 << 20) else None
        ts = ev_time(lambda: sp.run_spmv(alg, f, x, y, p=p), reps, 3, stream, flush)
        us = statistics.median(ts) * 1e3
        del flush
        if alg == sp.Algorithm.ParCrs:
            parcrs_us = us
        out[name] = {"conversion_ms": conv_ms, "spmv_us": us, "spmv_min_us": min(ts) * 1e3,
                     "gflops": 2 * nnz / us / 1e3, "gbs": byts / us / 1e3, "frac_of_hbm": byts / us / 1e3 / peak,
                     "algorithmic_bytes": byts}
        del f, y
        torch.cuda.empty_cache()
    for name, d in out.items():
        t_fmt = d["spmv_us"]
        d["break_even_vs_merge"] = (d["conversion_ms"] * 1e3 / (merge_us - t_fmt)) if t_fmt < merge_us and name != "merge" else None
        # the paper's break-even against the row-parallel CSR baseline: multiplies
        # after which a format's conversion is paid back by its faster SpMV
        d["break_even_vs_parcrs"] = (d["conversion_ms"] * 1e3 / (parcrs_us - t_fmt)) if parcrs_us and t_fmt < parcrs_us else None
        d["conversion_in_parcrs_spmvs"] = d["conversion_ms"] * 1e3 / parcrs_us if parcrs_us else None
    return out


def recorded_cpu_reference(cfg: int):
    """The reference's own bench_spmv / bench_convert (inc/bench.hpp:239-329) recorded on a B200 box's
    host cores by tools/cpu_reference_bench.py (profiles/cpu_reference/): per engine, the min of the
    protocol's multiplies and conversion seconds at the highest thread count."""
    base = os.path.join(ROOT, "profiles", "cpu_reference")
    out = {}
    for kind, fname in (("spmv", f"cfg{cfg}_spmv_all.json"), ("convert", f"cfg{cfg}_convert_all.json")):
        p = os.path.join(base, fname)
        if not os.path.exists(p):
            continue
        d = json.load(open(p))
        for rec in d["records"]:
            if rec["status"] != "ok":
                continue
            e = out.setdefault(rec["engine"], {"threads": rec["threads"], "host": d["host"]["cpu_model"]})
            if kind == "spmv":
                e["spmv_min_ms"] = rec["min_time_s"] * 1e3
                e["spmv_reps"] = d["protocol"]["spmv_reps"]
            else:
                e["conversion_s"] = rec["convert_time_s"]
    return out or None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=None, choices=[1, 2, 3, 4, 5],
                    help="BASELINE config (default: 2 on 1 GPU, 5 -- the iterated scale-26 matrix -- on N > 1)")
    ap.add_argument("--no-formats", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--exchange", default="fused", choices=["fused", "nccl"],
                    help="N > 1: exchange fused into the multiply (default) or NCCL all-gatherv")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.config is None:
        args.config = 2 if world == 1 else 5
    # SPMVLAB_BENCH_BACKEND=gloo (test only): N ranks as processes sharing fewer GPUs, synchronised
    # on the host (no kernel waits on another rank), to exercise the N > 1 flow on a 1-GPU box.
    backend = os.environ.get("SPMVLAB_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local %= max(1, torch.cuda.device_count())
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return

    import paper_2502_19284_b200 as sp
    sp.capi.load()
    L = sp.capi.load()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()
    peak, peak_kind = measured_peak()

    name, m, n, r, c, v = make_matrix(args.config, dev)
    nnz_total = v.numel()
    from paper_2502_19284_b200 import dist as sdist
    x = torch.rand(n, generator=torch.Generator(device=dev).manual_seed(7), device=dev, dtype=torch.float64)

    # N > 1: the same matrix on ONE GPU first (rank 0, before sharding), so the 1 -> N curve in
    # the line is on one matrix
    single_gpu = None
    if world > 1 and rank == 0 and m == n:
        f1 = sp.build_format(sp.Algorithm.Merge, sp.TripletMatrix(m, n, r, c, v), 1)
        y1 = torch.empty(m, dtype=torch.float64, device=dev)
        reps1 = max(3, min(args.steps, 20))
        ts = ev_time(lambda: sp.run_spmv(sp.Algorithm.Merge, f1, x, y1, p=1), reps1, 3, stream)
        ms1 = statistics.median(ts)
        single_gpu = {"ms_per_step": ms1, "gflops": 2.0 * nnz_total / (ms1 / 1e3) / 1e9, "steps": reps1,
                      "merge_panels": f1.info["merge_panels"]}
        del f1, y1
        sp.release_cached_memory()

    cuts = [0, m]
    if world > 1:
        cuts = sdist.shard_bounds(sdist.row_prefix(m, r), world)
        lr, lc, lv = sdist.shard_rows(r, c, v, cuts[rank], cuts[rank + 1])
        a = sp.TripletMatrix(cuts[rank + 1] - cuts[rank], n, lr, lc, lv)
    else:
        a = sp.TripletMatrix(m, n, r, c, v)
    m_loc = a.m

    # conversion (COO -> merge-CSR), event-timed, min of 3 (the first also warms the memory pools);
    # the multiply uses the first build (the later ones are timed and released)
    conv_ms = float("inf")
    fmt = None
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        built = sp.build_format(sp.Algorithm.Merge, a, 1)
        e1.record(stream)
        e1.synchronize()
        conv_ms = min(conv_ms, e0.elapsed_time(e1))
        if fmt is None:
            fmt = built
        del built
    if world > 1:
        del lr, lc, lv
        sp.release_cached_memory()
    y_full = torch.zeros(m, dtype=torch.float64, device=dev)
    y_loc = y_full[cuts[rank]:cuts[rank + 1]] if world > 1 else y_full

    sharded = sdist.ShardedSpMV(cuts, rank, lambda xf, yl: sp.run_spmv(sp.Algorithm.Merge, fmt, xf, yl, p=1))
    fused, fused_err = None, None
    if world > 1:
        try:  # collective; every rank agrees on success or falls back together
            fused = sdist.FusedExchangeSpMV(cuts, rank, fmt, n)
            fused.load(x)
        except Exception as ex:
            log(f"fused exchange unavailable: {ex}")
            fused, fused_err = None, str(ex)
    EXCH = {"fused": "fused: each merge warp tile copies its finished rows into every rank's next x (CUDA IPC "
                     "peer stores over NVLink)",
            "nccl": "NCCL all-gatherv (per-rank broadcasts) of the y slices"}

    def make_step(mode):
        if mode == "fused":
            return fused.step  # x_next = A_r x on every rank: multiply + peer stores + rank rendezvous
        if mode == "nccl":
            return lambda: sharded.step(x, y_full)  # local merge multiply + NCCL all-gatherv
        return lambda: sp.run_spmv(sp.Algorithm.Merge, fmt, x, y_loc, p=1)

    # A working set that fits the 126 MB L2 (cfg1: ~14 MB) would stay cached between steps: then the
    # L2 is flushed before every step (a 256 MiB write, outside the per-step event pair) and the
    # step times are summed.
    work_bytes = sp.storage_report(fmt).total() + 8 * n + 8 * m_loc
    flush = torch.empty(32 << 20, dtype=torch.float64, device=dev) if work_bytes < (256 << 20) else None
    l2_note = ("L2 flushed before every step (256 MiB write outside the timed events; working set "
               f"{work_bytes / 1e6:.1f} MB)") if flush is not None else "inputs larger than L2 (no flush)"

    def timed(fn, steps):
        """Device time of `steps` calls (max over ranks), after a barrier."""
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if flush is not None:
            ms = 0.0
            with torch.cuda.stream(stream):
                for _ in range(steps):
                    flush.fill_(0.0)
                    t0.record(stream)
                    fn()
                    t1.record(stream)
                    t1.synchronize()
                    ms += t0.elapsed_time(t1)
        else:
            t0.record(stream)
            for _ in range(steps):
                fn()
            t1.record(stream)
            torch.cuda.synchronize()
            ms = t0.elapsed_time(t1)
        if world > 1:
            import torch.distributed as dist
            tt = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt[0])
        return ms

    modes = ["local"] if world == 1 else (["fused", "nccl"] if fused is not None else ["nccl"])
    if world > 1 and args.exchange == "nccl":
        modes = ["nccl"] + [md for md in modes if md != "nccl"]
    primary = modes[0]
    exchange = "none (1 GPU)" if world == 1 else EXCH[primary] + (f" (fused unavailable: {fused_err})" if fused_err else "")
    step = make_step(primary)
    for _ in range(args.warmup):
        step()
    clocks = Clocks(local)
    clocks.start()
    launches0 = L.spmvlab_cuda_launch_count()
    elapsed_ms = timed(step, args.steps)
    launches = L.spmvlab_cuda_launch_count() - launches0
    clk = clocks.stop()
    if world > 1:
        import torch.distributed as dist
        tl = torch.tensor([float(launches)], dtype=torch.float64, device=dev)
        dist.all_reduce(tl, op=dist.ReduceOp.SUM)
        launches = int(tl[0])
    # dominant-kernel duration: a separate run with the library's per-launch event brackets (kept
    # out of the timed region above, where the extra event records would cost small kernels)
    L.spmvlab_cuda_kernel_timing(1)
    for _ in range(min(args.steps, 200)):
        step()
    torch.cuda.synchronize()
    L.spmvlab_cuda_kernel_timing(0)
    import ctypes as C
    kms, kl, kname = C.c_double(), C.c_uint64(), C.create_string_buffer(64)
    L.spmvlab_cuda_kernel_time(C.byref(kms), C.byref(kl), kname, 64)
    ms_step = elapsed_ms / args.steps
    value = 2.0 * nnz_total * args.steps / (elapsed_ms / 1e3) / 1e9

    # N > 1: per-iteration compute (the shard's multiply alone, no exchange, max over
    # ranks) and, for BOTH exchanges, the whole step and exchange = step - compute; plus the
    # 1-GPU step on the same matrix
    multi_gpu = None
    if world > 1:
        comp_fn = make_step("local")
        for _ in range(3):
            comp_fn()
        comp = timed(comp_fn, args.steps) / args.steps
        per = {}
        for md in modes:
            fn = make_step(md)
            for _ in range(3):
                fn()
            st = timed(fn, args.steps) / args.steps
            per[md] = {"step_ms": st, "exchange_ms": max(0.0, st - comp), "exchange": EXCH[md],
                       "gflops": 2.0 * nnz_total / (st / 1e3) / 1e9}
        multi_gpu = {"compute_ms_per_step": comp, "exchanges": per, "single_gpu": single_gpu,
                     "cuts": cuts, "note": "compute = the rank's shard multiply alone (max over ranks); "
                                           "exchange = step - compute; single_gpu = rank 0, whole matrix"}
        if single_gpu:
            multi_gpu["speedup_vs_1gpu"] = single_gpu["ms_per_step"] / ms_step

    # dominant kernel roofline (per launch, this rank).  Algorithmic bytes of the timed kernels: the
    # reference format (storage_report) + x once + y once; with K > 1 column panels the kernels read
    # the panel arrays instead (panel 0's row pointer over all m rows, the compressed pointers and
    # row ids of panels >= 1, the same col / data) and every row of a panel >= 1 reads and writes y
    # again, so those are the bytes counted.
    rep = sp.storage_report(fmt)
    ref_bytes = rep.total() + 8 * n + 8 * m_loc
    K = int(fmt.info["merge_panels"])
    nnz_loc = fmt.nnz()
    alg_bytes = ref_bytes
    if K > 1:  # the panel row pointers and row ids, the entries, x, y written by panel 0 and read +
        # written again for every row with entries in a later panel
        ptr_b = 4 * len(fmt.array("merge_panel_row_ptr")) + 4 * len(fmt.array("merge_panel_rows"))
        alg_bytes = ptr_b + 12 * nnz_loc + 8 * n + 8 * m_loc + 16 * int(fmt.info["merge_panel_row_visits"])
    k_ms = kms.value / max(1, kl.value)
    achieved = alg_bytes / (k_ms / 1e3) / 1e9
    kernel_name = kname.value.decode()
    roofline = {"bound": "hbm", "kernel": kernel_name + " + merge_fixup_kernel", "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "peak_kind": peak_kind, "kernel_ms": k_ms,
                "algorithmic_bytes_per_launch": alg_bytes, "reference_format_bytes": ref_bytes,
                "column_panels": K, "traffic": ncu_traffic(args.config, kernel_name),
                "share_of_step": k_ms / ms_step, "l2_sectors": l2_roofline(args.config, kernel_name, k_ms)}

    # End to end through the C ABI with host buffers: every step copies its own x in (pinned H2D),
    # multiplies, and copies its own y out (D2H).  Steps rotate over three streams with their own
    # staging buffers, so the H2D of later steps overlaps the multiply and D2H of earlier ones
    # (full-duplex PCIe) without waiting behind a stream's own D2H.
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    NS = 3
    e2e_streams = [torch.cuda.Stream(dev) for _ in range(NS)]
    x_host = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(NS)]
    for xh in x_host:
        xh.copy_(x.cpu())
    y_host = [torch.empty(m_loc, dtype=torch.float64).pin_memory() for _ in range(NS)]
    x_dev = [torch.empty_like(x) for _ in range(NS)]
    y_dev = [torch.empty(m_loc, dtype=torch.float64, device=dev) for _ in range(NS)]
    e2e_steps = max(6, min(args.steps, 200))

    def e2e_run(steps):
        start = torch.cuda.Event()
        start.record(stream)
        for s_ in e2e_streams:
            s_.wait_event(start)
        for k in range(steps):
            i = k % NS
            sp.run_spmv_host(sp.Algorithm.Merge, fmt, x_host[i], y_host[i], 1, x_dev[i], y_dev[i],
                             stream=e2e_streams[i])
        for s_ in e2e_streams:
            done = torch.cuda.Event()
            done.record(s_)
            stream.wait_event(done)

    e2e_run(4)
    torch.cuda.synchronize()
    t0.record(stream)
    e2e_run(e2e_steps)
    t1.record(stream)
    t1.synchronize()
    e2e_ms = t0.elapsed_time(t1)
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt[0])
    e2e = {"value": 2.0 * nnz_total * e2e_steps / (e2e_ms / 1e3) / 1e9, "unit": UNIT,
           "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * m_loc, "ms_per_step": e2e_ms / e2e_steps}

    # the application loop (spmvlab_cuda_iterate): 100 rescaled iterations with convergence norms,
    # as one CUDA graph and as a plain stream loop
    iterate = None
    if world == 1 and m == n:
        iters = 100
        normalize = bool(v.min() >= 0)  # unit-mass rescaling is meaningful for non-negative A
        work = torch.empty_like(x)
        side = torch.cuda.Stream(dev)
        res = {}
        for graph in (False, True):
            side.wait_stream(stream)
            xi = x.clone()
            sp.iterate(sp.Algorithm.Merge, fmt, xi, 3, normalize=normalize, graph=graph, work=work, stream=side)
            side.synchronize()
            t0.record(side)
            _, nb = sp.iterate(sp.Algorithm.Merge, fmt, xi, iters, normalize=normalize, graph=graph, work=work, stream=side)
            t1.record(side)
            t1.synchronize()
            res["graph" if graph else "stream"] = t0.elapsed_time(t1) / iters
        # the same loop keeping no norms (a rescaled loop then runs its mass inside the multiply)
        side.wait_stream(stream)
        xi = x.clone()
        sp.iterate(sp.Algorithm.Merge, fmt, xi, 3, normalize=normalize, norms=False, work=work, stream=side)
        side.synchronize()
        t0.record(side)
        sp.iterate(sp.Algorithm.Merge, fmt, xi, iters, normalize=normalize, norms=False, work=work, stream=side)
        t1.record(side)
        t1.synchronize()
        res["stream_no_norms"] = t0.elapsed_time(t1) / iters
        # the multiply back to back on the same stream (no L2 flush: the loop's own x and y stay in
        # the L2 between iterations for a small working set)
        side.wait_stream(stream)
        for _ in range(3):
            sp.run_spmv(sp.Algorithm.Merge, fmt, x, y_loc, p=1, stream=side)
        t0.record(side)
        for _ in range(iters):
            sp.run_spmv(sp.Algorithm.Merge, fmt, x, y_loc, p=1, stream=side)
        t1.record(side)
        t1.synchronize()
        spmv_b2b = t0.elapsed_time(t1) / iters
        iterate = {"engine": "merge", "iterations": iters, "normalize": normalize,
                   "ms_per_iteration": res, "spmv_ms": spmv_b2b,
                   "ratio_to_spmv": {k: t / spmv_b2b for k, t in res.items()},
                   "final_diff_l1": float(nb[-1, 0]), "final_mass": float(nb[-1, 1])}
        del work

    formats = None
    merge_us = ms_step * 1e3
    if world == 1 and not args.no_formats:
        del y_host, x_host
        formats = all_formats(sp, a, m, n, nnz_total, x, stream, peak, merge_us)
        cpu_rec = recorded_cpu_reference(args.config)
        for fname, d in (formats.items() if cpu_rec else ()):
            if fname in cpu_rec:
                d["cpu_reference"] = cpu_rec[fname]

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cb = cpu_reference(m, n, r, c, v, reps=50, warmup=3)
            cpu_baseline = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
            cpu_baseline["conversion_s"] = cb["conversion_s"]
        except Exception as ex:  # the checker is optional on a box without oracle/_ref
            cpu_baseline = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable",
                            "sample": f"failed: {ex}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded, generated on device)",
                "config": {"workload": CONFIG_DESC[args.config], "matrix": name, "n": n, "nnz": nnz_total,
                           "engine": "merge-CSR (spmv_merge)",
                           "parallelism": f"row-shard x{world}" if world > 1 else "1 GPU", "exchange": exchange,
                           "l2": l2_note, "conversion_ms": conv_ms,
                           "merge_path_partition": "at build time (one diagonal search per 32*IPT-item warp tile, "
                                                   "inside conversion_ms); the reference searches its p diagonals "
                                                   "inside spmv_merge (spmv_parallel.hpp:130-145)",
                           "merge_tile_ipt": int(fmt.info["merge_ipt"]), "column_panels": int(fmt.info["merge_panels"])},
                "roofline": roofline, "cpu_baseline": cpu_baseline, "e2e": e2e, "clocks": clk,
                "gpu_launches": launches, "formats": formats, "iterate": iterate}
        if multi_gpu is not None:
            line["multi_gpu"] = multi_gpu
        print(json.dumps(line), flush=True)
    if fused is not None:
        fused.close()  # collective
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
