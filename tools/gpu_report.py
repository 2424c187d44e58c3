"""Device benchmark report (the GPU counterpart of the reference CLI's bench/report subcommands,
proj/tools/spmvlab_cli.cpp:241-257): every engine on the chosen BASELINE configs through
paper_2502_19284_b200.report.bench_all, written as the reference's CSV / markdown plus the
extended GPU columns.

usage: python tools/gpu_report.py --configs 1,2 --threads 8 --out profiles/r01_report
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2502_19284_b200 as sp  # noqa: E402
from paper_2502_19284_b200 import gen, report  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2")
    ap.add_argument("--threads", default="8")
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "report"))
    args = ap.parse_args()
    peak_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak = float(json.load(open(peak_path))["hbm_gbs"]) if os.path.exists(peak_path) else None
    cfg = report.BenchConfig(threads=[int(t) for t in args.threads.split(",")], spmv_reps=args.reps,
                             peak_gbs=peak)
    recs = []
    for c in (int(x) for x in args.configs.split(",")):
        name, fn = gen.CONFIGS[c]
        m, n, r, cc, v = fn(torch.device("cuda"))
        recs += report.bench_all(sp.TripletMatrix(m, n, r, cc, v), name, cfg)
        del r, cc, v
        torch.cuda.empty_cache()
        print(f"{name}: {sum(1 for x in recs if x.matrix == name)} records", flush=True)
    open(args.out + ".csv", "w").write(report.emit_csv(recs, extended=True))
    open(args.out + ".md", "w").write(report.emit_markdown(recs, gpu_columns=True))
    print(report.emit_markdown(recs, gpu_columns=True))


if __name__ == "__main__":
    main()
