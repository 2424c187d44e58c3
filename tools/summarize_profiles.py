"""Summarise ncu captures into profiles/ (dev tool).

    python tools/summarize_profiles.py --round r01 --launches gpurun_out/launches.csv \
        --full gpurun_out/r01_merge_full.ncu-rep --kernel merge_spmv_wstage_kernel --config 2
"""
import argparse
import collections
import csv
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__cycles_elapsed.avg.per_second",
        "launch__grid_size", "launch__block_size", "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_requests.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(path, out, cmd):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        name = r[ki].split("(")[0].replace("void ", "").strip().split("::")[-1]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
    tot = sum(a[1] for a in agg.values())
    lines = [f"# ncu launch list (gpu__time_duration.sum, --clock-control none): {cmd}",
             "# cold-cache, serialised launches: compare SHARES, not absolutes", "kernel,launches,total_us,mean_us,share"]
    for k, (n, t) in agg.items():
        lines.append(f"{k},{n},{t / 1e3:.1f},{t / n / 1e3:.2f},{t / tot:.4f}")
    open(out, "w").write("\n".join(lines) + "\n")


def full(rep, out, kernel, config, summary):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    h, u, v = r[0], r[1], r[2]
    d = {n: (v[i], u[i]) for i, n in enumerate(h) if n in WANT}
    lines = [f"# ncu --set full of {kernel} (cfg{config}), one launch"] + [f"{k}: {d[k][0]} {d[k][1]}" for k in WANT if k in d]
    open(out, "w").write("\n".join(lines) + "\n")
    num = lambda k: float(d[k][0].replace(",", "")) * SCALE.get(d[k][1], 1)
    js = json.load(open(summary)) if os.path.exists(summary) else {}
    js[f"cfg{config}:{kernel}"] = {"dram_bytes_per_launch": num("dram__bytes_read.sum") + num("dram__bytes_write.sum"),
                                   "dram_read": num("dram__bytes_read.sum"), "dram_write": num("dram__bytes_write.sum"),
                                   "source": os.path.relpath(out, ROOT)}
    if "l1tex__m_xbar2l1tex_read_bytes.sum" in d:  # L2 -> SM bytes (gathers move whole 32 B sectors)
        js[f"cfg{config}:{kernel}"]["l2_to_sm_bytes_per_launch"] = num("l1tex__m_xbar2l1tex_read_bytes.sum")
    json.dump(js, open(summary, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--launches")
    ap.add_argument("--cmd", default="python bench.py --steps 20 --warmup 5 --no-formats --no-cpu")
    ap.add_argument("--full")
    ap.add_argument("--kernel")
    ap.add_argument("--config", type=int, default=2)
    a = ap.parse_args()
    prof = os.path.join(ROOT, "profiles")
    if a.launches:
        launches(a.launches, os.path.join(prof, f"{a.round}_launches_summary.csv"), a.cmd)
    if a.full:
        full(a.full, os.path.join(prof, f"{a.round}_{a.kernel}_ncu_full.txt"), a.kernel, a.config,
             os.path.join(prof, "ncu_summary.json"))
