"""Writes tests/golden/bicrs_golden.json: the REFERENCE's standalone ICRS / BICRS
(inc/bicrs.hpp: crs_to_icrs, triplet_to_bicrs, spmv_bicrs_seq + ReplayStats, bicrs_to_triplet)
run on a few matrices and element orders, plus corrupted streams and the ErrorKind the reference
replay raises for each.  Compiled here from /root/reference/proj/include.

Run in the development container:  python tests/golden/make_bicrs_golden.py
"""
import json
import os
import subprocess
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/proj/include"


def matrices():
    rng = np.random.default_rng(31)
    out = []
    out.append(("e4", 4, 4, [0, 0, 1, 3, 3], [0, 2, 1, 0, 3], [1.0, 2.0, 3.0, 4.0, 5.0]))
    out.append(("last_row_only", 6, 3, [5, 5], [0, 2], [1.0, 2.0]))
    out.append(("empty", 3, 5, [], [], []))
    m, n = 60, 45
    cells = rng.choice(m * n, 400, replace=False)
    out.append(("rand60x45", m, n, (cells // n).tolist(), (cells % n).tolist(),
                rng.uniform(-1, 1, 400).round(6).tolist()))
    m, n = 300, 1
    cells = rng.choice(m, 70, replace=False)
    out.append(("column", m, n, cells.tolist(), [0] * 70, rng.integers(1, 9, 70).astype(float).tolist()))
    return out


def orders(name, nnz, rows, cols):
    rng = np.random.default_rng(len(name) * 7 + nnz)
    idx = np.arange(nnz)
    res = {"identity": idx.tolist()}
    if nnz:
        res["colmajor"] = sorted(idx.tolist(), key=lambda k: (cols[k], rows[k]))
        res["random"] = rng.permutation(nnz).tolist()
    return res


DRIVER = r"""
#include <cstdio>
#include <cstring>
#include <iostream>
#include <spmvlab/bicrs.hpp>
#include <spmvlab/crs.hpp>
using namespace spmvlab;
static unsigned long long bits(double v) { unsigned long long b; std::memcpy(&b, &v, 8); return b; }
template <class M> void dump(const M& a, const DenseVector& x) {
  std::printf("inc");
  for (auto v : a.col_inc) std::printf(" %lld", (long long)v);
  std::printf("\njump");
  for (auto v : a.row_jump) std::printf(" %lld", (long long)v);
  std::printf("\n");
  try {
    ReplayStats st;
    auto y = spmv_bicrs_seq(a, x, &st);
    std::printf("y");
    for (double v : y) std::printf(" %016llx", bits(v));
    std::printf("\nstats %u %u\n", st.overflow_events, st.row_jumps_consumed);
    auto t = bicrs_to_triplet(a);
    std::printf("rows");
    for (auto v : t.row_ind) std::printf(" %u", v);
    std::printf("\ncols");
    for (auto v : t.col_ind) std::printf(" %u", v);
    std::printf("\n");
  } catch (const Error& e) {
    std::printf("err %d\nstats 0 0\nrows\ncols\n", (int)e.kind());
  }
}
int main() {
  int nm; std::cin >> nm;
  for (int q = 0; q < nm; ++q) {
    TripletMatrix a; size_t nnz; std::cin >> a.m >> a.n >> nnz;
    a.row_ind.resize(nnz); a.col_ind.resize(nnz); a.data.resize(nnz);
    for (auto& v : a.row_ind) std::cin >> v;
    for (auto& v : a.col_ind) std::cin >> v;
    for (auto& v : a.data) std::cin >> v;
    DenseVector x(a.n); for (auto& v : x) std::cin >> v;
    // ICRS from CRS, then corrupted copies
    auto icrs = crs_to_icrs(triplet_to_crs(a));
    dump(icrs, x);
    int no; std::cin >> no;
    for (int o = 0; o < no; ++o) {
      std::vector<index_t> ord(nnz); for (auto& v : ord) std::cin >> v;
      dump(triplet_to_bicrs(a, ord), x);
    }
    int nc; std::cin >> nc;  // corrupt BICRS streams given explicitly
    for (int c = 0; c < nc; ++c) {
      BicrsMatrix b; b.m = a.m; b.n = a.n; b.data = a.data;
      size_t ni, nj; std::cin >> ni >> nj;
      b.col_inc.resize(ni); b.row_jump.resize(nj);
      for (auto& v : b.col_inc) std::cin >> v;
      for (auto& v : b.row_jump) std::cin >> v;
      dump(b, x);
    }
  }
}
"""
KINDS = ["DimensionMismatch", "InvalidArgument", "CorruptFormat", "Overflow", "BadHeader", "UnsupportedFormat",
         "UnsupportedField", "UnsupportedSymmetry", "IndexOutOfRange", "DuplicateEntry", "ParseError", "Truncated",
         "BadMagic", "IoError"]


def corruptions(m, n, inc, jump):
    """Corrupted copies of a valid BICRS stream (inc, jump) hitting each replay check."""
    out = []
    if len(inc) < 3:
        return out
    out.append(("fewer_jumps", inc, jump[:-1]))                          # runs out of row jumps
    out.append(("extra_jump", inc, jump + [0]))                          # jumps left over
    out.append(("overshoot", [inc[0] + 2 * n + 1] + inc[1:], jump))      # exits [0, 2n)
    out.append(("negative_col", inc[:1] + [-(inc[0] + 1) - n * 0] + inc[2:], jump))  # column < 0
    out.append(("row_out", inc, [m + 3] + jump[1:]))                     # row out of bounds
    return out


def main():
    mats = matrices()
    lines = [str(len(mats))]
    plan = []
    for (name, m, n, r, c, v) in mats:
        x = np.random.default_rng(5).uniform(0.5, 1.5, n).round(6).tolist()
        lines += [f"{m} {n} {len(v)}", " ".join(map(str, r)), " ".join(map(str, c)), " ".join(repr(t) for t in v),
                  " ".join(repr(t) for t in x)]
        ords = orders(name, len(v), r, c)
        lines.append(str(len(ords)))
        for o in ords.values():
            lines.append(" ".join(map(str, o)))
        plan.append((name, m, n, r, c, v, x, list(ords)))
        lines.append("PLACEHOLDER_CORRUPT")
    # first pass: no corruptions, to learn the valid BICRS streams
    with tempfile.TemporaryDirectory() as td:
        src, exe = os.path.join(td, "d.cpp"), os.path.join(td, "d")
        open(src, "w").write(DRIVER)
        subprocess.check_call(["g++", "-std=c++20", "-O1", "-I" + REF, src, "-o", exe])

        def run(inp):
            return subprocess.run([exe], input=inp.encode(), capture_output=True, check=True).stdout.decode()

        first = run("\n".join(l if l != "PLACEHOLDER_CORRUPT" else "0" for l in lines) + "\n").splitlines()
        pos, valid_bicrs = 0, []
        for (name, m, n, r, c, v, x, on) in plan:
            pos += 6  # icrs dump
            inc = list(map(int, first[pos].split()[1:])) if on else []
            jump = list(map(int, first[pos + 1].split()[1:])) if on else []
            valid_bicrs.append((inc, jump))
            pos += 6 * len(on)
        out_lines, k = [], 0
        corr_names = []
        for l in lines:
            if l != "PLACEHOLDER_CORRUPT":
                out_lines.append(l)
                continue
            name, m, n = plan[k][0], plan[k][1], plan[k][2]
            cs = corruptions(m, n, *valid_bicrs[k])
            corr_names.append([cname for cname, _, _ in cs])
            out_lines.append(str(len(cs)))
            for _, inc, jump in cs:
                out_lines += [f"{len(inc)} {len(jump)}", " ".join(map(str, inc)), " ".join(map(str, jump))]
            k += 1
        out = run("\n".join(out_lines) + "\n").splitlines()

    def parse(block):
        d = {"col_inc": list(map(int, block[0].split()[1:])), "row_jump": list(map(int, block[1].split()[1:]))}
        if block[2].startswith("err"):
            d["error"] = KINDS[int(block[2].split()[1])]
            return d, 6
        d["y_bits"] = block[2].split()[1:]
        st = block[3].split()
        d["stats"] = [int(st[1]), int(st[2])]
        d["rows"] = list(map(int, block[4].split()[1:]))
        d["cols"] = list(map(int, block[5].split()[1:]))
        return d, 6

    res, pos = [], 0
    for i, (name, m, n, r, c, v, x, on) in enumerate(plan):
        entry = {"name": name, "m": m, "n": n, "rows": r, "cols": c, "vals": v, "x": x}
        entry["icrs"], used = parse(out[pos:pos + 7])
        pos += used
        entry["bicrs"] = {}
        for oname in on:
            d, used = parse(out[pos:pos + 7])
            pos += used
            d["order"] = orders(name, len(v), r, c)[oname]
            entry["bicrs"][oname] = d
        entry["corrupt"] = {}
        for cname in corr_names[i]:
            d, used = parse(out[pos:pos + 7])
            pos += used
            entry["corrupt"][cname] = d
        res.append(entry)
    json.dump(res, open(os.path.join(HERE, "bicrs_golden.json"), "w"))
    print("wrote bicrs_golden.json:", [(e["name"], len(e["bicrs"]), {k: v.get("error") for k, v in e["corrupt"].items()})
                                       for e in res])


if __name__ == "__main__":
    main()
