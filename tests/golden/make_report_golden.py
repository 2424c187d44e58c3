"""Generates tests/golden/report_golden.json: the reference's own report emitters
(emit_csv / emit_markdown, inc/bench.hpp:367-554, and detail::format_double = std::to_chars) run on
a fixed set of BenchRecords, compiled here straight from /root/reference/proj/include.

Run in the development container (needs g++ and /root/reference):
    python tests/golden/make_report_golden.py
"""
import json
import os
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/proj/include"

# (matrix, algorithm ordinal, threads, min_time, speedup, convert_time | None, convert_ratio | None,
#  density, status)
RECORDS = [
    ("rmat_s22", 0, 1, 0.0121473, 1.0, None, None, 3.7e-06, "ok"),
    ("rmat_s22", 2, 8, 0.000327812, 37.05567, 0.01056, 32.2, 3.7e-06, "ok"),
    ("rmat_s22", 2, 16, 0.000301, 40.3565, 0.0104, 31.5, 3.7e-06, "ok"),
    ("rmat_s22", 3, 8, 0.0006374, 19.0576, 0.01011, 30.83, 3.7e-06, "ok"),
    ("rmat_s22", 9, 8, 0.0003349, 37.05567, 0.00957, 29.18, 3.7e-06, "ok"),
    ("rmat_s22", 7, 8, 0.0, 0.0, None, None, 3.7e-06, "verify failed at element 17"),
    ("er_65536, tiny", 0, 1, 3.24e-05, 1.0, None, None, 0.000244, "ok"),
    ("er_65536, tiny", 1, 4, 1.99e-05, 1.628140703517588, 0.00455, 228.6, 0.000244, "ok"),
    ("er_65536, tiny", 4, 4, 4.27e-05, 0.7587822014051522, 0.00673, 338.1, 0.000244, "ok"),
    ("lap\nperm", 5, 2, 1e-07, 123456789.0, 1e16, 1e-05, 2.98e-07, "ok"),
]
DOUBLES = [0.0, 1.0, 100.0, 0.1, 1e-05, 1e-07, 123456.0, 1234567.0, 1e16, 1.5e16, 1e22, 2.5e-10,
           0.000327812, 3.7e-06, 37.05567, 1.0 / 3.0, 2.0 / 3.0 * 1e-300, 6.02214076e23, 1e100, 5e-324,
           1.7976931348623157e308, 12345678901234567.0, 0.001, 0.0001, 9.999999999999999e-05]


def _cxx_double(v):
    return repr(float(v))


def main():
    lines = ["#include <cstdio>", "#include <spmvlab/bench.hpp>", "using namespace spmvlab;", "int main() {",
             "  std::vector<BenchRecord> rs;"]
    for (mat, alg, th, mt, sp, ct, cr, de, st) in RECORDS:
        lines.append("  { BenchRecord r; r.matrix = " + json.dumps(mat) + f"; r.algorithm = static_cast<Algorithm>({alg});"
                     f" r.threads = {th}; r.min_time = {_cxx_double(mt)}; r.speedup = {_cxx_double(sp)};"
                     + (f" r.convert_time = {_cxx_double(ct)};" if ct is not None else "")
                     + (f" r.convert_ratio = {_cxx_double(cr)};" if cr is not None else "")
                     + f" r.density = {_cxx_double(de)}; r.status = " + json.dumps(st) + "; rs.push_back(r); }")
    lines += ['  std::string csv = emit_csv(rs), md = emit_markdown(rs);',
              '  std::printf("%zu\\n", csv.size()); std::fwrite(csv.data(), 1, csv.size(), stdout);',
              '  std::printf("%zu\\n", md.size()); std::fwrite(md.data(), 1, md.size(), stdout);']
    for d in DOUBLES:
        lines.append(f'  std::printf("%s\\n", detail::format_double({_cxx_double(d)}).c_str());')
    lines += ["  return 0;", "}"]
    with tempfile.TemporaryDirectory() as td:
        src = os.path.join(td, "g.cpp")
        exe = os.path.join(td, "g")
        open(src, "w").write("\n".join(lines) + "\n")
        subprocess.check_call(["g++", "-std=c++20", "-O1", "-I" + REF, src, "-o", exe])
        out = subprocess.check_output([exe])
    pos = 0

    def take_block():
        nonlocal pos
        nl = out.index(b"\n", pos)
        size = int(out[pos:nl])
        blk = out[nl + 1:nl + 1 + size].decode()
        pos = nl + 1 + size
        return blk

    csv = take_block()
    md = take_block()
    doubles = out[pos:].decode().splitlines()
    json.dump({"records": RECORDS, "csv": csv, "markdown": md,
               "doubles": [[repr(d), s] for d, s in zip(DOUBLES, doubles)]},
              open(os.path.join(HERE, "report_golden.json"), "w"), indent=1)
    print("wrote report_golden.json")


if __name__ == "__main__":
    main()
