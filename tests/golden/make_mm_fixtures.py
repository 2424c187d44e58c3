"""Writes tests/golden/mm/*.mtx (Matrix Market cases written for this repo: valid files of every
field / symmetry combination plus edge syntax, and malformed files for every documented error
kind) and tests/golden/mm/expected.json with the result of the REFERENCE parser
(read_matrix_market, inc/matrix_market.hpp:94-190, compiled here from /root/reference) on each:
either the entries in order or the ErrorKind name.

Run in the development container:  python tests/golden/make_mm_fixtures.py
"""
import json
import os
import subprocess
import tempfile

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "mm")
REF = "/root/reference/proj/include"

CASES = {
    # ---- valid
    "gen_real": "%%MatrixMarket matrix coordinate real general\n3 4 4\n1 1 2.5\n3 4 -1e-3\n2 2 7\n1 3 0.125\n",
    "gen_integer": "%%MatrixMarket matrix coordinate integer general\n2 2 3\n1 2 5\n2 1 -3\n2 2 12\n",
    "gen_pattern": "%%MatrixMarket matrix coordinate pattern general\n4 3 3\n4 3\n1 1\n2 3\n",
    "sym_real": "%%MatrixMarket matrix coordinate real symmetric\n4 4 4\n1 1 1.0\n3 1 2.0\n4 2 -0.5\n4 4 3\n",
    "sym_integer": "%%MatrixMarket matrix coordinate integer symmetric\n3 3 2\n2 1 4\n3 3 9\n",
    "sym_pattern": "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 3\n1 1\n3 2\n2 1\n",
    "comments_blank_crlf": "%%MatrixMarket matrix coordinate real general\r\n% a comment\r\n\r\n   % indented\r\n"
                           "\t \r\n2 2 2\r\n% between\r\n1 1 1.5\r\n\r\n2 2 -2.5\r\n% trailing comment\r\n\r\n",
    "banner_case_tabs": "%%MatrixMarket\tMATRIX  Coordinate   REAL\tGeneral\n2 3 2\n1 3\t4e2\n  2   1   -0\n",
    "no_final_newline": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 2 1\n2 1 2",
    "empty_matrix": "%%MatrixMarket matrix coordinate real general\n5 7 0\n",
    "zero_by_zero": "%%MatrixMarket matrix coordinate pattern general\n0 0 0\n",
    "single_entry": "%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 3.14159\n",
    "rectangular": "%%MatrixMarket matrix coordinate real general\n2 6 3\n1 6 1\n2 1 2\n2 5 3\n",
    "numbers": "%%MatrixMarket matrix coordinate real general\n6 1 6\n1 1 +1.5\n2 1 1E+300\n3 1 4.9e-324\n"
               "4 1 0x1.8p1\n5 1 -0.0\n6 1 .5\n",
    "dense_3x3": "%%MatrixMarket matrix coordinate real general\n3 3 9\n" +
                 "".join(f"{i} {j} {i * 10 + j}\n" for i in range(1, 4) for j in range(1, 4)),
    "leading_zeros": "%%MatrixMarket matrix coordinate real general\n003 003 002\n01 02 1\n003 1 2\n",
    # ---- malformed
    "bad_banner_prefix": "%MatrixMarket matrix coordinate real general\n1 1 0\n",
    "bad_banner_fields": "%%MatrixMarket matrix coordinate real\n1 1 0\n",
    "bad_object": "%%MatrixMarket vector coordinate real general\n1 1 0\n",
    "bad_format_word": "%%MatrixMarket matrix sparse real general\n1 1 0\n",
    "array_format": "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "complex_field": "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "hermitian": "%%MatrixMarket matrix coordinate real hermitian\n1 1 0\n",
    "skew_symmetric": "%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n2 1 1\n",
    "empty_file": "",
    "missing_size": "%%MatrixMarket matrix coordinate real general\n% only comments\n\n",
    "size_two_fields": "%%MatrixMarket matrix coordinate real general\n2 2\n",
    "size_signed": "%%MatrixMarket matrix coordinate real general\n+2 2 1\n1 1 1\n",
    "size_junk": "%%MatrixMarket matrix coordinate real general\n2x 2 1\n1 1 1\n",
    "dim_overflow": "%%MatrixMarket matrix coordinate real general\n2147483649 2 0\n",
    "dim_max_ok": "%%MatrixMarket matrix coordinate pattern general\n2147483648 1 1\n2147483648 1\n",
    "truncated": "%%MatrixMarket matrix coordinate real general\n3 3 3\n1 1 1\n2 2 2\n",
    "extra_entries": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1\n2 2 2\n",
    "wrong_field_count": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n",
    "pattern_with_value": "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 1 5\n",
    "bad_value": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.5x\n",
    "bad_index": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1.0 1 1\n",
    "zero_index": "%%MatrixMarket matrix coordinate real general\n2 2 1\n0 1 1\n",
    "row_out_of_range": "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n",
    "col_out_of_range": "%%MatrixMarket matrix coordinate integer general\n2 2 1\n1 3 1\n",
    "duplicate": "%%MatrixMarket matrix coordinate real general\n3 3 3\n1 2 1\n3 3 1\n1 2 5\n",
    "symmetric_duplicate": "%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n2 1 1\n1 2 1\n",
}

DRIVER = r"""
#include <cstdio>
#include <fstream>
#include <spmvlab/io.hpp>
int main(int argc, char** argv) {
  for (int a = 1; a < argc; ++a) {
    std::ifstream in(argv[a], std::ios::binary);
    try {
      spmvlab::MatrixHeader h;
      auto t = spmvlab::read_matrix_market(in, &h);
      std::printf("OK %u %u %d %d %u %zu\n", t.m, t.n, (int)h.field, (int)h.symmetry, h.declared_nnz, t.data.size());
      for (size_t k = 0; k < t.data.size(); ++k) {
        unsigned long long bits; std::memcpy(&bits, &t.data[k], 8);
        std::printf("%u %u %016llx\n", t.row_ind[k], t.col_ind[k], bits);
      }
    } catch (const spmvlab::Error& e) {
      std::printf("ERR %d\n", (int)e.kind());
    }
  }
}
"""
KINDS = ["DimensionMismatch", "InvalidArgument", "CorruptFormat", "Overflow", "BadHeader", "UnsupportedFormat",
         "UnsupportedField", "UnsupportedSymmetry", "IndexOutOfRange", "DuplicateEntry", "ParseError", "Truncated",
         "BadMagic", "IoError"]


def main():
    os.makedirs(HERE, exist_ok=True)
    names = sorted(CASES)
    for nm in names:
        with open(os.path.join(HERE, nm + ".mtx"), "w", newline="") as f:
            f.write(CASES[nm])
    with tempfile.TemporaryDirectory() as td:
        src, exe = os.path.join(td, "d.cpp"), os.path.join(td, "d")
        open(src, "w").write("#include <cstring>\n" + DRIVER)
        subprocess.check_call(["g++", "-std=c++20", "-O1", "-I" + REF, src, "-o", exe])
        out = subprocess.check_output([exe] + [os.path.join(HERE, nm + ".mtx") for nm in names]).decode().splitlines()
    exp, i = {}, 0
    for nm in names:
        head = out[i].split()
        i += 1
        if head[0] == "ERR":
            exp[nm] = {"error": KINDS[int(head[1])]}
            continue
        m, n, field, sym, decl, k = map(int, head[1:])
        ents = [out[i + q].split() for q in range(k)]
        i += k
        exp[nm] = {"m": m, "n": n, "field": ["real", "integer", "pattern"][field],
                   "symmetry": ["general", "symmetric"][sym], "declared_nnz": decl,
                   "rows": [int(e[0]) for e in ents], "cols": [int(e[1]) for e in ents],
                   "value_bits": [e[2] for e in ents]}
    json.dump(exp, open(os.path.join(HERE, "expected.json"), "w"), indent=0, sort_keys=True)
    print(f"wrote {len(names)} fixtures;",
          sum(1 for v in exp.values() if "error" in v), "error cases")


if __name__ == "__main__":
    main()
