"""Writes the SPMVLAB1 cache fixtures of tests/golden/cache/ with the REFERENCE's own cache_write
(oracle/_ref, inc/cache_io.hpp:58-66), plus malformed variants, and records the reference's
cache_read outcome (inc/cache_io.hpp:69-91) for each in expected.json.

    make -C oracle && python tests/golden/make_cache_fixtures.py
"""
import json
import os
import struct
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from matrices import e4, random_matrix  # noqa: E402
from oracle.oracle import CheckerError, Reference  # noqa: E402

OUT = os.path.join(HERE, "cache")


def main():
    os.makedirs(OUT, exist_ok=True)
    ref = Reference()
    files = {}
    m, n, r, c, v = e4()
    ref.cache_write(os.path.join(OUT, "e4.spmvlab1"), m, n, r, c, v)
    m, n, r, c, v = random_matrix(300, 200, 0.03, seed=8, dense_row_nnz=200, signed=True)
    ref.cache_write(os.path.join(OUT, "rand.spmvlab1"), m, n, r, c, v)
    ref.cache_write(os.path.join(OUT, "empty.spmvlab1"), 7, 3, np.zeros(0, np.uint32), np.zeros(0, np.uint32),
                    np.zeros(0))
    good = open(os.path.join(OUT, "rand.spmvlab1"), "rb").read()
    open(os.path.join(OUT, "bad_magic.spmvlab1"), "wb").write(b"SPMVLAB2" + good[8:])
    open(os.path.join(OUT, "truncated_body.spmvlab1"), "wb").write(good[:-13])
    open(os.path.join(OUT, "truncated_header.spmvlab1"), "wb").write(good[:20])
    hdr = lambda mm, nn, k: b"SPMVLAB1" + struct.pack("<QQQ", mm, nn, k)
    body = lambda rows, cols, vals: (b"".join(struct.pack("<Q", x) for x in rows) +
                                     b"".join(struct.pack("<Q", x) for x in cols) +
                                     b"".join(struct.pack("<d", x) for x in vals))
    open(os.path.join(OUT, "duplicate.spmvlab1"), "wb").write(hdr(4, 4, 3) + body([1, 2, 1], [3, 0, 3], [1.0, 2.0, 3.0]))
    open(os.path.join(OUT, "out_of_range.spmvlab1"), "wb").write(hdr(4, 4, 2) + body([1, 4], [0, 0], [1.0, 2.0]))
    open(os.path.join(OUT, "overflow_dim.spmvlab1"), "wb").write(hdr((1 << 31) + 1, 4, 0))
    # an index >= 2^32 is narrowed by static_cast<index_t> before validate (cache_io.hpp:86)
    open(os.path.join(OUT, "wide_index.spmvlab1"), "wb").write(hdr(4, 4, 1) + body([(1 << 32) + 2], [1], [5.0]))
    for name in sorted(os.listdir(OUT)):
        if not name.endswith(".spmvlab1"):
            continue
        try:
            mm, nn, rr, cc, vv = ref.cache_read(os.path.join(OUT, name))
            files[name] = {"code": 0, "m": mm, "n": nn, "nnz": len(vv)}
        except CheckerError as ex:
            files[name] = {"code": ex.code}
    json.dump(files, open(os.path.join(OUT, "expected.json"), "w"), indent=1, sort_keys=True)
    print(json.dumps(files, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
