"""The library's Matrix Market reader (host variant, no CUDA calls) against the REFERENCE parser's
results on the fixture set (tests/golden/mm, expected.json from tests/golden/make_mm_fixtures.py):
the same entries in the same order with bit-identical values, the same header, or the same
ErrorKind (models tests/test_matrix_io.cpp:55-126)."""
import json
import os

import numpy as np
import pytest

DIR = os.path.join(os.path.dirname(__file__), "golden", "mm")
EXPECTED = json.load(open(os.path.join(DIR, "expected.json")))


@pytest.mark.parametrize("name", sorted(EXPECTED))
def test_host_reader_matches_reference(name):
    from paper_2502_19284_b200 import engine as E
    exp = EXPECTED[name]
    path = os.path.join(DIR, name + ".mtx")
    if "error" in exp:
        with pytest.raises(E.Error) as e:
            E.read_matrix_market_host(path)
        assert e.value.kind == E.ErrorKind[exp["error"]], (name, str(e.value))
        return
    m, n, r, c, v, h = E.read_matrix_market_host(path)
    assert (m, n) == (exp["m"], exp["n"])
    assert (h.field, h.symmetry, h.declared_nnz) == (exp["field"], exp["symmetry"], exp["declared_nnz"])
    assert r.tolist() == exp["rows"] and c.tolist() == exp["cols"]
    assert [f"{b:016x}" for b in v.view(np.uint64).tolist()] == exp["value_bits"]


def test_missing_file_is_io_error():
    from paper_2502_19284_b200 import engine as E
    with pytest.raises(E.Error) as e:
        E.read_matrix_market_host(os.path.join(DIR, "does_not_exist.mtx"))
    assert e.value.kind == E.ErrorKind.IoError
