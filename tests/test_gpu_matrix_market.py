"""Device Matrix Market ingest (parse + device validate) and the load_matrix format sniffing
(inc/io.hpp:29-40) against the reference parser's results (tests/golden/mm/expected.json)."""
import json
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

DIR = os.path.join(os.path.dirname(__file__), "golden", "mm")
EXPECTED = json.load(open(os.path.join(DIR, "expected.json")))


@pytest.mark.parametrize("name", sorted(EXPECTED))
def test_device_reader_matches_reference(cuda, name):
    sp = cuda
    exp = EXPECTED[name]
    path = os.path.join(DIR, name + ".mtx")
    if "error" in exp:
        with pytest.raises(sp.Error) as e:
            sp.read_matrix_market(path)
        assert e.value.kind == sp.ErrorKind[exp["error"]], (name, str(e.value))
        with pytest.raises(sp.Error):
            sp.load_matrix(path)
        return
    a, h = sp.read_matrix_market(path, with_header=True)
    assert (a.m, a.n, h.field, h.symmetry) == (exp["m"], exp["n"], exp["field"], exp["symmetry"])
    assert a.row_ind.cpu().numpy().view(np.uint32).tolist() == exp["rows"]
    assert a.col_ind.cpu().numpy().view(np.uint32).tolist() == exp["cols"]
    assert [f"{b:016x}" for b in a.data.cpu().numpy().view(np.uint64).tolist()] == exp["value_bits"]
    b = sp.load_matrix(path)
    assert torch.equal(a.row_ind, b.row_ind) and torch.equal(a.data, b.data)


def test_load_matrix_sniffs_cache(cuda, tmp_path):
    """tests/test_matrix_io.cpp:191-200: a cache file and a text file of the same matrix load alike."""
    sp = cuda
    a = sp.read_matrix_market(os.path.join(DIR, "sym_real.mtx"))
    p = tmp_path / "m.spmvlab1"
    sp.cache_write(str(p), a)
    b = sp.load_matrix(str(p))
    assert (b.m, b.n) == (a.m, a.n)
    assert torch.equal(a.row_ind, b.row_ind) and torch.equal(a.col_ind, b.col_ind) and torch.equal(a.data, b.data)
    # and it multiplies: y = A * 1 by every engine equals the row sums
    f = sp.build_format(2, b, 1)
    y = sp.run_spmv(2, f, torch.ones(b.n, dtype=torch.float64, device="cuda"), p=1)
    want = torch.zeros(b.m, dtype=torch.float64, device="cuda").index_add_(0, b.row_ind.long(), b.data)
    assert torch.equal(y, want)
