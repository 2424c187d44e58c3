"""CPU checks of the drop-in boundary: the C-ABI library loads and exports every symbol that
include/spmvlab_cuda.h declares; host-side entry points (no GPU needed) match the oracle; the C++
drop-in header compiles; the package has no CPU fallback path."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "spmvlab_cuda.h")


def declared_functions():
    src = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|unsigned|uint64_t|const char\*)\s+(spmvlab_cuda_\w+)\(",
                                 src, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2502_19284_b200 import capi
    lib = C.CDLL(capi.lib_path())
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), f"{n} declared in spmvlab_cuda.h but not exported"
    assert set(names) == set(capi.EXPORTS)
    assert lib.spmvlab_cuda_abi_version() == 3


def test_library_is_sm100a():
    from paper_2502_19284_b200 import capi
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", capi.lib_path()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_entry_points_match_oracle(oracle):
    import paper_2502_19284_b200 as sp
    for n in (1, 4, 1000, 65536, 4194304, 1 << 31):
        for cap in (15, 16):
            for l2 in (64, 4096, 512 * 1024, 1 << 40):
                assert sp.select_block_size(n, cap, l2) == oracle.select_block_size(n, cap, l2)
    rng = np.random.default_rng(1)
    for _ in range(50):
        m = int(rng.integers(1, 300))
        prefix = np.concatenate([[0], np.cumsum(rng.integers(0, 30, m))]).astype(np.uint32)
        p, lb = int(rng.integers(1, 10)), int(rng.integers(0, 5))
        np.testing.assert_array_equal(sp.partition_rows_by_nnz(prefix, p, lb),
                                      oracle.partition_rows_by_nnz(prefix, p, lb))


def test_cpp_header_compiles(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text('#include "spmvlab_cuda/engine.hpp"\nint main(){return 0;}\n')
    r = subprocess.run(["g++", "-std=c++17", "-fsyntax-only", f"-I{ROOT}/include", "-I/usr/local/cuda/include",
                        str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_no_cpu_fallback_in_product():
    """The product package must not import or call the oracle (the checker)."""
    pkg = os.path.join(ROOT, "paper_2502_19284_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".hpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in txt.replace("Oracle", "").lower().replace("oracles.hpp", ""), f


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    from paper_2502_19284_b200 import capi
    monkeypatch.setattr(capi, "LIB", str(tmp_path / "nope.so"))
    monkeypatch.setattr(capi, "_lib", None)
    with pytest.raises(RuntimeError):
        capi.load()
