"""GPU parity of the iterated multiply (spmvlab_cuda_iterate): the cfg5 application loop
x <- A x on a column-normalised R-MAT with non-negative x0 (SURVEY.md §8e parity rule: compare the
iterates with the CPU oracle loop at iterations 1, 2 and 100), plus the per-iteration norms, the
unit-mass rescaling and the CUDA-graph form of the loop."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _matrix(scale=12):
    from paper_2502_19284_b200 import gen
    return gen.rmat_host(scale, 8, seed=21, normalize_columns=True)


def _oracle_loop(oracle, m, n, r, c, v, x0, iters, normalize=False):
    ref = oracle.build(0, m, n, r, c, v)
    xs, norms = [x0.copy()], []
    x = x0.copy()
    for _ in range(iters):
        y = oracle.spmv(ref, 0, x)
        mass = y.sum()
        res = np.abs(y - x).sum()  # residual ||A x_k - x_k||_1, before any rescale
        if normalize:
            y = y / mass
        norms.append((res, mass))
        xs.append(y.copy())
        x = y
    return xs, np.array(norms)


@pytest.mark.parametrize("graph", [False, True])
def test_seq_crs_iterates_bitwise(cuda, oracle, graph):
    """SeqCrs sums rows in the reference order, so every iterate is BITWISE the oracle's."""
    sp = cuda
    m, n, r, c, v = _matrix()
    x0 = np.random.default_rng(2).uniform(0.0, 1.0, n) + 1e-3
    xs, _ = _oracle_loop(oracle, m, n, r, c, v, x0, 100)
    f = sp.build_format(0, sp.TripletMatrix.from_host(m, n, r, c, v), 1)
    for k in (1, 2, 100):
        x = torch.from_numpy(x0).cuda()
        sp.iterate(0, f, x, k, graph=graph, norms=False)
        np.testing.assert_array_equal(x.cpu().numpy(), xs[k], err_msg=f"iteration {k}")


@pytest.mark.parametrize("alg", [2, 1, 3, 9, 6])
def test_engine_iterates_within_tolerance(cuda, oracle, alg):
    """Other engines: non-negative A and x, so sum|a x| = y and the normalised error bound is a
    per-entry relative bound; 1e-12 per iteration, accumulated over 100 iterations."""
    sp = cuda
    m, n, r, c, v = _matrix()
    x0 = np.random.default_rng(3).uniform(0.0, 1.0, n) + 1e-3
    xs, want = _oracle_loop(oracle, m, n, r, c, v, x0, 100)
    p = 4
    f = sp.build_format(alg, sp.TripletMatrix.from_host(m, n, r, c, v), p)
    for k in (1, 2, 100):
        x = torch.from_numpy(x0).cuda()
        _, nb = sp.iterate(alg, f, x, k, p=p)
        got = x.cpu().numpy()
        ok = np.abs(got - xs[k]) <= 1e-12 * k * np.abs(xs[k]) + 1e-300
        assert ok.all(), f"alg {alg} iteration {k}: max rel {np.max(np.abs(got - xs[k]) / np.maximum(xs[k], 1e-300))}"
        nb = nb.cpu().numpy()
        np.testing.assert_allclose(nb[:, 1], want[:k, 1], rtol=1e-11 * k)
        np.testing.assert_allclose(nb[:, 0], want[:k, 0], rtol=1e-9, atol=1e-12 * want[:k, 1].max())


def test_norms_and_leakage(cuda, oracle):
    """norms[k] = (||A x_k - x_k||_1, mass of A x_k); with empty columns the mass leaks, so it is
    non-increasing for a column-(sub)stochastic matrix."""
    sp = cuda
    m, n, r, c, v = _matrix()
    assert len(np.unique(c)) < n, "the test matrix should have empty columns"
    x0 = np.full(n, 1.0 / n)
    xs, want = _oracle_loop(oracle, m, n, r, c, v, x0, 20)
    f = sp.build_format(0, sp.TripletMatrix.from_host(m, n, r, c, v), 1)
    x = torch.from_numpy(x0).cuda()
    _, nb = sp.iterate(0, f, x, 20)
    nb = nb.cpu().numpy()
    np.testing.assert_allclose(nb, want, rtol=1e-12, atol=1e-18)
    assert np.all(np.diff(nb[:, 1]) <= 1e-14)


@pytest.mark.parametrize("graph", [False, True])
def test_normalized_iteration(cuda, oracle, graph):
    sp = cuda
    m, n, r, c, v = _matrix()
    x0 = np.random.default_rng(4).uniform(0.0, 1.0, n)
    x0 /= x0.sum()
    xs, want = _oracle_loop(oracle, m, n, r, c, v, x0, 30, normalize=True)
    f = sp.build_format(2, sp.TripletMatrix.from_host(m, n, r, c, v), 1)
    x = torch.from_numpy(x0).cuda()
    _, nb = sp.iterate(2, f, x, 30, normalize=True, graph=graph)
    got = x.cpu().numpy()
    np.testing.assert_allclose(got, xs[30], rtol=1e-10, atol=1e-300)
    assert abs(got.sum() - 1.0) < 1e-12
    np.testing.assert_allclose(nb.cpu().numpy()[:, 1], want[:, 1], rtol=1e-10)
    np.testing.assert_allclose(nb.cpu().numpy()[:, 0], want[:, 0], rtol=1e-9)


@pytest.mark.parametrize("panels", [1, 3])
@pytest.mark.parametrize("normalize", [False, True])
def test_loop_norms_with_column_panels(cuda, oracle, monkeypatch, panels, normalize):
    """The loop's one pass per iteration (deferred scale: the stored vector is A x_k, x_{k+1} =
    stored / mass_k) against the oracle loop, on a merge format with and without column panels."""
    sp = cuda
    m, n, r, c, v = _matrix(13)
    x0 = np.random.default_rng(6).uniform(0.0, 1.0, n) + 1e-3
    if normalize:
        x0 /= x0.sum()
    xs, want = _oracle_loop(oracle, m, n, r, c, v, x0, 12, normalize=normalize)
    monkeypatch.setenv("SPMVLAB_MERGE_PANELS", str(panels))
    f = sp.build_format(2, sp.TripletMatrix.from_host(m, n, r, c, v), 1)
    monkeypatch.delenv("SPMVLAB_MERGE_PANELS")
    assert f.info["merge_panels"] == panels
    for graph in (False, True):
        x = torch.from_numpy(x0).cuda()
        _, nb = sp.iterate(2, f, x, 12, normalize=normalize, graph=graph)
        got, nb = x.cpu().numpy(), nb.cpu().numpy()
        np.testing.assert_allclose(got, xs[12], rtol=2e-11, atol=1e-300)
        np.testing.assert_allclose(nb[:, 1], want[:, 1], rtol=1e-11)
        np.testing.assert_allclose(nb[:, 0], want[:, 0], rtol=1e-9)
        if normalize:
            assert abs(got.sum() - 1.0) < 1e-12


def test_graph_equals_stream_loop(cuda):
    """The captured graph runs the same kernels in the same order: bitwise equal results for the
    deterministic CRS engines (the blocked engines add into y with atomics, so their summation
    order -- not their accuracy -- varies from run to run)."""
    sp = cuda
    m, n, r, c, v = _matrix(13)
    x0 = torch.rand(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
    for alg in (0, 1, 2, 4, 7):
        f = sp.build_format(alg, sp.TripletMatrix.from_host(m, n, r, c, v), 2)
        a, na = sp.iterate(alg, f, x0.clone(), 7, p=2)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            b, nbb = sp.iterate(alg, f, x0.clone(), 7, p=2, graph=True, stream=s)
        s.synchronize()
        if alg <= 2:
            assert torch.equal(a, b) and torch.equal(na, nbb), alg
        else:
            torch.testing.assert_close(a, b, rtol=1e-12, atol=0)
            torch.testing.assert_close(na, nbb, rtol=1e-10, atol=0)


def test_iterate_errors(cuda):
    sp = cuda
    r = np.array([0, 1], dtype=np.uint32)
    c = np.array([0, 2], dtype=np.uint32)
    v = np.array([1.0, 2.0])
    f = sp.build_format(2, sp.TripletMatrix.from_host(2, 3, r, c, v), 1)
    with pytest.raises(sp.Error) as e:
        sp.iterate(2, f, torch.ones(3, dtype=torch.float64, device="cuda"), 2)
    assert e.value.kind == sp.ErrorKind.DimensionMismatch
