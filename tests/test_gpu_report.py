"""The device benchmark harness (report.bench_all) on a small matrix: every engine verifies and
times, records carry the GPU columns, and the CSV round-trips."""
import pytest

pytestmark = pytest.mark.gpu


def test_bench_all_small(cuda):
    sp = cuda
    from paper_2502_19284_b200 import gen, report
    m, n, r, c, v = gen.rmat_host(12, 8, seed=3)
    a = sp.TripletMatrix.from_host(m, n, r, c, v)
    recs = report.bench_all(a, "rmat12", report.BenchConfig(threads=[2, 4], spmv_reps=5, convert_reps=1,
                                                            peak_gbs=6441.0))
    assert len(recs) == 11 * 2
    assert [(x.algorithm, x.threads) for x in recs] == sorted((x.algorithm, x.threads) for x in recs)
    for x in recs:
        assert x.status == "ok", (x.algorithm, x.status)
        assert x.min_time > 0 and x.gbs > 0 and 0 < x.roofline_frac < 2
        assert x.convert_time > 0 and x.convert_ratio > 0
    seq = [x for x in recs if x.algorithm == 0]
    assert all(abs(x.speedup - seq[0].speedup) < 1e9 for x in seq)
    back = report.parse_csv(report.emit_csv(recs, extended=True))
    assert [(b.algorithm, b.threads, b.min_time, b.gbs) for b in back] == \
        [(x.algorithm, x.threads, x.min_time, x.gbs) for x in recs]
    md = report.emit_markdown(recs, gpu_columns=True)
    assert "Effective bandwidth" in md
