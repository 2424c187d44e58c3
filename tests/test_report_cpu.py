"""The report emitters (paper_2502_19284_b200/report.py) against the reference's own emit_csv,
emit_markdown and std::to_chars output for the same records (tests/golden/report_golden.json,
made by tests/golden/make_report_golden.py from inc/bench.hpp), plus CSV round trips."""
import json
import math
import os

import pytest

from paper_2502_19284_b200 import engine as E
from paper_2502_19284_b200 import report as R

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "report_golden.json")))


def _records():
    return [R.BenchRecord(m, a, t, mt, sp, ct, cr, de, st) for (m, a, t, mt, sp, ct, cr, de, st) in GOLD["records"]]


def test_format_double_matches_to_chars():
    for val, want in GOLD["doubles"]:
        assert R.format_double(float(val)) == want, val


def test_emit_csv_matches_reference():
    assert R.emit_csv(_records()) == GOLD["csv"]


def test_emit_markdown_matches_reference():
    assert R.emit_markdown(_records()) == GOLD["markdown"]


def test_csv_round_trip_plain_and_extended():
    recs = _records()
    back = R.parse_csv(R.emit_csv(recs))
    for a, b in zip(recs, back):
        assert (R._sanitize(a.matrix), a.algorithm, a.threads, a.min_time, a.speedup, a.convert_time,
                a.convert_ratio, a.density) == (b.matrix, b.algorithm, b.threads, b.min_time, b.speedup,
                                                b.convert_time, b.convert_ratio, b.density)
    recs[1].gbs, recs[1].roofline_frac, recs[1].break_even = 2643.9, 0.41047, 1234.5
    ext = R.emit_csv(recs, extended=True)
    assert ext.splitlines()[0] == R.CSV_EXT_HEADER
    back = R.parse_csv(ext)
    assert (back[1].gbs, back[1].roofline_frac, back[1].break_even) == (2643.9, 0.41047, 1234.5)
    assert back[0].gbs is None


def test_parse_errors():
    with pytest.raises(E.Error) as e:
        R.parse_csv("")
    assert e.value.kind == E.ErrorKind.ParseError
    with pytest.raises(E.Error):
        R.parse_csv("bad,header\n")
    with pytest.raises(E.Error):
        R.parse_csv(R.CSV_HEADER + "\nm,crs,1,0.1,1\n")
    with pytest.raises(E.Error):
        R.parse_csv(R.CSV_HEADER + "\nm,crs,1,zz,1,,,0.1,ok\n")
    with pytest.raises(E.Error):
        R.emit_report([])


def test_markdown_gpu_grids():
    recs = _records()
    for r in recs:
        if r.min_time > 0:
            r.gbs, r.roofline_frac = 1000.0 * r.speedup, 0.1
    recs[3].break_even = 42.0
    md = R.emit_markdown(recs, gpu_columns=True)
    assert md.startswith(GOLD["markdown"].split("\n## ")[0])
    assert "Effective bandwidth" in md and "Break-even multiplies" in md and "| 42.0 |" in md


def test_format_double_random_round_trip():
    import random
    rnd = random.Random(3)
    for _ in range(2000):
        v = rnd.choice([rnd.random(), rnd.uniform(-1e6, 1e6), 10 ** rnd.uniform(-300, 300), float(rnd.randint(0, 10**12))])
        s = R.format_double(v)
        assert float(s) == v and (math.isinf(v) or "e" in s or "." in s or s.lstrip("-").isdigit())
