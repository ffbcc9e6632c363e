"""The CETC-DM communication-volume model (dmsim.py:203-336).

Pinned by tests/golden/comm_cases.json, produced by the reference's own
comm_volume_* / comm_report / reports_to_csv / fit_scaling / format_volume
(tests/golden/make_comm_golden.py).  CPU tests evaluate the model on the
fixtures' reference labelings; the GPU test builds every report from the
device labeling and count.
"""
from __future__ import annotations

import json
import math
from pathlib import Path
from types import SimpleNamespace

import pytest

from conftest import SMALL_CASES
from paper_2403_02997_b200 import dm

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "comm_cases.json").read_text())
CASES = {c.name: c for c in SMALL_CASES}
NAMES = sorted(GOLD["graphs"])


def _graph_and_labeling(c):
    g = SimpleNamespace(n=c.n, m=c.m, row_offsets=c.row)
    lab = SimpleNamespace(level=c.level, max_level=c.max_level, horizontal_count=len(c.cover))
    return g, lab


def _report_dict(r):
    d = dict(vars(r)) if not hasattr(r, "__dataclass_fields__") else \
        {k: getattr(r, k) for k in r.__dataclass_fields__}
    if d["reduction"] == float("inf"):
        d["reduction"] = "inf"
    return d


@pytest.mark.parametrize("name", NAMES)
def test_volumes_match_reference(name):
    c = CASES[name]
    g, lab = _graph_and_labeling(c)
    for p, want in GOLD["graphs"][name].items():
        p = int(p)
        assert dm.comm_volume_previous(g, p) == want["previous"]
        assert list(dm.comm_volume_breakdown(g, lab, p)) == want["breakdown"]
        assert dm.comm_volume_cetc_dm(g, lab, p) == want["total"]
        rep = want["report"]
        assert dm.wedge_count(g) == rep["wedges"]
        assert rep["triangles"] == c.T


def test_labeling_mismatch_raises():
    c = CASES[NAMES[0]]
    g, lab = _graph_and_labeling(c)
    lab.level = lab.level[:-1]
    with pytest.raises(ValueError):
        dm.comm_volume_cetc_dm(g, lab, 2)


def test_csv_matches_reference():
    rows = []
    for name in [c.name for c in SMALL_CASES]:
        per_p = GOLD["graphs"][name]
        for p in sorted(per_p, key=int):
            r = dict(per_p[p]["report"])
            if r["reduction"] == "inf":
                r["reduction"] = float("inf")
            rows.append(dm.CommReport(**r))
    assert dm.reports_to_csv(rows) == GOLD["csv"]


def test_format_volume_and_ceil_log2():
    for bits, s in GOLD["format_volume"]:
        assert dm.format_volume(bits) == s, bits
    for x, b in GOLD["ceil_log2"]:
        assert dm.ceil_log2(x) == b
    with pytest.raises(ValueError):
        dm.ceil_log2(0)


def test_projected_volume():
    for n, m, k, p, ld, want in GOLD["projected"]:
        assert dm.projected_comm_volume(n, m, k, p, ld) == pytest.approx(want, rel=1e-15)


def test_fit_scaling_matches_reference():
    for f in GOLD["fits"]:
        got = dm.fit_scaling(f["xs"], f["ys"], f["kind"])
        assert got.kind == f["kind"]
        assert got.a == pytest.approx(f["a"], rel=1e-12)
        assert got.b == pytest.approx(f["b"], rel=1e-12, abs=1e-15)
        assert got.r_squared == pytest.approx(f["r_squared"], rel=1e-12, abs=1e-15)
        assert got.predict(f["predict_at"]) == pytest.approx(f["predict"], rel=1e-12)


def test_fit_scaling_errors():
    with pytest.raises(ValueError):
        dm.fit_scaling([1, 2, 3], [1, 2, 3], "linear")
    with pytest.raises(ValueError):
        dm.fit_scaling([1, 2], [1, 2])
    with pytest.raises(ValueError):
        dm.fit_scaling([1, 2, 3], [1, 0, 3])
    with pytest.raises(ValueError):
        dm.fit_scaling([0, 2, 3], [1, 2, 3], "power")
    assert math.isfinite(dm.fit_scaling([1, 2, 3], [2, 4, 8]).b)


@pytest.mark.gpu
def test_gpu_comm_reports():
    import paper_2403_02997_b200 as tb
    reports = []
    for c in SMALL_CASES:
        g = tb.normalize(tb.EdgeList(n=c.n, edges=c.pairs))
        per_p = GOLD["graphs"][c.name]
        for p in sorted(per_p, key=int):
            r = dm.comm_report(g, int(p), name=c.name)
            assert _report_dict(r) == per_p[p]["report"], (c.name, p)
            reports.append(r)
    assert dm.reports_to_csv(reports) == GOLD["csv"]
