"""The device study emits the reference CLI's run files.

The reference's pde_test1 preset at S=4, n_max=60, 6^3 cells is run through
driver.adaptive_run with a report.residual_sink.  The per-sample iteration
table must have the reference's rows (levels, sample ids, order) with counts
inside the preset's rounding envelope (+-1: the reference's own counts move by
that much under a different dot-product order, DESIGN.md "Rounding
envelope"); the residual histories of lockstep lanes match its values to
rounding; and two device runs must emit identical bytes (the reference's
acceptance criterion 8).  Byte-exact formatting is pinned on the CPU
(tests/test_report_cpu.py).
"""

import csv
import dataclasses

import numpy as np
import pytest

import paper_1705_02003_b200 as uq
from paper_1705_02003_b200.driver import adaptive_run
from paper_1705_02003_b200.report import emit_reports, residual_sink

from conftest import GOLDEN, ROOT

pytestmark = pytest.mark.gpu
REF = GOLDEN / "refrun_pde_test1"


def _run(out):
    cfg = dataclasses.replace(uq.PRESETS_3D["pde_test1"], cells=6, n_max=60)
    records, stop, grid = adaptive_run(cfg, residual_sink=residual_sink(out, cfg.ensemble_size),
                                       indicators=True)
    notes = [n for r in records for n in r.notes]
    emit_reports(cfg, records, stop, grid, out, notes, dump_residuals=True)
    return stop


def test_device_study_emits_reference_files(tmp_path):
    a, b = tmp_path / "a", tmp_path / "b"
    assert _run(a) == "budget_exhausted"
    mine = list(csv.reader((a / "iterations_by_level.csv").read_text().splitlines()))
    ref = list(csv.reader((REF / "iterations_by_level.csv").read_text().splitlines()))
    assert mine[0] == ref[0] and len(mine) == len(ref)
    for m, r in zip(mine[1:], ref[1:]):
        assert m[:3] == r[:3]                           # run, level, sample id
        assert abs(int(m[3]) - int(r[3])) <= 1          # iterations (envelope)
        assert (m[4] == "") == (r[4] == "")             # predicted on the same levels
        if r[4]:
            assert abs(float(m[4]) - float(r[4])) <= 2.0
    exact = sum(m[3] == r[3] for m, r in zip(mine[1:], ref[1:]))
    assert exact >= 0.8 * (len(ref) - 1)
    for name in ("residuals_level1_ens0.csv", "residuals_level1_ens11.csv"):
        m = list(csv.reader((a / name).read_text().splitlines()))
        r = list(csv.reader((REF / name).read_text().splitlines()))
        assert m[0] == r[0]
        n = min(len(m), len(r))  # the final iteration may differ by one (envelope)
        mv = np.array([[float(v) for v in row] for row in m[1:n]])
        rv = np.array([[float(v) for v in row] for row in r[1:n]])
        assert np.array_equal(mv[:, 0], rv[:, 0])
        np.testing.assert_allclose(mv[:, 1:], rv[:, 1:], rtol=1e-6, atol=1e-12 * rv[0, 1:].max())
    _run(b)
    files = sorted(p.name for p in a.iterdir())
    assert files == sorted(p.name for p in b.iterdir()) and len(files) > 10
    for name in files:
        assert (a / name).read_bytes() == (b / name).read_bytes(), name


def test_device_run_report_matches_reference(tmp_path):
    """r_table.csv and manifest.json of the device study (harness.py:741-782)
    against the reference CLI's: same levels, sample ids, coordinates, plans
    on level 1, counts in the envelope, anisotropy indicators to 1e-12, QoI-
    channel error indicators and surpluses to rounding; the manifest parses
    with the reference's own parse_manifest."""
    import json
    import sys

    out = tmp_path / "run"
    _run(out)
    mine = list(csv.reader((out / "r_table.csv").read_text().splitlines()))
    ref = list(csv.reader((REF / "r_table.csv").read_text().splitlines()))
    assert len(mine) == len(ref) and mine[0] == ref[0]
    for m, r in zip(mine[1:], ref[1:]):
        assert m[:5] == r[:5]
        for a, b in ((m[5], r[5]), (m[6], r[6])):
            assert (a == "") == (b == "")
            if b:
                assert abs(float(a) - float(b)) <= 0.05 * float(b)
    doc = json.loads((out / "manifest.json").read_text())["reports"][0]
    rep = json.loads((REF / "manifest.json").read_text())["reports"][0]
    assert doc["config"] == rep["config"]
    assert doc["stop_reason"] == rep["stop_reason"] and doc["notes"] == rep["notes"]
    assert len(doc["levels"]) == len(rep["levels"])
    for a, b in zip(doc["levels"], rep["levels"]):
        assert a["level"] == b["level"] and a["budget_truncated"] == b["budget_truncated"]
        assert [s["sample_id"] for s in a["samples"]] == [s["sample_id"] for s in b["samples"]]
        for sa, sb in zip(a["samples"], b["samples"]):
            assert sa["coords"] == sb["coords"]
            assert abs(sa["iterations"] - sb["iterations"]) <= 1
            assert abs(sa["indicator"] - sb["indicator"]) <= 1e-12 * abs(sb["indicator"])
        np.testing.assert_allclose(a["error_indicator"], b["error_indicator"], rtol=1e-5)
    pa, pb = doc["levels"][0]["plans"][0], rep["levels"][0]["plans"][0]
    assert (pa["ensembles"], pa["padding"]) == (pb["ensembles"], pb["padding"])
    assert abs(pa["R_l"] - pb["R_l"]) <= 0.05 * pb["R_l"]   # counts within the envelope
    na, nb = doc["grid"]["nodes"], rep["grid"]["nodes"]
    assert [(n["level"], n["index"], n["coords"]) for n in na] == \
        [(n["level"], n["index"], n["coords"]) for n in nb]
    qa = np.array([n["surpluses"]["qoi"] for n in na], dtype=float)
    qb = np.array([n["surpluses"]["qoi"] for n in nb], dtype=float)
    np.testing.assert_allclose(qa, qb, rtol=1e-6, atol=1e-9 * np.nanmax(np.abs(qb)))
    ref_pkg = ROOT / "baseline" / "_ref"
    if (ref_pkg / "uqgroup").exists():
        sys.path.insert(0, str(ref_pkg))
        try:
            from uqgroup.harness import parse_manifest
            (parsed,) = parse_manifest(out / "manifest.json")
        finally:
            sys.path.remove(str(ref_pkg))
        assert parsed.stop_reason == "budget_exhausted" and len(parsed.levels) == len(rep["levels"])
