"""report.py writes the reference CLI's files byte for byte.

Data parsed back from the reference's own outputs (tests/golden/refrun_pde_test1,
made by make_golden.py:refrun_outputs) is re-emitted through report.py and must
reproduce the reference's bytes exactly.
"""

import csv
from dataclasses import dataclass

import numpy as np

from paper_1705_02003_b200.report import fmt, residual_sink, write_iterations_by_level

from conftest import GOLDEN, ROOT

REF = GOLDEN / "refrun_pde_test1"


def test_residual_csv_bytes(tmp_path):
    for name in ("residuals_level1_ens0.csv", "residuals_level1_ens11.csv",
                 "residuals_level2_ens0.csv"):
        rows = list(csv.reader((REF / name).read_text().splitlines()))
        S = len(rows[0]) - 1
        history = [np.array([float(v) for v in r[1:]]) for r in rows[1:]]
        level = int(name.split("level")[1].split("_")[0])
        ens = int(name.split("ens")[1].split(".")[0])
        residual_sink(tmp_path, S)(level, ens, history)
        assert (tmp_path / name).read_bytes() == (REF / name).read_bytes()


@dataclass
class _Rec:
    level: int
    ids: list
    iterations: dict
    predicted: list | None


def test_iterations_by_level_bytes(tmp_path):
    rows = list(csv.reader((REF / "iterations_by_level.csv").read_text().splitlines()))[1:]
    recs = {}
    for run, level, sid, its, pred in rows:
        r = recs.setdefault(int(level), _Rec(int(level), [], {}, []))
        r.ids.append(int(sid))
        r.iterations[int(sid)] = int(its)
        r.predicted.append(None if pred == "" else float(pred))
    records = []
    for lv in sorted(recs):
        r = recs[lv]
        if all(p is None for p in r.predicted):
            r.predicted = None
        records.append(r)
    path = write_iterations_by_level(records, tmp_path)
    assert path.read_bytes() == (REF / "iterations_by_level.csv").read_bytes()


def test_fmt_matches_reference_rules():
    assert fmt(None) == "" and fmt(3) == "3" and fmt(0.1) == "0.1" and fmt(27.5) == "27.5"
    assert fmt(1e-300) == repr(1e-300)


@dataclass
class _PlanRec:
    level: int
    ensembles: tuple
    padding: tuple
    iterations: dict


def _ref_manifest():
    import json
    return json.loads((REF / "manifest.json").read_text())["reports"][0]


def test_r_table_bytes(tmp_path):
    """r_table.csv (harness.py:759-778) re-emitted from the reference run's own
    plans and counts through report.compute_R / write_r_table."""
    from paper_1705_02003_b200.report import write_r_table

    rep = _ref_manifest()
    recs = []
    for lv in rep["levels"]:
        (plan,) = lv["plans"]
        its = {s["sample_id"]: s["iterations"] for s in lv["samples"]}
        recs.append(_PlanRec(lv["level"], tuple(tuple(g) for g in plan["ensembles"]),
                             tuple(plan["padding"]), its))
    path = write_r_table(recs, tmp_path, rep["config"]["S"])
    assert path.read_bytes() == (REF / "r_table.csv").read_bytes()


def test_compute_R_matches_reference_rules():
    from paper_1705_02003_b200.report import compute_R

    # padded last slot excluded from the ideal cost; replicas still cost lanes
    per, tot = compute_R([([[1, 2], [3, 3]], [0, 1], [[3, 4], [5, 5]])])
    assert per == [(2 * 4 + 2 * 5) / (3 + 4 + 5)] and tot == per[0]
    per, tot = compute_R([([], [], []), ([[1]], [0], [[2.0]])])
    assert np.isnan(per[0]) and per[1] == 1.0 and tot == 1.0


def test_manifest_schema_parses_with_reference(tmp_path):
    """manifest.json in the reference's RunReport layout: the reference's own
    parse_manifest (baseline/_ref, staged by build()) reads what
    report.run_report / write_manifest emit for the reference run's data."""
    import sys

    import pytest

    from paper_1705_02003_b200 import configs
    from paper_1705_02003_b200.report import run_report, write_manifest
    from paper_1705_02003_b200.sparse_grid import SparseGrid

    ref_pkg = ROOT / "baseline" / "_ref"
    if not (ref_pkg / "uqgroup").exists():
        pytest.skip("reference not staged (tools/stage_reference.py)")
    rep = _ref_manifest()
    import dataclasses

    cfg = dataclasses.replace(configs.PRESETS_3D["pde_test1"], cells=6, n_max=60)
    grid = SparseGrid(rep["grid"]["dim"])
    grid._extend([(tuple(n["level"]), tuple(n["index"])) for n in rep["grid"]["nodes"]])
    for ch in ("qoi", "iterations"):
        grid.surplus[ch] = np.array([np.nan if n["surpluses"][ch] is None else
                                     n["surpluses"][ch] for n in rep["grid"]["nodes"]])

    @dataclass
    class Rec:
        level: int
        ids: list
        coords: np.ndarray
        predicted: object
        ensembles: tuple
        padding: tuple
        iterations: dict
        error_indicator: float
        budget_truncated: bool
        indicator: np.ndarray

    recs = []
    for lv in rep["levels"]:
        (plan,) = lv["plans"]
        sm = lv["samples"]
        pred = None if sm[0]["predicted_iterations"] is None else \
            [s["predicted_iterations"] for s in sm]
        recs.append(Rec(lv["level"], [s["sample_id"] for s in sm],
                        np.array([s["coords"] for s in sm]), pred,
                        tuple(tuple(g) for g in plan["ensembles"]), tuple(plan["padding"]),
                        {s["sample_id"]: s["iterations"] for s in sm}, lv["error_indicator"],
                        lv["budget_truncated"], np.array([s["indicator"] for s in sm])))
    mine = run_report(cfg, recs, rep["stop_reason"], grid, rep["notes"], dump_residuals=True)
    path = write_manifest(mine, tmp_path)
    # the reference run's own data re-emitted: every section equal to the reference's
    import json
    doc = json.loads(path.read_text())["reports"][0]
    for key in ("levels", "work_ratios", "predicted_speedups", "stop_reason", "notes", "grid",
                "config"):
        assert doc[key] == rep[key], key
    assert path.read_bytes() == (REF / "manifest.json").read_bytes()
    sys.path.insert(0, str(ref_pkg))
    try:
        from uqgroup.harness import parse_manifest
        (parsed,) = parse_manifest(path)
    finally:
        sys.path.remove(str(ref_pkg))
    assert parsed.work_ratios == rep["work_ratios"] and len(parsed.levels) == len(rep["levels"])
