"""report.py writes the reference CLI's files byte for byte.

Data parsed back from the reference's own outputs (tests/golden/refrun_pde_test1,
made by make_golden.py:refrun_outputs) is re-emitted through report.py and must
reproduce the reference's bytes exactly.
"""

import csv
from dataclasses import dataclass

import numpy as np

from paper_1705_02003_b200.report import fmt, residual_sink, write_iterations_by_level

from conftest import GOLDEN

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
