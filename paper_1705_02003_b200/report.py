"""Run outputs fed from the device results.

Byte-for-byte the reference's file formats, so a study run through the device
path emits the files the reference's CLI emits:

* per-ensemble lane residual histories ``residuals_level{L}_ens{k}.csv``
  (``cli.py:121-131``: header ``iteration,lane0..``, one row per iteration,
  floats as ``repr``) - the histories come from the device history buffer
  (``uqg_pcg`` ``hist_host``) through ``solve_plan(..., residual_sink)``;
* ``iterations_by_level.csv`` (``harness.py:784-797``: ``run, level,
  sample_id, iterations, predicted_iterations`` with the reference's ``_fmt``:
  ``repr`` for floats, ``str`` for ints, empty for None).

Files carry no timestamps; the device path is bitwise deterministic, so
repeated runs emit identical bytes (the reference's acceptance criterion 8).
"""

from __future__ import annotations

import csv
import io
from pathlib import Path

__all__ = ["residual_sink", "write_iterations_by_level", "fmt"]


def fmt(x) -> str:
    """The reference's cell formatting (``harness.py:753-758``)."""
    if x is None:
        return ""
    if isinstance(x, float):
        return repr(x)
    return str(x)


def residual_sink(out_dir, ensemble_size: int):
    """A ``residual_sink(level, ensemble, history)`` writing one CSV per
    ensemble into ``out_dir`` (``cli.py:121-131``)."""
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)

    def sink(level: int, ensemble: int, history) -> None:
        buf = io.StringIO()
        writer = csv.writer(buf, lineterminator="\n")
        writer.writerow(["iteration"] + [f"lane{s}" for s in range(ensemble_size)])
        for it, norms in enumerate(history):
            writer.writerow([it] + [repr(float(v)) for v in norms])
        (out_dir / f"residuals_level{level}_ens{ensemble}.csv").write_text(buf.getvalue())

    return sink


def write_iterations_by_level(runs, out_dir, name: str = "iterations_by_level.csv") -> Path:
    """``iterations_by_level.csv`` for one run's ``driver.LevelRecord`` list or
    several runs' lists (``harness.py:784-797``): samples of each level in
    generation order, predicted iterations empty on a natural-order level."""
    if runs and not isinstance(runs[0], (list, tuple)):
        runs = [runs]
    buf = io.StringIO()
    writer = csv.writer(buf, lineterminator="\n")
    writer.writerow(["run", "level", "sample_id", "iterations", "predicted_iterations"])
    for run_idx, records in enumerate(runs):
        for rec in records:
            for i, sid in enumerate(rec.ids):
                pred = None if rec.predicted is None else float(rec.predicted[i])
                writer.writerow([run_idx, rec.level, sid, fmt(rec.iterations[sid]), fmt(pred)])
    path = Path(out_dir) / name
    path.parent.mkdir(parents=True, exist_ok=True)
    path.write_text(buf.getvalue())
    return path
