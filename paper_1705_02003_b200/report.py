"""Run outputs fed from the device results.

Byte-for-byte the reference's file formats, so a study run through the device
path emits the files the reference's CLI emits:

* per-ensemble lane residual histories ``residuals_level{L}_ens{k}.csv``
  (``cli.py:121-131``: header ``iteration,lane0..``, one row per iteration,
  floats as ``repr``) - the histories come from the device history buffer
  (``uqg_pcg`` ``hist_host``) through ``solve_plan(..., residual_sink)``;
* ``iterations_by_level.csv`` (``harness.py:784-797``: ``run, level,
  sample_id, iterations, predicted_iterations`` with the reference's ``_fmt``:
  ``repr`` for floats, ``str`` for ints, empty for None);
* ``r_table.csv`` (``harness.py:759-778``): per-level and total work ratios
  R (``compute_R``, ``grouping.py:156-193``) of the executed plans from the
  device iteration counts - a function of the counts and plans only, so
  byte-identical to the reference's wherever the counts agree;
* ``manifest.json`` (``harness.py:780-782``, schema ``RunReport.to_dict``,
  ``harness.py:439-560``): config, per-level samples / plans / error
  indicator / prediction errors / budget flag, work ratios, stop reason,
  notes and the sparse grid with both channels' surpluses.  It parses with
  the reference's ``parse_manifest``; QoI-derived floats carry the device's
  rounding.

Files carry no timestamps; the device path is bitwise deterministic, so
repeated runs emit identical bytes (the reference's acceptance criterion 8).
"""

from __future__ import annotations

import csv
import io
import json
from pathlib import Path

import numpy as np

__all__ = ["residual_sink", "write_iterations_by_level", "fmt", "compute_R", "write_r_table",
           "run_report", "write_manifest", "emit_reports"]


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


def compute_R(levels):
    """Per-level and total work ratios (``grouping.py:156-193``): for each
    ``(ensembles, padding, slot_iterations)`` level, cost ``S * sum_k max_i
    I(k, i)`` (replica slots occupy lanes) over the ideal cost of the real
    samples; empty levels give NaN and are left out of the total."""
    per, num_t, den_t = [], 0.0, 0.0
    for ensembles, padding, iters in levels:
        if not ensembles:
            per.append(float("nan"))
            continue
        if len(iters) != len(ensembles):
            raise ValueError("iteration lists must match the plan's ensembles")
        S = len(ensembles[0])
        num = den = 0.0
        for pad, group_iters in zip(padding, iters):
            vals = np.asarray(group_iters, dtype=float)
            if vals.shape != (S,):
                raise ValueError(f"expected {S} slot iterations, got {vals.shape}")
            if not np.all(np.isfinite(vals)) or np.any(vals < 0):
                raise ValueError("slot iterations must be finite and non-negative")
            num += S * float(vals.max())
            den += float(vals[: S - pad].sum())
        if den <= 0:
            raise ValueError("level has zero ideal work; iteration counts all zero")
        per.append(num / den)
        num_t += num
        den_t += den
    return per, (num_t / den_t if den_t > 0 else float("nan"))


def _slot_iters(rec):
    return [[float(rec.iterations[sid]) for sid in g] for g in rec.ensembles]


def _level_ratio(rec) -> float:
    return float(compute_R([(rec.ensembles, rec.padding, _slot_iters(rec))])[1])


def write_r_table(runs, out_dir, sizes, strategy: str = "sur", speedups=None,
                  name: str = "r_table.csv") -> Path:
    """``r_table.csv`` (``harness.py:759-778``) for one or several runs' level
    records (the executed surrogate plans): one row per level with its real
    sample count, ensemble count and R_l, then the run's total R and the
    predicted speed-up (empty without a base curve)."""
    if runs and not isinstance(runs[0], (list, tuple)):
        runs, sizes, speedups = [runs], [sizes], [speedups]
    speedups = speedups or [None] * len(runs)
    buf = io.StringIO()
    writer = csv.writer(buf, lineterminator="\n")
    writer.writerow(["strategy", "S", "level", "n_samples", "n_ensembles", "R_l", "R",
                     "pred_speedup"])
    for records, size, sp in zip(runs, sizes, speedups):
        for rec in records:
            n_real = sum(len(g) for g in rec.ensembles) - sum(rec.padding)
            writer.writerow([strategy, size, rec.level, n_real, len(rec.ensembles),
                             fmt(_level_ratio(rec)), "", ""])
        total = compute_R([(r.ensembles, r.padding, _slot_iters(r)) for r in records])[1]
        writer.writerow([strategy, size, "", "", "", "", fmt(float(total)), fmt(sp)])
    path = Path(out_dir) / name
    path.parent.mkdir(parents=True, exist_ok=True)
    path.write_text(buf.getvalue())
    return path


def _config_dict(cfg, strategy: str, dump_residuals: bool) -> dict:
    """``RunConfig.to_dict`` (``harness.py:189-205``) for a reference preset;
    the 2D configs use the same keys plus the 2D operator's parameters."""
    conv = getattr(cfg, "sigma0_convention", "stddev")
    field = {"delta": cfg.delta, "sigma0": cfg.sigma0, "N": cfg.n_modes, "a_min": cfg.a_min,
             "a_hat": {"mode": cfg.a_hat_mode, "value": cfg.a_hat_value}, "a_y": cfg.a_y,
             "a_z": getattr(cfg, "a_z", 1.0), "nystrom_points": 513,
             "sigma0_convention": conv, "expansion": cfg.expansion}
    three_d = hasattr(cfg, "a_z")
    mesh = {"mesh_cells": cfg.cells, "quadrature": "gauss2"} if three_d else \
        {"mesh_cells": cfg.cells, "operator": "fv2d", "a2": cfg.a2}
    out = {"problem": cfg.name, "n_dims": cfg.n_modes, "S": cfg.ensemble_size, "tau": cfg.tau,
           "n_max": cfg.n_max, "initial_level": cfg.initial_level, "strategies": [strategy],
           "solver": {"tol": cfg.tol, "maxit": cfg.maxit}, "field": field, "mesh": mesh,
           "analytic": None, "base_curve": None, "dump_residuals": bool(dump_residuals)}
    if not three_d:
        out["max_total_level"] = cfg.max_total_level
    return out


def _grid_dict(grid) -> dict:
    """``HierGrid.to_json_dict`` (``hier_grid.py:421-436``)."""
    coords = grid.node_coords()
    nodes = []
    for p, (lv, ix) in enumerate(grid.nodes):
        nodes.append({
            "level": list(lv), "index": list(ix), "coords": [float(x) for x in coords[p]],
            "surpluses": {name: (float(arr[p]) if np.isfinite(arr[p]) else None)
                          for name, arr in grid.surplus.items()}})
    return {"dim": grid.dim, "domain": [list(d) for d in grid.domain], "nodes": nodes}


def run_report(cfg, records, stop_reason: str, grid, notes=(), strategy: str = "sur",
               dump_residuals: bool = False) -> dict:
    """One run in the reference's ``RunReport.to_dict`` layout."""
    levels = []
    for rec in records:
        pred = None if rec.predicted is None else np.asarray(rec.predicted, dtype=float)
        ind = getattr(rec, "indicator", None)
        samples = [{"sample_id": sid, "coords": [float(x) for x in rec.coords[i]],
                    "iterations": rec.iterations[sid],
                    "predicted_iterations": None if pred is None else float(pred[i]),
                    "indicator": None if ind is None else float(ind[i])}
                   for i, sid in enumerate(rec.ids)]
        err_mean = err_max = None
        if pred is not None:
            err = np.abs(pred - np.array([rec.iterations[sid] for sid in rec.ids]))
            err_mean, err_max = float(err.mean()), float(err.max())
        levels.append({
            "level": rec.level, "samples": samples,
            "plans": [{"strategy": strategy, "ensembles": [list(g) for g in rec.ensembles],
                       "padding": list(rec.padding), "R_l": _level_ratio(rec)}],
            "error_indicator": getattr(rec, "error_indicator", None),
            "mean_abs_prediction_error": err_mean, "max_abs_prediction_error": err_max,
            "budget_truncated": bool(getattr(rec, "budget_truncated", False))})
    total = compute_R([(r.ensembles, r.padding, _slot_iters(r)) for r in records])[1]
    return {"config": _config_dict(cfg, strategy, dump_residuals), "levels": levels,
            "work_ratios": {strategy: float(total)}, "predicted_speedups": None,
            "stop_reason": stop_reason, "notes": list(notes), "grid": _grid_dict(grid)}


def write_manifest(reports, out_dir, name: str = "manifest.json") -> Path:
    """``manifest.json`` (``harness.py:780-782``): ``{"reports": [...]}``,
    indent 1, trailing newline."""
    if isinstance(reports, dict):
        reports = [reports]
    path = Path(out_dir) / name
    path.parent.mkdir(parents=True, exist_ok=True)
    path.write_text(json.dumps({"reports": list(reports)}, indent=1) + "\n")
    return path


def emit_reports(cfg, records, stop_reason: str, grid, out_dir, notes=(),
                 dump_residuals: bool = False) -> dict:
    """The reference's ``emit_reports`` (``harness.py:741-797``) for one device
    run: ``r_table.csv``, ``manifest.json`` and ``iterations_by_level.csv``."""
    out_dir = Path(out_dir)
    rep = run_report(cfg, records, stop_reason, grid, notes, dump_residuals=dump_residuals)
    return {"table": write_r_table(records, out_dir, cfg.ensemble_size),
            "manifest": write_manifest(rep, out_dir),
            "iterations": write_iterations_by_level(records, out_dir)}
