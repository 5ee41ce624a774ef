"""Adaptive study loop around the device solve (host; reference ``harness.py:575-701``).

Level 1 is the initial grid grouped in generation order; every later level is
grouped by the iteration surrogate fitted through the previous level ("sur",
``harness.py:613-629``) on the device, solved level-batched on the device, and
its per-sample iterations and QoIs refit both surrogates before refinement.
With ``world > 1`` the groups of each level are dealt round-robin to ranks
(``dist.py``) and the per-sample results are allgathered before the refit -
the only collective of the run.
"""

from __future__ import annotations

from dataclasses import dataclass, field as dc_field

import numpy as np

from .configs import StudyConfig
from .grouping import group_by_key, group_natural
from .solve import EnsembleSolver
from .sparse_grid import SparseGrid

QOI, ITER = "qoi", "iterations"


@dataclass
class LevelRecord:
    level: int
    ids: list
    coords: np.ndarray
    predicted: np.ndarray | None
    ensembles: tuple
    padding: tuple
    iterations: dict
    qois: dict
    notes: list = dc_field(default_factory=list)
    # run-report fields (harness.py:439-524): QoI-channel error indicator after
    # the level's fit, the budget flag of the refinement that made the level,
    # and the per-sample anisotropy indicator (adaptive_run(indicators=True))
    error_indicator: float | None = None
    budget_truncated: bool = False
    indicator: np.ndarray | None = None


def sample_set(cfg: StudyConfig) -> np.ndarray:
    """Seeded synthetic U[-1,1]^M samples for configs the grid cannot reach (C5)."""
    return np.random.default_rng(0).uniform(-1.0, 1.0, (cfg.synthetic_samples, cfg.n_modes))


def adaptive_run(cfg: StudyConfig, solver: EnsembleSolver | None = None, shard=None,
                 max_levels: int | None = None, device_keys: bool = False,
                 residual_sink=None, indicators: bool = False):
    """Run the grouped adaptive loop; returns (records, stop_reason, grid).

    ``shard``: optional callable(plan, coords_by_id) -> (iters, qois, notes)
    replacing ``solver.solve_plan`` (multi-GPU sharded solve + allgather).
    ``device_keys``: fit and evaluate the iteration surrogate on the GPU
    (``SparseGrid.fit_device`` / ``evaluate_device``; bit-identical surpluses
    and keys on this channel; the QoI channel, whose surpluses steer
    refinement, stays on the host BLAS path).
    ``residual_sink(level, ensemble, history)``: per-ensemble lane residual
    histories, as the reference's ``adaptive_run(residual_sink=...)``
    (``report.residual_sink`` writes the reference's CSVs).
    ``indicators``: record each sample's anisotropy indicator on the device
    (``harness.py:616``; the run report's ``indicator`` column).  The
    reference's budget notes ("level L truncated to the n_max=... sample
    budget") are appended to the notes of the level whose refinement
    truncated the next one, so concatenated notes keep the reference's order.
    """
    if solver is None and shard is None:
        solver = cfg.make_solver()
    if residual_sink is not None:
        if shard is not None:
            raise ValueError("residual histories are recorded by the single-device solve only")
        solve = lambda plan, coords: solver.solve_plan(plan, coords, residual_sink)  # noqa: E731
    else:
        solve = shard or solver.solve_plan
    S = cfg.ensemble_size
    grid = SparseGrid(cfg.n_modes)
    batch = grid.add_initial_levels(cfg.initial_level)
    if len(batch) > cfg.n_max:
        raise ValueError(f"n_max={cfg.n_max} is smaller than the {len(batch)}-point initial grid")
    cap = cfg.max_levels if max_levels is None else max_levels
    records, level, stop, truncated = [], 0, None, False
    probe = None
    if indicators:
        from .field import anisotropy_indicators

        op = solver.op
        probe = (op.field, op.indicator_points())
        probe = probe + (op.field.mode_values(probe[1]),)
    while True:
        level += 1
        start = len(grid) - len(batch)
        ids = list(range(start, len(grid)))
        coords = grid.node_coords()[start:]
        coords_by_id = {sid: coords[i] for i, sid in enumerate(ids)}
        predicted = None
        if level == 1:
            plan = group_natural(ids, S, level, "sur")
        else:
            predicted = (grid.evaluate_device if device_keys else grid.evaluate)(
                ITER, coords, n_nodes=start)
            plan = group_by_key(ids, {sid: float(predicted[i]) for i, sid in enumerate(ids)}, S,
                                level, "sur")
        ind = None if probe is None else anisotropy_indicators(probe[0], coords, probe[1],
                                                                probe[2])
        iters, qois, notes = solve(plan, coords_by_id)
        grid.fit(QOI, {sid: qois[sid] for sid in ids})
        (grid.fit_device if device_keys else grid.fit)(ITER, {sid: iters[sid] for sid in ids})
        records.append(LevelRecord(level, ids, coords, predicted, plan.ensembles, plan.padding,
                                   iters, qois, list(notes), grid.error_indicator(QOI),
                                   truncated, ind))
        if level >= cap:
            stop = "level_cap"
            break
        new, exhausted = grid.refine(cfg.tau, QOI, cfg.n_max)
        if not new:
            stop = "budget_exhausted" if exhausted else "tolerance_met"
            break
        truncated = exhausted
        if truncated:
            records[-1].notes.append(
                f"level {level + 1} truncated to the n_max={cfg.n_max} sample budget")
        batch = new
    return records, stop, grid
