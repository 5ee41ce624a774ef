"""Oracle: one level's solve over a grouping plan (TEST INFRA ONLY).

Restates ``harness._PdeProblem.solve_plan`` (``harness.py:399-431``) for the
2D operator: per group, assemble -> Jacobi-PCG -> QoI; record iterations and
QoI for the first occurrence of each sample id only (replica slots do real
lane work but are discarded, ``harness.py:427-430``); note unconverged groups
(``harness.py:421-426``).
"""

from __future__ import annotations

import numpy as np

from . import fv2d, pcg


def solve_plan(mesh, field, table, ensembles, coords_by_id, tol, maxit, a2="const",
               level=0, keep_history=False):
    iters, qois, notes, hists = {}, {}, [], []
    for k, group in enumerate(ensembles):
        ys = np.array([coords_by_id[sid] for sid in group])
        sysm = fv2d.assemble(mesh, field, ys, table, a2)
        res = pcg.pcg(sysm.row_offsets, sysm.col_indices, sysm.values, sysm.rhs,
                      tol=tol, maxit=maxit, history=keep_history)
        if keep_history:
            hists.append(res.history)
        if not res.converged.all():
            bad = int((~res.converged).sum())
            notes.append(f"level {level} ensemble {k}: {bad} lane(s) hit maxit ({maxit}) unconverged")
        for s, sid in enumerate(group):
            if sid not in iters:
                iters[sid] = int(res.iterations[s])
                qois[sid] = fv2d.qoi(res.solution[s])
    if keep_history:
        return iters, qois, notes, hists
    return iters, qois, notes
