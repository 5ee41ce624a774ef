"""Multi-GPU sharding of a level's groups + the one collective of the study.

Each rank (one process per GPU, ``torch.distributed``) runs the identical host
loop, so every rank builds the identical plan.  Groups are independent
(``ensemble.py:1-8``; ``harness.py:631-633``), so group k is solved by rank
``k % world`` - round-robin over the cost-sorted plan balances ascending
predicted costs - with no communication on the solve path.  After the level,
one allgather of fixed-size rows (group index, per-lane iterations, converged
flags, QoIs) gives every rank the full per-sample results for the surrogate
refit (``harness.py:658-660``).  Kernel geometry never depends on the rank
count, so 1-GPU and N-GPU results are bit-identical.
"""

from __future__ import annotations

import numpy as np

from .solve import LevelSolveResult

__all__ = ["my_groups", "pack_rows", "unpack_rows", "ShardedSolver"]


def my_groups(n_groups: int, rank: int, world: int) -> list[int]:
    return list(range(rank, n_groups, world))


def pack_rows(groups: list[int], res: LevelSolveResult, rows: int, S: int) -> np.ndarray:
    """(rows, 1 + 3S) float64: [k, iters..., converged..., qoi...]; k=-1 pads.

    Iteration counts are small integers, exact in float64.
    """
    out = np.zeros((rows, 1 + 3 * S))
    out[:, 0] = -1
    for r, k in enumerate(groups):
        out[r, 0] = k
        out[r, 1:1 + S] = res.iterations[r]
        out[r, 1 + S:1 + 2 * S] = res.converged[r]
        out[r, 1 + 2 * S:] = res.qoi[r]
    return out


def unpack_rows(gathered: np.ndarray, n_groups: int, S: int) -> LevelSolveResult:
    it = np.zeros((n_groups, S), dtype=int)
    cv = np.zeros((n_groups, S), dtype=bool)
    q = np.zeros((n_groups, S))
    seen = np.zeros(n_groups, dtype=bool)
    for row in gathered.reshape(-1, gathered.shape[-1]):
        k = int(row[0])
        if k < 0:
            continue
        it[k] = row[1:1 + S].astype(int)
        cv[k] = row[1 + S:1 + 2 * S] != 0
        q[k] = row[1 + 2 * S:]
        seen[k] = True
    if not seen.all():
        raise RuntimeError(f"allgather lost groups {np.flatnonzero(~seen).tolist()}")
    return LevelSolveResult(it, cv, np.zeros_like(cv), it.max(axis=1), q)


class ShardedSolver:
    """``solve_plan`` over torch.distributed ranks.

    ``solve_groups(samples (k,S,M)) -> LevelSolveResult`` does the local solve
    (``EnsembleSolver2D.solve_groups`` on a GPU); ``collect(plan, result)``
    applies the first-occurrence rule (``EnsembleSolver2D.collect``).
    """

    def __init__(self, solve_groups, collect, process_group=None, device=None):
        import torch.distributed as dist

        self.dist = dist
        self.pg = process_group
        self.rank = dist.get_rank(process_group)
        self.world = dist.get_world_size(process_group)
        self.solve_groups = solve_groups
        self.collect = collect
        self.device = device
        self.last_local_groups = 0

    def solve_plan(self, plan, coords_by_id, residual_sink=None):
        import torch

        K, S = len(plan.ensembles), plan.ensemble_size
        mine = my_groups(K, self.rank, self.world)
        self.last_local_groups = len(mine)
        rows = -(-K // self.world)
        if mine:
            samples = np.array([[coords_by_id[sid] for sid in plan.ensembles[k]] for k in mine],
                               dtype=np.float64)
            local = pack_rows(mine, self.solve_groups(samples), rows, S)
        else:
            local = pack_rows([], None, rows, S)
        t = torch.from_numpy(local)
        if self.device is not None:
            t = t.to(self.device)
        bufs = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(bufs, t, group=self.pg)
        gathered = np.stack([b.cpu().numpy() for b in bufs])
        return self.collect(plan, unpack_rows(gathered, K, S), residual_sink)
