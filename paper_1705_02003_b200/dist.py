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

__all__ = ["my_groups", "pack_rows", "unpack_rows", "ShardedSolver", "LevelShard"]


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


class LevelShard:
    """Device-resident sharding of ONE level's plan (the bench's strong-scaling
    step and ``EnsembleSolver.run_level_device(shard=...)``).

    Every rank has built the identical plan ``groups [K*S]`` on its own device
    (same keys, same sort).  Rank r solves groups k = r, r+W, r+2W, ... (round
    robin over the cost-sorted plan, ``my_groups``), then ONE
    ``all_gather_into_tensor`` of fixed-size float64 rows
    ``[k, ensemble_iterations, iterations[S], converged[S], qoi[S]]`` (k = -1
    pads a short rank) gives every rank the whole level's results, scattered
    back into plan order on the device - the input of the surrogate refit
    (``harness.py:658-660``).  Nothing is communicated on the solve path.

    ``coll_device``: where the collective runs (the rank's GPU under NCCL;
    ``cpu`` under gloo).  After each call ``last_load`` holds, per rank, the
    number of groups and the sum of their ensemble iterations (the load
    balance of the cost-sorted plan).
    """

    def __init__(self, rank: int, world: int, process_group=None, coll_device=None,
                 force_collective: bool = False):
        self.rank, self.world, self.pg = int(rank), int(world), process_group
        self.coll_device = coll_device
        # issue the all-gather even with one rank (the single-GPU NCCL check in
        # tests/test_gpu_dist.py: same tensors, dtypes and call as N ranks make)
        self.force_collective = bool(force_collective)
        self.last_load = None

    @classmethod
    def from_env(cls, process_group=None, coll_device=None):
        import torch.distributed as dist
        return cls(dist.get_rank(process_group), dist.get_world_size(process_group),
                   process_group, coll_device)

    def mine(self, K: int):
        return my_groups(K, self.rank, self.world)

    def solve(self, solve_fn, groups, K: int, S: int):
        """``solve_fn(lane_ids [g*S] int32, g) -> (iters [g*S], conv [g*S],
        ens [g], qoi [g*S])`` solves this rank's g groups; returns the level's
        (iters [K*S] int32, conv [K*S] bool, ens [K] int32, qoi [K*S] f64) on
        ``groups.device``."""
        import torch
        import torch.distributed as dist

        dev = groups.device
        sel = torch.arange(self.rank, K, self.world, device=dev, dtype=torch.long)
        g = int(sel.numel())
        rows = -(-K // self.world)
        width = 2 + 3 * S
        local = torch.full((rows, width), -1.0, dtype=torch.float64, device=dev)
        if g:
            lanes = groups.view(K, S).index_select(0, sel).reshape(-1).contiguous()
            it, cv, en, q = solve_fn(lanes, g)
            local[:g, 0] = sel.to(torch.float64)
            local[:g, 1] = en.to(torch.float64)
            local[:g, 2:2 + S] = it.view(g, S).to(torch.float64)
            local[:g, 2 + S:2 + 2 * S] = cv.view(g, S).to(torch.float64)
            local[:g, 2 + 2 * S:] = q.view(g, S)
        cdev = self.coll_device or dev
        send = local.to(cdev)
        allr = torch.empty((self.world * rows, width), dtype=torch.float64, device=cdev)
        if self.world > 1 or self.force_collective:
            dist.all_gather_into_tensor(allr, send, group=self.pg)
        else:
            allr.copy_(send)
        allr = allr.to(dev)
        valid = allr[:, 0] >= 0
        got = allr[valid]
        k = got[:, 0].long()
        if got.shape[0] != K or not torch.equal(torch.sort(k).values,
                                                torch.arange(K, device=dev)):
            raise RuntimeError("allgather lost or duplicated groups")
        ens = torch.empty((K,), dtype=torch.int32, device=dev)
        ens[k] = got[:, 1].to(torch.int32)
        it = torch.empty((K, S), dtype=torch.int32, device=dev)
        it[k] = got[:, 2:2 + S].to(torch.int32)
        cv = torch.empty((K, S), dtype=torch.bool, device=dev)
        cv[k] = got[:, 2 + S:2 + 2 * S] != 0
        q = torch.empty((K, S), dtype=torch.float64, device=dev)
        q[k] = got[:, 2 + 2 * S:]
        owner = (k % self.world)
        self.last_load = {
            "groups": torch.bincount(owner, minlength=self.world).tolist(),
            "group_iterations": torch.zeros(self.world, dtype=torch.float64, device=dev)
            .index_add_(0, owner, got[:, 1]).long().tolist()}
        return it.reshape(-1), cv.reshape(-1), ens, q.reshape(-1)
