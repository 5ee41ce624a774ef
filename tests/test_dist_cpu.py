"""Multi-rank sharding + allgather on CPU (gloo, world size 2).

The GPU solve is replaced by a deterministic stand-in with the same signature
(``solve_groups(samples) -> LevelSolveResult``); what is tested is the host
logic around it: round-robin group ownership, fixed-size row packing, the
allgather, reassembly and the first-occurrence rule for replica slots.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1705_02003_b200.dist import ShardedSolver, my_groups, pack_rows, unpack_rows
from paper_1705_02003_b200.grouping import GroupingPlan
from paper_1705_02003_b200.solve import EnsembleSolver2D, LevelSolveResult


def fake_solve(samples):
    K, S, M = samples.shape
    it = (np.abs(samples).sum(axis=2) * 100).astype(int) + 1
    q = (samples ** 2).sum(axis=2)
    return LevelSolveResult(it, np.ones((K, S), bool), np.zeros((K, S), bool), it.max(axis=1), q)


def collect(plan, res, sink=None):
    return EnsembleSolver2D.collect(type("X", (), {"maxit": 10})(), plan, res, sink)


def make_plan(n, S, M, seed=0):
    rng = np.random.default_rng(seed)
    ids = list(range(100, 100 + n))
    coords = {i: rng.uniform(-1, 1, M) for i in ids}
    K = -(-n // S)
    ens, pad = [], []
    for k in range(K):
        g = ids[k * S:(k + 1) * S]
        p = S - len(g)
        ens.append(tuple(g + [g[-1]] * p))
        pad.append(p)
    return GroupingPlan(3, S, tuple(ens), tuple(pad), "sur"), coords


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, S, M, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan, coords = make_plan(n, S, M)
        sh = ShardedSolver(fake_solve, collect)
        iters, qois, notes = sh.solve_plan(plan, coords)
        q.put((rank, sh.last_local_groups, iters, qois))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,S", [(37, 8), (5, 4), (64, 16)])
def test_sharded_solve_equals_single_rank(n, S):
    M, world = 3, 2
    plan, coords = make_plan(n, S, M)
    samples = np.array([[coords[s] for s in g] for g in plan.ensembles])
    want = collect(plan, fake_solve(samples))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, S, M, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    K = len(plan.ensembles)
    for rank, local, iters, qois in got:
        assert local == len(my_groups(K, rank, world))
        assert iters == want[0]
        assert qois == want[1]


def test_pack_unpack_roundtrip():
    plan, coords = make_plan(29, 8, 2)
    samples = np.array([[coords[s] for s in g] for g in plan.ensembles])
    res = fake_solve(samples)
    K = len(plan.ensembles)
    rows = [pack_rows(my_groups(K, r, 3),
                      LevelSolveResult(res.iterations[my_groups(K, r, 3)],
                                       res.converged[my_groups(K, r, 3)], None, None,
                                       res.qoi[my_groups(K, r, 3)]), -(-K // 3), 8)
            for r in range(3)]
    back = unpack_rows(np.stack(rows), K, 8)
    assert np.array_equal(back.iterations, res.iterations)
    assert np.array_equal(back.qoi, res.qoi)


def test_round_robin_covers_all_groups_once():
    for K in (1, 7, 8, 100):
        for W in (1, 2, 4, 8):
            seen = sorted(k for r in range(W) for k in my_groups(K, r, W))
            assert seen == list(range(K))


# ---------------------------------------------------------------------------
# LevelShard: the bench's strong-scaling step (device-resident plan, one
# all_gather_into_tensor) with a deterministic stand-in for the GPU solve

def _fake_solve_tensors(coords_t, S):
    import torch

    def solve(lanes, g):
        y = coords_t[lanes.long()]                       # [g*S, M]
        it = (y.abs().sum(dim=1) * 100).to(torch.int32) + 1
        q = (y ** 2).sum(dim=1)
        cv = it < 250
        en = it.view(g, S).max(dim=1).values
        return it, cv, en, q
    return solve


def _level_worker(rank, world, port, n, S, M, q):
    import torch

    from paper_1705_02003_b200.dist import LevelShard

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(1)
        coords = torch.from_numpy(rng.uniform(-1, 1, (n, M)))
        K = -(-n // S)
        order = torch.from_numpy(rng.permutation(n)).to(torch.int32)
        groups = torch.cat([order, order[-1:].repeat(K * S - n)])   # a plan with padding
        sh = LevelShard.from_env()
        it, cv, en, qq = sh.solve(_fake_solve_tensors(coords, S), groups, K, S)
        q.put((rank, it.tolist(), cv.tolist(), en.tolist(), qq.tolist(), sh.last_load))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,S,world", [(37, 8, 2), (5, 4, 2), (130, 16, 3)])
def test_level_shard_equals_single_rank(n, S, world):
    import torch

    from paper_1705_02003_b200.dist import LevelShard

    M = 3
    rng = np.random.default_rng(1)
    coords = torch.from_numpy(rng.uniform(-1, 1, (n, M)))
    K = -(-n // S)
    order = torch.from_numpy(rng.permutation(n)).to(torch.int32)
    groups = torch.cat([order, order[-1:].repeat(K * S - n)])
    want = LevelShard(0, 1).solve(_fake_solve_tensors(coords, S), groups, K, S)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_level_worker, args=(r, world, port, n, S, M, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, it, cv, en, qq, load in got:
        assert it == want[0].tolist() and cv == want[1].tolist()
        assert en == want[2].tolist() and qq == want[3].tolist()   # bitwise
        assert load["groups"] == [len(my_groups(K, r, world)) for r in range(world)]
        assert sum(load["group_iterations"]) == int(want[2].sum())
