"""Multi-rank path on the GPU box: the C1 study with each level's groups sharded
over 2 ranks (one allgather per level) reproduces the single-rank reference
golden; one bench level sharded over 2 ranks (the strong-scaling bench step)
is bit-identical to one rank; and `bench.py` runs under torchrun with N=2.  Both ranks share cuda:0
with gloo (UQG_BENCH_SHARE_GPU=1) because the box has one GPU; no rank's
kernels wait on another's, so this is safe."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return str(s.getsockname()[1])


def _torchrun(args, env_extra, timeout=900):
    env = dict(os.environ, UQG_BENCH_SHARE_GPU="1", **env_extra)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", _port(), *args]
    return subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=timeout)


def test_sharded_study_matches_single_rank_golden(tmp_path, c1_golden):
    out = tmp_path / "dist.json"
    r = _torchrun([str(ROOT / "tools" / "dist_study.py"), "--config", "C1", "--out", str(out)], {})
    assert r.returncode == 0, r.stderr[-3000:]
    doc = json.loads(out.read_text())
    assert doc["world"] == 2
    assert len(doc["levels"]) == len(c1_golden["levels"])
    for got, gold in zip(doc["levels"], c1_golden["levels"]):
        assert got["ids"] == gold["ids"]
        assert got["ensembles"] == gold["ensembles"]
        assert max(abs(a - b) for a, b in zip(got["iterations"], gold["iterations"])) <= 1
        assert max(abs(a - b) / abs(b) for a, b in zip(got["qoi"], gold["qoi"])) <= 1e-8


def test_sharded_level_bitwise_equals_single_rank(tmp_path):
    """The bench's strong-scaling step (LevelShard over 2 ranks) returns the
    whole level bit-identical to one rank's run_level_device."""
    import numpy as np
    import torch

    from paper_1705_02003_b200.configs import get

    out = tmp_path / "lvl.json"
    r = _torchrun([str(ROOT / "tools" / "dist_level.py"), "--config", "C1", "--out", str(out)], {})
    assert r.returncode == 0, r.stderr[-3000:]
    doc = json.loads(out.read_text())
    assert doc["world"] == 2
    cfg = get("C1")
    z = np.load(ROOT / "bench_workloads" / "C1.npz")
    solver = cfg.make_solver()
    dev = torch.device("cuda", 0)
    groups, pad, it, cv, en, q = solver.run_level_device(
        torch.from_numpy(z["coords"]).to(dev), len(z["coords"]), cfg.ensemble_size,
        torch.from_numpy(z["keys"]).to(dev))
    assert doc["groups"] == groups.tolist()
    assert doc["iters"] == it.tolist() and doc["conv"] == cv.tolist()
    assert doc["ens"] == en.tolist()
    assert doc["qoi"] == q.tolist()  # bitwise
    K = pad.numel()
    assert doc["load"]["groups"] == [len(range(0, K, 2)), len(range(1, K, 2))]


def test_nccl_collectives_on_one_gpu(tmp_path):
    """The NCCL calls the N-GPU step makes - init with device_id, the level's
    all_gather_into_tensor of float64 rows on the device, barrier, MAX
    all-reduce - executed by one rank on the box's GPU (NCCL refuses two ranks
    on one device): same results as the plain single-process level."""
    import numpy as np
    import torch

    from paper_1705_02003_b200.configs import get

    out = tmp_path / "nccl.json"
    env = {k: v for k, v in os.environ.items() if k != "UQG_BENCH_SHARE_GPU"}
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", _port(),
           str(ROOT / "tools" / "dist_level.py"), "--config", "C1", "--out", str(out),
           "--force-collective"]
    r = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    doc = json.loads(out.read_text())
    assert doc["world"] == 1 and doc["backend"] == "nccl"
    cfg = get("C1")
    z = np.load(ROOT / "bench_workloads" / "C1.npz")
    dev = torch.device("cuda", 0)
    solver = cfg.make_solver()
    groups, pad, it, cv, en, q = solver.run_level_device(
        torch.from_numpy(z["coords"]).to(dev), len(z["coords"]), cfg.ensemble_size,
        torch.from_numpy(z["keys"]).to(dev))
    assert doc["groups"] == groups.tolist() and doc["iters"] == it.tolist()
    assert doc["ens"] == en.tolist() and doc["qoi"] == q.tolist()
    assert doc["load"]["groups"] == [len(doc["ens"])]


def test_bench_runs_with_two_ranks():
    r = _torchrun([str(ROOT / "bench.py"), "--gpus", "2", "--config", "C1", "--steps", "2",
                   "--warmup", "3"], {})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "strong"
    assert sum(d["shards"]["groups_per_rank"]) == 22  # the C1 level's groups, split over 2
    assert d["parity"]["ok"], d["parity"]


def test_bench_weak_scaling_opt_in():
    r = _torchrun([str(ROOT / "bench.py"), "--gpus", "2", "--config", "C1", "--steps", "2",
                   "--warmup", "3", "--scaling", "weak"], {})
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    assert d["scaling"] == "weak" and d["value"] > 0
