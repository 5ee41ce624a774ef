"""Run an adaptive study with the level's groups sharded over torch.distributed
ranks (one allgather per level) and write rank 0's per-level results.

    torchrun --nproc-per-node N tools/dist_study.py --config C1 --out out.json

With UQG_BENCH_SHARE_GPU=1 every rank uses cuda:0 and the gloo backend (for a
1-GPU box; ranks never wait on each other's kernels).  Otherwise NCCL, one GPU
per rank.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    share = os.environ.get("UQG_BENCH_SHARE_GPU") == "1"
    local = 0 if share else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if share:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    from paper_1705_02003_b200.configs import get
    from paper_1705_02003_b200.dist import ShardedSolver
    from paper_1705_02003_b200.driver import adaptive_run

    cfg = get(a.config)
    solver = cfg.make_solver()
    sharded = ShardedSolver(solver.solve_groups, solver.collect,
                            device=None if share else dev)
    records, stop, _ = adaptive_run(cfg, solver, shard=sharded.solve_plan)
    if dist.get_rank() == 0:
        doc = [{"level": r.level, "ids": r.ids, "ensembles": [list(g) for g in r.ensembles],
                "iterations": [r.iterations[s] for s in r.ids],
                "qoi": [r.qois[s] for s in r.ids]} for r in records]
        Path(a.out).write_text(json.dumps({"world": dist.get_world_size(), "stop": stop,
                                           "levels": doc}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
