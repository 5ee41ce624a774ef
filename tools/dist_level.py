"""One bench workload level solved with its groups sharded over torch.distributed
ranks (``dist.LevelShard``: round robin + one all_gather_into_tensor) - the
bench's strong-scaling step - writing rank 0's whole-level results.

    torchrun --nproc-per-node N tools/dist_level.py --config C1 --out out.json

With UQG_BENCH_SHARE_GPU=1 every rank uses cuda:0 and gloo (1-GPU box).
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
    ap.add_argument("--force-collective", action="store_true",
                    help="issue the all-gather (and a barrier / MAX all-reduce as bench.py "
                         "does) even with one rank: the single-GPU NCCL check")
    a = ap.parse_args()
    import numpy as np
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
    from paper_1705_02003_b200.dist import LevelShard

    cfg = get(a.config)
    z = np.load(ROOT / "bench_workloads" / f"{cfg.name}.npz")
    coords, keys = z["coords"], z["keys"]
    solver = cfg.make_solver()
    shard = LevelShard.from_env(coll_device=torch.device("cpu") if share else dev)
    shard.force_collective = a.force_collective
    d_c = torch.from_numpy(coords).to(dev)
    d_k = torch.from_numpy(keys).to(dev) if keys.size else None
    groups, pad, it, cv, en, q = solver.run_level_device(d_c, len(coords), cfg.ensemble_size, d_k,
                                                         shard)
    if a.force_collective:  # the bench's other collectives, same tensors and devices
        dist.barrier()
        tt = torch.tensor([1.25], device=shard.coll_device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        assert float(tt.item()) == 1.25
    if dist.get_rank() == 0:
        Path(a.out).write_text(json.dumps({
            "world": dist.get_world_size(), "groups": groups.tolist(), "iters": it.tolist(),
            "conv": cv.tolist(), "ens": en.tolist(), "qoi": q.tolist(), "load": shard.last_load,
            "backend": dist.get_backend()}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
