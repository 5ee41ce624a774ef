"""One warm-up + one timed level step of a bench workload, for ncu captures.

    python tools/profile_step.py [--config C2] [--wave G]

Prints the step time; meant to be wrapped by ncu (never a bench number).
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--wave", type=int, default=None)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--maxit", type=int, default=None,
                    help="cap PCG iterations per group (KL / assembly captures at C4/C5)")
    a = ap.parse_args()
    import torch

    import bench
    import paper_1705_02003_b200 as uq
    from paper_1705_02003_b200.configs import get

    cfg = get(a.config)
    f = uq.build_field(**cfg.field_kwargs())
    solver = uq.EnsembleSolver2D(f, cfg.cells, cfg.tol, cfg.maxit, cfg.a2,
                                 max_groups_per_wave=a.wave)
    ids, coords, keys, _ = bench.make_workload(cfg, solver)
    if a.maxit:
        solver.maxit, solver.tol = a.maxit, 1e-300
    dev = torch.device("cuda", 0)
    d_c = torch.from_numpy(coords).to(dev)
    d_k = None if keys is None else torch.from_numpy(keys).to(dev)
    solver.run_level_device(d_c, len(ids), cfg.ensemble_size, d_k)
    torch.cuda.synchronize()
    for _ in range(a.steps):
        t0 = time.perf_counter()
        out = solver.run_level_device(d_c, len(ids), cfg.ensemble_size, d_k)
        torch.cuda.synchronize()
        print(f"step {time.perf_counter() - t0:.3f}s groups={out[1].numel()} "
              f"group_iters={int(out[4].sum())}")


if __name__ == "__main__":
    main()
