"""Time the persistent small-batch solves (C1 shape) against the number of
groups, for one UQG_PCG_PERSISTENT mode (set in the environment):

    UQG_PCG_PERSISTENT=3 python tools/persistent_probe.py

Prints per K: ms per solve (device-resident samples, median of 5) and us per
iteration of the slowest group.  Tuning tool; not a bench value.
"""

from __future__ import annotations

import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import numpy as np
    import torch

    import paper_1705_02003_b200 as uq
    from paper_1705_02003_b200 import _lib

    cfg = uq.CONFIGS["C1"]
    s = cfg.make_solver()
    mode = os.environ.get("UQG_PCG_PERSISTENT", "auto")
    for K in (1, 2, 4, 7, 8, 14, 22):
        ys = np.random.default_rng(K).uniform(-1, 1, (K * cfg.ensemble_size, cfg.n_modes))
        d = _lib.to_dev(ys)
        out = s.solve_wave(d, K, cfg.ensemble_size)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            out = s.solve_wave(d, K, cfg.ensemble_size)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        its = int(out[3].max())
        ms = float(np.median(ts)) * 1e3
        print(f"mode {mode} K={K:2d}: {ms:7.3f} ms, max its {its}, {ms * 1e3 / its:6.2f} us/it")


if __name__ == "__main__":
    main()
