"""Probe: does splitting one level's groups over two concurrent PCG solves
(two contexts, two streams, two host threads) raise throughput?  Tuning tool.

    python tools/two_stream_probe.py [--config C2] [--reps 2]
"""

from __future__ import annotations

import argparse
import ctypes
import sys
import threading
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--parts", type=int, nargs="+", default=[2])
    args = ap.parse_args()
    import torch

    import bench
    from paper_1705_02003_b200 import _lib
    from paper_1705_02003_b200.configs import get
    from paper_1705_02003_b200.grouping import group_by_key

    cfg = get(args.config)
    solver = cfg.make_solver()
    ids, coords, keys, _ = bench.make_workload(cfg, solver)
    S = cfg.ensemble_size
    plan = group_by_key(ids, {i: float(k) for i, k in zip(ids, keys)}, S)
    samples = np.array([[coords[ids.index(s)] for s in g] for g in plan.ensembles])
    G = len(samples)
    op = solver.op
    lib = _lib.load()
    dev = _lib.device()
    d_y = _lib.to_dev(samples.reshape(G * S, -1))
    a = torch.empty(G * op.n_coef * S, dtype=torch.float64, device=dev)
    F = op.n_faces
    tx = torch.empty(G * F * S, dtype=torch.float64, device=dev)
    dinv = torch.empty(G * op.n_dofs * S, dtype=torch.float64, device=dev)
    op.coefficients(d_y, None, G, S, a)
    op.assemble_faces(a, G, S, tx, None, dinv)
    torch.cuda.synchronize()
    N = op.n_dofs

    def solve(ctx, stream, g0, g1, out):
        n = g1 - g0
        x = torch.empty(n * N * S, dtype=torch.float64, device=dev)
        it = torch.empty(n * S, dtype=torch.int32, device=dev)
        cv = torch.empty(n * S, dtype=torch.uint8, device=dev)
        fz = torch.empty(n * S, dtype=torch.uint8, device=dev)
        en = torch.empty(n, dtype=torch.int32, device=dev)
        rows = ctypes.c_int(0)
        rc = lib.uqg_pcg_fv2d(ctx, cfg.cells, S, n, tx[g0 * F * S:].data_ptr(), None,
                              float(op.field.a_y), None, float(op.rhs_const),
                              dinv[g0 * N * S:].data_ptr(), float(cfg.tol), int(cfg.maxit),
                              x.data_ptr(), it.data_ptr(), cv.data_ptr(), fz.data_ptr(),
                              en.data_ptr(), None, 0, ctypes.byref(rows), stream)
        out.append((rc, it))

    ctxs = [_lib.ctx()]
    streams = [torch.cuda.Stream()]
    for _ in range(max(args.parts) - 1):
        c = ctypes.c_void_p()
        _lib.check(lib.uqg_ctx_create(torch.cuda.current_device(), ctypes.byref(c)))
        ctxs.append(c.value)
        streams.append(torch.cuda.Stream())
    for rep in range(args.reps):
        out = []
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        solve(ctxs[0], streams[0].cuda_stream, 0, G, out)
        torch.cuda.synchronize()
        t_one = time.perf_counter() - t0
        line = f"rep {rep}: one solve {t_one * 1e3:.0f} ms"
        for k in args.parts:
            out = []
            bounds = [G * i // k for i in range(k + 1)]
            t0 = time.perf_counter()
            th = [threading.Thread(target=solve, args=(ctxs[i], streams[i].cuda_stream,
                                                        bounds[i], bounds[i + 1], out))
                  for i in range(k)]
            for t in th:
                t.start()
            for t in th:
                t.join()
            torch.cuda.synchronize()
            assert all(rc == 0 for rc, _ in out), out
            line += f", {k} concurrent parts {(time.perf_counter() - t0) * 1e3:.0f} ms"
        print(line + f" ({G} groups)", flush=True)


if __name__ == "__main__":
    main()
