"""Benchmark: ensemble sample-solves/s of one adaptive level (BASELINE.json metric).

One *step* = the hot path over one level's batch of samples: device stable
sort of the surrogate keys + chunking into width-S groups, KL coefficient at
every node, sample-interleaved assembly of every group's operator, batched
Jacobi-PCG of all groups to their own termination, per-lane QoI.  The
workload (default C2: n=256, M=4, S=16, rtol 1e-8, adaptive grid to total
level 5) is the last adaptive level of the study: levels 1..L-1 are solved in
the untimed setup to fit the iteration surrogate that keys the final level.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

N>1 (torchrun): weak scaling - rank r solves the final level's sample set
reflected through the sign pattern of r's bits (same grid, same shape of
work, distinct samples), no collective on the solve path; the step time is
the max over ranks.  Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
WORKLOADS = ROOT / "bench_workloads"
# BASELINE.json's metric, verbatim (value = ensemble sample-solves/s; the
# SpMV/PCG HBM GB/s vs peak part is reported in `roofline` / `pcg_loop`)
METRIC = "ensemble sample-solves/s at 1/2/4/8 B200; SpMV+PCG HBM GB/s vs peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--separate-kernel-timing", action="store_true",
                    help="(default behaviour; kept for old command lines) value from "
                         "un-instrumented steps, kernel breakdown from a profiled pass")
    ap.add_argument("--max-iters", type=int, default=None,
                    help="throughput mode: run exactly this many PCG iterations per group "
                         "(value = sample-iterations/s); for C4/C5 where full solves take minutes")
    ap.add_argument("--max-samples", type=int, default=None,
                    help="use only the first samples of the workload")
    ap.add_argument("--wave", type=int, default=None,
                    help="max groups per device wave (default: as many as fit in HBM)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# workload

def bytes_model(cfg, op=None, kx=1):
    """Algorithmic bytes per group per launch (DESIGN.md / SURVEY.md 8d).

    CSR operator: the SURVEY 8d figures.  Face-form FV2D operator (``op.faces``):
    the operator stream is ``op.n_op`` doubles per lane (faces) instead of nnz
    values + the int32 graph - the same formula with the smaller operator.
    ``kx`` > 1 (deferred solution update, ``uqg_pcg_x_defer``): the direction
    class moves 4 vector passes per iteration plus, every kx-th iteration, the
    flush (x read + write, kx p reads): (4 + (2 + kx) / kx) passes.
    """
    S, N, nnz = cfg.ensemble_size, cfg.n_dofs, cfg.nnz
    if op is not None and getattr(op, "faces", False):
        n_op, graph = op.n_op, 0
    else:
        n_op, graph = nnz, 4 * nnz + 4 * (N + 1)
    spmv = 8 * S * n_op + graph + 16 * S * N
    update = 4 * 8 * S * N      # read r, Ap, dinv; write r
    if kx > 1:
        direction = int((4 + (2 + kx) / kx) * 8 * S * N)
    else:
        direction = 6 * 8 * S * N   # read x, p, r, dinv; write x, p (x += alpha p deferred here)
    return {"spmv": spmv, "update": update, "dir": direction,
            # SURVEY 8d's algorithmic bytes per PCG iteration (13 vector passes) and
            # the bytes this implementation actually moves (12 passes)
            "pcg_iter": 8 * S * (n_op + 13 * N) + graph,
            "pcg_iter_moved": spmv + update + direction,
            "operator": "fv2d faces" if graph == 0 else "csr",
            **({"flush": kx} if kx > 1 else {})}


def make_workload(cfg, solver=None):
    """(ids, coords (n,M), keys (n,) or None) of the final adaptive level."""
    path = WORKLOADS / f"{cfg.name}.npz"
    if path.exists():
        z = np.load(path)
        keys = z["keys"] if z["keys"].size else None
        return z["ids"].tolist(), z["coords"], keys, json.loads(str(z["meta"]))
    from paper_1705_02003_b200.driver import adaptive_run, sample_set
    if cfg.synthetic_samples:
        coords = sample_set(cfg)
        ids, keys, meta = list(range(len(coords))), None, {"source": "seeded U[-1,1]^M, rng 0"}
    else:
        # the study's last level: its samples and the surrogate keys that grouped it
        t0 = time.time()
        records, stop, grid = adaptive_run(cfg, solver)
        last = records[-1]
        ids, coords = list(last.ids), np.asarray(last.coords)
        keys = None if last.predicted is None else np.asarray(last.predicted)
        meta = {"source": f"adaptive study solved on device: levels "
                          f"{[len(r.ids) for r in records]} samples ({stop}, "
                          f"{time.time() - t0:.1f}s); workload = level {last.level}",
                "levels": [len(r.ids) for r in records]}
    if int(os.environ.get("RANK", "0")) == 0:  # every rank computes the same; one writes
        WORKLOADS.mkdir(exist_ok=True)
        tmp = path.with_suffix(".tmp.npz")
        np.savez(tmp, ids=np.array(ids), coords=coords,
                 keys=np.array([]) if keys is None else keys, meta=json.dumps(meta))
        os.replace(tmp, path)
    return ids, coords, keys, meta


def reflect(coords, rank):
    """Rank-specific reflection y_d -> -y_d for the set bits of rank (weak scaling)."""
    if rank == 0:
        return coords
    signs = np.array([-1.0 if (rank >> d) & 1 else 1.0 for d in range(coords.shape[1])])
    return coords * signs


# ---------------------------------------------------------------------------
# clocks

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.proc, self.lines = index, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.index)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU legs (oracle = the reference algorithm restated; test infra, used here
# only as the timed CPU baseline)

_CPU_SETUP = {}


def _cpu_setup(cfg_name):
    """One-time per-process setup of the CPU path (field, mesh, mode table) -
    excluded from the timed steps like the device arm's."""
    if cfg_name not in _CPU_SETUP:
        from threadpoolctl import threadpool_limits

        from oracle import fv2d as ofv, field2d
        from paper_1705_02003_b200.configs import get

        cfg = get(cfg_name)
        with threadpool_limits(limits=1):
            fld = field2d.KL2D.select(**cfg.field_kwargs())
            mesh = ofv.Mesh2D(cfg.cells)
            _CPU_SETUP[cfg_name] = (cfg, fld, mesh, fld.mode_table(mesh.node_points))
    return _CPU_SETUP[cfg_name]


def _cpu_warm(cfg_name):
    _cpu_setup(cfg_name)
    return os.getpid()


def _cpu_group_worker(args):
    cfg_name, samples = args
    from threadpoolctl import threadpool_limits

    from oracle import fv2d as ofv, pcg as opcg

    cfg, fld, mesh, table = _cpu_setup(cfg_name)
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        sysm = ofv.assemble(mesh, fld, samples, table, cfg.a2)
        res = opcg.pcg(sysm.row_offsets, sysm.col_indices, sysm.values, sysm.rhs, tol=cfg.tol,
                       maxit=cfg.maxit)
        q = [ofv.qoi(u) for u in res.solution]
        return time.perf_counter() - t0, res.ensemble_iterations, q


def cpu_plan(cfg, coords, keys):
    from oracle import grouping as ogrp
    ids = list(range(len(coords)))
    if keys is None:
        return ogrp.natural(ids, cfg.ensemble_size)[0]
    return ogrp.by_key(ids, dict(zip(ids, keys)), cfg.ensemble_size)[0]


def cpu_baseline(cfg, coords, keys):
    """Oracle port, 1 thread, one median-cost group of the same level."""
    ens = cpu_plan(cfg, coords, keys)
    g = ens[len(ens) // 2]
    dt, its, _ = _cpu_group_worker((cfg.name, coords[list(g)]))
    S = cfg.ensemble_size
    return {"value": S / dt, "unit": "sample-solves/s", "cores": 1, "kind": "port",
            "sample": f"1 group (S={S}) of the {cfg.name} final level (group {len(ens) // 2} of "
                      f"{len(ens)} in surrogate order): 2D KL + assembly + Jacobi-PCG "
                      f"({its} iterations) + QoI, oracle/ numpy+scipy, 1 thread, {dt:.1f}s"}


def run_reference(args, cfg):
    """--impl reference: the CPU path on all host cores (multiprocessing, 1 thread each)."""
    import multiprocessing as mproc

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    ids, coords, keys, meta = make_workload(cfg)
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    ens = cpu_plan(cfg, coords, keys)
    t_group = time.perf_counter() - t0
    P = max(1, min(cores, len(ens)))
    steps = max(1, min(args.steps, 3))
    times, done = [], 0
    ctx = mproc.get_context("spawn")
    with ctx.Pool(P) as pool:
        # untimed warm-up: worker start-up and the per-process setup
        warm = 1 if args.warmup > 0 else 0
        if warm:
            pool.map(_cpu_warm, [cfg.name] * P, chunksize=1)
        for st in range(steps):
            chosen = [ens[(st * P + j) % len(ens)] for j in range(P)]
            t0 = time.perf_counter()
            out = pool.map(_cpu_group_worker, [(cfg.name, coords[list(g)]) for g in chosen])
            times.append(time.perf_counter() - t0 + t_group)
            done += P * cfg.ensemble_size
    total = sum(times)
    value = done / total
    S = cfg.ensemble_size
    line = {
        "impl": "reference", "metric": METRIC, "value": value,
        "unit": "sample-solves/s", "n_gpus": args.gpus, "steps": steps, "warmup": warm,
        "ms_per_step": 1e3 * total / steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg.name} final adaptive level, {P} groups per step",
                   "n": cfg.cells, "M": cfg.n_modes, "S": S, "rtol": cfg.tol},
        "cpu_baseline": {"value": value, "unit": "sample-solves/s", "cores": P, "kind": "port",
                         "sample": f"{P} groups x S={S} per step (one group per process, "
                                   "1 BLAS thread each) of the final level; oracle/ restatement "
                                   "of uqgroup's path (reference is pure Python; its 2D operator "
                                   "does not exist, see DESIGN.md)"},
        "e2e": {"value": value, "unit": "sample-solves/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm

def main():
    args = parse()
    from paper_1705_02003_b200.configs import get
    cfg = get(args.config)
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # Test hook (not used by the driver): UQG_BENCH_SHARE_GPU=1 puts every rank on
    # cuda:0 with gloo, to exercise the N>1 code path on a 1-GPU box (no rank's
    # kernels ever wait on another rank's, so sharing a GPU is safe).
    share = os.environ.get("UQG_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_1705_02003_b200 as uq
    from paper_1705_02003_b200 import _lib
    from paper_1705_02003_b200.build import needs_build, build

    if needs_build():
        build()
    field = uq.build_field(**cfg.field_kwargs())
    solver = uq.EnsembleSolver2D(field, cfg.cells, cfg.tol, cfg.maxit, cfg.a2,
                                 max_groups_per_wave=args.wave)
    ids, coords, keys, meta = make_workload(cfg, solver)
    if args.max_iters:
        # throughput mode (C4/C5: a full solve of a level takes minutes): every
        # group runs exactly max_iters PCG iterations; `value` then counts
        # sample-iterations, not sample-solves, and says so in `unit`
        solver.maxit = args.max_iters
        solver.tol = 1e-300
    if args.max_samples and len(ids) > args.max_samples:
        ids, coords = ids[: args.max_samples], coords[: args.max_samples]
        keys = None if keys is None else keys[: args.max_samples]
    # weak scaling: rank r solves the mirror images of the level's samples and
    # groups them by the keys of their originals (same sort work, same costs shape)
    coords = reflect(coords, rank)
    n, S = len(ids), cfg.ensemble_size
    dev = _lib.device()
    coll_dev = torch.device("cpu") if share else dev  # gloo test hook collects on the host
    d_coords = torch.from_numpy(np.ascontiguousarray(coords)).to(dev)
    d_keys = None if keys is None else torch.from_numpy(np.ascontiguousarray(keys)).to(dev)
    lib, ctx = _lib.load(), _lib.ctx()
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    def step():
        out = solver.run_level_device(d_coords, n, S, d_keys)
        if world > 1:
            # the study's one collective: per-slot iterations + QoIs of every rank's
            # groups allgathered (NCCL) for the surrogate refit (harness.py:658-660)
            groups, pad, it, cv, en, q = out
            mine = torch.cat([it.double(), q]).to(coll_dev)
            allv = torch.empty(world * mine.numel(), dtype=mine.dtype, device=coll_dev)
            dist.all_gather_into_tensor(allv, mine)
        return out

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    import ctypes
    NK = 10

    def timed(profile: bool):
        """K timed steps; per-launch CUDA-event kernel timing when `profile`."""
        ms = (ctypes.c_double * NK)()
        cnt = (ctypes.c_longlong * NK)()
        lib.uqg_ctx_profile_read(ctx, ms, cnt, 1)
        lib.uqg_ctx_profile(ctx, int(profile))
        launches0 = lib.uqg_ctx_launch_count(ctx)
        times, group_iters, last = [], 0, None
        with ClockSampler(torch.cuda.current_device()) as clocks:
            for _ in range(args.steps):
                barrier()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                last = step()
                e1.record(stream)
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1)
                if world > 1:
                    tt = torch.tensor([t], device=coll_dev)
                    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                    t = float(tt.item())
                times.append(t)
                group_iters += int(last[4].sum().item())
                barrier()
        launches = lib.uqg_ctx_launch_count(ctx) - launches0
        lib.uqg_ctx_profile_read(ctx, ms, cnt, 1)
        lib.uqg_ctx_profile(ctx, 0)
        return times, group_iters, launches, ms, cnt, clocks, last

    # value from un-instrumented steps (the library solves a level's groups as
    # concurrent parts on several streams); the per-kernel times for the
    # roofline from an identical profiled pass on ONE stream, so each launch's
    # duration is that kernel's alone (UQG_SOLVE_STREAMS=1; same results).
    times, group_iters, launches, _, _, clocks, last = timed(False)
    prev = os.environ.get("UQG_SOLVE_STREAMS")
    os.environ["UQG_SOLVE_STREAMS"] = "1"
    try:
        _, prof_iters, _, ms, cnt, _, _ = timed(True)
    finally:
        if prev is None:
            os.environ.pop("UQG_SOLVE_STREAMS", None)
        else:
            os.environ["UQG_SOLVE_STREAMS"] = prev
    assert prof_iters == group_iters
    groups, pad, it, cv, en, q = last
    conv_all = bool(cv.all().item())

    # ---- end to end through the public API: host inputs, host results -------
    e2e_steps = args.e2e_steps or args.steps
    e2e_t = []
    for _ in range(e2e_steps):
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plan, iters, qois, notes = solver.solve_level(ids, coords, S, keys=keys, level=99)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if world > 1:
            tt = torch.tensor([dt], device=coll_dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
        e2e_t.append(dt)
    K = len(plan.ensembles)
    h2d = coords.nbytes + (0 if keys is None else 8 * n)
    d2h = 8 * (K * S * 4 + K)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    total_ms = sum(times)
    value = world * n * len(times) / (total_ms / 1e3)
    unit = "sample-solves/s"
    if args.max_iters:  # throughput mode: sample-iterations per second
        value *= args.max_iters
        unit = f"sample-iterations/s (throughput mode: {args.max_iters} PCG iterations per group)"
    bm = bytes_model(cfg, solver.op, int(lib.uqg_pcg_x_defer()))
    peaks = {}
    pk = ROOT / "MEASURED_PEAKS.json"
    if pk.exists():
        peaks = json.loads(pk.read_text())
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    traffic_all = {}
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        traffic_all = json.loads(tf.read_text())
    # per-kernel rooflines of the three PCG kernels; the line's "roofline" is the
    # one with the largest measured time share (the dominant kernel)
    spmv_name = "pcg_spmv_fv2d_kernel" if bm["operator"] != "csr" else "pcg_spmv_tma_kernel"
    per = {}
    dir_name = "pcg_dir_kernel" + (" + pcg_flush_kernel" if "flush" in bm else "")
    for key, idx, kname in (("spmv", 3, spmv_name), ("update", 4, "pcg_update_kernel"),
                            ("dir", 5, dir_name)):
        t_ms = ms[idx]
        gbs = group_iters * bm[key] / (t_ms / 1e3) / 1e9 if t_ms else None
        tr = traffic_all.get(f"{cfg.name}:{kname}", {})
        per[key] = {"kernel": kname, "ms": t_ms, "achieved": gbs,
                    "frac": gbs / peak if gbs else None,
                    "bytes_per_group_launch": bm[key],
                    "traffic": tr.get("dram_bytes_per_launch"),
                    "traffic_algorithmic_same_launch": tr.get("algorithmic_bytes_per_launch"),
                    "traffic_source": tr.get("source")}
    if cnt[3] and not cnt[4] and not cnt[5]:
        # small batches: the whole solve is ONE persistent launch (cluster or
        # cooperative kernel; SpMV, update and direction as phases of each
        # iteration, x updated in place) - its roofline is the loop's
        bm1 = bytes_model(cfg, solver.op, 1)
        b_it = bm1["spmv"] + bm1["update"] + bm1["dir"]
        gbs = group_iters * b_it / (ms[3] / 1e3) / 1e9 if ms[3] else None
        tr = traffic_all.get(f"{cfg.name}:pcg_persistent_kernel", {})
        per = {"persistent": {
            "kernel": "pcg_persistent_kernel (whole solve; per group-iteration: SpMV + update "
                      "+ direction phases)",
            "ms": ms[3], "achieved": gbs, "frac": gbs / peak if gbs else None,
            "bytes_per_group_launch": b_it,
            "traffic": tr.get("dram_bytes_per_launch"),
            "traffic_algorithmic_same_launch": tr.get("algorithmic_bytes_per_launch"),
            "traffic_source": tr.get("source")}}
    dom = max(per, key=lambda k: per[k]["ms"] or 0.0)
    loop_ms = ms[3] + ms[4] + ms[5]
    loop_gbs = group_iters * bm["pcg_iter"] / (loop_ms / 1e3) / 1e9 if loop_ms else None
    step_gbs = group_iters * bm["pcg_iter"] / (total_ms / 1e3) / 1e9
    kern = {name: {"ms": ms[k], "launches": int(cnt[k])} for k, name in enumerate(
        ["kl", "assemble", "pcg_init", "pcg_spmv", "pcg_update", "pcg_dir", "dot_qoi", "group",
         "spmv", "other"]) if cnt[k]}
    line = {
        "metric": METRIC,
        "value": value,
        "unit": unit,
        "n_gpus": world,
        "steps": len(times),
        "warmup": max(3, args.warmup),
        "ms_per_step": total_ms / len(times),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{cfg.name}: final adaptive level ({n} samples/rank, {K} groups "
                               f"of S={S}) - group sort + KL + assembly + batched Jacobi-PCG + QoI",
                   "n": cfg.cells, "unknowns": cfg.n_dofs, "M": cfg.n_modes, "S": S,
                   "rtol": cfg.tol, "delta": cfg.delta, "sigma": cfg.sigma0,
                   "parallelism": f"groups sharded weak x{world}",
                   "l2": "inputs larger than L2 (operator+vectors of all groups ~"
                         f"{solver.bytes_per_group(S) * K / 1e9:.1f} GB per step)",
                   "workload_source": meta.get("source")},
        "gpu_launches": int(launches),
        "e2e": {"value": world * n * len(e2e_t) / sum(e2e_t) * (args.max_iters or 1),
                "unit": unit,
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        "roofline": {"bound": "hbm", "kernel": per[dom]["kernel"], "operator": bm["operator"],
                     "achieved": per[dom]["achieved"], "peak": peak, "unit": "GB/s",
                     "frac": per[dom]["frac"], "traffic": per[dom]["traffic"],
                     "traffic_algorithmic_same_launch": per[dom]["traffic_algorithmic_same_launch"],
                     "traffic_source": per[dom]["traffic_source"],
                     "peak_source": peak_src,
                     # also against the 8 TB/s HBM3e specification
                     "peak_spec": 8000.0,
                     "frac_spec": (per[dom]["achieved"] / 8000.0) if per[dom]["achieved"] else None,
                     "bytes_per_group_launch": per[dom]["bytes_per_group_launch"],
                     "group_launches": group_iters,
                     "timing": "per-launch CUDA events on the launching stream, profiled pass "
                               "with the level on one stream (UQG_SOLVE_STREAMS=1)",
                     "time_share": (per[dom]["ms"] / sum(ms[k] for k in range(NK))
                                    if sum(ms[k] for k in range(NK)) else None),
                     "pcg_kernels": per},
        "pcg_loop": {"achieved_gbs": loop_gbs, "frac": loop_gbs / peak if loop_gbs else None,
                     "bytes_per_group_iter": bm["pcg_iter"],
                     "moved_gbs": (loop_gbs * bm["pcg_iter_moved"] / bm["pcg_iter"])
                     if loop_gbs else None,
                     "moved_bytes_per_group_iter": bm["pcg_iter_moved"], "step_gbs": step_gbs,
                     "group_iterations": group_iters},
        "kernels": kern,
        "all_converged": conv_all,
        "clocks": clocks.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, coords, keys)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
