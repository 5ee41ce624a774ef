"""Benchmark: ensemble sample-solves/s of one adaptive level (BASELINE.json metric).

One *step* = the hot path over one level's batch of samples: device stable
sort of the surrogate keys + chunking into width-S groups, KL coefficient at
every node, sample-interleaved assembly of every group's operator, batched
Jacobi-PCG of all groups to their own termination, per-lane QoI.  The
workload (default C3: n=512, M=6, sigma=1.5, S=32, rtol 1e-8 - the config
BASELINE.json's 1/2/4/8-GPU metric is quoted on) is the study's last adaptive
level (``bench_workloads/C3.npz``: its samples and the surrogate keys that
grouped it).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3]
                    [--impl ours|reference] [--scaling strong|weak]

N>1 (torchrun, one rank per GPU, NCCL): strong scaling by default - every
rank builds the identical plan, solves the groups k = rank (mod N) of it
(``dist.LevelShard``) and one ``all_gather_into_tensor`` returns the whole
level's iterations and QoIs to every rank (the input of the surrogate
refit); the step time is the max over ranks.  ``--scaling weak`` gives every
rank a mirrored copy of the whole level instead.  Prints ONE JSON line on
rank 0.  ``--impl reference`` times the reference's CPU path (the oracle
port: uqgroup's algorithm with scipy csr_matvec and numpy dots) on every host
core on the same workload and config.
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
from types import SimpleNamespace

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
WORKLOADS = ROOT / "bench_workloads"
GOLDEN = ROOT / "tests" / "golden"
# BASELINE.json's metric, verbatim (value = ensemble sample-solves/s; the
# SpMV/PCG HBM GB/s vs peak part is reported in `roofline` / `pcg_loop`)
METRIC = "ensemble sample-solves/s at 1/2/4/8 B200; SpMV+PCG HBM GB/s vs peak"

# CPU legs: PCG iterations timed per group (None = full solve).  Full solves
# of a C2-C5 group take 15 s to many minutes on one core, so the
# CPU legs time a fixed number of iterations per group and project the full
# solve with the reference's own iteration count for that group
# (tests/golden, from uqgroup's ensemble_pcg) - BASELINE.md 4.
REF_ITERS = {"C1": None, "C2": 40, "C3": 8, "C4": 3, "C5": 2}      # --impl reference, per step
BASE_ITERS = {"C1": None, "C2": None, "C3": 30, "C4": 6, "C5": 3}  # cpu_baseline (1 core)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N>1: strong = the level's groups sharded over ranks + one allgather "
                         "(default); weak = every rank solves a mirrored copy of the level")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--prof-steps", type=int, default=1,
                    help="steps of the profiled (per-launch CUDA events, one stream) pass")
    ap.add_argument("--separate-kernel-timing", action="store_true",
                    help="(default behaviour; kept for old command lines)")
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
            # kx > 1, per kernel: pcg_dir_kernel reads p, r, dinv and writes p
            # every iteration; pcg_flush_kernel reads each iteration's p once and
            # reads + writes x once per flush launch
            "dir_only": (4 if kx > 1 else 6) * 8 * S * N,
            "flush_p": 8 * S * N, "flush_x": 16 * S * N,
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
                 "-lms", "20", "-i", str(self.index)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            # wait for the first sample, so short timed regions (C1: ~0.1 s)
            # are sampled from their start
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.01)
            self.lines.clear()
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
# shared by both arms: the config dict, the reference's results, the host

def l2_note(cfg, K) -> str:
    """L2 policy of the timed region (no flush between steps): the level's
    face operator + 5 vectors per group against the 126 MB L2."""
    gb = 8 * cfg.ensemble_size * ((cfg.cells - 1) * cfg.cells + 5 * cfg.n_dofs) * K / 1e9
    if gb > 0.126:
        return (f"inputs larger than L2 (face operator + 5 vectors per group: {gb:.2f} GB per "
                "level, streamed every iteration)")
    return (f"working set {gb:.3f} GB fits in L2; no flush: each step recomputes every input "
            "from the sample coordinates (KL, assembly, PCG from x = 0)")


def config_dict(cfg, n, K, world, scaling, meta, extra=None):
    """The `config` object of the JSON line - identical for both arms."""
    d = {"workload": f"{cfg.name}: final adaptive level ({n} samples, {K} groups of "
                     f"S={cfg.ensemble_size}) - group sort + KL + assembly + batched "
                     "Jacobi-PCG + QoI",
         "n": cfg.cells, "unknowns": cfg.n_dofs, "M": cfg.n_modes, "S": cfg.ensemble_size,
         "rtol": cfg.tol, "delta": cfg.delta, "sigma": cfg.sigma0,
         "parallelism": (f"groups round-robin over {world} GPU(s) + 1 allgather"
                         if scaling == "strong" else f"weak x{world} (mirrored level per rank)"),
         "workload_source": meta.get("source"),
         "l2": l2_note(cfg, K)}
    d.update(extra or {})
    return d


def golden_level(cfg_name, ids, coords):
    """The reference's own results for this workload's level - uqgroup's
    ``group_by_key`` + ``ensemble_pcg`` on the oracle 2D operator, committed by
    ``tests/golden/make_golden.py`` - or None when no fixture covers it.
    Returns {ensembles, iterations {sid: it}, qoi {sid: q}, ensemble_iterations [K]}."""
    ids = [int(i) for i in ids]
    if cfg_name in ("C1", "C2"):
        path = GOLDEN / f"{cfg_name.lower()}_adaptive.json"
        if not path.exists():
            return None
        lv = json.loads(path.read_text())["levels"][-1]
        if lv["ids"] != ids or not np.array_equal(np.asarray(lv["coords"]), coords):
            return None
        return {"ensembles": [list(g) for g in lv["ensembles"]],
                "iterations": dict(zip(lv["ids"], lv["iterations"])),
                "qoi": dict(zip(lv["ids"], lv["qoi"])),
                "ensemble_iterations": lv["ensemble_iterations"], "source": path.name}
    if cfg_name == "C3":
        path = GOLDEN / "c3_level.json"
        if not path.exists():
            return None
        doc = json.loads(path.read_text())
        it, q = {}, {}
        for grp, res in zip(doc["ensembles"], doc["groups"]):
            for s, sid in enumerate(grp):
                if sid not in it:
                    it[sid], q[sid] = res["iterations"][s], res["qoi"][s]
        if sorted(it) != sorted(ids):
            return None
        return {"ensembles": doc["ensembles"], "iterations": it, "qoi": q,
                "ensemble_iterations": [r["ensemble_iterations"] for r in doc["groups"]],
                "source": path.name}
    return None


def parity(gold, ensembles, iters, qois):
    """GPU level vs the reference's: plan identity, per-sample iteration and
    QoI differences (north_star gates: +-1, 1e-8 relative)."""
    if gold is None:
        return None
    same_plan = [list(g) for g in ensembles] == gold["ensembles"]
    d_it = max(abs(iters[s] - gold["iterations"][s]) for s in gold["iterations"])
    d_q = max(abs(qois[s] - gold["qoi"][s]) / abs(gold["qoi"][s]) for s in gold["qoi"])
    return {"reference": f"tests/golden/{gold['source']} (uqgroup group_by_key + ensemble_pcg)",
            "samples": len(gold["iterations"]), "groups": len(gold["ensembles"]),
            "identical_plan": bool(same_plan), "max_iter_diff": int(d_it),
            "max_qoi_rel": float(d_q),
            "ok": bool(same_plan and d_it <= 1 and d_q <= 1e-8)}


def host_info():
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.lower().startswith("model name"):
                model = ln.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return {"cpu_model": model, "cpu_count": os.cpu_count()}


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


REF_PKG = ROOT / "baseline" / "_ref"


def _reference_solver():
    """The reference's own ``EnsembleCsrMatrix`` / ``ensemble_pcg``
    (``ensemble.py:52-281``, unmodified, installed in baseline/_ref by
    tools/stage_reference.py; it travels to the GPU box), or None when it is
    not staged - then the oracle's restatement (oracle/pcg.py) is timed."""
    if not (REF_PKG / "uqgroup").exists():
        return None
    if str(REF_PKG) not in sys.path:
        sys.path.append(str(REF_PKG))
    try:
        from uqgroup import ensemble as ref_ens
    except Exception:  # noqa: BLE001 - fall back to the port
        return None
    return ref_ens


def cpu_path_kind() -> str:
    return "reference" if _reference_solver() is not None else "port"


def _cpu_group_worker(args):
    """One group through the CPU path, 1 thread: the 2D assembly restated in
    oracle/ (the reference has no 2D operator) and the reference's own
    ``ensemble_pcg`` (baseline/_ref; else oracle/pcg.py).  ``maxit`` None:
    full solve.  Otherwise the PCG runs ``maxit`` iterations, and its
    initialisation (Jacobi inverse, r = b, norms) is timed separately by a
    maxit=0 run, so the per-iteration time excludes it."""
    cfg_name, samples, maxit = args
    from threadpoolctl import threadpool_limits

    from oracle import fv2d as ofv, pcg as opcg

    cfg, fld, mesh, table = _cpu_setup(cfg_name)
    ref = _reference_solver()

    def solve(sysm, k):
        if ref is None:
            return opcg.pcg(sysm.row_offsets, sysm.col_indices, sysm.values, sysm.rhs,
                            tol=cfg.tol, maxit=k)
        mat = ref.EnsembleCsrMatrix(sysm.row_offsets, sysm.col_indices, sysm.values)
        r = ref.ensemble_pcg(mat, sysm.rhs, tol=cfg.tol, maxit=k)
        return SimpleNamespace(ensemble_iterations=r.ensemble_iterations,
                               iterations=r.iterations_per_lane, solution=r.solution)

    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        sysm = ofv.assemble(mesh, fld, samples, table, cfg.a2)
        t_asm = time.perf_counter() - t0
        t_init = 0.0
        if maxit is not None:
            t0 = time.perf_counter()
            solve(sysm, 0)
            t_init = time.perf_counter() - t0
        t0 = time.perf_counter()
        res = solve(sysm, cfg.maxit if maxit is None else maxit)
        t_pcg = time.perf_counter() - t0
        t0 = time.perf_counter()
        q = [ofv.qoi(u) for u in res.solution]
        t_qoi = time.perf_counter() - t0
    # fixed-iteration runs: the PCG's initialisation counts as setup, so
    # "pcg" is exactly iters_run iterations
    return {"setup": t_asm + t_init + t_qoi, "pcg": t_pcg - t_init,
            "iters_run": int(res.ensemble_iterations), "full": maxit is None,
            "iterations": [int(v) for v in res.iterations], "qoi": q}


def _projected_seconds(r, its_full):
    """Full-solve seconds of a group from a fixed-iteration sample: setup +
    per-iteration time x the group's full iteration count."""
    if r["full"]:
        return r["setup"] + r["pcg"]
    return r["setup"] + r["pcg"] / max(1, r["iters_run"]) * its_full


def cpu_plan(cfg, coords, keys):
    from oracle import grouping as ogrp
    ids = list(range(len(coords)))
    if keys is None:
        return ogrp.natural(ids, cfg.ensemble_size)[0]
    return ogrp.by_key(ids, dict(zip(ids, keys)), cfg.ensemble_size)[0]


def full_iterations(cfg, plan_rows, gold, keys, max_iters):
    """Per-group full-solve iteration counts used to project fixed-iteration
    CPU samples: the reference's own counts (golden) when they cover the
    workload, else the surrogate's prediction (max key of the group)."""
    if max_iters:
        return [max_iters] * len(plan_rows), f"throughput mode: {max_iters} iterations per group"
    if gold is not None:
        return list(gold["ensemble_iterations"]), f"reference counts, tests/golden/{gold['source']}"
    if keys is not None:
        return ([int(np.ceil(max(keys[j] for j in g))) for g in plan_rows],
                "surrogate-predicted counts (max key per group)")
    return None, "no full iteration counts for this workload"


def cpu_baseline(cfg, ids, coords, keys, gold, max_iters, gpu_rows=None):
    """Oracle port, 1 thread, the median-cost group of the same level (bounded
    ~10-30 s: a full solve at C1/C2, BASE_ITERS iterations projected with the
    reference's iteration count at C3-C5)."""
    ens = cpu_plan(cfg, coords, keys)
    k = len(ens) // 2
    g = ens[k]
    maxit = BASE_ITERS.get(cfg.name)
    if max_iters:
        maxit = min(maxit or max_iters, max_iters)
    r = _cpu_group_worker((cfg.name, coords[list(g)], maxit))
    full, src = full_iterations(cfg, ens, gold, keys, max_iters)
    S = cfg.ensemble_size
    out = {"unit": "sample-solves/s" if not max_iters else "sample-iterations/s", "cores": 1,
           "kind": cpu_path_kind(), "projected": not r["full"], **host_info()}
    if full is None and not r["full"]:
        out.update(value=None, sample="no iteration counts to project a full solve")
        return out
    t = _projected_seconds(r, full[k] if full else r["iters_run"])
    out["value"] = S / t * (max_iters or 1)
    how = ("full solve" if r["full"] else
           f"{r['iters_run']} PCG iterations timed ({r['pcg']:.1f}s) + setup {r['setup']:.1f}s, "
           f"projected to {full[k]} iterations ({src})")
    out["sample"] = (f"group {k} of {len(ens)} (S={S}, median in surrogate order) of the {cfg.name} "
                     f"final level: 2D KL + assembly (oracle/) + Jacobi-PCG ("
                     + ("uqgroup ensemble_pcg, baseline/_ref" if cpu_path_kind() == "reference"
                        else "oracle/pcg.py") + f") + QoI, 1 thread; {how}")
    if r["full"] and gpu_rows is not None:
        it_g, q_g = gpu_rows(k)
        out["parity_vs_gpu"] = {
            "group": k, "max_iter_diff": int(max(abs(a - b) for a, b in zip(it_g, r["iterations"]))),
            "max_qoi_rel": float(max(abs(a - b) / abs(b) for a, b in zip(q_g, r["qoi"])))}
    return out


def run_reference(args, cfg):
    """--impl reference: the CPU path on all host cores (multiprocessing, one
    process per core, 1 BLAS thread each) on the SAME workload and config as
    the GPU arm.  Each step solves a stratified sample of the level's groups
    (every (K/P)-th group in surrogate order, shifted by one per step; never a
    cheapest prefix), one group per process; at C2-C5 each group runs
    REF_ITERS PCG iterations and the step projects the WHOLE level's time from
    the per-iteration rate and every group's full iteration count (the
    reference's own counts, tests/golden) over P cores with perfect load
    balance - which favours the reference."""
    import multiprocessing as mproc

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    ids, coords, keys, meta = make_workload(cfg)
    if args.max_samples and len(ids) > args.max_samples:
        ids, coords = ids[: args.max_samples], coords[: args.max_samples]
        keys = None if keys is None else keys[: args.max_samples]
    n, S = len(ids), cfg.ensemble_size
    cores = os.cpu_count() or 1
    ens = cpu_plan(cfg, coords, keys)
    K = len(ens)
    gold = golden_level(cfg.name, ids, coords)
    full, src = full_iterations(cfg, ens, gold, keys, args.max_iters)
    P = max(1, min(cores, K))
    maxit = REF_ITERS.get(cfg.name)
    if args.max_iters:
        maxit = min(maxit or args.max_iters, args.max_iters)
    if full is None and maxit is not None:
        print(json.dumps({"impl": "reference", "unavailable": src}), flush=True)
        return
    times, samples = [], []
    ctx = mproc.get_context("spawn")
    with ctx.Pool(P) as pool:
        pool.map(_cpu_warm, [cfg.name] * P, chunksize=1)  # worker start-up + per-process setup

        def one(st):
            if maxit is None:  # full solves of the whole level (C1): its wall time
                chosen = list(range(K))
                t0 = time.perf_counter()
                rs = pool.map(_cpu_group_worker, [(cfg.name, coords[list(ens[k])], None)
                                                  for k in chosen], chunksize=1)
                return n / (time.perf_counter() - t0), chosen, rs
            chosen = sorted({(j * K // P + st) % K for j in range(P)})
            rs = pool.map(_cpu_group_worker, [(cfg.name, coords[list(ens[k])], maxit)
                                              for k in chosen], chunksize=1)
            t_iter = sum(r["pcg"] / max(1, r["iters_run"]) for r in rs) / len(rs)
            t_setup = sum(r["setup"] for r in rs) / len(rs)
            level_s = (t_setup * K + t_iter * sum(full)) / P
            return n / level_s * (args.max_iters or 1), chosen, rs

        for st in range(args.warmup):
            one(K - 1 - st)
        t0 = time.perf_counter()
        for st in range(args.steps):
            v, chosen, rs = one(st)
            times.append(v)
            samples.append(chosen)
        wall = time.perf_counter() - t0
    value = float(np.mean(times))
    unit = "sample-solves/s" if not args.max_iters else \
        f"sample-iterations/s (throughput mode: {args.max_iters} PCG iterations per group)"
    how = ("full solves of every group" if maxit is None else
           f"{maxit} PCG iterations per group timed, the whole level projected with every "
           f"group's full iteration count ({src}) over {P} cores")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": unit,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / max(1, args.steps), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (committed bench workload; see DESIGN.md)",
        "config": config_dict(cfg, n, K, world, args.scaling, meta),
        "cpu_baseline": {
            "value": value, "unit": unit, "cores": P,
            "kind": cpu_path_kind(), "projected": maxit is not None,
            "sample": f"per step {len(samples[0]) if samples else 0} of {K} groups (stratified: "
                      f"every {K / P:.1f}th in surrogate order, offset = step), one per process, "
                      f"1 BLAS thread each; {how}; " + (
                          "uqgroup's own EnsembleCsrMatrix/ensemble_pcg from baseline/_ref "
                          "(unmodified) on the 2D assembly restated in oracle/ (the reference "
                          "has no 2D operator, DESIGN.md)" if cpu_path_kind() == "reference"
                          else "oracle/ restatement of uqgroup's path (baseline/_ref not "
                          "staged)"),
            "step_values": times, **host_info()},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
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
            # NCCL's init log (ranks, transports, NVLS) goes to stderr for the record
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_1705_02003_b200 as uq
    from paper_1705_02003_b200 import _lib
    from paper_1705_02003_b200.build import needs_build, build
    from paper_1705_02003_b200.dist import LevelShard

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
    strong = args.scaling == "strong"
    if not strong:
        # weak scaling: rank r solves the mirror images of the level's samples and
        # groups them by the keys of their originals (same sort work, same costs shape)
        coords = reflect(coords, rank)
    n, S = len(ids), cfg.ensemble_size
    K = -(-n // S)
    dev = _lib.device()
    coll_dev = torch.device("cpu") if share else dev  # gloo test hook collects on the host
    shard = LevelShard(rank, world, None, coll_dev) if (strong and world > 1) else None
    d_coords = torch.from_numpy(np.ascontiguousarray(coords)).to(dev)
    d_keys = None if keys is None else torch.from_numpy(np.ascontiguousarray(keys)).to(dev)
    lib, ctx = _lib.load(), _lib.ctx()
    stream = torch.cuda.current_stream()
    mine = list(range(rank, K, world)) if shard is not None else list(range(K))

    def barrier():
        if world > 1:
            dist.barrier()

    def step():
        out = solver.run_level_device(d_coords, n, S, d_keys, shard)
        if world > 1 and not strong:
            # weak mode: the study's one collective on each rank's own level
            groups, pad, it, cv, en, q = out
            m = torch.cat([it.double(), q]).to(coll_dev)
            allv = torch.empty(world * m.numel(), dtype=m.dtype, device=coll_dev)
            dist.all_gather_into_tensor(allv, m)
        return out

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    import ctypes
    NK = _lib.NKERN  # UQG_NKERN

    def timed(profile: bool, steps: int):
        """`steps` timed steps; per-launch CUDA-event kernel timing when `profile`."""
        ms = (ctypes.c_double * NK)()
        cnt = (ctypes.c_longlong * NK)()
        lib.uqg_ctx_profile_read(ctx, ms, cnt, 1)
        lib.uqg_ctx_profile(ctx, int(profile))
        launches0 = lib.uqg_ctx_launch_count(ctx)
        times, local_iters, local_flush, last = [], 0, 0, None
        kx = max(1, int(lib.uqg_pcg_x_defer()))
        with ClockSampler(torch.cuda.current_device()) as clocks:
            for _ in range(steps):
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
                # this rank's group-iterations (its own kernels' work)
                en_mine = last[4][mine].long()
                local_iters += int(en_mine.sum().item())
                local_flush += int(((en_mine + kx - 1) // kx).sum().item())
                barrier()
        launches = lib.uqg_ctx_launch_count(ctx) - launches0
        lib.uqg_ctx_profile_read(ctx, ms, cnt, 1)
        lib.uqg_ctx_profile(ctx, 0)
        return times, local_iters, local_flush, launches, ms, cnt, clocks, last

    # value from un-instrumented steps (the library solves a level's groups as
    # concurrent parts on several streams); the per-kernel times for the
    # roofline from an identical profiled pass on ONE stream, so each launch's
    # duration is that kernel's alone (UQG_SOLVE_STREAMS=1; same results).
    times, local_iters, _, launches, _, _, clocks, last = timed(False, args.steps)
    prev = os.environ.get("UQG_SOLVE_STREAMS")
    os.environ["UQG_SOLVE_STREAMS"] = "1"
    try:
        prof_steps = max(1, min(args.prof_steps, args.steps))
        _, prof_iters, prof_flush, _, ms, cnt, _, _ = timed(True, prof_steps)
    finally:
        if prev is None:
            os.environ.pop("UQG_SOLVE_STREAMS", None)
        else:
            os.environ["UQG_SOLVE_STREAMS"] = prev
    assert prof_iters * args.steps == local_iters * prof_steps
    groups, pad, it, cv, en, q = last
    conv_all = bool(cv.all().item())
    load = shard.last_load if shard is not None else None

    # ---- end to end through the public API: host inputs, host results -------
    e2e_steps = args.e2e_steps or args.steps
    e2e_t = []
    for _ in range(e2e_steps):
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plan, iters, qois, notes = solver.solve_level(ids, coords, S, keys=keys, level=99,
                                                      shard=shard)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if world > 1:
            tt = torch.tensor([dt], device=coll_dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
        e2e_t.append(dt)
    h2d = coords.nbytes + (0 if keys is None else 8 * n)
    d2h = 8 * (K * S * 4 + K)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    total_ms = sum(times)
    per_step = n if strong else world * n
    value = per_step * len(times) / (total_ms / 1e3)
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
    # per-kernel rooflines of the PCG kernels (group-iterations of THIS rank's
    # groups in the profiled pass); the line's "roofline" is the single
    # kernel with the largest measured time share (the dominant kernel)
    spmv_name = "pcg_spmv_fv2d_kernel" if bm["operator"] != "csr" else "pcg_spmv_tma_kernel"
    per = {}
    kernels = [("spmv", 3, spmv_name, prof_iters, prof_iters * bm["spmv"]),
               ("update", 4, "pcg_update_kernel", prof_iters, prof_iters * bm["update"]),
               ("dir", 5, "pcg_dir_kernel", prof_iters, prof_iters * bm["dir_only"])]
    if "flush" in bm:
        kernels.append(("flush", 10, "pcg_flush_kernel", prof_flush,
                        prof_iters * bm["flush_p"] + prof_flush * bm["flush_x"]))
    for key, idx, kname, glaunch, nbytes in kernels:
        t_ms = ms[idx]
        gbs = nbytes / (t_ms / 1e3) / 1e9 if t_ms else None
        tr = traffic_all.get(f"{cfg.name}:{kname}", {})
        gpl = tr.get("groups_per_launch") or 1
        per[key] = {"kernel": kname, "ms": t_ms, "achieved": gbs,
                    "frac": gbs / peak if gbs else None,
                    "group_launches": glaunch,
                    "bytes_per_group_launch": nbytes / glaunch if glaunch else None,
                    # ncu DRAM bytes of one launch over `groups_per_launch` groups,
                    # per group-launch like bytes_per_group_launch
                    "traffic": (tr["dram_bytes_per_launch"] / gpl
                                if tr.get("dram_bytes_per_launch") else None),
                    "traffic_algorithmic_same_launch": (
                        tr["algorithmic_bytes_per_launch"] / gpl
                        if tr.get("algorithmic_bytes_per_launch") else None),
                    "traffic_unit": "bytes per group-launch",
                    "traffic_source": tr.get("source")}
    if cnt[3] and not cnt[4] and not cnt[5]:
        # small batches: the whole solve is ONE persistent launch (cluster or
        # cooperative kernel; SpMV, update and direction as phases of each
        # iteration, x updated in place) - its roofline is the loop's
        bm1 = bytes_model(cfg, solver.op, 1)
        b_it = bm1["spmv"] + bm1["update"] + bm1["dir"]
        gbs = prof_iters * b_it / (ms[3] / 1e3) / 1e9 if ms[3] else None
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
    loop_ms = ms[3] + ms[4] + ms[5] + ms[10]
    loop_gbs = prof_iters * bm["pcg_iter"] / (loop_ms / 1e3) / 1e9 if loop_ms else None
    step_gbs = local_iters * bm["pcg_iter"] / (total_ms / 1e3) / 1e9
    kern = {name: {"ms": ms[k], "launches": int(cnt[k])} for k, name in enumerate(
        ["kl", "assemble", "pcg_init", "pcg_spmv", "pcg_update", "pcg_dir", "dot_qoi", "group",
         "spmv", "other", "pcg_flush"]) if cnt[k]}
    all_ms = sum(ms[k] for k in range(NK))

    # ---- parity of this run's level against the reference's results ----------
    g_host = groups.cpu().numpy().reshape(K, S)
    ens_ids = [[int(ids[j]) for j in row] for row in g_host]
    it_h = it.cpu().numpy().reshape(K, S)
    q_h = q.cpu().numpy().reshape(K, S)
    first_it, first_q = {}, {}
    for k_, row in enumerate(ens_ids):
        for s_, sid in enumerate(row):
            if sid not in first_it:
                first_it[sid], first_q[sid] = int(it_h[k_, s_]), float(q_h[k_, s_])
    gold = None if (args.max_iters or args.max_samples or not strong and world > 1) else \
        golden_level(cfg.name, ids, coords)
    par = parity(gold, ens_ids, first_it, first_q)

    line = {
        "metric": METRIC,
        "value": value,
        "unit": unit,
        "n_gpus": world,
        "steps": len(times),
        "warmup": max(3, args.warmup),
        "ms_per_step": total_ms / len(times),
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (committed bench workload; see DESIGN.md)",
        "config": config_dict(cfg, n, K, world, args.scaling, meta),
        "gpu_launches": int(launches),
        "e2e": {"value": per_step * len(e2e_t) / sum(e2e_t) * (args.max_iters or 1),
                "unit": unit, "steps": len(e2e_t),
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        "roofline": {"bound": "hbm", "kernel": per[dom]["kernel"], "operator": bm["operator"],
                     "achieved": per[dom]["achieved"], "peak": peak, "unit": "GB/s",
                     "frac": per[dom]["frac"], "traffic": per[dom]["traffic"],
                     "traffic_algorithmic_same_launch": per[dom]["traffic_algorithmic_same_launch"],
                     "traffic_unit": "bytes per group-launch (ncu DRAM bytes of one launch / "
                                     "its groups)",
                     "traffic_source": per[dom]["traffic_source"],
                     "peak_source": peak_src,
                     # also against the 8 TB/s HBM3e specification
                     "peak_spec": 8000.0,
                     "frac_spec": (per[dom]["achieved"] / 8000.0) if per[dom]["achieved"] else None,
                     "bytes_per_group_launch": per[dom]["bytes_per_group_launch"],
                     "group_launches": per[dom].get("group_launches", prof_iters),
                     "timing": f"per-launch CUDA events on the launching stream, {prof_steps} "
                               "profiled step(s) with the level on one stream "
                               "(UQG_SOLVE_STREAMS=1)",
                     "time_share": per[dom]["ms"] / all_ms if all_ms else None,
                     "pcg_kernels": per},
        "pcg_loop": {"achieved_gbs": loop_gbs, "frac": loop_gbs / peak if loop_gbs else None,
                     "bytes_per_group_iter": bm["pcg_iter"],
                     "moved_gbs": (loop_gbs * bm["pcg_iter_moved"] / bm["pcg_iter"])
                     if loop_gbs else None,
                     "moved_bytes_per_group_iter": bm["pcg_iter_moved"], "step_gbs": step_gbs,
                     "group_iterations": local_iters},
        "kernels": kern,
        "all_converged": conv_all,
        "parity": par,
        "clocks": clocks.summary(),
    }
    if load is not None:
        gi = load["group_iterations"]
        line["shards"] = {"groups_per_rank": load["groups"], "group_iterations_per_rank": gi,
                          "imbalance_max_over_mean": max(gi) / (sum(gi) / len(gi)) if sum(gi)
                          else None}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(
            cfg, ids, coords, keys, gold, args.max_iters,
            lambda k_: (it_h[k_].tolist(), q_h[k_].tolist()))
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
