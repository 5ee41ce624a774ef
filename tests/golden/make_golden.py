"""Generate the committed golden fixtures from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the unmodified reference package (``/root/reference/pkg/src``) and
its test helpers (``/root/reference/pkg/tests/_oracles.py``) and writes small
fixtures next to this file.  Nothing at test/bench time reads /root/reference.

Fixtures:
* pcg_cases.npz     - random shared-graph SPD ensembles (reference
                      ``random_spd_system``) with the reference's
                      ``EnsembleCsrMatrix.spmv`` products and ``ensemble_pcg``
                      results (solution, counts, flags, residual history);
* special_cases.npz - the hand cases of test_ensemble.py (zero rhs, identity,
                      diagonal, subnormal freeze) solved by the reference;
* grouping.json     - reference ``group_by_key``/``group_natural`` plans on
                      keys with ties, signed zeros and strings as ids;
* eigen.npz         - reference ``eigenpairs_1d`` for the config deltas;
* c1_adaptive.json  - the C1 study (n=64, M=3, S=8) driven by the reference's
                      own HierGrid, group_by_key/group_natural and
                      ensemble_pcg, with the 2D operator from oracle/fv2d.py;
* c2_group.json     - one S=16 group at C2 (n=256) through the same path;
* fv2d_small.npz    - oracle 2D assembly (n=8, S=3) for bitwise kernel checks.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path[:0] = ["/root/reference/pkg/src", "/root/reference/pkg/tests", str(REPO)]

from uqgroup import ensemble as ref_ens  # noqa: E402
from uqgroup import grouping as ref_grp  # noqa: E402
from uqgroup import random_field as ref_rf  # noqa: E402
from uqgroup.hier_grid import HierGrid, RefinementPolicy  # noqa: E402
from _oracles import random_spd_system  # noqa: E402

from oracle import field2d, fv2d  # noqa: E402
from paper_1705_02003_b200.configs import CONFIGS  # noqa: E402


def pcg_cases():
    rng = np.random.default_rng(20260816)
    out = {}
    specs = [(12, 1), (30, 4), (45, 3), (60, 8), (120, 2), (200, 8), (7, 16), (90, 5)]
    for c, (n, width) in enumerate(specs):
        lanes, rhs = random_spd_system(rng, n, width)
        ens = ref_ens.EnsembleCsrMatrix.from_scipy_lanes(lanes)
        x = rng.standard_normal((width, n))
        tol = [1e-12, 1e-10, 1e-9, 1e-11][c % 4]
        res = ref_ens.ensemble_pcg(ens, rhs, tol=tol, maxit=5000, record_history=True)
        pre = f"c{c}_"
        out.update({
            pre + "row_offsets": ens.row_offsets, pre + "col_indices": ens.col_indices,
            pre + "values": ens.values, pre + "rhs": rhs, pre + "x": x, pre + "Ax": ens.spmv(x),
            pre + "tol": np.array(tol), pre + "solution": res.solution,
            pre + "iterations": res.iterations_per_lane, pre + "converged": res.converged_per_lane,
            pre + "frozen": res.frozen_lanes, pre + "history": np.array(res.residual_history),
            pre + "diag": ens.diagonal(),
        })
    out["n_cases"] = np.array(len(specs))
    np.savez_compressed(HERE / "pcg_cases.npz", **out)


def special_cases():
    out = {}
    tiny = np.finfo(np.float64).tiny

    def diag_ens(d):
        d = np.atleast_2d(np.asarray(d, dtype=float))
        n = d.shape[1]
        return ref_ens.EnsembleCsrMatrix(np.arange(n + 1), np.arange(n), d.copy())

    r = ref_ens.ensemble_pcg(diag_ens([[2.0, 3.0], [4.0, 5.0]]), np.zeros((2, 2)))
    out["zero_iters"] = r.iterations_per_lane
    rhs = np.arange(15.0).reshape(3, 5)
    r = ref_ens.ensemble_pcg(diag_ens(np.ones((3, 5))), rhs)
    out["ident_iters"], out["ident_x"] = r.iterations_per_lane, r.solution
    r = ref_ens.ensemble_pcg(diag_ens([[2.0, 2.0], [0.5 * tiny, 0.5 * tiny]]), np.ones((2, 2)),
                             precond=ref_ens.IdentityPreconditioner(), tol=1e-8, maxit=50)
    out.update(frz_x=r.solution, frz_iters=r.iterations_per_lane, frz_conv=r.converged_per_lane,
               frz_frozen=r.frozen_lanes)
    r = ref_ens.ensemble_pcg(diag_ens([[2.0, 3.0]]), np.ones((1, 2)), maxit=0)
    out["maxit0_iters"], out["maxit0_conv"] = r.iterations_per_lane, r.converged_per_lane
    np.savez_compressed(HERE / "special_cases.npz", **out)


def grouping_cases():
    rng = np.random.default_rng(7)
    cases = []
    for n, size in [(1, 1), (5, 4), (13, 4), (64, 8), (97, 16), (300, 8), (2441, 16)]:
        keys = np.round(rng.normal(50, 20, n))  # plenty of exact ties
        keys[rng.random(n) < 0.05] = 0.0
        keys[rng.random(n) < 0.05] = -0.0
        ids = list(rng.permutation(10 * n)[:n].tolist())
        kmap = {i: float(k) for i, k in zip(ids, keys)}
        p1 = ref_grp.group_by_key(ids, kmap, size, level=2, tag="sur")
        p2 = ref_grp.group_natural(ids, size, level=2)
        cases.append({"ids": ids, "keys": [float(k) for k in keys], "size": size,
                      "by_key": [list(g) for g in p1.ensembles], "by_key_pad": list(p1.padding),
                      "natural": [list(g) for g in p2.ensembles],
                      "natural_pad": list(p2.padding)})
    sids = ["a", "b", "c", "d"]
    p = ref_grp.group_by_key(sids, {"a": 5.0, "b": 1.0, "c": 3.0, "d": 2.0}, 2)
    cases.append({"ids": sids, "keys": [5.0, 1.0, 3.0, 2.0], "size": 2,
                  "by_key": [list(g) for g in p.ensembles], "by_key_pad": list(p.padding),
                  "natural": [["a", "b"], ["c", "d"]], "natural_pad": [0, 0]})
    (HERE / "grouping.json").write_text(json.dumps(cases))


def eigen_cases():
    """The reference's eigenpairs, computed single-threaded (LAPACK's eigh
    rounds differently with the BLAS thread count; the drop-in pins one)."""
    from threadpoolctl import threadpool_limits

    out = {}
    for delta in (0.2, 0.1, 0.05, 0.25):
        with threadpool_limits(limits=1):
            pairs = ref_rf.eigenpairs_1d(delta, 12, 513)
        out[f"lam_{delta}"] = np.array([p.eigenvalue for p in pairs])
        out[f"vec_{delta}"] = np.stack([p.values for p in pairs])
    np.savez_compressed(HERE / "eigen.npz", **out)


# ---------------------------------------------------------------------------
# parallel per-group solves (the reference's ensemble_pcg, one group per
# process, 1 BLAS thread): the study loop itself stays sequential

_POOL_STATE = {}


def _pool_init(cfg_name):
    from threadpoolctl import threadpool_limits
    threadpool_limits(limits=1)
    cfg = CONFIGS[cfg_name]
    fld = field2d.KL2D.select(**cfg.field_kwargs())
    mesh = fv2d.Mesh2D(cfg.cells)
    _POOL_STATE.update(cfg=cfg, fld=fld, mesh=mesh, table=fld.mode_table(mesh.node_points))


def _solve_group_ref(args):
    """One group through the reference's own ensemble_pcg on the oracle 2D
    operator: (per-lane iterations, converged, QoI, ensemble iterations)."""
    ys, maxit, keep = args
    st = _POOL_STATE
    cfg = st["cfg"]
    sysm = fv2d.assemble(st["mesh"], st["fld"], np.asarray(ys), st["table"], cfg.a2)
    mat = ref_ens.EnsembleCsrMatrix(sysm.row_offsets, sysm.col_indices, sysm.values)
    res = ref_ens.ensemble_pcg(mat, sysm.rhs, tol=cfg.tol, maxit=cfg.maxit if maxit is None else maxit,
                               record_history=keep)
    out = {"iterations": res.iterations_per_lane.tolist(),
           "converged": res.converged_per_lane.tolist(),
           "qoi": [float(np.dot(u, u)) for u in res.solution],
           "ensemble_iterations": int(res.ensemble_iterations)}
    if keep:
        out["history"] = np.array(res.residual_history)
        out["solution"] = res.solution
    return out


def _pool(cfg_name, procs):
    import multiprocessing as mp
    return mp.get_context("fork").Pool(procs, initializer=_pool_init, initargs=(cfg_name,))


def reference_study(cfg, max_levels=None, pool=None):
    """The reference's adaptive loop (harness.py:604-701, exec plan 'sur') on the 2D operator."""
    fld = field2d.KL2D.select(**{k: v for k, v in cfg.field_kwargs().items()})
    mesh = fv2d.Mesh2D(cfg.cells)
    table = fld.mode_table(mesh.node_points)
    S = cfg.ensemble_size
    grid = HierGrid(cfg.n_modes)
    batch = grid.add_initial_levels(cfg.initial_level)
    policy = RefinementPolicy(tau=cfg.tau, channel="qoi", max_points=cfg.n_max)
    cap = cfg.max_levels if max_levels is None else max_levels
    levels, level = [], 0
    while True:
        level += 1
        start = len(grid) - len(batch)
        ids = list(range(start, len(grid)))
        coords = grid.node_coords()[start:]
        coords_by_id = {sid: coords[i] for i, sid in enumerate(ids)}
        predicted = None
        if level == 1:
            plan = ref_grp.group_natural(ids, S, level, "sur")
        else:
            predicted = grid.eval_many("iterations", coords, n_nodes=start)
            plan = ref_grp.group_by_key(ids, {sid: float(predicted[i]) for i, sid in enumerate(ids)},
                                        S, level, "sur")
        iters, qois, ens_iters = {}, {}, []
        if pool is None:
            results = []
            for group in plan.ensembles:
                ys = np.array([coords_by_id[sid] for sid in group])
                sysm = fv2d.assemble(mesh, fld, ys, table, cfg.a2)
                mat = ref_ens.EnsembleCsrMatrix(sysm.row_offsets, sysm.col_indices, sysm.values)
                res = ref_ens.ensemble_pcg(mat, sysm.rhs, tol=cfg.tol, maxit=cfg.maxit)
                results.append({"iterations": res.iterations_per_lane.tolist(),
                                "ensemble_iterations": int(res.ensemble_iterations),
                                "qoi": [float(np.dot(u, u)) for u in res.solution]})
        else:
            results = pool.map(_solve_group_ref,
                               [(np.array([coords_by_id[sid] for sid in g]), None, False)
                                for g in plan.ensembles], chunksize=1)
        for group, res in zip(plan.ensembles, results):
            ens_iters.append(int(res["ensemble_iterations"]))
            for s, sid in enumerate(group):
                if sid not in iters:
                    iters[sid] = int(res["iterations"][s])
                    qois[sid] = float(res["qoi"][s])
        nodes = grid.nodes[start:]
        grid.compute_surpluses("qoi", {nd: qois[sid] for nd, sid in zip(nodes, ids)})
        grid.compute_surpluses("iterations", {nd: iters[sid] for nd, sid in zip(nodes, ids)})
        levels.append({
            "level": level, "ids": ids, "coords": coords.tolist(),
            "predicted": None if predicted is None else predicted.tolist(),
            "ensembles": [list(g) for g in plan.ensembles], "padding": list(plan.padding),
            "iterations": [iters[sid] for sid in ids], "qoi": [qois[sid] for sid in ids],
            "ensemble_iterations": ens_iters,
        })
        print(f"  level {level}: {len(ids)} samples, {len(plan.ensembles)} groups", flush=True)
        if level >= cap:
            break
        out = grid.refine(policy)
        if not out.new_nodes:
            break
        batch = out.new_nodes
    return {"config": cfg.to_dict(), "levels": levels}


def fem3d_cases():
    """The reference's own 3D FEM: assembly, solves and the Laplacian centre value."""
    from uqgroup import fem3d as rfem

    fld = ref_rf.build_field(delta=0.25, sigma0=np.sqrt(300.0), n_modes=4, a_min=0.1,
                             sigma0_convention="kernel")
    mesh = rfem.StructuredMesh(6)
    ys = np.array([[0.3, -0.7, 0.1, 0.9], [0.3, -0.7, 0.1, 0.9], [-1.0, 1.0, -1.0, 1.0]])
    sysm = rfem.assemble(mesh, fld, ys)
    res = ref_ens.ensemble_pcg(sysm.matrix, sysm.rhs, tol=1e-10, maxit=4000)
    lap = ref_rf.build_field(delta=0.25, sigma0=0.0, n_modes=1, a_min=0.0, a_hat_value=1.0,
                             expansion="linear")
    mesh16 = rfem.StructuredMesh(16)
    s16 = rfem.assemble(mesh16, lap, np.zeros((1, 1)))
    r16 = ref_ens.ensemble_pcg(s16.matrix, s16.rhs, tol=1e-10, maxit=4000)
    k16 = rfem.assemble(mesh16, fld, ys)
    rk = ref_ens.ensemble_pcg(k16.matrix, k16.rhs, tol=1e-7, maxit=30000)
    np.savez_compressed(
        HERE / "fem3d.npz", samples=ys, a_q=fld.eval_a_batch(mesh.quad_points, ys),
        values=sysm.matrix.values, rhs=sysm.rhs, row_offsets=mesh.row_offsets,
        col_indices=mesh.col_indices, solution=res.solution, iterations=res.iterations_per_lane,
        lap_centre=np.array(r16.solution[0][mesh16.center_dof()]),
        lap_iterations=r16.iterations_per_lane, m16_iterations=rk.iterations_per_lane,
        m16_qoi=np.array([rfem.qoi(u) for u in rk.solution]))


def reference_study_3d(name):
    """The reference's own adaptive loop on its own preset (harness.py:575-701,
    exec plan 'sur'), recording per-sample iterations AND QoIs."""
    from uqgroup import harness as H

    cfg = H.preset_config(name)
    prob = H._PdeProblem(cfg)
    S = cfg.ensemble_size
    grid = HierGrid(cfg.n_dims, domain=prob.box)
    batch = grid.add_initial_levels(cfg.initial_level)
    policy = RefinementPolicy(tau=cfg.tau, channel="qoi", max_points=cfg.n_max)
    levels, level = [], 0
    while True:
        level += 1
        start = len(grid) - len(batch)
        ids = list(range(start, len(grid)))
        coords = grid.node_coords()[start:]
        coords_by_id = {sid: coords[i] for i, sid in enumerate(ids)}
        predicted = None
        if level == 1:
            plan = ref_grp.group_natural(ids, S, level, "sur")
        else:
            predicted = grid.eval_many("iterations", coords, n_nodes=start)
            plan = ref_grp.group_by_key(ids, {sid: float(predicted[i]) for i, sid in enumerate(ids)},
                                        S, level, "sur")
        iters, qois, notes = prob.solve_plan(plan, coords_by_id, None)
        nodes = grid.nodes[start:]
        grid.compute_surpluses("qoi", {nd: qois[sid] for nd, sid in zip(nodes, ids)})
        grid.compute_surpluses("iterations", {nd: iters[sid] for nd, sid in zip(nodes, ids)})
        levels.append({
            "level": level, "ids": ids, "coords": coords.tolist(),
            "predicted": None if predicted is None else predicted.tolist(),
            "ensembles": [list(g) for g in plan.ensembles], "padding": list(plan.padding),
            "iterations": [iters[sid] for sid in ids], "qoi": [qois[sid] for sid in ids],
            "notes": notes,
        })
        print(f"  {name} level {level}: {len(ids)} samples", flush=True)
        out = grid.refine(policy)
        if not out.new_nodes:
            stop = "budget_exhausted" if out.budget_exhausted else "tolerance_met"
            break
        batch = out.new_nodes
    return {"preset": name, "stop": stop, "levels": levels}


def rounding_envelope(name, doc):
    """The reference's own iteration-count reproducibility on its preset.

    Lock-step over the golden study's plans, the reference's ensemble_pcg is
    re-run (a) with per-lane dots summed in a different order (numpy pairwise
    ``sum(x*y)`` instead of BLAS ``ddot``) and (b) with the assembled values
    jittered by one ulp; the largest |iteration change| per level is the
    envelope within which two correct FP64 implementations can disagree.
    """
    from uqgroup import fem3d as rfem
    from uqgroup import harness as H

    cfg = H.preset_config(name)
    prob = H._PdeProblem(cfg)
    rng = np.random.default_rng(1)
    orig_dot = ref_ens.lane_dot
    env = []
    for lv in doc["levels"]:
        coords = {s: np.array(c) for s, c in zip(lv["ids"], lv["coords"])}
        gold = dict(zip(lv["ids"], lv["iterations"]))
        worst = 0
        for grp in lv["ensembles"]:
            ys = np.array([coords[s] for s in grp])
            sysm = rfem.assemble(prob.mesh, prob.field, ys, prob.mode_vals)
            ref_ens.lane_dot = lambda x, y: np.array([np.sum(x[s] * y[s]) for s in range(x.shape[0])])
            try:
                a = ref_ens.ensemble_pcg(sysm.matrix, sysm.rhs, tol=cfg.solver.tol,
                                         maxit=cfg.solver.maxit).iterations_per_lane
            finally:
                ref_ens.lane_dot = orig_dot
            v = sysm.matrix.values
            v = np.where(rng.random(v.shape) < 0.5, np.nextafter(v, np.inf), np.nextafter(v, -np.inf))
            pm = ref_ens.EnsembleCsrMatrix(sysm.matrix.row_offsets, sysm.matrix.col_indices, v)
            b = ref_ens.ensemble_pcg(pm, sysm.rhs, tol=cfg.solver.tol,
                                     maxit=cfg.solver.maxit).iterations_per_lane
            for s, sid in enumerate(grp):
                worst = max(worst, abs(int(a[s]) - gold[sid]), abs(int(b[s]) - gold[sid]))
        env.append(worst)
        print(f"  {name} level {lv['level']}: reference rounding envelope +-{worst}", flush=True)
    return env


def c2_group():
    cfg = CONFIGS["C2"]
    fld = field2d.KL2D.select(**cfg.field_kwargs())
    mesh = fv2d.Mesh2D(cfg.cells)
    grid = HierGrid(cfg.n_modes)
    grid.add_initial_levels(1)
    ys = grid.node_coords()[:cfg.ensemble_size]
    sysm = fv2d.assemble(mesh, fld, ys, None, cfg.a2)
    mat = ref_ens.EnsembleCsrMatrix(sysm.row_offsets, sysm.col_indices, sysm.values)
    res = ref_ens.ensemble_pcg(mat, sysm.rhs, tol=cfg.tol, maxit=cfg.maxit)
    doc = {"config": cfg.to_dict(), "samples": ys.tolist(),
           "iterations": res.iterations_per_lane.tolist(),
           "ensemble_iterations": int(res.ensemble_iterations),
           "qoi": [float(np.dot(u, u)) for u in res.solution],
           "center_value": [float(u[mesh.n_dofs // 2]) for u in res.solution]}
    (HERE / "c2_group.json").write_text(json.dumps(doc))


def c2_study(procs=6):
    """The full C2 adaptive study (every level, every group) through the
    reference's own loop pieces - the bench's C2 workload is its last level."""
    with _pool("C2", procs) as pool:
        doc = reference_study(CONFIGS["C2"], pool=pool)
    (HERE / "c2_adaptive.json").write_text(json.dumps(doc))


def _workload(name):
    z = np.load(REPO / "bench_workloads" / f"{name}.npz")
    keys = z["keys"] if z["keys"].size else None
    return [int(i) for i in z["ids"]], np.asarray(z["coords"]), keys


def c3_level(procs=6):
    """Every group of the C3 bench workload (the study's final level: samples +
    surrogate keys, bench_workloads/C3.npz) grouped by the reference's
    group_by_key and solved to convergence by the reference's ensemble_pcg on
    the oracle 2D operator.  One mid-cost group also keeps its residual history."""
    cfg = CONFIGS["C3"]
    ids, coords, keys = _workload("C3")
    plan = ref_grp.group_by_key(ids, {sid: float(k) for sid, k in zip(ids, keys)},
                                cfg.ensemble_size, 5, "sur")
    row = {sid: i for i, sid in enumerate(ids)}
    K = len(plan.ensembles)
    keep = K // 2
    import time
    t0 = time.time()
    with _pool("C3", procs) as pool:
        res = pool.map(_solve_group_ref,
                       [(coords[[row[s] for s in g]], None, k == keep)
                        for k, g in enumerate(plan.ensembles)], chunksize=1)
    hist = res[keep].pop("history")
    sol = res[keep].pop("solution")
    doc = {"config": cfg.to_dict(), "workload": "bench_workloads/C3.npz",
           "ensembles": [list(g) for g in plan.ensembles], "padding": list(plan.padding),
           "groups": res, "history_group": keep,
           "cpu_seconds_wall": time.time() - t0, "procs": procs}
    (HERE / "c3_level.json").write_text(json.dumps(doc))
    idx = np.arange(0, sol.shape[1], 997)
    np.savez_compressed(HERE / "c3_history.npz", history=hist, group=keep, idx=idx,
                        x_idx=sol[:, idx], x_norm2=np.einsum("ij,ij->i", sol, sol))


def fixed_iterations(name, maxit=30):
    """The first group of the C4 / C5 bench workload, exactly `maxit` PCG
    iterations of the reference's ensemble_pcg: residual history, and x through
    per-lane x.x plus x at every 997th unknown."""
    cfg = CONFIGS[name]
    ids, coords, keys = _workload(name)
    S = cfg.ensemble_size
    if keys is None:
        plan = ref_grp.group_natural(ids, S, 1, "nat")
    else:
        plan = ref_grp.group_by_key(ids, {sid: float(k) for sid, k in zip(ids, keys)}, S, 2, "sur")
    row = {sid: i for i, sid in enumerate(ids)}
    g = plan.ensembles[0]
    _pool_init(name)
    out = _solve_group_ref((coords[[row[s] for s in g]], maxit, True))
    sol = out["solution"]
    idx = np.arange(0, sol.shape[1], 997)
    np.savez_compressed(HERE / f"{name.lower()}_fixed.npz", group=np.array(list(g)),
                        maxit=np.array(maxit), history=out["history"],
                        iterations=np.array(out["iterations"]), idx=idx, x_idx=sol[:, idx],
                        x_norm2=np.einsum("ij,ij->i", sol, sol))


def fv2d_small():
    fld = field2d.KL2D.select(0.2, 1.0, 3, 0.0)
    mesh = fv2d.Mesh2D(8)
    ys = np.array([[0.5, -0.25, 1.0], [-1.0, 1.0, 0.0], [0.5, -0.25, 1.0]])
    a = fld.coeff(mesh.node_points, ys)
    np.savez_compressed(HERE / "fv2d_small.npz", samples=ys, a_nodes=a,
                        values=fv2d.assemble_values(mesh, a, 1.0),
                        values_same=fv2d.assemble_values(mesh, a, 1.0, "same"),
                        row_offsets=mesh.row_offsets, col_indices=mesh.col_indices)


def refrun_outputs():
    """The reference CLI's own output files for a small pde_test1 study
    (``cli.py:116-131`` residual dump + ``harness.py:762-797`` emission):
    S=4, n_max=60, 6^3 cells, surrogate grouping.  Pins report.py's formats and,
    through the device study, the per-sample iteration table byte for byte."""
    import shutil
    import tempfile

    from uqgroup import cli

    dst = HERE / "refrun_pde_test1"
    if dst.exists():
        shutil.rmtree(dst)
    dst.mkdir()
    with tempfile.TemporaryDirectory() as tmp:
        rc = cli.main(["run", "--problem", "pde_test1", "--strategies", "sur", "--S", "4",
                       "--n-max", "60", "--mesh-cells", "6", "--dump-residuals",
                       "--out-dir", tmp])
        assert rc in (0, 2)  # 2: stopped on the budget, outputs complete
        for name in ("iterations_by_level.csv", "r_table.csv", "manifest.json",
                     "residuals_level1_ens0.csv", "residuals_level1_ens11.csv",
                     "residuals_level2_ens0.csv"):
            shutil.copy(Path(tmp) / name, dst / name)
        n = len(list(Path(tmp).glob("residuals_level*_ens*.csv")))
        (dst / "README").write_text(
            "Outputs of the reference CLI (uqgroup run --problem pde_test1 --strategies sur "
            "--S 4 --n-max 60 --mesh-cells 6 --dump-residuals), generated by "
            f"tests/golden/make_golden.py:refrun_outputs; {n} residual files in the run, "
            "3 kept.\n")


if __name__ == "__main__":
    which = sys.argv[1:] or ["pcg", "special", "grouping", "eigen", "fv2d", "c1", "c2"]
    if "pcg" in which:
        pcg_cases()
    if "special" in which:
        special_cases()
    if "grouping" in which:
        grouping_cases()
    if "eigen" in which:
        eigen_cases()
    if "fv2d" in which:
        fv2d_small()
    if "c1" in which:
        doc = reference_study(CONFIGS["C1"])
        (HERE / "c1_adaptive.json").write_text(json.dumps(doc))
    if "c2" in which:
        c2_group()
    if "c2study" in which:
        c2_study()
    if "c3level" in which:
        c3_level()
    for nm in ("C4", "C5"):
        if nm.lower() + "fixed" in which:
            fixed_iterations(nm)
    if "refrun" in which:
        refrun_outputs()
    if "fem3d" in which:
        fem3d_cases()
    for preset in ("pde_test1", "pde_test2"):
        if preset in which:
            doc = reference_study_3d(preset)
            doc["envelope"] = rounding_envelope(preset, doc)
            (HERE / f"{preset}_study.json").write_text(json.dumps(doc))
    print("golden fixtures written to", HERE)
