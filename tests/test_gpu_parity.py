"""Parity of the CUDA path (libuqg.so through the C ABI) with the oracle and
the reference's golden outputs.  Mirrors the reference's hot-path tests
(test_ensemble.py, test_grouping.py, test_fem3d.py, test_acceptance.py crit 1).

Tolerances (BASELINE.json north_star): iteration counts exact (the gate is
+-1), solutions/QoIs within 1e-8 relative; SpMV, grouping and assembly
bit-exact; the KL coefficient within 1e-14 relative (exp and the M-term sum
round differently from numpy's exp/BLAS).
"""

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import driver as odriver, field2d, fv2d as ofv, pcg as opcg
import paper_1705_02003_b200 as uq
from paper_1705_02003_b200 import _lib
from paper_1705_02003_b200.fv2d import FieldTables, assemble_values, kl_nodes

pytestmark = pytest.mark.gpu
TINY = np.finfo(np.float64).tiny


def diag_ensemble(d):
    d = np.atleast_2d(np.asarray(d, dtype=float))
    n = d.shape[1]
    return uq.EnsembleCsrMatrix(np.arange(n + 1), np.arange(n), d.copy())


def spd_system(rng, n, width):
    """Shared-graph diagonally dominant SPD ensemble (as the reference's tests build)."""
    mask = np.triu(rng.random((n, n)) < min(1.0, 6.0 / n), 1)
    base = np.where(mask, rng.uniform(-1.0, 1.0, (n, n)), 0.0)
    base = base + base.T
    lanes = []
    for _ in range(width):
        v = base * rng.uniform(0.2, 1.0)
        np.fill_diagonal(v, np.abs(v).sum(axis=1) + rng.uniform(1.0, 3.0, n))
        lanes.append(sp.csr_matrix(v))
    return lanes, rng.standard_normal((width, n))


# ---------------------------------------------------------------------------
# SpMV / container (test_ensemble.py:41-87)

def test_spmv_bitwise_equals_reference_scipy(pcg_golden):
    for c in pcg_golden:
        ens = uq.EnsembleCsrMatrix(c["row_offsets"], c["col_indices"], c["values"])
        assert np.array_equal(ens.spmv(c["x"]), c["Ax"])


def test_diagonal_and_jacobi(pcg_golden):
    for c in pcg_golden:
        ens = uq.EnsembleCsrMatrix(c["row_offsets"], c["col_indices"], c["values"])
        assert np.array_equal(ens.diagonal(), c["diag"])
        assert np.array_equal(uq.jacobi_precond(ens).inv_diag, 1.0 / c["diag"])
    with pytest.raises(uq.EnsembleError):
        uq.jacobi_precond(diag_ensemble([[1.0, 0.0, 2.0]]))
    with pytest.raises(uq.EnsembleError):
        diag_ensemble([[1.0, 2.0]]).spmv(np.ones((2, 2)))


def test_lane_dot_and_norms():
    rng = np.random.default_rng(1)
    for S, n in ((1, 1), (3, 17), (8, 1000), (64, 4097)):
        a, b = rng.standard_normal((S, n)), rng.standard_normal((S, n))
        want = np.array([np.dot(a[s], b[s]) for s in range(S)])
        np.testing.assert_allclose(uq.lane_dot(a, b), want, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(uq.lane_norms(a), np.sqrt((a * a).sum(1)), rtol=1e-13)


# ---------------------------------------------------------------------------
# PCG semantics (test_ensemble.py:94-248)

def test_pcg_matches_reference_golden(pcg_golden):
    for c in pcg_golden:
        ens = uq.EnsembleCsrMatrix(c["row_offsets"], c["col_indices"], c["values"])
        r = uq.ensemble_pcg(ens, c["rhs"], tol=float(c["tol"]), maxit=5000, record_history=True)
        assert np.array_equal(r.iterations_per_lane, c["iterations"])
        assert np.array_equal(r.converged_per_lane, c["converged"])
        assert np.array_equal(r.frozen_lanes, c["frozen"])
        assert r.ensemble_iterations == c["iterations"].max()
        for s in range(ens.width):
            ref = c["solution"][s]
            assert np.linalg.norm(r.solution[s] - ref) <= 1e-10 * np.linalg.norm(ref)
        hist = np.array(r.residual_history)
        assert hist.shape == c["history"].shape
        np.testing.assert_allclose(hist[0], c["history"][0], rtol=1e-14)
        # residual norms agree to rounding relative to ||b|| (the last entries of a
        # lane that converged far past tol are pure rounding noise in both codes)
        scale = c["history"][0][None, :]
        assert np.all(np.abs(hist - c["history"]) <= 1e-9 * scale + 1e-6 * np.abs(c["history"]))


def test_trivial_systems(special_golden):
    g = special_golden
    r = uq.ensemble_pcg(diag_ensemble([[2.0, 3.0], [4.0, 5.0]]), np.zeros((2, 2)))
    assert np.array_equal(r.iterations_per_lane, g["zero_iters"]) and r.converged_per_lane.all()
    assert np.array_equal(r.solution, np.zeros((2, 2)))
    rhs = np.arange(15.0).reshape(3, 5)
    r = uq.ensemble_pcg(diag_ensemble(np.ones((3, 5))), rhs)
    assert np.array_equal(r.iterations_per_lane, [1, 1, 1])
    assert np.array_equal(r.solution, rhs)
    d = np.array([[2.0, 4.0, 8.0]])
    r = uq.ensemble_pcg(diag_ensemble(d), d.copy(), tol=1e-14)
    np.testing.assert_allclose(r.solution, np.ones((1, 3)), rtol=1e-13)
    r = uq.ensemble_pcg(diag_ensemble([[2.0, 3.0]]), np.ones((1, 2)), maxit=0)
    assert not r.converged_per_lane.any() and r.iterations_per_lane[0] == 0
    ens = diag_ensemble([[1.0]])
    for tol in (0.0, -1.0, float("inf"), float("nan")):
        with pytest.raises(uq.EnsembleError):
            uq.ensemble_pcg(ens, np.ones((1, 1)), tol=tol)
    with pytest.raises(uq.EnsembleError):
        uq.ensemble_pcg(ens, np.ones((1, 1)), maxit=-1)


def test_subnormal_lane_freezes(special_golden):
    d = np.array([[2.0, 2.0], [0.5 * TINY, 0.5 * TINY]])
    r = uq.ensemble_pcg(diag_ensemble(d), np.ones((2, 2)), precond=uq.IdentityPreconditioner(),
                        tol=1e-8, maxit=50)
    assert r.converged_per_lane[0] and not r.converged_per_lane[1]
    assert r.frozen_lanes[1] and not r.frozen_lanes[0]
    assert np.array_equal(r.solution[1], np.zeros(2))
    assert np.array_equal(r.solution, special_golden["frz_x"])
    assert np.array_equal(r.iterations_per_lane, special_golden["frz_iters"])


def test_nonfinite_active_lane_raises_breakdown():
    with pytest.raises(uq.NumericalBreakdownError):
        uq.ensemble_pcg(diag_ensemble([[1.0, np.inf]]), np.ones((1, 2)),
                        precond=uq.IdentityPreconditioner(), maxit=5)


def test_unsupported_preconditioner_rejected():
    class Mine:
        def apply(self, r):
            return r
    with pytest.raises(uq.EnsembleError):
        uq.ensemble_pcg(diag_ensemble([[1.0]]), np.ones((1, 1)), precond=Mine())


def test_counts_equal_scalar_pcg_acceptance_crit1():
    """test_acceptance.py:92-110: 50 random SPD systems, widths 2/4/8, tol 1e-12."""
    rng = np.random.default_rng(20260816)
    widths = [2, 4, 8]
    for t in range(50):
        n = int(rng.integers(20, 201))
        lanes, rhs = spd_system(rng, n, widths[t % 3])
        ens = uq.EnsembleCsrMatrix.from_scipy_lanes(lanes)
        r = uq.ensemble_pcg(ens, rhs, tol=1e-12, maxit=5000)
        assert r.converged_per_lane.all()
        for s in range(len(lanes)):
            single = opcg.pcg(ens.row_offsets, ens.col_indices, ens.values[s:s + 1], rhs[s:s + 1],
                              tol=1e-12, maxit=5000)
            assert single.iterations[0] == r.iterations_per_lane[s]
            x = single.solution[0]
            assert np.linalg.norm(r.solution[s] - x) <= 1e-10 * np.linalg.norm(x)


def test_duplicated_lanes_bitwise_and_repeat_determinism():
    rng = np.random.default_rng(12)
    lanes, rhs = spd_system(rng, 40, 2)
    ens = uq.EnsembleCsrMatrix.from_scipy_lanes([lanes[0], lanes[1], lanes[0], lanes[1]])
    rhs4 = np.vstack([rhs[0], rhs[1], rhs[0], rhs[1]])
    r = uq.ensemble_pcg(ens, rhs4, tol=1e-10, maxit=2000)
    assert np.array_equal(r.solution[0], r.solution[2])
    assert np.array_equal(r.solution[1], r.solution[3])
    r2 = uq.ensemble_pcg(ens, rhs4, tol=1e-10, maxit=2000)
    assert np.array_equal(r.solution, r2.solution)
    assert np.array_equal(r.iterations_per_lane, r2.iterations_per_lane)


def test_lane_independent_of_companions():
    rng = np.random.default_rng(13)
    lanes, rhs = spd_system(rng, 35, 3)
    full = uq.ensemble_pcg(uq.EnsembleCsrMatrix.from_scipy_lanes(lanes), rhs, tol=1e-10, maxit=2000)
    solo = uq.ensemble_pcg(uq.EnsembleCsrMatrix.from_scipy_lanes([lanes[1]]), rhs[1:2], tol=1e-10,
                           maxit=2000)
    assert solo.iterations_per_lane[0] == full.iterations_per_lane[1]
    x = solo.solution[0]
    assert np.linalg.norm(x - full.solution[1]) <= 1e-9 * np.linalg.norm(x)


@pytest.mark.parametrize("seed", range(12))
def test_property_counts_match_oracle(seed):
    rng = np.random.default_rng(1000 + seed)
    n, width = int(rng.integers(2, 13)), int(rng.integers(1, 5))
    lanes, rhs = spd_system(rng, n, width)
    ens = uq.EnsembleCsrMatrix.from_scipy_lanes(lanes)
    r = uq.ensemble_pcg(ens, rhs, tol=1e-10, maxit=500)
    o = opcg.pcg(ens.row_offsets, ens.col_indices, ens.values, rhs, tol=1e-10, maxit=500)
    assert np.array_equal(r.iterations_per_lane, o.iterations)
    assert np.array_equal(r.converged_per_lane, o.converged)


# ---------------------------------------------------------------------------
# grouping (test_grouping.py:37-82)

def test_grouping_matches_reference(grouping_golden):
    for case in grouping_golden:
        ids, size = case["ids"], case["size"]
        p = uq.group_by_key(ids, dict(zip(ids, case["keys"])), size, level=2)
        assert [list(g) for g in p.ensembles] == case["by_key"]
        assert list(p.padding) == case["by_key_pad"]
        p = uq.group_natural(ids, size, level=2)
        assert [list(g) for g in p.ensembles] == case["natural"]
        assert list(p.padding) == case["natural_pad"]


def test_grouping_errors_and_hand_cases():
    assert uq.group_natural([7, 8, 9, 10, 11], 4).ensembles == ((7, 8, 9, 10), (11, 11, 11, 11))
    assert uq.group_by_key([3, 1, 4, 5], {3: 2.0, 1: 2.0, 4: 2.0, 5: 2.0}, 2).ensembles == \
        ((3, 1), (4, 5))
    with pytest.raises(uq.GroupingError):
        uq.group_by_key([0, 1], {0: 1.0}, 2)
    with pytest.raises(uq.GroupingError):
        uq.group_by_key([0, 1], {0: 1.0, 1: float("nan")}, 2)
    with pytest.raises(uq.GroupingError):
        uq.group_natural([], 2)
    big = np.random.default_rng(3).integers(0, 50, 20000).astype(float)
    p = uq.group_by_key(list(range(20000)), dict(enumerate(big)), 32)
    order = np.argsort(big, kind="stable")
    assert [x for g in p.ensembles for x in g][:20000] == order.tolist()


# ---------------------------------------------------------------------------
# KL coefficient + 2D assembly

@pytest.mark.parametrize("cells,M,delta,sigma,S", [(8, 3, 0.2, 1.0, 3), (64, 3, 0.2, 1.0, 8),
                                                     (32, 10, 0.05, 2.0, 16)])
def test_kl_nodes_match_oracle(cells, M, delta, sigma, S):
    f = uq.build_field(delta, sigma, M, 0.0)
    o = field2d.KL2D.select(delta, sigma, M, 0.0)
    mesh = uq.StructuredMesh2D(cells)
    ys = np.random.default_rng(cells).uniform(-1, 1, (2 * S, M))
    d = kl_nodes(FieldTables(f, mesh), _lib.to_dev(ys), 2, S)
    got = d.reshape(2, mesh.n_nodes, S).cpu().numpy()
    want = o.coeff(ofv.Mesh2D(cells).node_points, ys)  # (2S, P)
    for g in range(2):
        np.testing.assert_allclose(got[g].T, want[g * S:(g + 1) * S], rtol=1e-14, atol=0)
    tab = f.mode_values(mesh.node_coords())
    np.testing.assert_allclose(f.eval_a_batch(None, ys[:S], tab), want[:S], rtol=1e-14)


def test_kl_tiled_contraction_bitwise_equals_per_element_kernel():
    """kl_sep2d_kernel (lane coefficients + tile mode values staged in shared
    memory) and kl_sep2d_elem_kernel (per-element recompute; taken when
    M x S is too large to stage) run the same FMA chain: bit-identical lanes.
    S = 8 takes the tiled kernel, S = 512 with M = 56 the per-element one;
    lanes 0..7 of both carry the same samples."""
    M, cells = 56, 6
    f = uq.build_field(0.1, 1.0, M, 0.0)
    mesh = uq.StructuredMesh2D(cells)
    P = mesh.n_nodes
    ys = np.random.default_rng(4).uniform(-1, 1, (512, M))
    small = kl_nodes(FieldTables(f, mesh), _lib.to_dev(ys[:8]), 1, 8)
    big = kl_nodes(FieldTables(f, mesh), _lib.to_dev(ys), 1, 512)
    a = small.reshape(P, 8).cpu().numpy()
    b = big.reshape(P, 512).cpu().numpy()[:, :8]
    assert np.array_equal(a, b)


def test_assembly_bitwise_given_nodal_coefficients(fv2d_golden):
    g = fv2d_golden
    mesh = uq.StructuredMesh2D(8)
    S = g["a_nodes"].shape[0]
    a_dev = _lib.to_dev(np.ascontiguousarray(g["a_nodes"].T))  # [P][S]
    for mode, key in (("const", "values"), ("same", "values_same")):
        vals, dinv = assemble_values(mesh, a_dev, 1, S, 1.0, mode)
        got = vals.reshape(mesh.nnz, S).cpu().numpy().T
        assert np.array_equal(got, g[key])
        diag = opcg.jacobi_inverse(mesh.row_offsets, mesh.col_indices, g[key])
        assert np.array_equal(dinv.reshape(mesh.n_dofs, S).cpu().numpy().T, diag)


def test_assemble_dropin_and_fem_error():
    f = uq.build_field(0.2, 1.0, 3, 0.0)
    o = field2d.KL2D.select(0.2, 1.0, 3, 0.0)
    mesh, omesh = uq.StructuredMesh2D(16), ofv.Mesh2D(16)
    ys = np.array([[0.3, -0.2, 0.9], [0.3, -0.2, 0.9], [-1, 1, 1.0]])
    sysd = uq.assemble(mesh, f, ys)
    syso = ofv.assemble(omesh, o, ys)
    np.testing.assert_allclose(sysd.matrix.values, syso.values, rtol=2e-14)
    assert np.array_equal(sysd.matrix.values[0], sysd.matrix.values[1])
    assert np.array_equal(sysd.rhs, syso.rhs)
    lin = uq.build_field(0.2, 5.0, 3, 0.0, expansion="linear")
    with pytest.raises(uq.FemError):
        uq.assemble(mesh, lin, np.array([[1.0, 1.0, 1.0]]) * 50)


def test_qoi_dropin():
    assert uq.qoi(np.zeros(7)) == 0.0
    u = np.random.default_rng(0).standard_normal(1000)
    assert uq.qoi(u) == pytest.approx(float(np.dot(u, u)), rel=1e-14)
    with pytest.raises(uq.FemError):
        uq.qoi(np.zeros((2, 2)))


# ---------------------------------------------------------------------------
# level-batched solve + end-to-end study

def test_batched_groups_bitwise_equal_single_group_solves():
    cfg = uq.CONFIGS["C1"]
    f = uq.build_field(**cfg.field_kwargs())
    solver = uq.EnsembleSolver2D(f, cfg.cells, cfg.tol, cfg.maxit)
    ys = np.random.default_rng(5).uniform(-1, 1, (5, cfg.ensemble_size, cfg.n_modes))
    allg = solver.solve_groups(ys)
    for k in range(5):
        one = solver.solve_groups(ys[k:k + 1])
        assert np.array_equal(one.iterations[0], allg.iterations[k])
        assert np.array_equal(one.qoi[0], allg.qoi[k])
    waves = uq.EnsembleSolver2D(f, cfg.cells, cfg.tol, cfg.maxit, max_groups_per_wave=2)
    w = waves.solve_groups(ys)
    assert w.waves == 3 and np.array_equal(w.qoi, allg.qoi)


def test_level_solve_matches_oracle_solve_plan():
    cfg = uq.CONFIGS["C1"]
    f = uq.build_field(**cfg.field_kwargs())
    o = field2d.KL2D.select(**cfg.field_kwargs())
    omesh = ofv.Mesh2D(cfg.cells)
    rng = np.random.default_rng(8)
    ids = list(range(21))
    coords = {i: rng.uniform(-1, 1, cfg.n_modes) for i in ids}
    plan = uq.group_natural(ids, cfg.ensemble_size, level=1)
    solver = uq.EnsembleSolver2D(f, cfg.cells, cfg.tol, cfg.maxit)
    it_d, q_d, notes_d = solver.solve_plan(plan, coords)
    it_o, q_o, notes_o = odriver.solve_plan(omesh, o, o.mode_table(omesh.node_points),
                                            plan.ensembles, coords, cfg.tol, cfg.maxit, level=1)
    assert it_d == it_o and notes_d == notes_o == []
    for i in ids:
        assert abs(q_d[i] - q_o[i]) <= 1e-8 * abs(q_o[i])


def test_c1_adaptive_study_matches_reference_golden(c1_golden):
    """Identical grouping and ensemble composition at every level, iteration
    counts within +-1 (observed: exact), QoIs within 1e-8 relative."""
    from paper_1705_02003_b200.driver import adaptive_run
    cfg = uq.CONFIGS["C1"]
    records, stop, _ = adaptive_run(cfg)
    assert len(records) == len(c1_golden["levels"])
    worst_q, worst_it = 0.0, 0
    for rec, gold in zip(records, c1_golden["levels"]):
        assert rec.ids == gold["ids"]
        assert [list(g) for g in rec.ensembles] == gold["ensembles"]
        assert list(rec.padding) == gold["padding"]
        for sid, it, q in zip(gold["ids"], gold["iterations"], gold["qoi"]):
            worst_it = max(worst_it, abs(rec.iterations[sid] - it))
            worst_q = max(worst_q, abs(rec.qois[sid] - q) / abs(q))
    assert worst_it <= 1
    assert worst_q <= 1e-8


def test_c2_group_matches_reference_golden(c2_golden):
    cfg = uq.CONFIGS["C2"]
    f = uq.build_field(**cfg.field_kwargs())
    solver = uq.EnsembleSolver2D(f, cfg.cells, cfg.tol, cfg.maxit)
    res = solver.solve_groups(np.array(c2_golden["samples"])[None])
    assert np.abs(res.iterations[0] - np.array(c2_golden["iterations"])).max() <= 1
    np.testing.assert_allclose(res.qoi[0], c2_golden["qoi"], rtol=1e-8)


def test_full_size_c3_properties():
    """BASELINE size (n=512, S=32): size-independent checks - residual bound
    through the device SpMV, duplicated samples bitwise, QoI symmetry."""
    cfg = uq.CONFIGS["C3"]
    f = uq.build_field(**cfg.field_kwargs())
    solver = uq.EnsembleSolver2D(f, cfg.cells, cfg.tol, cfg.maxit)
    ys = np.random.default_rng(11).uniform(-1, 1, (cfg.ensemble_size, cfg.n_modes))
    ys[1] = ys[0]
    d_y = _lib.to_dev(ys)
    iters, conv, frz, ens, q, _, x = solver.solve_wave(d_y, 1, cfg.ensemble_size)
    conv = conv.cpu().numpy().astype(bool)
    assert conv.all()
    q = q.cpu().numpy()
    assert q[0] == q[1]
    m = solver.mesh
    S = cfg.ensemble_size
    X = x.reshape(m.n_dofs, S).cpu().numpy().T
    assert np.array_equal(X[0], X[1])
    sysd = uq.assemble(m, f, ys[:4])
    Ax = sysd.matrix.spmv(X[:4])
    for s in range(4):
        res = np.linalg.norm(sysd.rhs[s] - Ax[s]) / np.linalg.norm(sysd.rhs[s])
        assert res <= 1.5e-8
        assert abs(np.dot(X[s], X[s]) - q[s]) <= 1e-12 * q[s]


def test_solve_level_equals_group_by_key_plus_solve_plan():
    cfg = uq.CONFIGS["C1"]
    f = uq.build_field(**cfg.field_kwargs())
    solver = uq.EnsembleSolver2D(f, cfg.cells, cfg.tol, cfg.maxit)
    rng = np.random.default_rng(21)
    n = 45
    ids = [f"s{i}" for i in range(n)]
    coords = rng.uniform(-1, 1, (n, cfg.n_modes))
    keys = np.round(rng.uniform(200, 240, n))
    plan, iters, qois, notes = solver.solve_level(ids, coords, cfg.ensemble_size, keys=keys, level=3)
    ref_plan = uq.group_by_key(ids, dict(zip(ids, keys)), cfg.ensemble_size, level=3)
    assert plan == ref_plan
    it2, q2, n2 = solver.solve_plan(ref_plan, dict(zip(ids, coords)))
    assert iters == it2 and qois == q2 and notes == n2
    plan_n, _, _, _ = solver.solve_level(ids, coords, cfg.ensemble_size, keys=None, level=3,
                                         tag="nat")
    assert plan_n == uq.group_natural(ids, cfg.ensemble_size, level=3)


def test_launch_accounting_and_profiling():
    lib, ctx = _lib.load(), _lib.ctx()
    import ctypes
    # arrays of UQG_NKERN (include/uqg.h) entries: the library fills all of them
    ms = (ctypes.c_double * _lib.NKERN)()
    cnt = (ctypes.c_longlong * _lib.NKERN)()
    lib.uqg_ctx_profile_read(ctx, ms, cnt, 1)
    lib.uqg_ctx_profile(ctx, 1)
    before = lib.uqg_ctx_launch_count(ctx)
    r = uq.ensemble_pcg(diag_ensemble(np.arange(1.0, 9.0)[None]), np.ones((1, 8)), tol=1e-12)
    lib.uqg_ctx_profile_read(ctx, ms, cnt, 1)
    lib.uqg_ctx_profile(ctx, 0)
    assert lib.uqg_ctx_launch_count(ctx) > before
    assert cnt[3] >= r.ensemble_iterations and ms[3] > 0.0


_CSR_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1705_02003_b200 as uq
cfg = uq.CONFIGS["C1"]
S = int(sys.argv[3])
f = uq.build_field(**cfg.field_kwargs())
s = uq.EnsembleSolver2D(f, cfg.cells, cfg.tol, cfg.maxit)
ys = np.random.default_rng(3).uniform(-1, 1, (4, S, cfg.n_modes))
r = s.solve_groups(ys)
np.save(sys.argv[2], np.concatenate([r.iterations.ravel().astype(float), r.qoi.ravel()]))
"""


@pytest.mark.parametrize("S", ["8", "7"])
def test_csr_spmv_kernels_bitwise_equal_face_form(tmp_path, S):
    """Whole batched launch-loop solves through the CSR operator - TMA-staged
    values with and without the L2 band prefetch (S even), the register-gather
    kernel (S odd: 1 lane per thread) - and through the face-form operator
    produce identical bits."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parents[1])
    out = {}
    for tag, faces, band in (("csr_band", "0", "1"), ("csr", "0", "0"), ("faces", "1", "1")):
        env = dict(os.environ, UQG_BAND_HINT=band, UQG_PCG_PERSISTENT="0", UQG_FV2D_FACES=faces)
        dst = tmp_path / f"{tag}.npy"
        subprocess.run([sys.executable, "-c", _CSR_SCRIPT, root, str(dst), S], env=env, check=True)
        out[tag] = np.load(dst)
    assert np.array_equal(out["csr_band"], out["faces"])
    assert np.array_equal(out["csr"], out["faces"])


def test_empty_plan_and_level():
    """Edge cases as the reference handles them: an empty plan solves nothing
    (harness.py:409 loops over no ensembles); an empty level cannot be grouped
    (grouping.py:100-101, 115-116)."""
    from paper_1705_02003_b200.grouping import GroupingPlan
    cfg = uq.CONFIGS["C1"]
    solver = uq.EnsembleSolver2D(uq.build_field(**cfg.field_kwargs()), cfg.cells, cfg.tol,
                                 cfg.maxit)
    assert solver.solve_plan(GroupingPlan(1, 4, (), (), "sur"), {}) == ({}, {}, [])
    with pytest.raises(uq.GroupingError):
        solver.solve_level([], np.zeros((0, cfg.n_modes)), 4)


def test_lane_limit_raises_cleanly():
    """S > 512 lanes (kMaxLanes: one tile row per 256-thread block at most) is
    rejected with EnsembleError instead of launching."""
    d = np.ones((513, 3))
    with pytest.raises(uq.EnsembleError):
        uq.ensemble_pcg(diag_ensemble(d), np.ones((513, 3)))
    r = uq.ensemble_pcg(diag_ensemble(np.ones((512, 3))), np.ones((512, 3)))
    assert r.converged_per_lane.all()


def test_dropped_solver_leaves_no_workspace_behind():
    """A solver's workspace is registered with the library context only while
    its wave runs: after the solver is dropped and torch reuses that memory,
    other library calls (here the drop-in lane_dot) must not carve scratch out
    of it (regression: an intermittent lane_dot mismatch)."""
    import gc

    import torch

    cfg = uq.CONFIGS["C1"]
    f = uq.build_field(**cfg.field_kwargs())
    for faces in (True, False):
        solver = uq.EnsembleSolver2D(f, cfg.cells, cfg.tol, cfg.maxit, faces=faces)
        solver.solve_groups(np.random.default_rng(0).uniform(-1, 1, (2, 8, cfg.n_modes)))
        nbytes = solver._ws.numel()
        del solver
        gc.collect()
        guard = torch.full((nbytes // 8,), 7.0, dtype=torch.float64, device=_lib.device())
        rng = np.random.default_rng(3)
        a, b = rng.standard_normal((64, 4097)), rng.standard_normal((64, 4097))
        got = uq.lane_dot(a, b)
        np.testing.assert_allclose(got, np.einsum("sn,sn->s", a, b), rtol=1e-12)
        assert bool((guard == 7.0).all())


def test_interleaved_entry_points_are_deterministic():
    """Level solves of two mesh sizes (faces and CSR), drop-in ensemble_pcg
    and lane_dot calls interleaved, solvers created and dropped between
    rounds: every round reproduces the first round's results bit for bit
    (workspace reuse, growth and context state leave no trace)."""
    import gc

    cfg = uq.CONFIGS["C1"]
    f = uq.build_field(**cfg.field_kwargs())
    rng = np.random.default_rng(4)
    ys_small = rng.uniform(-1, 1, (3, 8, cfg.n_modes))
    ys_big = rng.uniform(-1, 1, (2, 16, cfg.n_modes))
    lanes, rhs = spd_system(np.random.default_rng(9), 40, 3)
    ens = uq.EnsembleCsrMatrix.from_scipy_lanes(lanes)
    a, b = rng.standard_normal((16, 3000)), rng.standard_normal((16, 3000))

    def one_round():
        out = []
        for cells, ys, faces in ((cfg.cells, ys_small, True), (96, ys_big, False),
                                 (96, ys_big, True), (cfg.cells, ys_small, False)):
            s = uq.EnsembleSolver2D(f, cells, cfg.tol, cfg.maxit, faces=faces)
            r = s.solve_groups(ys)
            out += [r.iterations.ravel().astype(float), r.qoi.ravel()]
            res = uq.ensemble_pcg(ens, rhs, tol=1e-10, maxit=300)
            out += [res.solution.ravel(), uq.lane_dot(a, b)]
            del s
            gc.collect()
        return np.concatenate(out)

    first = one_round()
    for _ in range(3):
        assert np.array_equal(one_round(), first)
