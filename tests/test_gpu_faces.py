"""Face form of the 2D FV operator (uqg_assemble_fv2d_faces / uqg_spmv_fv2d /
uqg_pcg_fv2d) against the CSR form of the same matrix.

The face form re-derives each CSR row from the face transmissibilities with
the same products in the same column order, so the bar is bit-identity with
the CSR path - which the rest of the suite pins to the oracle and to the
reference's golden outputs (test_gpu_parity.py).
"""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_1705_02003_b200 as uq
from paper_1705_02003_b200 import _lib
from paper_1705_02003_b200.fv2d import StructuredMesh2D, assemble_faces, assemble_values

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _nodes(rng, cells, G, S):
    a = np.exp(rng.standard_normal((G, (cells + 1) ** 2, S)))  # positive, lognormal
    return _lib.to_dev(np.ascontiguousarray(a).ravel())


@pytest.mark.parametrize("cells,S,G", [(2, 1, 1), (5, 3, 2), (17, 8, 3), (64, 16, 2),
                                       (33, 32, 1), (9, 2, 5)])
@pytest.mark.parametrize("a2", ["const", "same"])
def test_face_spmv_and_dinv_bitwise_equal_csr(cells, S, G, a2):
    rng = np.random.default_rng(cells * 100 + S)
    mesh = StructuredMesh2D(cells)
    a = _nodes(rng, cells, G, S)
    a_y = 0.7
    vals, dinv_csr = assemble_values(mesh, a, G, S, a_y, a2)
    tx, ty, dinv = assemble_faces(mesh, a, G, S, a_y, a2)
    assert (ty is None) == (a2 == "const")
    assert np.array_equal(dinv.cpu().numpy(), dinv_csr.cpu().numpy())
    N = mesh.n_dofs
    x = _lib.to_dev(rng.standard_normal(G * N * S))
    y_csr = x.new_empty(G * N * S)
    y_fac = x.new_empty(G * N * S)
    rowptr, col = mesh.device()
    _lib.call("uqg_spmv", _lib.ctx(), N, mesh.nnz, 5, S, G, _lib.ptr(rowptr), _lib.ptr(col),
              _lib.ptr(vals), _lib.ptr(x), _lib.ptr(y_csr), _lib.stream())
    _lib.call("uqg_spmv_fv2d", _lib.ctx(), cells, S, G, _lib.ptr(tx), _lib.ptr(ty), a_y,
              _lib.ptr(x), _lib.ptr(y_fac), _lib.stream())
    assert np.array_equal(y_fac.cpu().numpy(), y_csr.cpu().numpy())


def test_face_entry_points_validate_arguments():
    with pytest.raises(uq.EnsembleError):
        _lib.call("uqg_spmv_fv2d", _lib.ctx(), 1, 1, 1, None, None, 1.0, None, None, None)
    mesh = StructuredMesh2D(4)
    a = _nodes(np.random.default_rng(0), 4, 1, 2)
    tx = a.new_empty(mesh.n_dofs * 4)
    with pytest.raises(uq.EnsembleError):  # a2_same needs ty
        _lib.call("uqg_assemble_fv2d_faces", _lib.ctx(), 4, 1, 2, _lib.ptr(a), 1.0, 1,
                  _lib.ptr(tx), None, None, _lib.stream())


_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1705_02003_b200 as uq
cfg = uq.CONFIGS["C1"]
f = uq.build_field(**cfg.field_kwargs())
out = []
for a2 in ("const", "same"):
    for faces in (False, True):
        s = uq.EnsembleSolver2D(f, cfg.cells, cfg.tol, cfg.maxit, a2=a2, faces=faces)
        ys = np.random.default_rng(5).uniform(-1, 1, (6, cfg.ensemble_size, cfg.n_modes))
        r = s.solve_groups(ys, record_history=True)
        h = np.concatenate([np.concatenate(g) for g in r.histories])
        out.append(np.concatenate([r.iterations.ravel().astype(float), r.qoi.ravel(),
                                   r.converged.ravel().astype(float), h]))
np.save(sys.argv[2], np.array(out, dtype=object), allow_pickle=True)
"""


_VARIANTS = {  # solve-loop variants (all must give the CSR bits)
    "reg": {},                                            # default launch loop
    "graph": {"UQG_PCG_GRAPH": "1"},                      # launch loop as one graph launch
}


@pytest.mark.parametrize("persistent,variant", [
    ("0", "reg"), ("1", "reg"), ("2", "reg")] + [("0", v) for v in _VARIANTS if v != "reg"])
def test_face_pcg_bitwise_equal_csr_pcg(tmp_path, persistent, variant):
    """Whole batched solves (iterations, QoIs, residual histories) through the
    launch loop (0), the cooperative (1) and the cluster (2) persistent kernel,
    and the graph launch loop."""
    env = dict(os.environ, UQG_PCG_PERSISTENT=persistent, **_VARIANTS[variant])
    dst = tmp_path / "r.npy"
    subprocess.run([sys.executable, "-c", _SCRIPT, str(ROOT), str(dst)], env=env, check=True)
    out = np.load(dst, allow_pickle=True)
    csr_c, fac_c, csr_s, fac_s = out
    assert np.array_equal(csr_c, fac_c)
    assert np.array_equal(csr_s, fac_s)
    assert not np.array_equal(csr_c, csr_s)  # the random y coefficient does change the solve


def test_deferred_x_update_bitwise(tmp_path):
    """x += alpha_j p_j applied kx iterations at a time (UQG_X_DEFER; pcg_update
    FLUSH iterations + pcg_flush) rounds in the same order as the per-iteration
    update: every kx gives the bits of kx = 1, CSR and face operator, launch loop."""
    outs = {}
    for kx in ("1", "2", "3", "4", "8"):
        for graph in ("0", "1"):  # host-polled / graph launch loop
            env = dict(os.environ, UQG_PCG_PERSISTENT="0", UQG_X_DEFER=kx, UQG_PCG_GRAPH=graph)
            dst = tmp_path / f"x{kx}{graph}.npy"
            subprocess.run([sys.executable, "-c", _SCRIPT, str(ROOT), str(dst)], env=env,
                           check=True)
            outs[kx + graph] = np.load(dst, allow_pickle=True)
    for key in outs:
        for a, b in zip(outs[key], outs["10"]):
            assert np.array_equal(a, b), key


@pytest.mark.parametrize("S", [6, 64, 130, 512])
def test_face_pcg_wide_ensembles_bitwise(S):
    """Wide and non-power-of-two ensembles (lane padding Lp > L, one row per
    tile at S = 512): face-form solve == CSR solve, bit for bit."""
    f = uq.build_field(0.2, 1.0, 3, 0.0)
    ys = np.random.default_rng(S).uniform(-1, 1, (2, S, 3))
    out = []
    for faces in (False, True):
        s = uq.EnsembleSolver2D(f, 24, 1e-8, 3000, faces=faces)
        r = s.solve_groups(ys)
        out.append((r.iterations, r.qoi, r.converged))
    for a, b in zip(*out):
        assert np.array_equal(a, b)


_PARTS_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1705_02003_b200 as uq
cfg = uq.CONFIGS["C2"]
f = uq.build_field(**cfg.field_kwargs())
out = []
for a2 in ("const", "same"):
    s = uq.EnsembleSolver2D(f, cfg.cells, cfg.tol, cfg.maxit, a2=a2)
    ys = np.random.default_rng(11).uniform(-1, 1, (21, cfg.ensemble_size, cfg.n_modes))
    r = s.solve_groups(ys)
    out.append(np.concatenate([r.iterations.ravel().astype(float), r.qoi.ravel(),
                               r.ensemble_iterations.astype(float)]))
np.save(sys.argv[2], np.concatenate(out))
"""


def test_concurrent_parts_bitwise(tmp_path):
    """A level solved as 1, 2 or 3 concurrent parts on separate streams
    (UQG_SOLVE_STREAMS; C2 size, 21 groups: > 1 GB per part and iteration;
    constant and random y-faces) gives identical results."""
    outs = {}
    for k in ("1", "2", "3"):
        env = dict(os.environ, UQG_SOLVE_STREAMS=k)
        dst = tmp_path / f"p{k}.npy"
        subprocess.run([sys.executable, "-c", _PARTS_SCRIPT, str(ROOT), str(dst)], env=env,
                       check=True)
        outs[k] = np.load(dst)
    assert np.array_equal(outs["2"], outs["1"]) and np.array_equal(outs["3"], outs["1"])


_MAXIT_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1705_02003_b200 as uq
cfg = uq.CONFIGS["C1"]
f = uq.build_field(**cfg.field_kwargs())
out = []
for faces in (False, True):
    s = uq.EnsembleSolver2D(f, cfg.cells, cfg.tol, 37, faces=faces)   # maxit 37: 1 mod 4
    ys = np.random.default_rng(2).uniform(-1, 1, (5, cfg.ensemble_size, cfg.n_modes))
    r = s.solve_groups(ys)
    out.append(np.concatenate([r.iterations.ravel().astype(float), r.qoi.ravel(),
                               r.converged.ravel().astype(float)]))
np.save(sys.argv[2], np.array(out))
"""


def test_maxit_termination_with_deferred_update(tmp_path):
    """Groups stopped by maxit (unconverged lanes report the iterations run)
    with a pending deferred-update tail: identical for kx = 1 and 4, CSR and
    face operator, launch loop and persistent kernel."""
    outs = {}
    for tag, env_extra in (("loop1", {"UQG_PCG_PERSISTENT": "0", "UQG_X_DEFER": "1"}),
                           ("loop4", {"UQG_PCG_PERSISTENT": "0", "UQG_X_DEFER": "4"}),
                           ("graph4", {"UQG_PCG_PERSISTENT": "0", "UQG_X_DEFER": "4",
                                       "UQG_PCG_GRAPH": "1"}),
                           ("persistent", {})):
        dst = tmp_path / f"{tag}.npy"
        subprocess.run([sys.executable, "-c", _MAXIT_SCRIPT, str(ROOT), str(dst)],
                       env=dict(os.environ, **env_extra), check=True)
        outs[tag] = np.load(dst)
    ref = outs["loop1"]
    n = ref.shape[1] // 3
    assert (ref[0][:n] == 37).any() and not ref[0][2 * n:].all()  # some lanes hit maxit
    for tag in ("loop4", "graph4", "persistent"):
        assert np.array_equal(outs[tag], ref), tag
    assert np.array_equal(ref[0], ref[1])  # CSR == faces


@pytest.mark.parametrize("cells,S", [(2, 1), (3, 3), (7, 5), (17, 1), (33, 2)])
@pytest.mark.parametrize("maxit", [0, 1, 3000])
def test_small_and_odd_meshes_match_oracle(cells, S, maxit):
    """Edge shapes through the default (face-form) level solve: one-cell and
    few-cell meshes, single-lane and odd ensembles, a padded last group, and
    maxit 0 / 1 (unconverged lanes) - iterations and notes equal to the oracle's
    solve_plan, QoIs within 1e-8, and bit-identical to the CSR path."""
    sys.path.insert(0, str(ROOT))
    from oracle import driver as odriver, field2d, fv2d as ofv

    cfg = uq.CONFIGS["C1"]
    f = uq.build_field(**cfg.field_kwargs())
    o = field2d.KL2D.select(**cfg.field_kwargs())
    omesh = ofv.Mesh2D(cells)
    rng = np.random.default_rng(cells * 100 + S)
    ids = list(range(2 * S + 1))
    coords = {i: rng.uniform(-1, 1, cfg.n_modes) for i in ids}
    plan = uq.group_natural(ids, S, level=1)
    got = {}
    for faces in (True, False):
        solver = uq.EnsembleSolver2D(f, cells, cfg.tol, maxit, faces=faces)
        got[faces] = solver.solve_plan(plan, coords)
    it_d, q_d, notes_d = got[True]
    it_o, q_o, notes_o = odriver.solve_plan(omesh, o, o.mode_table(omesh.node_points),
                                            plan.ensembles, coords, cfg.tol, maxit, level=1)
    assert it_d == it_o and notes_d == notes_o
    if maxit == 0:
        assert notes_o and all(v == 0 for v in it_o.values())
    for i in ids:
        assert abs(q_d[i] - q_o[i]) <= 1e-8 * abs(q_o[i])
    assert got[False][0] == it_d and got[False][2] == notes_d
    assert all(got[False][1][i] == q_d[i] for i in ids)


_CLUSTER_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1705_02003_b200 as uq
out = []
for cells, G in ((128, 5), (128, 1), (512, 2)):      # chunks of m + 1 rows at S = 32
    f = uq.build_field(0.1, 1.5, 6, 0.0)
    s = uq.EnsembleSolver2D(f, cells, 1e-8, 400 if cells == 512 else 30000)
    ys = np.random.default_rng(cells + G).uniform(-1, 1, (G, 32, 6))
    ys[0, 1] = ys[0, 0]
    r = s.solve_groups(ys)
    out.append(np.concatenate([r.iterations.ravel().astype(float), r.qoi.ravel(),
                               r.converged.ravel().astype(float),
                               r.ensemble_iterations.astype(float)]))
np.save(sys.argv[2], np.concatenate(out))
"""


def test_cluster_multicast_face_spmv_bitwise(tmp_path):
    """UQG_FACE_CLUSTER=1 (thread-block clusters of two CTAs on adjacent chunks, band tiles
    fetched once by TMA multicast, full / empty mbarriers across the CTAs) gives the plain
    face kernel's bits for whole solves: n = 128 and n = 512 at S = 32 (chunks of m + 1 rows),
    several groups and a single group, converged and maxit-limited."""
    outs = {}
    for k in ("0", "1"):
        env = dict(os.environ, UQG_FACE_CLUSTER=k)
        dst = tmp_path / f"c{k}.npy"
        subprocess.run([sys.executable, "-c", _CLUSTER_SCRIPT, str(ROOT), str(dst)], env=env,
                       check=True, timeout=900)
        outs[k] = np.load(dst)
    assert np.array_equal(outs["0"], outs["1"])
