"""Pin the CPU oracle against the reference's own outputs (golden fixtures).

When /root/reference is importable (build container) the oracle is also
compared live against the reference modules; on the GPU box those tests skip
and the committed fixtures carry the pin.
"""

import sys

import numpy as np
import pytest

from oracle import field2d, fv2d, grouping, pcg

REF = "/root/reference/pkg/src"


def _ref():
    try:
        sys.path.insert(0, REF)
        import uqgroup  # noqa: F401
        return uqgroup
    except Exception:
        pytest.skip("reference package not present on this host")
    finally:
        if sys.path and sys.path[0] == REF:
            sys.path.pop(0)


def test_spmv_oracle_matches_reference_scipy_bitwise(pcg_golden):
    for c in pcg_golden:
        ax = pcg.spmv(c["row_offsets"], c["col_indices"], c["values"], c["x"])
        assert np.array_equal(ax, c["Ax"])
        seq = pcg.spmv_sequential(c["row_offsets"], c["col_indices"], c["values"], c["x"])
        assert np.array_equal(seq, c["Ax"])  # scipy == sequential non-FMA CSR sum


def test_pcg_oracle_matches_reference_bitwise(pcg_golden):
    for c in pcg_golden:
        r = pcg.pcg(c["row_offsets"], c["col_indices"], c["values"], c["rhs"], tol=float(c["tol"]),
                    maxit=5000, history=True)
        assert np.array_equal(r.iterations, c["iterations"])
        assert np.array_equal(r.converged, c["converged"])
        assert np.array_equal(r.frozen, c["frozen"])
        assert np.array_equal(r.solution, c["solution"])
        assert np.array_equal(np.array(r.history), c["history"])


def test_oracle_diagonal(pcg_golden):
    for c in pcg_golden:
        inv = pcg.jacobi_inverse(c["row_offsets"], c["col_indices"], c["values"])
        assert np.array_equal(inv, 1.0 / c["diag"])


def test_oracle_special_cases(special_golden):
    g = special_golden
    tiny = np.finfo(np.float64).tiny
    r = pcg.pcg(np.arange(3), np.arange(2), np.array([[2.0, 3.0], [4.0, 5.0]]), np.zeros((2, 2)))
    assert np.array_equal(r.iterations, g["zero_iters"])
    rhs = np.arange(15.0).reshape(3, 5)
    r = pcg.pcg(np.arange(6), np.arange(5), np.ones((3, 5)), rhs)
    assert np.array_equal(r.iterations, g["ident_iters"]) and np.array_equal(r.solution, g["ident_x"])
    d = np.array([[2.0, 2.0], [0.5 * tiny, 0.5 * tiny]])
    r = pcg.pcg(np.arange(3), np.arange(2), d, np.ones((2, 2)), inv_diag=np.ones((2, 2)), tol=1e-8,
                maxit=50)
    assert np.array_equal(r.solution, g["frz_x"]) and np.array_equal(r.frozen, g["frz_frozen"])
    assert np.array_equal(r.iterations, g["frz_iters"])
    with pytest.raises(pcg.Breakdown):
        pcg.pcg(np.arange(3), np.arange(2), np.array([[1.0, np.inf]]), np.ones((1, 2)),
                inv_diag=np.ones((1, 2)), maxit=5)


def test_grouping_oracle_matches_reference(grouping_golden):
    for case in grouping_golden:
        ids, size = case["ids"], case["size"]
        keys = dict(zip(ids, case["keys"]))
        ens, pad = grouping.by_key(ids, keys, size)
        assert [list(g) for g in ens] == case["by_key"] and list(pad) == case["by_key_pad"]
        ens, pad = grouping.natural(ids, size)
        assert [list(g) for g in ens] == case["natural"] and list(pad) == case["natural_pad"]


def test_nystrom_oracle_matches_reference(eigen_golden):
    for delta in (0.2, 0.1, 0.05, 0.25):
        modes = field2d.nystrom_1d(delta, 12, 513)
        assert np.array_equal([m.eigenvalue for m in modes], eigen_golden[f"lam_{delta}"])
        assert np.array_equal(np.stack([m.values for m in modes]), eigen_golden[f"vec_{delta}"])


def test_pair_selection_matches_brute_force():
    f = field2d.KL2D.select(0.1, 1.5, 12, 0.0)
    lam = [m.eigenvalue for m in field2d.nystrom_1d(0.1, 8, 513)]
    best = sorted(((lam[p] * lam[q], (p, q)) for p in range(8) for q in range(8)),
                  key=lambda t: (-t[0], t[1]))[:12]
    assert f.modes == tuple(m for _, m in best)
    np.testing.assert_allclose(f.eigenvalues, [2.25 * v for v, _ in best], rtol=1e-15)
    assert f.modes[1:3] == ((0, 1), (1, 0))  # lexicographic tie-break of the symmetric pair


def test_fv2d_operator_properties(fv2d_golden):
    g = fv2d_golden
    mesh = fv2d.Mesh2D(8)
    assert np.array_equal(mesh.row_offsets, g["row_offsets"])
    assert np.array_equal(mesh.col_indices, g["col_indices"])
    vals = fv2d.assemble_values(mesh, g["a_nodes"], 1.0)
    assert np.array_equal(vals, g["values"])
    assert np.array_equal(vals[0], vals[2])  # duplicated samples -> bit-identical lanes
    for s in range(3):
        A = pcg.lane_mats(mesh.row_offsets, mesh.col_indices, vals)[s].toarray()
        assert np.array_equal(A, A.T)  # exactly symmetric
        assert np.all(np.linalg.eigvalsh(A) > 0)
    # constant coefficient 1 -> the classic 5-point Laplacian (h^2-scaled)
    ones = np.ones((1, mesh.n_nodes))
    A = pcg.lane_mats(mesh.row_offsets, mesh.col_indices, fv2d.assemble_values(mesh, ones, 1.0))[0]
    m = mesh.m
    T = np.diag(np.full(m, 2.0)) - np.diag(np.ones(m - 1), 1) - np.diag(np.ones(m - 1), -1)
    lap = np.kron(T, np.eye(m)) + np.kron(np.eye(m), T)
    assert np.array_equal(A.toarray(), lap)


def test_fv2d_poisson_centre_value():
    """-lap u = 1 on the unit square: u(1/2,1/2) = 0.0736713532... (series)."""
    mesh = fv2d.Mesh2D(64)
    ones = np.ones((1, mesh.n_nodes))
    vals = fv2d.assemble_values(mesh, ones, 1.0)
    rhs = np.full((1, mesh.n_dofs), mesh.h ** 2)
    r = pcg.pcg(mesh.row_offsets, mesh.col_indices, vals, rhs, tol=1e-12, maxit=5000)
    k = np.arange(1, 200, 2, dtype=float)
    ii, jj = np.meshgrid(k, k, indexing="ij")
    sgn = np.where(((ii - 1) / 2 + (jj - 1) / 2) % 2 == 0, 1.0, -1.0)
    series = 16.0 / np.pi ** 4 * (sgn / (ii * jj * (ii ** 2 + jj ** 2))).sum()
    centre = r.solution[0][(mesh.m // 2) * mesh.m + mesh.m // 2]
    assert abs(centre - series) < 2e-4


def test_oracle_live_against_reference():
    uq = _ref()
    rng = np.random.default_rng(99)
    n, S = 40, 3
    lanes = []
    base = np.triu(np.where(rng.random((n, n)) < 0.15, rng.uniform(-1, 1, (n, n)), 0.0), 1)
    base = base + base.T
    for _ in range(S):
        v = base * rng.uniform(0.2, 1.0)
        np.fill_diagonal(v, np.abs(v).sum(axis=1) + 1.0)
        lanes.append(v)
    import scipy.sparse as sp
    ens = uq.EnsembleCsrMatrix.from_scipy_lanes([sp.csr_matrix(v) for v in lanes])
    rhs = rng.standard_normal((S, n))
    a = uq.ensemble_pcg(ens, rhs, tol=1e-10, maxit=500)
    b = pcg.pcg(ens.row_offsets, ens.col_indices, ens.values, rhs, tol=1e-10, maxit=500)
    assert np.array_equal(a.solution, b.solution)
    assert np.array_equal(a.iterations_per_lane, b.iterations)
    f = uq.build_field(0.2, 1.0, 3, 0.0)  # 3D reference field: eigenpairs shared
    assert np.array_equal([p.eigenvalue for p in f.factors],
                          [m.eigenvalue for m in field2d.nystrom_1d(0.2, len(f.factors))])
