"""3D trilinear FEM host setup against the reference's
golden outputs: graph, element tables, load, 3D mode selection, study keys."""

import json

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1705_02003_b200 import build_field
from paper_1705_02003_b200.fem3d import StructuredMesh3D
from paper_1705_02003_b200.sparse_grid import SparseGrid


@pytest.fixture(scope="module")
def fem3d_golden():
    with np.load(GOLDEN / "fem3d.npz") as z:
        return {k: z[k] for k in z.files}


def test_graph_and_load_match_reference(fem3d_golden):
    g = fem3d_golden
    mesh = StructuredMesh3D(6)
    assert np.array_equal(mesh.row_offsets, g["row_offsets"])
    assert np.array_equal(mesh.col_indices, g["col_indices"])
    assert np.all(g["rhs"] == mesh.load)  # bit-identical constant load h^3
    assert StructuredMesh3D(16).nnz == 79507  # test_fem3d.py:43-49
    assert StructuredMesh3D(16).n_dofs == 15 ** 3


def test_element_tables_reproduce_reference_row_stencil():
    """Constant unit coefficient: one interior row = the 27-point trilinear
    Laplacian stencil (test_fem3d.py:84-105) scaled by h."""
    m = 8
    mesh = StructuredMesh3D(m)
    kx = mesh.elem_mats[0].sum(axis=0) + mesh.kyz(1.0, 1.0)  # a = 1 at every quad point
    k1 = {-1: -1.0, 0: 2.0, 1: -1.0}
    m1 = {-1: 1.0 / 6.0, 0: 4.0 / 6.0, 1: 1.0 / 6.0}
    # assemble the centre row by hand from the element matrices
    c = (4, 4, 4)
    row = {}
    for ex in (3, 4):
        for ey in (3, 4):
            for ez in (3, 4):
                a = (c[0] - ex) * 4 + (c[1] - ey) * 2 + (c[2] - ez)
                for b in range(8):
                    j = (ex + (b >> 2), ey + ((b >> 1) & 1), ez + (b & 1))
                    off = tuple(jj - cc for jj, cc in zip(j, c))
                    row[off] = row.get(off, 0.0) + kx[a, b]
    for (dx, dy, dz), v in row.items():
        want = (k1[dx] * m1[dy] * m1[dz] + m1[dx] * k1[dy] * m1[dz] + m1[dx] * m1[dy] * k1[dz]) / m
        assert abs(v - want) < 1e-15


def test_3d_mode_selection_known_answer():
    """test_random_field.py:94-100: four modes, eigenvalues [1.00882, 0.563383 x3]."""
    f = build_field(0.25, np.sqrt(300.0), 4, 0.1, sigma0_convention="kernel", dim=3)
    assert f.modes == ((0, 0, 0), (0, 0, 1), (0, 1, 0), (1, 0, 0))
    np.testing.assert_allclose(f.eigenvalues, [1.00882, 0.563383, 0.563383, 0.563383], atol=2e-4)


def test_quad_tables_rebuild_dense_mode_table():
    f = build_field(0.25, np.sqrt(300.0), 4, 0.1, sigma0_convention="kernel", dim=3)
    m = 5
    mesh = StructuredMesh3D(m)
    dense = f.mode_values(mesh.quad_points)
    qt = f.quad_tables(m)
    e = np.arange(m ** 3)
    ex, ey, ez = e // (m * m), (e // m) % m, e % m
    for k, (p, q, r) in enumerate(f.modes):
        for qq in range(8):
            rec = (qt[p][2 * ex + (qq >> 2)] * qt[q][2 * ey + ((qq >> 1) & 1)]) * qt[r][2 * ez + (qq & 1)]
            assert np.array_equal(rec, dense[k][e * 8 + qq])


@pytest.mark.parametrize("preset", ["pde_test1", "pde_test2"])
def test_sparse_grid_reproduces_reference_study_keys(preset):
    doc = json.loads((GOLDEN / f"{preset}_study.json").read_text())
    g = SparseGrid(4)
    batch = g.add_initial_levels(1)
    for lv in doc["levels"]:
        start = len(g) - len(batch)
        ids = list(range(start, len(g)))
        assert ids == lv["ids"]
        coords = g.node_coords()[start:]
        assert np.array_equal(coords, np.array(lv["coords"]))
        if lv["predicted"] is not None:
            assert np.array_equal(g.evaluate("iterations", coords, n_nodes=start),
                                  np.array(lv["predicted"]))
        g.fit("qoi", dict(zip(ids, lv["qoi"])))
        g.fit("iterations", dict(zip(ids, lv["iterations"])))
        batch, _ = g.refine(1e-3, "qoi", 600)
        if not batch:
            break
