"""3D trilinear hexahedral FEM ensemble operator - the reference's own operator
(``fem3d.py``), assembled on the GPU ("next" row 1).

-div(diag(a(x,y), a_y, a_z) grad u) = 1 on [0,1]^3, u = 0 on the boundary,
m cells per direction, (m-1)^3 interior unknowns numbered z fastest.

Host setup (once per mesh) restates ``StructuredMesh`` (``fem3d.py:57-126``):
the shared 27-point CSR graph (``:97-108``), the reference-element tables
``_elem_mats[0]`` (x-direction, per quadrature point) and the constant
``a_y, a_z`` part (``:112``, ``:160``), the f = 1 load (``:114``, ``:168-174``)
- computed with the reference's own numpy expressions, so the tables are
bit-identical.  The device does the per-sample work:

* ``uqg_kl_eval_sep3d``  - a(x_q, y) at the 8 Gauss points of every element,
  mode values rebuilt from 1D tables (``random_field.py:145-166``);
* ``uqg_assemble_fem3d`` - per lane, every nonzero (i, j) sums its element
  contributions K_e(a, b) = sum_q a_q Dx[q,a,b] + Kyz[a,b] in increasing
  element order - the order ``np.bincount`` accumulates the (element, a, b)
  pairs in (``fem3d.py:163-166``) - and writes [nnz][S] plus 1/diag.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import FemError
from .field import GAUSS

__all__ = ["StructuredMesh3D", "shape_data"]


def shape_data():
    """Trilinear shape gradients at the 8 Gauss points (``fem3d.py:33-51``).

    Corners and quadrature points are both bit-ordered (x, y, z), z fastest.
    Returns dphi (3, 8q, 8a).
    """
    corners = np.array([[dx, dy, dz] for dx in (0, 1) for dy in (0, 1) for dz in (0, 1)])
    signs = 2.0 * corners - 1.0
    qpts = signs * GAUSS
    dphi = np.empty((3, 8, 8))
    for q in range(8):
        one = 1.0 + signs * qpts[q]
        for d in range(3):
            others = [i for i in range(3) if i != d]
            dphi[d, q] = signs[:, d] * one[:, others].prod(axis=1) / 8.0
    return dphi


class StructuredMesh3D:
    """Uniform hex mesh of the unit cube: graph, element tables, load."""

    def __init__(self, cells: int):
        if cells < 2:
            raise FemError(f"need at least 2 cells per direction, got {cells}")
        m = self.cells = int(cells)
        self.h = 1.0 / m
        k = m - 1
        self.n_dofs = k ** 3
        self.n_elems = m ** 3
        self.n_quad = 8 * self.n_elems
        # 27-point graph: neighbours (dx, dy, dz) in lexicographic order give
        # ascending columns (dof = ((ix-1) k + (iy-1)) k + (iz-1)).
        idx = np.arange(1, m)
        ix, iy, iz = (a.ravel() for a in np.meshgrid(idx, idx, idx, indexing="ij"))
        offs = np.array([(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)])
        jx = ix[:, None] + offs[None, :, 0]
        jy = iy[:, None] + offs[None, :, 1]
        jz = iz[:, None] + offs[None, :, 2]
        keep = (jx >= 1) & (jx <= k) & (jy >= 1) & (jy <= k) & (jz >= 1) & (jz <= k)
        cols = ((jx - 1) * k + (jy - 1)) * k + (jz - 1)
        self.col_indices = cols[keep].astype(np.int32)
        self.row_offsets = np.zeros(self.n_dofs + 1, dtype=np.int32)
        np.cumsum(keep.sum(axis=1), out=self.row_offsets[1:])
        self.nnz = int(self.row_offsets[-1])
        # reference-element tables (fem3d.py:112): (3, 8q, 8a, 8b) scaled by h/2
        dphi = shape_data()
        self.elem_mats = dphi[:, :, :, None] * dphi[:, :, None, :] * (self.h / 2.0)
        # f = 1 load: every interior node collects h^3/8 from its 8 elements
        load = 0.0
        for _ in range(8):
            load += self.h ** 3 / 8.0
        self.load = load
        self._dev = None

    def kyz(self, a_y: float, a_z: float) -> np.ndarray:
        """Constant second/third-direction element matrix (``fem3d.py:160``)."""
        return a_y * self.elem_mats[1].sum(axis=0) + a_z * self.elem_mats[2].sum(axis=0)

    def quad_points(self) -> np.ndarray:
        """(E*8, 3) Gauss points, element-major, q bit-ordered (``fem3d.py:93-95``)."""
        m = self.cells
        ex, ey, ez = np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij")
        elems = np.stack([ex.ravel(), ey.ravel(), ez.ravel()], axis=1)
        corners = np.array([[dx, dy, dz] for dx in (0, 1) for dy in (0, 1) for dz in (0, 1)])
        qref = (2.0 * corners - 1.0) * GAUSS
        centers = (elems + 0.5) * self.h
        return (centers[:, None, :] + qref[None, :, :] * (self.h / 2.0)).reshape(-1, 3)

    def interior_node_coords(self) -> np.ndarray:
        ax = np.arange(1, self.cells) * self.h
        g = np.meshgrid(ax, ax, ax, indexing="ij")
        return np.stack([a.ravel() for a in g], axis=1)

    def center_dof(self) -> int:
        c = self.interior_node_coords()
        return int(np.argmin(((c - 0.5) ** 2).sum(axis=1)))

    def device(self):
        if self._dev is None:
            self._dev = (_lib.to_dev(self.row_offsets), _lib.to_dev(self.col_indices),
                         _lib.to_dev(np.ascontiguousarray(self.elem_mats[0])))
        return self._dev
