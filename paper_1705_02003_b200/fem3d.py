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

__all__ = ["StructuredMesh3D", "StructuredMesh", "assemble", "shape_data"]


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

    def __init__(self, cells: int, quadrature: str = "gauss2"):
        if cells < 2:
            raise FemError(f"need at least 2 cells per direction, got {cells}")
        if quadrature != "gauss2":
            raise FemError(f"unsupported quadrature {quadrature!r}")
        self.quadrature = quadrature
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

    @property
    def quad_points(self) -> np.ndarray:
        """(E*8, 3) Gauss points, element-major, q bit-ordered (``fem3d.py:93-95``)."""
        if getattr(self, "_qp", None) is None:
            self._qp = self._quad_points()
        return self._qp

    def _quad_points(self) -> np.ndarray:
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


StructuredMesh = StructuredMesh3D  # the reference's name (fem3d.py:57)


def assemble(mesh: StructuredMesh3D, field, samples, mode_vals=None):
    """Drop-in for the reference's ``assemble`` (``fem3d.py:138-175``) on its
    own 3D operator: the width-S ensemble system assembled on the GPU
    (``uqg_kl_eval_sep3d`` + ``uqg_assemble_fem3d``), the matrix kept
    device-resident as ``[nnz][S]`` (host values materialise lazily).

    ``mode_vals`` is accepted for signature parity; the device rebuilds the
    mode values at the Gauss points from separable 1D tables (bit-identical
    to ``field.mode_values(mesh.quad_points)``).  Raises ``FemError`` on a
    non-positive coefficient (``:153-154``) before returning.
    """
    from .ensemble import EnsembleCsrMatrix
    from .fv2d import AssembledEnsembleSystem
    from .solve import FEM3DOperator

    ys = np.atleast_2d(np.asarray(samples, dtype=np.float64))
    S = len(ys)
    if getattr(field, "dim", 3) != 3:
        raise FemError("the 3D operator needs a 3D field (build_field(..., dim=3))")
    if ys.shape[1] != field.n_modes:
        raise FemError(f"samples must have {field.n_modes} columns, got {ys.shape[1]}")
    if field.a_y <= 0 or field.a_z <= 0:
        raise FemError("non-positive diffusion coefficient at a quadrature point")
    torch = _lib._torch()
    op = FEM3DOperator(field, mesh.cells, mesh=mesh)
    _lib.call("uqg_status_clear", _lib.ctx(), _lib.stream())
    a = torch.empty((mesh.n_quad * S,), dtype=torch.float64, device=_lib.device())
    op.coefficients(_lib.to_dev(ys), None, 1, S, a)
    if _lib.status_sync() & 1:
        raise FemError("non-positive diffusion coefficient at a quadrature point")
    vals = torch.empty((mesh.nnz * S,), dtype=torch.float64, device=_lib.device())
    op.assemble(a, 1, S, vals, None)
    rowptr, col, _ = mesh.device()
    mat = EnsembleCsrMatrix.from_device(mesh.row_offsets, mesh.col_indices, rowptr, col, vals, S)
    rhs = np.full((S, mesh.n_dofs), mesh.load)
    return AssembledEnsembleSystem(matrix=mat, rhs=rhs, samples=ys.copy())
