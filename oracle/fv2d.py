"""Oracle: 2D 5-point finite-volume ensemble operator (TEST INFRA ONLY).

-div(diag(a1, a2) grad u) = 1 on the unit square, u = 0 on the boundary,
vertex-centred FV on an n x n cell grid (h = 1/n), (n-1)^2 interior unknowns.
This restatement defines the BASELINE.json operator, which the reference does
not contain; it follows the reference's 3D FEM contract (``fem3d.py:57-175``):

* dofs are interior nodes numbered lexicographically, second coordinate fastest
  (``fem3d.py:78-82``: z fastest);
* one shared, column-sorted CSR graph per mesh (``fem3d.py:97-108``);
* per-lane values depend on that lane's sample only, so duplicated samples give
  bit-identical lanes (``fem3d.py:10-12``);
* the coefficient is sampled at nodes through ``KL2D.coeff`` (``eval_a_batch``),
  a non-positive value raises (``fem3d.py:153-154``);
* load f = 1 integrates to h^2 per control volume; ``qoi`` is ``u . u``
  (``fem3d.py:178-183``).

Pinned arithmetic (the device kernel reproduces it bit for bit):
* x-face transmissibility between nodes a, b:  ``(2.0 * a) * b / (a + b)``
  (harmonic mean; the h/h factors cancel in 2D);
* y-face transmissibility: the constant ``a_y`` (reference convention: only the
  first direction is random, ``fem3d.py:158-160``), or, with ``a2="same"``, the
  harmonic mean of a1 along y;
* row (i,j), neighbours W=(i-1,j), S=(i,j-1), N=(i,j+1), E=(i+1,j):
  ``diag = ((Tw + Te) + Ts) + Tn``, off-diagonals ``-T``; boundary neighbours
  are dropped from the graph but their T stays in the diagonal.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .field2d import KL2D


@dataclass
class Mesh2D:
    cells: int

    def __post_init__(self):
        n = self.cells
        if n < 2:
            raise ValueError("need at least 2 cells per direction")
        self.h = 1.0 / n
        self.m = n - 1  # interior nodes per direction
        self.n_dofs = self.m * self.m
        self.n_nodes = (n + 1) * (n + 1)
        axis = np.arange(n + 1) * self.h
        gi, gj = np.meshgrid(axis, axis, indexing="ij")
        self.node_points = np.stack([gi.ravel(), gj.ravel()], axis=1)  # node id = i*(n+1)+j
        m = self.m
        ii, jj = np.meshgrid(np.arange(1, n), np.arange(1, n), indexing="ij")
        ii, jj = ii.ravel(), jj.ravel()
        dof = np.arange(self.n_dofs)
        # stencil slots in CSR (ascending column) order: W, S, C, N, E
        self._present = np.stack([ii > 1, jj > 1, np.ones_like(ii, bool), jj < m, ii < m], axis=1)
        cols = np.stack([dof - m, dof - 1, dof, dof + 1, dof + m], axis=1)
        self.col_indices = cols[self._present].astype(np.int32)
        self.row_offsets = np.concatenate([[0], np.cumsum(self._present.sum(axis=1))]).astype(np.int32)
        self.nnz = int(self.row_offsets[-1])
        self._ii, self._jj = ii, jj

    def interior_points(self) -> np.ndarray:
        ii, jj = self._ii, self._jj
        return np.stack([ii * self.h, jj * self.h], axis=1)


def _harm(a, b):
    return 2.0 * a * b / (a + b)


def assemble_values(mesh: Mesh2D, a_nodes: np.ndarray, a_y: float, a2: str = "const") -> np.ndarray:
    """(S, P) nodal a1 -> (S, nnz) CSR values in the shared graph's order."""
    n = mesh.cells
    S = a_nodes.shape[0]
    grid = a_nodes.reshape(S, n + 1, n + 1)  # [s, i, j]
    ii, jj = mesh._ii, mesh._jj
    tw = _harm(grid[:, ii - 1, jj], grid[:, ii, jj])
    te = _harm(grid[:, ii, jj], grid[:, ii + 1, jj])
    if a2 == "const":
        ts = np.full_like(tw, a_y)
        tn = ts
    elif a2 == "same":
        ts = _harm(grid[:, ii, jj - 1], grid[:, ii, jj])
        tn = _harm(grid[:, ii, jj], grid[:, ii, jj + 1])
    else:
        raise ValueError(a2)
    diag = ((tw + te) + ts) + tn
    slots = np.stack([-tw, -ts, diag, -tn, -te], axis=2)  # (S, N, 5)
    return slots[:, mesh._present]


@dataclass
class System2D:
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray  # (S, nnz)
    rhs: np.ndarray  # (S, N)
    samples: np.ndarray


def assemble(mesh: Mesh2D, field: KL2D, samples, table=None, a2: str = "const") -> System2D:
    """Width-S ensemble system for the sample rows (fem3d.py:138-175 contract)."""
    ys = np.atleast_2d(np.asarray(samples, dtype=float))
    a = field.coeff(mesh.node_points, ys, table)
    if np.any(a <= 0) or field.a_y <= 0:
        raise ValueError("non-positive diffusion coefficient")
    vals = assemble_values(mesh, a, field.a_y, a2)
    rhs = np.full((len(ys), mesh.n_dofs), mesh.h * mesh.h)
    return System2D(mesh.row_offsets, mesh.col_indices, vals, rhs, ys.copy())


def qoi(u) -> float:
    u = np.asarray(u, dtype=float)
    return float(np.dot(u, u))
