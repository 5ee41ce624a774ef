"""2D 5-point finite-volume ensemble operator: mesh (host setup) + device assembly.

Drop-in for the reference's ``fem3d`` entry points on the BASELINE.json
operator (-div(diag(a1, a2) grad u) = 1 on the unit square, u = 0 on the
boundary; operator definition pinned in ``oracle/fv2d.py`` and DESIGN.md):

* ``StructuredMesh2D`` <- ``StructuredMesh`` (``fem3d.py:57-126``): interior
  dofs (second coordinate fastest), the shared column-sorted CSR graph, node
  coordinates; built once per mesh on the host, uploaded once;
* ``assemble``         <- ``assemble`` (``fem3d.py:138-175``): KL coefficient at
  the nodes (``uqg_kl_eval_sep2d``) and the sample-interleaved values
  ``[nnz][S]`` (``uqg_assemble_fv2d``) on the GPU; ``FemError`` on a
  non-positive coefficient;
* ``qoi``              <- ``qoi`` (``fem3d.py:178-183``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .ensemble import EnsembleCsrMatrix
from .errors import FemError

__all__ = ["StructuredMesh2D", "AssembledEnsembleSystem", "assemble", "qoi"]


class StructuredMesh2D:
    def __init__(self, cells: int):
        if cells < 2:
            raise FemError(f"need at least 2 cells per direction, got {cells}")
        n = self.cells = int(cells)
        self.h = 1.0 / n
        m = n - 1
        self.n_dofs = m * m
        self.n_nodes = (n + 1) ** 2
        self.nnz = 5 * self.n_dofs - 4 * m
        i = np.repeat(np.arange(1, n), m)  # row r = (i-1)*m + (j-1)
        j = np.tile(np.arange(1, n), m)
        r = np.arange(self.n_dofs)
        stencil_cols = np.stack([r - m, r - 1, r, r + 1, r + m], axis=1)
        keep = np.stack([i > 1, j > 1, np.ones_like(i, dtype=bool), j < m, i < m], axis=1)
        self.col_indices = stencil_cols[keep].astype(np.int32)
        self.row_offsets = np.zeros(self.n_dofs + 1, dtype=np.int32)
        np.cumsum(keep.sum(axis=1), out=self.row_offsets[1:])
        self._dev = None

    def node_coords(self) -> np.ndarray:
        ax = np.arange(self.cells + 1) * self.h
        return np.stack(np.meshgrid(ax, ax, indexing="ij"), axis=-1).reshape(-1, 2)

    def interior_node_coords(self) -> np.ndarray:
        ax = np.arange(1, self.cells) * self.h
        return np.stack(np.meshgrid(ax, ax, indexing="ij"), axis=-1).reshape(-1, 2)

    def center_dof(self) -> int:
        c = self.interior_node_coords()
        return int(np.argmin(((c - 0.5) ** 2).sum(axis=1)))

    def device(self):
        """(rowptr, col) on the device, uploaded once.

        Both arrays carry 4 ints of zeroed slack after their last entry (the
        staged SpMV bulk-copies 16-byte aligned spans; ``band_hint``)."""
        if self._dev is None:
            pad = np.zeros(4, dtype=np.int32)
            ro = _lib.to_dev(np.concatenate([self.row_offsets, pad]))
            ci = _lib.to_dev(np.concatenate([self.col_indices, pad]))
            self._dev = (ro[: self.n_dofs + 1], ci[: self.nnz])
        return self._dev

    def band_hint(self):
        """Row bands holding the columns of a tile of rows [r0, r0+R): the
        x-neighbours [r0-m, r0-m+R), the row and its y-neighbours
        [r0-1, r0+R+1), [r0+m, r0+m+R) (m = cells - 1)."""
        m = self.cells - 1
        return [-m, -1, m], [0, 2, 0]


@dataclass
class AssembledEnsembleSystem:
    matrix: EnsembleCsrMatrix
    rhs: np.ndarray  # (S, n_dofs)
    samples: np.ndarray


class FieldTables:
    """Device constants of one (field, mesh) pair: separable 1D node tables."""

    def __init__(self, field, mesh: StructuredMesh2D):
        self.table = _lib.to_dev(field.node_tables(mesh.cells))
        self.n_factors = len(field.factors)
        consts = field._device_consts()
        self.sqrt_lam, self.mode_p, self.mode_q = consts["sqrt_lam"], consts["mode_p"], consts["mode_q"]
        self.ahat, self.expansion = field.codes()
        self.field, self.cells = field, mesh.cells


def kl_nodes(tables: FieldTables, d_samples, G: int, S: int, out=None, lane_ids=None):
    """a at all (n+1)^2 nodes -> device [G][P][S].

    Lane g*S+s uses sample row ``lane_ids[g*S+s]`` of ``d_samples`` (device
    int32), or row g*S+s when ``lane_ids`` is None.
    """
    f = tables.field
    P = (tables.cells + 1) ** 2
    if out is None:
        out = d_samples.new_empty((G * P * S,))
    _lib.call("uqg_kl_eval_sep2d", _lib.ctx(), tables.cells, _lib.ptr(tables.table),
              tables.n_factors, _lib.ptr(tables.mode_p), _lib.ptr(tables.mode_q),
              _lib.ptr(tables.sqrt_lam), f.n_modes, _lib.ptr(d_samples), _lib.ptr(lane_ids), G, S,
              float(f.a_min),
              tables.ahat, float(f.a_hat_value), tables.expansion, _lib.ptr(out), _lib.stream(),
              invalid=FemError)
    return out


def assemble_values(mesh: StructuredMesh2D, a_nodes, G: int, S: int, a_y: float, a2: str = "const",
                    vals=None, dinv=None, want_dinv=True):
    """Device [G][nnz][S] values (+ [G][N][S] Jacobi inverse diagonal)."""
    if a2 not in ("const", "same"):
        raise FemError(f"unknown second-direction mode {a2!r}")
    rowptr, _ = mesh.device()
    if vals is None:
        vals = a_nodes.new_empty((G * mesh.nnz * S,))
    if want_dinv and dinv is None:
        dinv = a_nodes.new_empty((G * mesh.n_dofs * S,))
    _lib.call("uqg_assemble_fv2d", _lib.ctx(), mesh.cells, G, S, _lib.ptr(a_nodes), float(a_y),
              int(a2 == "same"), _lib.ptr(rowptr), _lib.ptr(vals),
              _lib.ptr(dinv) if want_dinv else None, _lib.stream(), invalid=FemError)
    return vals, dinv


def n_faces(mesh: StructuredMesh2D) -> int:
    """Face slots per group of the face form: (m+1)*m (x-faces; y-faces alike)."""
    m = mesh.cells - 1
    return (m + 1) * m


def assemble_faces(mesh: StructuredMesh2D, a_nodes, G: int, S: int, a_y: float,
                   a2: str = "const", tx=None, ty=None, dinv=None):
    """Face form of the same operator (``uqg_assemble_fv2d_faces``): device
    tx [G][(m+1)m][S], ty (None unless a2 == "same"), dinv [G][N][S]."""
    if a2 not in ("const", "same"):
        raise FemError(f"unknown second-direction mode {a2!r}")
    F = n_faces(mesh)
    if tx is None:
        tx = a_nodes.new_empty((G * F * S,))
    if a2 == "same" and ty is None:
        ty = a_nodes.new_empty((G * F * S,))
    if a2 != "same":
        ty = None
    if dinv is None:
        dinv = a_nodes.new_empty((G * mesh.n_dofs * S,))
    _lib.call("uqg_assemble_fv2d_faces", _lib.ctx(), mesh.cells, G, S, _lib.ptr(a_nodes),
              float(a_y), int(a2 == "same"), _lib.ptr(tx), _lib.ptr(ty), _lib.ptr(dinv),
              _lib.stream(), invalid=FemError)
    return tx, ty, dinv


def assemble(mesh: StructuredMesh2D, field, samples, mode_vals=None, a2: str = "const"
             ) -> AssembledEnsembleSystem:
    """Width-S ensemble system for the sample rows, assembled on the GPU.

    ``mode_vals`` is accepted for signature parity with ``fem3d.assemble``; the
    device rebuilds mode values from the separable node tables instead.
    """
    ys = np.atleast_2d(np.asarray(samples, dtype=float))
    S = len(ys)
    if ys.shape[1] != field.n_modes:
        raise FemError(f"samples must have {field.n_modes} columns, got {ys.shape[1]}")
    if field.a_y <= 0:
        raise FemError("non-positive diffusion coefficient a_y")
    tables = FieldTables(field, mesh)
    _lib.status_sync()
    a = kl_nodes(tables, _lib.to_dev(ys), 1, S)
    if _lib.status_sync() & 1:
        raise FemError("non-positive diffusion coefficient at a mesh node")
    vals, _ = assemble_values(mesh, a, 1, S, field.a_y, a2, want_dinv=False)
    rowptr, col = mesh.device()
    mat = EnsembleCsrMatrix.from_device(mesh.row_offsets, mesh.col_indices, rowptr, col, vals, S)
    rhs = np.full((S, mesh.n_dofs), mesh.h * mesh.h)
    return AssembledEnsembleSystem(matrix=mat, rhs=rhs, samples=ys.copy())


def qoi(u) -> float:
    """Squared l2 norm of one lane solution, on the device (``fem3d.py:178-183``)."""
    u = np.asarray(u, dtype=float)
    if u.ndim != 1:
        raise FemError(f"qoi expects a single lane vector, got shape {u.shape}")
    d = _lib.to_dev(u)
    out = d.new_empty((1,))
    _lib.call("uqg_lane_dot", _lib.ctx(), len(u), 1, 1, _lib.ptr(d), _lib.ptr(d), _lib.ptr(out),
              _lib.stream())
    return float(out.cpu().numpy()[0])
