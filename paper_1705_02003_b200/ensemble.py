"""Drop-in for ``uqgroup.ensemble`` backed by libuqg.so (sm_100a).

Same names, arguments, return types and errors as the reference module
(``ensemble.py:27-281``); the arithmetic runs on the GPU:

* ``EnsembleCsrMatrix`` keeps the shared graph plus sample-interleaved values
  ``[nnz][S]`` resident on the device; host ``values`` (S, nnz) are
  materialised lazily (tests, ``lane(s)`` views);
* ``spmv`` is ``uqg_spmv`` (bitwise equal to scipy ``csr_matvec`` per lane);
* ``lane_dot``/``lane_norms`` are ``uqg_lane_dot`` (deterministic tree);
* ``jacobi_precond`` is ``uqg_jacobi_dinv``;
* ``ensemble_pcg`` is ``uqg_pcg``: the whole loop (alpha/beta, freezing,
  per-lane convergence, termination) runs on the device.

Only ``JacobiPreconditioner`` / ``IdentityPreconditioner`` (or ``None`` =
Jacobi) are accepted: an arbitrary Python preconditioner object would need a
CPU callback inside the device loop, which this build deliberately lacks.
"""

from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np
import scipy.sparse as sp

from . import _lib
from .errors import EnsembleError, NumericalBreakdownError

__all__ = [
    "EnsembleError",
    "NumericalBreakdownError",
    "EnsembleCsrMatrix",
    "lane_norms",
    "lane_dot",
    "JacobiPreconditioner",
    "IdentityPreconditioner",
    "jacobi_precond",
    "LaneSolveResult",
    "ensemble_pcg",
]


class EnsembleCsrMatrix:
    """Shared-graph CSR matrix with a lane axis (reference ``ensemble.py:52-137``).

    Host construction validates exactly like the reference (``:65-80``).
    ``from_device`` wraps values already resident on the GPU in the
    ``[nnz][S]`` layout (what ``assemble`` produces).
    """

    def __init__(self, row_offsets, col_indices, values):
        ro = np.ascontiguousarray(row_offsets, dtype=np.int32)
        ci = np.ascontiguousarray(col_indices, dtype=np.int32)
        vals = np.ascontiguousarray(values, dtype=np.float64)
        if ro.ndim != 1 or ro[0] != 0:
            raise EnsembleError("row_offsets must be 1-D and start at 0")
        if vals.ndim != 2:
            raise EnsembleError("values must have shape (lanes, nnz)")
        nnz = ci.shape[0]
        if ro[-1] != nnz or vals.shape[1] != nnz:
            raise EnsembleError("row_offsets, col_indices and values disagree on nnz")
        if np.any(np.diff(ro) < 0):
            raise EnsembleError("row_offsets must be non-decreasing")
        n = len(ro) - 1
        if nnz and (ci.min() < 0 or ci.max() >= n):
            raise EnsembleError("column index out of range")
        self.row_offsets, self.col_indices = ro, ci
        self._host_vals = vals
        self._width = vals.shape[0]
        self._dev = None  # (rowptr, col, vals[nnz][S]) device tensors

    @classmethod
    def from_device(cls, row_offsets, col_indices, d_rowptr, d_col, d_vals, width):
        self = cls.__new__(cls)
        self.row_offsets = np.ascontiguousarray(row_offsets, dtype=np.int32)
        self.col_indices = np.ascontiguousarray(col_indices, dtype=np.int32)
        self._host_vals = None
        self._width = int(width)
        self._dev = (d_rowptr, d_col, d_vals)
        return self

    @classmethod
    def from_scipy_lanes(cls, mats: Sequence) -> "EnsembleCsrMatrix":
        """Stack scalar CSR matrices with identical graphs (``ensemble.py:90-104``)."""
        csr = [sp.csr_matrix(m) for m in mats]
        for m in csr:
            m.sort_indices()
        head = csr[0]
        for m in csr[1:]:
            if m.shape != head.shape or not (
                np.array_equal(m.indptr, head.indptr) and np.array_equal(m.indices, head.indices)
            ):
                raise EnsembleError("lane matrices must share one sparsity graph")
        return cls(head.indptr, head.indices, np.vstack([m.data for m in csr]))

    # -- shape --------------------------------------------------------------
    @property
    def n_rows(self) -> int:
        return len(self.row_offsets) - 1

    @property
    def nnz(self) -> int:
        return len(self.col_indices)

    @property
    def width(self) -> int:
        return self._width

    @property
    def max_row_len(self) -> int:
        if self.n_rows == 0:
            return 0
        return int(np.diff(self.row_offsets).max())

    # -- storage ------------------------------------------------------------
    def device(self):
        """(rowptr, col, vals[nnz][S]) device tensors, uploaded on first use."""
        if self._dev is None:
            self._dev = (_lib.to_dev(self.row_offsets), _lib.to_dev(self.col_indices),
                         _lib.lanes_to_dev(self._host_vals))
        return self._dev

    @property
    def values(self) -> np.ndarray:
        if self._host_vals is None:
            self._host_vals = _lib.dev_to_lanes(self._dev[2], self.width, self.nnz)
        return self._host_vals

    def lane(self, s: int) -> sp.csr_matrix:
        n = self.n_rows
        return sp.csr_matrix((self.values[s], self.col_indices, self.row_offsets), shape=(n, n))

    # -- compute (device) ---------------------------------------------------
    def spmv(self, x) -> np.ndarray:
        """Lane-wise product (S, n) -> (S, n), bitwise scipy per lane (``:116-128``)."""
        x = np.asarray(x, dtype=np.float64)
        if x.shape != (self.width, self.n_rows):
            raise EnsembleError(f"vector has shape {x.shape}, expected {(self.width, self.n_rows)}")
        ro, ci, vals = self.device()
        dx = _lib.lanes_to_dev(x)
        dy = dx.new_empty(dx.shape)
        _lib.call("uqg_spmv", _lib.ctx(), self.n_rows, self.nnz, self.max_row_len, self.width, 1,
                  _lib.ptr(ro),
                  _lib.ptr(ci), _lib.ptr(vals), _lib.ptr(dx), _lib.ptr(dy), _lib.stream())
        return _lib.dev_to_lanes(dy, self.width, self.n_rows)

    def diagonal(self) -> np.ndarray:
        """Per-lane main diagonal (S, n); absent entries read zero (``:130-137``)."""
        ro, ci, vals = self.device()
        d = vals.new_empty((self.n_rows * self.width,))
        _lib.call("uqg_diagonal", _lib.ctx(), self.n_rows, self.nnz, self.width, 1, _lib.ptr(ro),
                  _lib.ptr(ci), _lib.ptr(vals), _lib.ptr(d), _lib.stream())
        return _lib.dev_to_lanes(d, self.width, self.n_rows)


def _check_vector(width: int, n: int, x, name: str) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (width, n):
        raise EnsembleError(f"{name} has shape {x.shape}, expected {(width, n)}")
    return x


def lane_dot(x, y) -> np.ndarray:
    """Per-lane inner products (``ensemble.py:155-161``), on the device."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if x.shape != y.shape or x.ndim != 2:
        raise EnsembleError(f"mismatched ensemble vectors: {x.shape} vs {y.shape}")
    S, n = x.shape
    dx, dy = _lib.lanes_to_dev(x), _lib.lanes_to_dev(y)
    out = dx.new_empty((S,))
    _lib.call("uqg_lane_dot", _lib.ctx(), n, S, 1, _lib.ptr(dx), _lib.ptr(dy), _lib.ptr(out),
              _lib.stream())
    return out.cpu().numpy()


def lane_norms(x) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 2:
        raise EnsembleError("ensemble vectors must be 2-D (lanes, entries)")
    return np.sqrt(lane_dot(x, x))


class IdentityPreconditioner:
    """z = r (``ensemble.py:164-166``); the device loop uses no scaling."""

    def apply(self, r):
        return np.array(r, dtype=np.float64, copy=True)


class JacobiPreconditioner:
    """z = D^-1 r per lane (``ensemble.py:169-176``); keeps a device copy."""

    def __init__(self, inv_diag, _dev=None, _shape=None):
        self._host = None if inv_diag is None else np.asarray(inv_diag, dtype=np.float64)
        self._dev = _dev  # [n][S] device tensor
        self._shape = _shape if _dev is not None else None  # (S, n) of the device copy

    @property
    def inv_diag(self) -> np.ndarray:
        if self._host is None:
            S, n = self._shape
            self._host = _lib.dev_to_lanes(self._dev, S, n)
        return self._host

    def device(self, width: int, n: int):
        """The [n][S] device copy for a (width, n) solve.  A preconditioner
        reused with another system shape raises ``EnsembleError`` (the
        reference's numpy broadcast fails there too) instead of letting the
        solver read past the copy."""
        if self._dev is None:
            self._dev = _lib.lanes_to_dev(_check_vector(width, n, self._host, "inv_diag"))
            self._shape = (width, n)
        if self._shape != (width, n):
            raise EnsembleError(f"inv_diag has shape {self._shape}, expected {(width, n)}")
        return self._dev

    def apply(self, r):
        r = np.asarray(r, dtype=np.float64)
        S, n = r.shape
        return _lib.dev_to_lanes(_lib.lanes_to_dev(r) * self.device(S, n), S, n)


def jacobi_precond(mat: EnsembleCsrMatrix) -> JacobiPreconditioner:
    """1/diag on the device; ``EnsembleError`` if any lane diagonal <= 0 (``:179-183``)."""
    mat = _as_matrix(mat)
    ro, ci, vals = mat.device()
    d = vals.new_empty((mat.n_rows * mat.width,))
    _lib.call("uqg_jacobi_dinv", _lib.ctx(), mat.n_rows, mat.nnz, mat.width, 1, _lib.ptr(ro),
              _lib.ptr(ci), _lib.ptr(vals), _lib.ptr(d), _lib.stream())
    return JacobiPreconditioner(None, d, (mat.width, mat.n_rows))


class LaneSolveResult:
    """Outcome of one ensemble solve (``ensemble.py:186-202``).

    ``solution`` is downloaded from the device on first access.
    """

    def __init__(self, x_dev, width, n, iterations, ens_iters, converged, frozen, history):
        self._x_dev, self._shape, self._solution = x_dev, (width, n), None
        self.iterations_per_lane = iterations
        self.ensemble_iterations = ens_iters
        self.converged_per_lane = converged
        self.frozen_lanes = frozen
        self.residual_history = history

    @property
    def solution(self) -> np.ndarray:
        if self._solution is None:
            self._solution = _lib.dev_to_lanes(self._x_dev, *self._shape)
        return self._solution

    @property
    def solution_device(self):
        return self._x_dev


def _as_matrix(mat) -> EnsembleCsrMatrix:
    if isinstance(mat, EnsembleCsrMatrix):
        return mat
    # duck-typed reference EnsembleCsrMatrix (uqgroup.ensemble)
    return EnsembleCsrMatrix(mat.row_offsets, mat.col_indices, mat.values)


def run_pcg(N, nnz, S, G, d_rowptr, d_col, d_vals, d_rhs, rhs_const, d_dinv, tol, maxit,
            record_history=False, max_row_len=0):
    """Batched device PCG over G groups; returns device/host result pieces."""
    def call(*tail):
        return _lib.load().uqg_pcg(
            _lib.ctx(), N, nnz, int(max_row_len), S, G, _lib.ptr(d_rowptr), _lib.ptr(d_col),
            _lib.ptr(d_vals), _lib.ptr(d_rhs), float(rhs_const), _lib.ptr(d_dinv), float(tol),
            int(maxit), *tail)
    return _pcg_loop(call, N, S, G, maxit, record_history)


def run_pcg_fv2d(n_cells, S, G, d_tx, d_ty, a_y, d_rhs, rhs_const, d_dinv, tol, maxit,
                 record_history=False):
    """``run_pcg`` on the face form of the 2D FV operator (``uqg_pcg_fv2d``):
    same results bit for bit, a third of the SpMV traffic."""
    def call(*tail):
        return _lib.load().uqg_pcg_fv2d(
            _lib.ctx(), n_cells, S, G, _lib.ptr(d_tx), _lib.ptr(d_ty), float(a_y), _lib.ptr(d_rhs),
            float(rhs_const), _lib.ptr(d_dinv), float(tol), int(maxit), *tail)
    return _pcg_loop(call, (n_cells - 1) ** 2, S, G, maxit, record_history)


def _pcg_loop(call, N, S, G, maxit, record_history):
    torch = _lib._torch()
    dev = _lib.device()
    x = torch.empty((G * N * S,), dtype=torch.float64, device=dev)
    iters = torch.empty((G * S,), dtype=torch.int32, device=dev)
    conv = torch.empty((G * S,), dtype=torch.uint8, device=dev)
    frz = torch.empty((G * S,), dtype=torch.uint8, device=dev)
    ens = torch.empty((G,), dtype=torch.int32, device=dev)
    cap = min(int(maxit), 4096)
    while True:
        hist = np.empty(((cap + 1) * G * S,)) if record_history else None
        rows = ctypes.c_int(0)
        rc = call(_lib.ptr(x), _lib.ptr(iters), _lib.ptr(conv), _lib.ptr(frz), _lib.ptr(ens),
                  hist.ctypes.data if hist is not None else None, cap, ctypes.byref(rows),
                  _lib.stream())
        if rc == _lib.UQG_ECAPACITY and cap < maxit:
            cap = int(maxit)
            continue
        _lib.check(rc)
        break
    hist_rows = hist.reshape(cap + 1, G, S)[: rows.value] if hist is not None else None
    return x, iters, conv, frz, ens, hist_rows


def ensemble_pcg(mat, rhs, precond=None, tol: float = 1e-7, maxit: int = 1000,
                 record_history: bool = False) -> LaneSolveResult:
    """Ensemble Jacobi-PCG on the device (reference ``ensemble.py:205-281``)."""
    if not (tol > 0) or not np.isfinite(tol):
        raise EnsembleError(f"tol must be positive and finite, got {tol}")
    if maxit < 0:
        raise EnsembleError(f"maxit must be >= 0, got {maxit}")
    mat = _as_matrix(mat)
    S, n = mat.width, mat.n_rows
    b = _check_vector(S, n, rhs, "rhs")
    if precond is None:
        precond = jacobi_precond(mat)
    if isinstance(precond, IdentityPreconditioner):
        d_dinv = None
    elif isinstance(precond, JacobiPreconditioner):
        d_dinv = precond.device(S, n)
    else:
        raise EnsembleError(
            f"unsupported preconditioner {type(precond).__name__}: the device solver supports "
            "Jacobi and identity only")
    ro, ci, vals = mat.device()
    d_b = _lib.lanes_to_dev(b)
    x, iters, conv, frz, ens, hist = run_pcg(n, mat.nnz, S, 1, ro, ci, vals, d_b, 0.0, d_dinv,
                                             tol, maxit, record_history, mat.max_row_len)
    history = None
    if record_history:
        history = [hist[k, 0].copy() for k in range(hist.shape[0])]
    return LaneSolveResult(
        x, S, n,
        iters.cpu().numpy().astype(int),
        int(ens.cpu().numpy()[0]),
        conv.cpu().numpy().astype(bool),
        frz.cpu().numpy().astype(bool),
        history,
    )
