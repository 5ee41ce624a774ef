"""Oracle: ensemble Jacobi-PCG with per-lane convergence (TEST INFRA ONLY).

Restates ``ensemble.py:116-281`` of the reference on plain arrays:
``row_offsets``/``col_indices`` (shared graph) and ``values`` of shape (S, nnz).
Arithmetic sources are the reference's own: per-lane scipy ``csr_matvec``
(``ensemble.py:116-128``) and per-lane ``numpy.dot`` (``ensemble.py:155-161``),
so this oracle agrees with the reference bit for bit (checked by
``tests/golden/make_golden.py``).

Semantics (``ensemble.py:205-281``): x0 = 0; lanes converge when
||r|| <= tol*||b|| (zero rhs at iteration 0); converged lanes keep iterating
with the ensemble; p'Ap <= DBL_MIN freezes a lane (alpha = beta = 0 from then
on); a non-finite residual in an active lane raises; unconverged lanes report
the number of iterations run.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

DBL_MIN = np.finfo(np.float64).tiny


class Breakdown(RuntimeError):
    pass


def lane_mats(row_offsets, col_indices, values):
    n = len(row_offsets) - 1
    return [sp.csr_matrix((values[s], col_indices, row_offsets), shape=(n, n)) for s in range(values.shape[0])]


def spmv(row_offsets, col_indices, values, x):
    """(S, nnz) x (S, N) -> (S, N), one scipy csr_matvec per lane."""
    return np.stack([m.dot(x[s]) for s, m in enumerate(lane_mats(row_offsets, col_indices, values))])


def spmv_sequential(row_offsets, col_indices, values, x):
    """Numpy restatement of csr_matvec's order: per row, 0 + v0*x0 + v1*x1 + ...

    No fused multiply-add; used to pin the claim that scipy == sequential sum.
    """
    ro = np.asarray(row_offsets, dtype=np.int64)
    lens = np.diff(ro)
    S, n = x.shape
    acc = np.zeros((S, n))
    for k in range(int(lens.max(initial=0))):
        rows = np.flatnonzero(lens > k)
        idx = ro[rows] + k
        acc[:, rows] = acc[:, rows] + values[:, idx] * x[:, col_indices[idx]]
    return acc


def dots(a, b):
    return np.array([np.dot(a[s], b[s]) for s in range(a.shape[0])])


def jacobi_inverse(row_offsets, col_indices, values):
    """1/diag per lane (ensemble.py:130-137,179-183); absent diagonal reads 0."""
    n = len(row_offsets) - 1
    rows = np.repeat(np.arange(n), np.diff(row_offsets))
    on = col_indices == rows
    d = np.zeros((values.shape[0], n))
    d[:, rows[on]] = values[:, on]
    if np.any(d <= 0):
        raise ValueError("Jacobi needs strictly positive lane diagonals")
    return 1.0 / d


@dataclass
class Result:
    solution: np.ndarray
    iterations: np.ndarray
    ensemble_iterations: int
    converged: np.ndarray
    frozen: np.ndarray
    history: list | None


def pcg(row_offsets, col_indices, values, rhs, inv_diag=None, tol=1e-7, maxit=1000,
        history=False) -> Result:
    """inv_diag=None -> Jacobi from the matrix; pass np.ones for the identity."""
    if not (tol > 0 and np.isfinite(tol)) or maxit < 0:
        raise ValueError("bad tol/maxit")
    b = np.asarray(rhs, dtype=np.float64)
    S = b.shape[0]
    mats = lane_mats(row_offsets, col_indices, values)
    if inv_diag is None:
        inv_diag = jacobi_inverse(row_offsets, col_indices, values)

    x = np.zeros_like(b)
    r = b.copy()
    bn = np.sqrt(dots(b, b))
    thr = tol * bn
    its = np.zeros(S, dtype=int)
    conv = bn <= thr
    frz = np.zeros(S, dtype=bool)
    hist = [bn.copy()] if history else None
    z = r * inv_diag
    p = z.copy()
    rz = dots(r, z)
    k = 0
    while k < maxit and not np.all(conv | frz):
        k += 1
        ap = np.stack([m.dot(p[s]) for s, m in enumerate(mats)])
        pap = dots(p, ap)
        frz |= pap <= DBL_MIN
        live = ~frz
        alpha = np.zeros(S)
        alpha[live] = rz[live] / pap[live]
        x += alpha[:, None] * p
        r -= alpha[:, None] * ap
        rn = np.sqrt(dots(r, r))
        if hist is not None:
            hist.append(rn.copy())
        if not np.all(np.isfinite(rn[live])):
            raise Breakdown(f"non-finite residual at iteration {k}")
        hit = live & ~conv & (rn <= thr)
        its[hit] = k
        conv |= hit
        if np.all(conv | frz):
            break
        z = r * inv_diag
        rz_next = dots(r, z)
        beta = np.zeros(S)
        ok = live & (rz > 0)
        beta[ok] = rz_next[ok] / rz[ok]
        p = z + beta[:, None] * p
        rz = rz_next
    its[~conv] = k
    return Result(x, its, int(its.max(initial=0)), conv, frz, hist)
