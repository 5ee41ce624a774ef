"""Oracle: truncated KL diffusion coefficient on the unit square (TEST INFRA ONLY).

Restates, for two spatial dimensions, the reference's KL machinery:

* ``nystrom_1d``      <- ``random_field.py:59-92``  (eigenpairs_1d)
* ``KL2D.select``     <- ``random_field.py:174-251`` (build_field; triples -> pairs)
* ``KL2D.mode_table`` <- ``random_field.py:135-143`` (mode_values; np.interp factors)
* ``KL2D.coeff``      <- ``random_field.py:145-166`` (eval_a_batch) and
                         ``random_field.py:121-133`` (a_hat)

The covariance exp(-|x-x'|_1/delta) on [0,1]^2 is separable, so 2D modes are
products e_p(x0) e_q(x1) of 1D Nystrom modes, selected by descending product
eigenvalue with ties broken lexicographically on (p, q).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.linalg
from threadpoolctl import threadpool_limits


@dataclass(frozen=True)
class Mode1D:
    eigenvalue: float
    grid: np.ndarray
    values: np.ndarray

    def at(self, x) -> np.ndarray:
        return np.interp(x, self.grid, self.values)


def nystrom_1d(delta: float, count: int, grid_points: int = 513) -> list[Mode1D]:
    """Leading eigenpairs of exp(-|x-x'|/delta) on [0,1] (random_field.py:59-92).

    Trapezoid-weighted Nystrom matrix, symmetrised by W^1/2, dense ``eigh``;
    eigenfunctions rescaled by W^-1/2 and oriented positive at x=0 (or at their
    largest-magnitude entry when they vanish there).
    """
    if delta <= 0 or grid_points < 64 or not 1 <= count <= grid_points:
        raise ValueError("bad Nystrom parameters")
    xs = np.linspace(0.0, 1.0, grid_points)
    step = xs[1] - xs[0]
    wts = np.full(grid_points, step)
    wts[[0, -1]] = step / 2.0
    root = np.sqrt(wts)
    kern = np.exp(-np.abs(xs[:, None] - xs[None, :]) / delta)
    with threadpool_limits(limits=1):  # as paper_1705_02003_b200.field: thread-independent bits
        lam, vec = scipy.linalg.eigh(root[:, None] * kern * root[None, :])
    picked = np.argsort(lam)[::-1][:count]
    modes = []
    for col in picked:
        f = vec[:, col] / root
        ref = f[0] if f[0] != 0 else f[np.argmax(np.abs(f))]
        if ref < 0:
            f = -f
        modes.append(Mode1D(float(lam[col]), xs, np.ascontiguousarray(f)))
    return modes


@dataclass(frozen=True)
class KL2D:
    delta: float
    sigma0: float
    a_min: float
    a_hat_mode: str
    a_hat_value: float
    a_y: float
    expansion: str
    eigenvalues: np.ndarray
    modes: tuple  # ((p, q), ...)
    factors: tuple  # Mode1D, ...

    @property
    def n_modes(self) -> int:
        return len(self.modes)

    @staticmethod
    def select(delta, sigma0, n_modes, a_min, a_hat_mode="constant", a_hat_value=1.0,
               a_y=1.0, nystrom_points=513, sigma0_convention="stddev",
               expansion="log") -> "KL2D":
        """Pair-product mode selection (random_field.py:211-251 with pairs)."""
        if n_modes < 1 or sigma0 < 0 or a_min < 0:
            raise ValueError("bad field parameters")
        scale = {"stddev": sigma0 ** 2, "kernel": sigma0}[sigma0_convention]
        n1 = min(max(2, n_modes), nystrom_points)
        while True:
            facs = nystrom_1d(delta, n1, nystrom_points)
            lam = [f.eigenvalue for f in facs]
            cands = sorted(((lam[p] * lam[q], (p, q)) for p in range(n1) for q in range(n1)),
                           key=lambda c: (-c[0], c[1]))
            if len(cands) < n_modes:
                if n1 == nystrom_points:
                    raise ValueError("not enough 1D modes")
                n1 = min(2 * n1, nystrom_points)
                continue
            kept = cands[:n_modes]
            # an excluded pair using an index >= n1 is bounded by lam[n1-1]*lam[0]
            if kept[-1][0] >= lam[n1 - 1] * lam[0] or n1 == nystrom_points:
                break
            n1 = min(2 * n1, nystrom_points)
        return KL2D(delta, sigma0, a_min, a_hat_mode, a_hat_value, a_y, expansion,
                    np.array([scale * v for v, _ in kept]), tuple(m for _, m in kept),
                    tuple(facs))

    def a_hat(self, y: np.ndarray) -> np.ndarray:
        y = np.atleast_2d(np.asarray(y, dtype=float))
        if self.a_hat_mode == "constant":
            return np.full(len(y), self.a_hat_value)
        if self.a_hat_mode == "test2":
            # random_field.py:126-132: radius thresholds use sqrt(3) verbatim
            rad = np.sqrt((y ** 2).sum(axis=1))
            d = math.sqrt(3.0)
            return self.a_hat_value * np.where(rad < d / 4.0, 1.0, np.where(rad < d / 2.0, 100.0, 10.0))
        raise ValueError(self.a_hat_mode)

    def mode_table(self, points: np.ndarray) -> np.ndarray:
        """(P,2) -> (M,P): e_p(x0) * e_q(x1) via linear interpolation."""
        pts = np.asarray(points, dtype=float)
        out = np.empty((self.n_modes, len(pts)))
        for m, (p, q) in enumerate(self.modes):
            out[m] = self.factors[p].at(pts[:, 0]) * self.factors[q].at(pts[:, 1])
        return out

    def coeff(self, points, samples, table=None) -> np.ndarray:
        """(S, P) coefficient a(x, y) = a_min + a_hat(y) * exp(sum sqrt(lam) b(x) y)."""
        ys = np.atleast_2d(np.asarray(samples, dtype=float))
        if ys.shape[1] != self.n_modes:
            raise ValueError("sample width != n_modes")
        if table is None:
            table = self.mode_table(points)
        expo = (ys * np.sqrt(self.eigenvalues)) @ table
        if self.expansion == "log":
            expo = np.exp(expo)
        elif self.expansion == "linear":
            expo = 1.0 + expo
        else:
            raise ValueError(self.expansion)
        return self.a_min + self.a_hat(ys)[:, None] * expo
