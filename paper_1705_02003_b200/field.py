"""Truncated-KL diffusion coefficient for the 2D ensemble operator.

Host-side setup (one-time per field/mesh) plus the device
evaluation of the coefficient (row 1):

* ``eigenpairs_1d``  - Nystrom eigenpairs of exp(-|x-x'|/delta) on [0,1]
  (reference ``random_field.py:59-92``; dense ``scipy.linalg.eigh``, host);
* ``build_field``    - 2D separable mode selection by descending product
  eigenvalue, lexicographic (p, q) tie-break, with the reference's "enough 1D
  modes" doubling rule (``random_field.py:174-251`` restated for pairs);
* ``KLField2D.eval_a_batch`` - a(x, y) = a_min + a_hat(y) f(sum sqrt(lam) b(x) y)
  on the GPU through ``uqg_kl_eval_table`` (``random_field.py:145-166``);
* ``KLField2D.node_tables`` - the 1D factor values at the grid abscissae that
  let ``uqg_kl_eval_sep2d`` rebuild every mode value on the fly.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.linalg

from . import _lib
from .errors import FieldError

__all__ = ["Eigenpair1D", "eigenpairs_1d", "KLField2D", "build_field"]


@dataclass(frozen=True)
class Eigenpair1D:
    eigenvalue: float
    grid: np.ndarray
    values: np.ndarray

    def __call__(self, x) -> np.ndarray:
        return np.interp(x, self.grid, self.values)


def eigenpairs_1d(delta: float, count: int, grid_points: int = 513) -> list[Eigenpair1D]:
    if delta <= 0:
        raise FieldError(f"correlation length delta must be positive, got {delta}")
    if grid_points < 64:
        raise FieldError(f"grid_points must be >= 64, got {grid_points}")
    if not 1 <= count <= grid_points:
        raise FieldError(f"count must be in [1, {grid_points}], got {count}")
    grid = np.linspace(0.0, 1.0, grid_points)
    h = grid[1] - grid[0]
    w = np.full(grid_points, h)
    w[0] = w[-1] = h / 2.0
    sw = np.sqrt(w)
    kmat = sw[:, None] * np.exp(-np.abs(grid[:, None] - grid[None, :]) / delta) * sw[None, :]
    evals, evecs = scipy.linalg.eigh(kmat)
    out = []
    for k in np.argsort(evals)[::-1][:count]:
        v = evecs[:, k] / sw
        lead = v[0] if v[0] != 0 else v[np.argmax(np.abs(v))]
        out.append(Eigenpair1D(float(evals[k]), grid, np.ascontiguousarray(-v if lead < 0 else v)))
    return out


_AHAT = {"constant": 0, "test2": 1}
_EXPANSION = {"log": 0, "linear": 1}


@dataclass(frozen=True)
class KLField2D:
    """2D analogue of ``KLDiffusionField`` (``random_field.py:95-171``).

    ``modes[m] = (p, q)`` selects b_m(x) = e_p(x0) e_q(x1); eigenvalues carry
    the sigma0 scaling; ``a_y`` is the constant second-direction coefficient.
    """

    delta: float
    sigma0: float
    a_min: float
    a_hat_mode: str
    a_hat_value: float
    a_y: float
    expansion: str
    eigenvalues: np.ndarray
    modes: tuple
    factors: tuple

    @property
    def n_modes(self) -> int:
        return len(self.modes)

    def a_hat(self, y) -> np.ndarray:
        y = np.atleast_2d(np.asarray(y, dtype=float))
        if self.a_hat_mode == "constant":
            return np.full(len(y), self.a_hat_value)
        d = np.sqrt(3.0)
        r = np.sqrt((y ** 2).sum(axis=1))
        return self.a_hat_value * np.where(r < d / 4.0, 1.0, np.where(r < d / 2.0, 100.0, 10.0))

    def mode_values(self, points) -> np.ndarray:
        """(P, 2) -> (M, P) host table (setup, ``random_field.py:135-143``)."""
        pts = np.asarray(points, dtype=float)
        if pts.ndim != 2 or pts.shape[1] != 2:
            raise FieldError(f"points must have shape (P, 2), got {pts.shape}")
        tab = np.empty((self.n_modes, len(pts)))
        for m, (p, q) in enumerate(self.modes):
            tab[m] = self.factors[p](pts[:, 0]) * self.factors[q](pts[:, 1])
        return tab

    # -- device -------------------------------------------------------------
    def _device_consts(self):
        cache = self.__dict__.get("_dev_cache")
        if cache is None:
            cache = {
                "sqrt_lam": _lib.to_dev(np.sqrt(self.eigenvalues)),
                "mode_p": _lib.to_dev(np.array([p for p, _ in self.modes], dtype=np.int32)),
                "mode_q": _lib.to_dev(np.array([q for _, q in self.modes], dtype=np.int32)),
            }
            object.__setattr__(self, "_dev_cache", cache)
        return cache

    def codes(self) -> tuple[int, int]:
        try:
            return _AHAT[self.a_hat_mode], _EXPANSION[self.expansion]
        except KeyError as err:
            raise FieldError(f"unknown mode {err.args[0]!r}") from None

    def eval_a_batch(self, points, samples, mode_vals=None) -> np.ndarray:
        """Coefficient on points for many samples: (S, P), computed on the GPU."""
        ys = np.atleast_2d(np.asarray(samples, dtype=float))
        if ys.shape[1] != self.n_modes:
            raise FieldError(f"samples must have {self.n_modes} columns, got {ys.shape[1]}")
        if mode_vals is None:
            mode_vals = self.mode_values(points)
        ahat_code, exp_code = self.codes()
        P = mode_vals.shape[1]
        d_modes = _lib.to_dev(np.asarray(mode_vals, dtype=np.float64))
        d_y = _lib.to_dev(ys)
        out = d_y.new_empty((len(ys) * P,))
        _lib.call("uqg_kl_eval_table", _lib.ctx(), _lib.ptr(d_modes), P, self.n_modes,
                  _lib.ptr(self._device_consts()["sqrt_lam"]), _lib.ptr(d_y), len(ys),
                  float(self.a_min), ahat_code, float(self.a_hat_value), exp_code, _lib.ptr(out),
                  _lib.stream(), invalid=FieldError)
        return out.reshape(len(ys), P).cpu().numpy()

    def node_tables(self, cells: int) -> np.ndarray:
        """[n_factors][cells+1] factor values at x_i = i*h (h = 1/cells)."""
        x = np.arange(cells + 1) * (1.0 / cells)
        return np.stack([f(x) for f in self.factors])


def build_field(delta: float, sigma0: float, n_modes: int, a_min: float,
                a_hat_mode: str = "constant", a_hat_value: float = 1.0, a_y: float = 1.0,
                nystrom_points: int = 513, sigma0_convention: str = "stddev",
                expansion: str = "log") -> KLField2D:
    if n_modes < 1:
        raise FieldError(f"n_modes must be >= 1, got {n_modes}")
    if sigma0 < 0:
        raise FieldError(f"sigma0 must be >= 0, got {sigma0}")
    if a_min < 0:
        raise FieldError(f"a_min must be >= 0, got {a_min}")
    if sigma0_convention not in ("stddev", "kernel"):
        raise FieldError(f"unknown sigma0 convention {sigma0_convention!r}")
    if a_hat_mode not in _AHAT:
        raise FieldError(f"unknown a_hat mode {a_hat_mode!r}")
    if expansion not in _EXPANSION:
        raise FieldError(f"unknown expansion {expansion!r}")
    scale = sigma0 ** 2 if sigma0_convention == "stddev" else sigma0
    n1 = min(max(2, n_modes), nystrom_points)
    while True:
        facs = eigenpairs_1d(delta, n1, nystrom_points)
        lam = np.array([f.eigenvalue for f in facs])
        ranked = sorted(((lam[p] * lam[q], (p, q)) for p in range(n1) for q in range(n1)),
                        key=lambda e: (-e[0], e[1]))
        if len(ranked) < n_modes:
            if n1 == nystrom_points:
                raise FieldError(f"cannot form {n_modes} 2D modes from {n1} 1D modes")
            n1 = min(2 * n1, nystrom_points)
            continue
        chosen = ranked[:n_modes]
        if chosen[-1][0] >= lam[n1 - 1] * lam[0] or n1 == nystrom_points:
            break
        n1 = min(2 * n1, nystrom_points)
    return KLField2D(delta, sigma0, a_min, a_hat_mode, a_hat_value, a_y, expansion,
                     np.array([scale * v for v, _ in chosen]), tuple(m for _, m in chosen),
                     tuple(facs))
