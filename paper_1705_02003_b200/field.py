"""Truncated-KL diffusion coefficient (2D for the BASELINE operator, 3D for the
reference's FEM presets).

Host-side setup (one-time per field/mesh) plus the device
evaluation of the coefficient (row 1):

* ``eigenpairs_1d``  - Nystrom eigenpairs of exp(-|x-x'|/delta) on [0,1]
  (reference ``random_field.py:59-92``; dense ``scipy.linalg.eigh``, host);
* ``build_field``    - separable mode selection by descending product
  eigenvalue, lexicographic index tie-break, with the reference's "enough 1D
  modes" doubling rule (``random_field.py:174-251``; pairs for dim=2, the
  reference's own triples for dim=3);
* ``KLField.eval_a_batch`` - a(x, y) = a_min + a_hat(y) f(sum sqrt(lam) b(x) y)
  on the GPU through ``uqg_kl_eval_table`` (``random_field.py:145-166``);
* ``KLField.node_tables`` / ``quad_tables`` - the 1D factor values at the grid
  abscissae that let ``uqg_kl_eval_sep2d`` / ``uqg_kl_eval_sep3d`` rebuild every
  mode value on the fly.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.linalg
from threadpoolctl import threadpool_limits

from . import _lib
from .errors import FieldError

__all__ = ["Eigenpair1D", "eigenpairs_1d", "KLField", "KLField2D", "build_field",
           "GAUSS"]

GAUSS = 1.0 / np.sqrt(3.0)  # 2-point Gauss abscissa (fem3d.py:26)


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
    # LAPACK's eigh rounds differently with the BLAS thread count (OpenBLAS
    # blocks by thread): pinned to one thread, the field - and every bit
    # downstream of it - is the same on every host and under torchrun (which
    # sets OMP_NUM_THREADS=1), so N-GPU results equal 1-GPU results bitwise.
    # The reference's eigenpairs equal these bits when it runs single-threaded
    # too (tests/golden/eigen.npz is generated that way).
    with threadpool_limits(limits=1):
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
class KLField:
    """Analogue of ``KLDiffusionField`` (``random_field.py:95-171``) in 2 or 3 dims.

    ``modes[m]`` is a tuple of 1D factor ids (one per spatial dimension): the
    m-th mode is b_m(x) = prod_d e_{modes[m][d]}(x_d); eigenvalues carry the
    sigma0 scaling; ``a_y`` / ``a_z`` are the constant coefficients of the
    other directions (only the first is random, ``fem3d.py:158-160``).
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
    a_z: float = 1.0

    @property
    def n_modes(self) -> int:
        return len(self.modes)

    @property
    def dim(self) -> int:
        return len(self.modes[0])

    def a_hat(self, y) -> np.ndarray:
        y = np.atleast_2d(np.asarray(y, dtype=float))
        if self.a_hat_mode == "constant":
            return np.full(len(y), self.a_hat_value)
        d = np.sqrt(3.0)
        r = np.sqrt((y ** 2).sum(axis=1))
        return self.a_hat_value * np.where(r < d / 4.0, 1.0, np.where(r < d / 2.0, 100.0, 10.0))

    def mode_values(self, points) -> np.ndarray:
        """(P, dim) -> (M, P) host table (setup, ``random_field.py:135-143``)."""
        pts = np.asarray(points, dtype=float)
        if pts.ndim != 2 or pts.shape[1] != self.dim:
            raise FieldError(f"points must have shape (P, {self.dim}), got {pts.shape}")
        tab = np.empty((self.n_modes, len(pts)))
        for m, ids in enumerate(self.modes):
            v = self.factors[ids[0]](pts[:, 0])
            for d in range(1, self.dim):
                v = v * self.factors[ids[d]](pts[:, d])
            tab[m] = v
        return tab

    # -- device -------------------------------------------------------------
    def _device_consts(self):
        cache = self.__dict__.get("_dev_cache")
        if cache is None:
            ids = np.array(self.modes, dtype=np.int32)  # (M, dim)
            cache = {"sqrt_lam": _lib.to_dev(np.sqrt(self.eigenvalues))}
            for d, name in enumerate(("mode_p", "mode_q", "mode_r")[: self.dim]):
                cache[name] = _lib.to_dev(np.ascontiguousarray(ids[:, d]))
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

    def quad_tables(self, cells: int) -> np.ndarray:
        """[n_factors][2*cells] factor values at the 1D Gauss abscissae of the
        hex mesh: entry 2*e + bit is (e + 0.5) h + (+-1/sqrt3)(h/2), computed with
        the reference's expression for quad_points (``fem3d.py:93-95``)."""
        h = 1.0 / cells
        centers = (np.arange(cells) + 0.5) * h
        signs = np.array([-1.0, 1.0]) * GAUSS
        x = (centers[:, None] + signs[None, :] * (h / 2.0)).ravel()
        return np.stack([f(x) for f in self.factors])


KLField2D = KLField  # backwards-compatible name for the 2D field


def anisotropy_indicators(field: KLField, samples, probe_points, mode_vals=None) -> np.ndarray:
    """Worst local anisotropy ratio per sample on the GPU (batched form of
    ``anisotropy_indicator``, ``random_field.py:254-270``): for each sample
    row, max over the probe points of max(a, a_hi) / min(a, a_lo) with
    a_hi = max(a_y, a_z), a_lo = min(a_y, a_z) (a_z only in 3D)."""
    ys = np.atleast_2d(np.asarray(samples, dtype=float))
    if ys.shape[1] != field.n_modes:
        raise FieldError(f"samples must have {field.n_modes} columns, got {ys.shape[1]}")
    if mode_vals is None:
        mode_vals = field.mode_values(probe_points)
    others = (field.a_y, field.a_z) if field.dim == 3 else (field.a_y,)
    ahat_code, exp_code = field.codes()
    P = mode_vals.shape[1]
    d_modes = _lib.to_dev(np.ascontiguousarray(mode_vals, dtype=np.float64))
    d_y = _lib.to_dev(ys)
    out = d_y.new_empty((len(ys),))
    _lib.call("uqg_anisotropy_indicator", _lib.ctx(), _lib.ptr(d_modes), P, field.n_modes,
              _lib.ptr(field._device_consts()["sqrt_lam"]), _lib.ptr(d_y), len(ys),
              float(field.a_min), ahat_code, float(field.a_hat_value), exp_code,
              float(max(others)), float(min(others)), _lib.ptr(out), _lib.stream(),
              invalid=FieldError)
    return out.cpu().numpy()


def anisotropy_indicator(field: KLField, y, probe_points, mode_vals=None) -> float:
    """Single-sample drop-in for ``anisotropy_indicator`` (``random_field.py:254``)."""
    return float(anisotropy_indicators(field, np.asarray(y, dtype=float)[None, :], probe_points,
                                       mode_vals)[0])


def build_field(delta: float, sigma0: float, n_modes: int, a_min: float,
                a_hat_mode: str = "constant", a_hat_value: float = 1.0, a_y: float = 1.0,
                nystrom_points: int = 513, sigma0_convention: str = "stddev",
                expansion: str = "log", dim: int = 2, a_z: float = 1.0) -> KLField:
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
    if dim not in (2, 3):
        raise FieldError(f"dim must be 2 or 3, got {dim}")
    scale = sigma0 ** 2 if sigma0_convention == "stddev" else sigma0
    n1 = min(max(2, n_modes), nystrom_points)
    while True:
        facs = eigenpairs_1d(delta, n1, nystrom_points)
        lam = np.array([f.eigenvalue for f in facs])
        if dim == 2:
            ranked = [(lam[p] * lam[q], (p, q)) for p in range(n1) for q in range(n1)]
        else:
            ranked = [(lam[p] * lam[q] * lam[r], (p, q, r))
                      for p in range(n1) for q in range(n1) for r in range(n1)]
        ranked.sort(key=lambda e: (-e[0], e[1]))
        if len(ranked) < n_modes:
            if n1 == nystrom_points:
                raise FieldError(f"cannot form {n_modes} {dim}D modes from {n1} 1D modes")
            n1 = min(2 * n1, nystrom_points)
            continue
        chosen = ranked[:n_modes]
        # an excluded product with an index >= n1 is at most lam[n1-1] * lam[0]^(dim-1)
        if chosen[-1][0] >= lam[n1 - 1] * lam[0] ** (dim - 1) or n1 == nystrom_points:
            break
        n1 = min(2 * n1, nystrom_points)
    return KLField(delta, sigma0, a_min, a_hat_mode, a_hat_value, a_y, expansion,
                   np.array([scale * v for v, _ in chosen]), tuple(m for _, m in chosen),
                   tuple(facs), a_z)
