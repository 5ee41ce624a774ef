"""Host-side adaptive hierarchical sparse grid (the caller of the hot path).

The paper's contribution - the iteration surrogate that produces the grouping
keys - is kept unchanged (BASELINE.json north_star) and stays on the host
(keys must be bit-identical to the reference's, which
only host BLAS guarantees).  This module restates the subset of
``hier_grid.HierGrid`` (``hier_grid.py:151-451``) the adaptive driver needs:

* 1D rule: level 0 = {-1, +1} (indices 0, 1), level l>=1 = odd i, coordinate
  i*2^(1-l)-1, hat half-width 2^(1-l) (``hier_grid.py:4-14``);
* nodes ordered canonically by (total level, level vector, index vector)
  (``hier_grid.py:81-84``), initial grid = every node of total level <= L
  (``:237-253``);
* surpluses fitted cohort by cohort in ascending total level, subtracting the
  interpolant of all strictly lower total levels (``:277-315``);
* prefix evaluation ``basis @ surplus`` (``:317-359``), domain <-> canonical
  affine maps (``:225-233``);
* classic refinement of the frontier with |surplus| >= tau under a point
  budget (``:379-406``; children per ``:111-128``).

The numpy expressions that produce surpluses and keys are the reference's, in
the same order, so keys agree bit for bit on the same host BLAS.
"""

from __future__ import annotations

import itertools

import numpy as np

__all__ = ["SparseGrid"]


def _pair_coord(level: int, index: int) -> float:
    return index * 2.0 ** (1 - level) - 1.0


def _level_indices(level: int):
    return (0, 1) if level == 0 else tuple(range(1, 2 ** level, 2))


def _compositions(total: int, parts: int):
    if parts == 1:
        yield (total,)
        return
    for head in range(total + 1):
        for tail in _compositions(total - head, parts - 1):
            yield (head,) + tail


def _key(node):
    lv, ix = node
    return (sum(lv), lv, ix)


def _children(node):
    lv, ix = node
    kids = set()
    for d, (l, i) in enumerate(zip(lv, ix)):
        opts = ((1, 1),) if l == 0 else ((l + 1, 2 * i - 1), (l + 1, 2 * i + 1))
        for nl, ni in opts:
            kids.add((lv[:d] + (nl,) + lv[d + 1:], ix[:d] + (ni,) + ix[d + 1:]))
    return kids


class SparseGrid:
    """Nodes are ((levels...), (indices...)) tuples in generation order."""

    def __init__(self, dim: int, domain=None):
        self.dim = dim
        self.domain = tuple(domain) if domain is not None else ((-1.0, 1.0),) * dim
        self.nodes: list = []
        self._index: dict = {}
        self._hw = np.empty((0, dim))
        self._ctr = np.empty((0, dim))
        self._tot = np.empty((0,), dtype=int)
        self.surplus: dict[str, np.ndarray] = {}
        self.frontier: list[int] = []

    def __len__(self):
        return len(self.nodes)

    def _lo_hi(self):
        return (np.array([d[0] for d in self.domain]), np.array([d[1] for d in self.domain]))

    def node_coords(self) -> np.ndarray:
        lo, hi = self._lo_hi()
        return lo + (self._ctr + 1.0) * 0.5 * (hi - lo)

    def to_canonical(self, y) -> np.ndarray:
        lo, hi = self._lo_hi()
        return 2.0 * (y - lo) / (hi - lo) - 1.0

    def _extend(self, new):
        for nd in new:
            self._index[nd] = len(self.nodes)
            self.nodes.append(nd)
        if not new:
            return
        lv = np.array([nd[0] for nd in new], dtype=float)
        ix = np.array([nd[1] for nd in new], dtype=float)
        h = 2.0 ** (1.0 - lv)
        self._hw = np.vstack([self._hw, h])
        self._ctr = np.vstack([self._ctr, ix * h - 1.0])
        self._tot = np.concatenate([self._tot, np.array([sum(nd[0]) for nd in new])])
        for ch in self.surplus:
            self.surplus[ch] = np.concatenate([self.surplus[ch], np.full(len(new), np.nan)])

    def add_initial_levels(self, max_total: int):
        new = []
        for tot in range(max_total + 1):
            for lv in _compositions(tot, self.dim):
                for ix in itertools.product(*[_level_indices(l) for l in lv]):
                    new.append((tuple(lv), tuple(ix)))
        new.sort(key=_key)
        self._extend(new)
        self.frontier = list(range(len(new)))
        return new

    def basis(self, pts_canonical, cols) -> np.ndarray:
        c, w = self._ctr[cols], self._hw[cols]
        out = np.empty((len(pts_canonical), len(cols)))
        step = max(1, 2 ** 22 // max(1, c.size))
        for a in range(0, len(pts_canonical), step):
            t = 1.0 - np.abs(pts_canonical[a:a + step, None, :] - c[None, :, :]) / w[None, :, :]
            np.maximum(t, 0.0, out=t)
            out[a:a + step] = t.prod(axis=2)
        return out

    def fit(self, channel: str, values_by_pos: dict):
        """Surpluses of the frontier cohort from values at frontier positions."""
        c = self.surplus.setdefault(channel, np.full(len(self.nodes), np.nan))
        cohorts: dict[int, list[int]] = {}
        for pos in self.frontier:
            cohorts.setdefault(int(self._tot[pos]), []).append(pos)
        for tot in sorted(cohorts):
            grp = cohorts[tot]
            v = np.array([float(values_by_pos[p]) for p in grp])
            prior = np.flatnonzero(self._tot < tot)
            if prior.size:
                v = v - self.basis(self._ctr[grp], prior) @ c[prior]
            c[grp] = v

    def evaluate(self, channel: str, points, n_nodes: int | None = None) -> np.ndarray:
        c = self.surplus[channel]
        n = len(self.nodes) if n_nodes is None else n_nodes
        c = c[:n]
        if not np.all(np.isfinite(c)):
            raise ValueError(f"channel {channel!r} has unfitted surpluses")
        return self.basis(self.to_canonical(np.asarray(points, dtype=float)), np.arange(n)) @ c

    def evaluate_device(self, channel: str, points, n_nodes: int | None = None) -> np.ndarray:
        """``evaluate`` on the GPU (``uqg_surrogate_eval``).  On the iteration
        channel (integer data on the dyadic grid) every term is exact, so the
        keys equal the host's bit for bit; on other channels they agree to
        rounding."""
        c = self.surplus[channel]
        n = len(self.nodes) if n_nodes is None else n_nodes
        c = c[:n]
        if not np.all(np.isfinite(c)):
            raise ValueError(f"channel {channel!r} has unfitted surpluses")
        pts = self.to_canonical(np.asarray(points, dtype=float))
        return self._basis_dot_device(pts, self._ctr[:n], self._hw[:n], c)

    @staticmethod
    def _basis_dot_device(pts_canonical, centers, widths, surplus) -> np.ndarray:
        """``basis(pts, nodes) @ surplus`` on the GPU (one CTA per point, the
        basis formed as hier_grid.py:317-328 forms it)."""
        from . import _lib

        pts = np.ascontiguousarray(pts_canonical, dtype=np.float64)
        n_pts, n = len(pts), len(surplus)
        if n_pts == 0:
            return np.zeros(0)
        if n == 0:
            return np.zeros(n_pts)
        # keep the device copies referenced until the kernel has run (a temporary
        # freed before the launch could be handed to the next allocation)
        d_pts = _lib.to_dev(pts)
        out = d_pts.new_empty((n_pts,))
        d_ctr = _lib.to_dev(np.ascontiguousarray(centers, dtype=np.float64))
        d_hw = _lib.to_dev(np.ascontiguousarray(widths, dtype=np.float64))
        d_c = _lib.to_dev(np.ascontiguousarray(surplus, dtype=np.float64))
        _lib.call("uqg_surrogate_eval", _lib.ctx(), _lib.ptr(d_pts), n_pts, pts.shape[1],
                  _lib.ptr(d_ctr), _lib.ptr(d_hw), _lib.ptr(d_c), n, _lib.ptr(out), _lib.stream())
        return out.cpu().numpy()

    def fit_device(self, channel: str, values_by_pos: dict):
        """``fit`` with each cohort's prior-interpolant subtraction on the GPU
        (``hier_grid.py:277-315``): the cohorts still run in
        ascending total level, each one's ``basis(cohort, prior) @ surplus``
        evaluated by ``uqg_surrogate_eval`` over the gathered prior nodes.  On
        the iteration channel every term is an exact dyadic product, so the
        surpluses equal ``fit``'s bit for bit; on other channels they agree to
        rounding (the sum order differs from host BLAS)."""
        c = self.surplus.setdefault(channel, np.full(len(self.nodes), np.nan))
        cohorts: dict[int, list[int]] = {}
        for pos in self.frontier:
            cohorts.setdefault(int(self._tot[pos]), []).append(pos)
        for tot in sorted(cohorts):
            grp = cohorts[tot]
            v = np.array([float(values_by_pos[p]) for p in grp])
            prior = np.flatnonzero(self._tot < tot)
            if prior.size:
                v = v - self._basis_dot_device(self._ctr[grp], self._ctr[prior],
                                               self._hw[prior], c[prior])
            c[grp] = v

    def error_indicator(self, channel: str) -> float:
        if not self.frontier:
            return 0.0
        return float(np.max(np.abs(self.surplus[channel][np.asarray(self.frontier)])))

    def refine(self, tau: float, channel: str, max_points: int):
        c = self.surplus[channel]
        cand = set()
        for pos in self.frontier:
            if abs(c[pos]) >= tau:
                cand.update(k for k in _children(self.nodes[pos]) if k not in self._index)
        ordered = sorted(cand, key=_key)
        room = max_points - len(self.nodes)
        exhausted = len(ordered) > room
        if exhausted:
            ordered = ordered[: max(0, room)]
        if ordered:
            self._extend(ordered)
            n = len(self.nodes)
            self.frontier = list(range(n - len(ordered), n))
        return ordered, exhausted
