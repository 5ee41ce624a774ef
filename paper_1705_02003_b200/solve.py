"""Level-batched device solve: the B200 replacement of ``_PdeProblem.solve_plan``.

Reference (``harness.py:399-431``): for each group of a plan, assemble ->
``ensemble_pcg`` -> QoI, one group after another, on one CPU core.

Here all groups of a level (or as many as fit in HBM, "waves") are solved by
ONE set of launches: samples [G][S][M] are uploaded once, the KL coefficient
and the sample-interleaved operator of every group are built on the device,
and one batched PCG runs every group to its own termination (a finished group
turns later launches into no-ops), followed by the per-lane QoI.  Per-lane
arithmetic and the reduction trees do not depend on G, so results are
bit-identical to solving the groups one at a time.

Only iterations, convergence flags and QoIs come back to the host; the
first-occurrence rule for replica slots (``harness.py:427-430``) and the
"hit maxit" notes (``harness.py:421-426``) are applied on the host.
"""

from __future__ import annotations

import contextlib
import ctypes
import os
from dataclasses import dataclass, field as dc_field

import numpy as np

from . import _lib
from .ensemble import run_pcg, run_pcg_fv2d
from .errors import FemError
from .fem3d import StructuredMesh3D
from .fv2d import (FieldTables, StructuredMesh2D, assemble_faces, assemble_values, kl_nodes,
                   n_faces)

__all__ = ["LevelSolveResult", "EnsembleSolver", "EnsembleSolver2D", "EnsembleSolver3D",
           "FV2DOperator", "FEM3DOperator"]


@dataclass
class LevelSolveResult:
    iterations: np.ndarray      # (K, S) per-slot iterations
    converged: np.ndarray       # (K, S) bool
    frozen: np.ndarray          # (K, S) bool
    ensemble_iterations: np.ndarray  # (K,)
    qoi: np.ndarray             # (K, S)
    histories: list | None = None    # per group: list of (S,) residual norms
    waves: int = 1
    stats: dict = dc_field(default_factory=dict)


# ---------------------------------------------------------------------------
# operators: how a group's coefficient and matrix are built on the device

class FV2DOperator:
    """BASELINE.json's 2D 5-point FV operator (``fv2d.py``).

    ``faces`` (default; ``UQG_FV2D_FACES=0`` selects CSR): the solve stores
    the operator once per face (``uqg_assemble_fv2d_faces``) and runs
    ``uqg_pcg_fv2d`` - the same matrix and the same bits as the CSR path, with
    the SpMV streaming 1-2 face arrays instead of 5 value arrays.
    """

    max_row_len = 5

    def __init__(self, field, cells: int, a2: str = "const", faces: bool | None = None):
        if field.dim != 2:
            raise FemError("the 2D operator needs a 2D field")
        self.field, self.a2 = field, a2
        self.mesh = StructuredMesh2D(cells)
        self.tables = FieldTables(field, self.mesh)
        self.n_dofs, self.nnz, self.n_coef = self.mesh.n_dofs, self.mesh.nnz, self.mesh.n_nodes
        self.rhs_const = self.mesh.h * self.mesh.h
        if faces is None:
            faces = os.environ.get("UQG_FV2D_FACES", "1") != "0"
        self.faces = bool(faces)
        self.n_faces = n_faces(self.mesh)

    @property
    def n_op(self) -> int:
        """Operator doubles per group and lane (CSR values or faces)."""
        if self.faces:
            return self.n_faces * (2 if self.a2 == "same" else 1)
        return self.nnz

    def assemble_faces(self, a, G, S, tx, ty, dinv):
        return assemble_faces(self.mesh, a, G, S, self.field.a_y, self.a2, tx=tx, ty=ty,
                              dinv=dinv)

    def graph(self):
        return self.mesh.device()

    def band_hint(self):
        return self.mesh.band_hint()

    def indicator_points(self):
        """Probe points of the anisotropy indicator: the KL nodes."""
        return self.mesh.node_coords()

    def coefficients(self, d_samples, lane_ids, G, S, out):
        kl_nodes(self.tables, d_samples, G, S, out=out, lane_ids=lane_ids)

    def assemble(self, a, G, S, vals, dinv):
        assemble_values(self.mesh, a, G, S, self.field.a_y, self.a2, vals=vals, dinv=dinv)


class FEM3DOperator:
    """The reference's 3D trilinear FEM (``fem3d.py:138-175``), on the device."""

    max_row_len = 27

    def __init__(self, field, cells: int, mesh: StructuredMesh3D | None = None):
        if field.dim != 3:
            raise FemError("the 3D operator needs a 3D field")
        if field.a_y <= 0 or field.a_z <= 0:
            raise FemError("non-positive diffusion coefficient a_y / a_z")
        self.field = field
        self.mesh = m = mesh if mesh is not None else StructuredMesh3D(cells)
        self.n_dofs, self.nnz, self.n_coef = m.n_dofs, m.nnz, m.n_quad
        self.rhs_const = m.load
        self.qtab = _lib.to_dev(field.quad_tables(cells))
        self.kyz = _lib.to_dev(np.ascontiguousarray(m.kyz(field.a_y, field.a_z)))
        self.consts = field._device_consts()
        self.codes = field.codes()

    def graph(self):
        rowptr, col, _ = self.mesh.device()
        return rowptr, col

    def indicator_points(self):
        """Probe points of the anisotropy indicator: the Gauss points
        (``harness.py:393-397``)."""
        return self.mesh.quad_points

    def coefficients(self, d_samples, lane_ids, G, S, out):
        f, c = self.field, self.consts
        _lib.call("uqg_kl_eval_sep3d", _lib.ctx(), self.mesh.cells, _lib.ptr(self.qtab),
                  len(f.factors), _lib.ptr(c["mode_p"]), _lib.ptr(c["mode_q"]),
                  _lib.ptr(c["mode_r"]), _lib.ptr(c["sqrt_lam"]), f.n_modes, _lib.ptr(d_samples),
                  _lib.ptr(lane_ids), G, S, float(f.a_min), self.codes[0], float(f.a_hat_value),
                  self.codes[1], _lib.ptr(out), _lib.stream(), invalid=FemError)

    def assemble(self, a, G, S, vals, dinv):
        rowptr, _, dx = self.mesh.device()
        _lib.call("uqg_assemble_fem3d", _lib.ctx(), self.mesh.cells, G, S, _lib.ptr(a),
                  _lib.ptr(dx), _lib.ptr(self.kyz), _lib.ptr(rowptr), _lib.ptr(vals),
                  _lib.ptr(dinv), _lib.stream(), invalid=FemError)


class EnsembleSolver:
    """Device solver for one (operator, solver-config) pair."""

    def __init__(self, operator, tol: float = 1e-8, maxit: int = 30000,
                 mem_fraction: float = 0.8, max_groups_per_wave: int | None = None):
        self.op = operator
        self.field, self.mesh = operator.field, operator.mesh
        self.tol, self.maxit = float(tol), int(maxit)
        self.mem_fraction = mem_fraction
        self.max_groups_per_wave = max_groups_per_wave
        self._bufs = {}
        self._pins = {}
        self._ws = None
        self._waves = {}

    # -- memory planning ----------------------------------------------------
    def bytes_per_group(self, S: int) -> int:
        o = self.op
        n_op = getattr(o, "n_op", o.nnz)
        per = 8 * S * (n_op + 2 * o.n_dofs + o.n_coef)       # operator, dinv, x, coefficient
        per += _lib.load().uqg_pcg_workspace_bytes(o.n_dofs, o.nnz, S, 1)  # r, p, Ap, ...
        return int(per)

    def wave_size(self, S: int, K: int) -> int:
        """Groups per device wave: as many as fit in ``mem_fraction`` of the
        HBM this solver can use (free + what it already holds).  Measured
        once per ensemble width (``torch.cuda.mem_get_info`` is a device
        query); ``release()`` forgets it."""
        g = self._waves.get(S)
        if g is None:
            torch = _lib._torch()
            free, _ = torch.cuda.mem_get_info()
            held = sum(t.numel() * t.element_size() for t in self._bufs.values())
            held += 0 if self._ws is None else self._ws.numel()
            budget = (free + held) * self.mem_fraction
            g = max(1, int(budget // self.bytes_per_group(S)))
            if self.max_groups_per_wave:
                g = min(g, self.max_groups_per_wave)
            self._waves[S] = g
        return min(g, K)

    def _pinned(self, name, n):
        """Grow-only pinned host float64 staging buffer (first n entries)."""
        torch = _lib._torch()
        t = self._pins.get(name)
        if t is None or t.numel() < n:
            t = torch.empty((max(n, 1024),), dtype=torch.float64).pin_memory()
            self._pins[name] = t
        return t[:n]

    def _buf(self, name, n, dtype):
        torch = _lib._torch()
        t = self._bufs.get(name)
        if t is None or t.numel() < n or t.dtype != dtype:
            self._bufs.pop(name, None)
            t = torch.empty((n,), dtype=dtype, device=_lib.device())
            self._bufs[name] = t
        return t[:n]

    @contextlib.contextmanager
    def _workspace(self, G, S):
        """The solver's PCG workspace, registered with the library context for
        one wave only: the context never keeps the address of a tensor that a
        dropped solver would hand back to torch's allocator for reuse."""
        torch = _lib._torch()
        m = self.op
        need = int(_lib.load().uqg_pcg_workspace_bytes(m.n_dofs, m.nnz, S, G)) + (1 << 20)
        if self._ws is None or self._ws.numel() < need:
            self._ws = None
            self._ws = torch.empty((need,), dtype=torch.uint8, device=_lib.device())
        _lib.call("uqg_ctx_set_workspace", _lib.ctx(), _lib.ptr(self._ws), self._ws.numel())
        try:
            yield
        finally:
            _lib.call("uqg_ctx_set_workspace", _lib.ctx(), None, 0)

    def release(self):
        self._bufs.clear()
        self._waves.clear()
        if self._ws is not None:
            _lib.call("uqg_ctx_set_workspace", _lib.ctx(), None, 0)
            self._ws = None

    # -- solve --------------------------------------------------------------
    def _check_inputs(self):
        """The one host synchronisation before a wave's PCG: the reference
        rejects a non-positive coefficient in ``assemble`` before any solve
        (``fem3d.py:153-154``) and a non-finite key in ``group_by_key``
        (``grouping.py:115-120``); the device status word carries both."""
        from .errors import GroupingError

        st = _lib.status_sync()
        if st & 2:
            raise GroupingError("grouping keys must be finite")
        if st & 1:
            raise FemError("non-positive diffusion coefficient at a mesh node")

    def solve_wave(self, d_samples, G: int, S: int, record_history: bool = False, lane_ids=None,
                   clear_status: bool = True):
        """One batched launch set over G groups; samples already on the device.

        ``lane_ids`` (device int32 [G*S]) maps lanes to rows of ``d_samples``
        (the device grouping plan); None = rows in lane order.
        ``clear_status=False``: the caller cleared the device status word
        itself and queued work whose bits must reach this wave's check (the
        level pipeline's device grouping).
        Returns device tensors (iters, conv, frozen, ens, qoi, hist, x).
        """
        torch = _lib._torch()
        o = self.op
        if clear_status:
            _lib.call("uqg_status_clear", _lib.ctx(), _lib.stream())
        a = self._buf("a", G * o.n_coef * S, torch.float64)
        dinv = self._buf("dinv", G * o.n_dofs * S, torch.float64)
        o.coefficients(d_samples, lane_ids, G, S, a)
        if getattr(o, "faces", False):
            F = o.n_faces
            tx = self._buf("vals", G * F * S, torch.float64)
            ty = self._buf("ty", G * F * S, torch.float64) if o.a2 == "same" else None
            o.assemble_faces(a, G, S, tx, ty, dinv)
            self._check_inputs()
            with self._workspace(G, S):
                x, iters, conv, frz, ens, hist = run_pcg_fv2d(
                    o.mesh.cells, S, G, tx, ty, o.field.a_y, None, o.rhs_const, dinv, self.tol,
                    self.maxit, record_history)
                return self._finish(x, iters, conv, frz, ens, hist, G, S)
        vals = self._buf("vals", G * o.nnz * S, torch.float64)
        o.assemble(a, G, S, vals, dinv)
        self._check_inputs()
        rowptr, col = o.graph()
        # banded-graph hint: the SpMV bulk-prefetches each tile's p bands into L2
        # (UQG_SPMV_TMA=3 stages them in shared memory instead); UQG_BAND_HINT=0
        # disables it.  Results are identical either way.
        hint = (o.band_hint() if hasattr(o, "band_hint") and
                os.environ.get("UQG_BAND_HINT", "1") != "0" else None)
        if hint:
            starts, extras = hint
            _lib.call("uqg_ctx_set_band_hint", _lib.ctx(), len(starts),
                      (ctypes.c_int * len(starts))(*starts), (ctypes.c_int * len(extras))(*extras),
                      1)
        try:
            with self._workspace(G, S):
                x, iters, conv, frz, ens, hist = run_pcg(
                    o.n_dofs, o.nnz, S, G, rowptr, col, vals, None, o.rhs_const, dinv, self.tol,
                    self.maxit, record_history, max_row_len=o.max_row_len)
                return self._finish(x, iters, conv, frz, ens, hist, G, S)
        finally:
            if hint:
                _lib.call("uqg_ctx_set_band_hint", _lib.ctx(), 0, None, None, 0)

    def _finish(self, x, iters, conv, frz, ens, hist, G, S):
        torch = _lib._torch()
        o = self.op
        q = torch.empty((G * S,), dtype=torch.float64, device=_lib.device())
        _lib.call("uqg_lane_dot", _lib.ctx(), o.n_dofs, S, G, _lib.ptr(x), _lib.ptr(x), _lib.ptr(q),
                  _lib.stream())
        return iters, conv, frz, ens, q, hist, x

    def solve_groups(self, samples, record_history: bool = False) -> LevelSolveResult:
        """samples: host (K, S, M) array or device float64 tensor of that shape."""
        torch = _lib._torch()
        if isinstance(samples, np.ndarray):
            samples = np.asarray(samples, dtype=np.float64)
            K, S, M = samples.shape
        else:
            K, S, M = samples.shape
        if M != self.field.n_modes:
            raise FemError(f"samples must have {self.field.n_modes} columns, got {M}")
        if self.field.a_y <= 0:
            raise FemError("non-positive diffusion coefficient a_y")
        gw = self.wave_size(S, K)
        out = {k: [] for k in ("it", "cv", "fz", "en", "q")}
        hists = [] if record_history else None
        waves = 0
        for k0 in range(0, K, gw):
            g = min(gw, K - k0)
            chunk = samples[k0:k0 + g]
            d_y = _lib.to_dev(chunk.reshape(g * S, M)) if isinstance(chunk, np.ndarray) \
                else chunk.reshape(g * S, M).contiguous()
            iters, conv, frz, ens, q, hist, _ = self.solve_wave(d_y, g, S, record_history)
            out["it"].append(iters.reshape(g, S))
            out["cv"].append(conv.reshape(g, S))
            out["fz"].append(frz.reshape(g, S))
            out["en"].append(ens)
            out["q"].append(q.reshape(g, S))
            if record_history:
                hists.extend([[hist[r, gi].copy() for r in range(int(ens[gi].item()) + 1)]
                              for gi in range(g)])
            waves += 1
        cat = {k: torch.cat(v).cpu().numpy() for k, v in out.items()}
        return LevelSolveResult(cat["it"].astype(int), cat["cv"].astype(bool),
                                cat["fz"].astype(bool), cat["en"].astype(int), cat["q"], hists,
                                waves)

    def run_groups_device(self, d_coords, lane_ids, G: int, S: int, clear_status: bool = True):
        """Solve G groups whose lanes read rows ``lane_ids`` [G*S] of the
        device samples ``d_coords`` [n][M], in waves that fit in HBM; returns
        device (iters [G*S], conv [G*S], ens [G], qoi [G*S])."""
        torch = _lib._torch()
        gw = self.wave_size(S, G)
        parts = {k: [] for k in ("it", "cv", "en", "q")}
        for k0 in range(0, G, gw):
            g = min(gw, G - k0)
            it, cv, _, en, q, _, _ = self.solve_wave(d_coords, g, S,
                                                     lane_ids=lane_ids[k0 * S:(k0 + g) * S],
                                                     clear_status=clear_status and k0 == 0)
            parts["it"].append(it)
            parts["cv"].append(cv)
            parts["en"].append(en)
            parts["q"].append(q)
        cat = {k: (v[0] if len(v) == 1 else torch.cat(v)) for k, v in parts.items()}
        return cat["it"], cat["cv"], cat["en"], cat["q"]

    def run_level_device(self, d_coords, n: int, S: int, d_keys=None, shard=None):
        """The whole level on the device: group (sort + chunk) -> KL -> assemble
        -> PCG -> QoI.  ``d_coords`` [n][M] and ``d_keys`` [n] (None = natural
        order) are device tensors; returns device tensors
        (groups [K*S], padding [K], iters [K*S], conv [K*S], ens [K], qoi [K*S]).

        ``shard`` (``dist.LevelShard``, world > 1): this rank solves its
        round-robin share of the plan's groups and one allgather returns the
        whole level's results on every rank.
        """
        from .grouping import device_group

        _lib.call("uqg_status_clear", _lib.ctx(), _lib.stream())
        groups, pad = device_group(n, S, d_keys, sync=False)
        K = pad.numel()
        if shard is None or (shard.world == 1 and not getattr(shard, "force_collective", False)):
            it, cv, en, q = self.run_groups_device(d_coords, groups, K, S, clear_status=False)
        else:
            it, cv, en, q = shard.solve(
                lambda lanes, g: self.run_groups_device(d_coords, lanes, g, S, clear_status=False),
                groups, K, S)
        return groups, pad, it, cv, en, q

    def solve_level(self, ids, coords, size: int, keys=None, level: int = 1, tag: str = "sur",
                    shard=None):
        """Public end-to-end entry: host ids / coords (n, M) / keys (n,) in,
        grouping plan and per-sample results out - ``group_by_key`` (or
        ``group_natural`` when ``keys`` is None) fused with ``solve_plan`` on
        the device.  Returns (plan, iters dict, qois dict, notes).
        ``shard``: ``dist.LevelShard`` for a multi-GPU level (same results).
        """
        from .grouping import GroupingPlan

        torch = _lib._torch()
        ids = list(ids)
        coords = np.ascontiguousarray(coords, dtype=np.float64)
        n = len(ids)
        if coords.shape != (n, self.field.n_modes):
            raise FemError(f"coords must have shape ({n}, {self.field.n_modes})")
        dev = _lib.device()
        M = coords.shape[1]
        # inputs through a reused pinned staging buffer (pinning per call costs
        # more than the copy itself at small levels)
        stage = self._pinned("in", n * M + (n if keys is not None else 0))
        stage[:n * M].copy_(torch.from_numpy(coords.reshape(-1)))
        d_c = stage[:n * M].to(dev, non_blocking=True).view(n, M)
        d_k = None
        if keys is not None:
            stage[n * M:].copy_(torch.from_numpy(np.ascontiguousarray(keys, dtype=np.float64)))
            d_k = stage[n * M:].to(dev, non_blocking=True)
        groups, pad, it, cv, en, q = self.run_level_device(d_c, n, size, d_k, shard)
        d_out = torch.cat([groups.double(), pad.double(), it.double(), cv.double(), q])
        h_out = self._pinned("out", d_out.numel())
        h_out.copy_(d_out, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        host = h_out.numpy()
        K = pad.numel()
        KS = K * size
        g_idx = host[:KS].astype(np.int64).reshape(K, size)
        plan = GroupingPlan(level, size, tuple(tuple(ids[j] for j in row) for row in g_idx),
                            tuple(int(p) for p in host[KS:KS + K]), tag)
        o = KS + K
        res = LevelSolveResult(host[o:o + KS].astype(int).reshape(K, size),
                               host[o + KS:o + 2 * KS].reshape(K, size) != 0, None, None,
                               host[o + 2 * KS:o + 3 * KS].reshape(K, size))
        iters, qois, notes = self.collect(plan, res)
        return plan, iters, qois, notes

    def solve_plan(self, plan, coords_by_id, residual_sink=None):
        """Drop-in for ``_PdeProblem.solve_plan`` (``harness.py:399-431``)."""
        groups = plan.ensembles
        if not groups:  # the reference's loop over no ensembles
            return {}, {}, []
        samples = np.array([[coords_by_id[sid] for sid in grp] for grp in groups], dtype=np.float64)
        res = self.solve_groups(samples, record_history=residual_sink is not None)
        return self.collect(plan, res, residual_sink)

    def collect(self, plan, res: LevelSolveResult, residual_sink=None):
        iters, qois, notes = {}, {}, []
        for k, grp in enumerate(plan.ensembles):
            if residual_sink is not None:
                residual_sink(plan.level, k, res.histories[k])
            if not res.converged[k].all():
                bad = int((~res.converged[k]).sum())
                notes.append(f"level {plan.level} ensemble {k}: {bad} lane(s) hit maxit "
                             f"({self.maxit}) unconverged")
            for s, sid in enumerate(grp):
                if sid not in iters:
                    iters[sid] = int(res.iterations[k, s])
                    qois[sid] = float(res.qoi[k, s])
        return iters, qois, notes


class EnsembleSolver2D(EnsembleSolver):
    """Level-batched solver on BASELINE.json's 2D 5-point FV operator."""

    def __init__(self, field, cells: int, tol: float = 1e-8, maxit: int = 30000,
                 a2: str = "const", mem_fraction: float = 0.8,
                 max_groups_per_wave: int | None = None, faces: bool | None = None):
        super().__init__(FV2DOperator(field, cells, a2, faces), tol, maxit, mem_fraction,
                         max_groups_per_wave)
        self.tables, self.a2 = self.op.tables, a2


class EnsembleSolver3D(EnsembleSolver):
    """Level-batched solver on the reference's 3D trilinear FEM operator
    (``harness._PdeProblem``: ``fem3d.py`` + ``ensemble_pcg``)."""

    def __init__(self, field, cells: int, tol: float = 1e-7, maxit: int = 30000,
                 mem_fraction: float = 0.8, max_groups_per_wave: int | None = None):
        super().__init__(FEM3DOperator(field, cells), tol, maxit, mem_fraction,
                         max_groups_per_wave)
