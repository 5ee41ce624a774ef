"""The five BASELINE.json workloads (C1..C5) as concrete, recorded parameters.

Decisions for what BASELINE.json leaves open (DESIGN.md "Config gaps",
SURVEY.md Appendix B): a1 = exp(KL) (a_min = 0, a_hat = 1, stddev sigma
convention), a2 = a_y = 1 (the reference randomises only the first direction,
``fem3d.py:158-160``); f = 1; Jacobi; rtol 1e-8 on ||r||/||b||; the grid is the
reference's hierarchical rule on [-1,1]^M, the initial grid is total level 0
(2^M corners) and "adaptive grid to level L" caps refinement passes at total
level L.  tau is relative to nothing in BASELINE.json; it is set per config and
recorded.  C4/C5 cannot run the reference loop as stated (2^10 / 2^20 corner
nodes at level 0), so their sample sets are budgeted (``n_max``) or synthetic.
"""

from __future__ import annotations

from dataclasses import asdict, dataclass

__all__ = ["StudyConfig", "CONFIGS", "get"]


@dataclass(frozen=True)
class StudyConfig:
    name: str
    cells: int
    n_modes: int
    delta: float
    sigma0: float
    ensemble_size: int
    max_total_level: int
    tau: float
    n_max: int
    initial_level: int = 0
    tol: float = 1e-8
    maxit: int = 30000
    a_min: float = 0.0
    a_hat_mode: str = "constant"
    a_hat_value: float = 1.0
    a_y: float = 1.0
    sigma0_convention: str = "stddev"
    expansion: str = "log"
    a2: str = "const"
    synthetic_samples: int = 0  # >0: seeded U[-1,1]^M sample set instead of a grid (C5)

    @property
    def n_dofs(self) -> int:
        return (self.cells - 1) ** 2

    @property
    def nnz(self) -> int:
        m = self.cells - 1
        return 5 * m * m - 4 * m

    @property
    def n_nodes(self) -> int:
        return (self.cells + 1) ** 2

    @property
    def max_levels(self) -> int:
        return self.max_total_level - self.initial_level + 1

    def field_kwargs(self) -> dict:
        return dict(delta=self.delta, sigma0=self.sigma0, n_modes=self.n_modes, a_min=self.a_min,
                    a_hat_mode=self.a_hat_mode, a_hat_value=self.a_hat_value, a_y=self.a_y,
                    sigma0_convention=self.sigma0_convention, expansion=self.expansion)

    def to_dict(self) -> dict:
        return asdict(self)

    def make_solver(self, **kw):
        from .field import build_field
        from .solve import EnsembleSolver2D
        return EnsembleSolver2D(build_field(**self.field_kwargs()), self.cells, self.tol,
                                self.maxit, self.a2, **kw)


@dataclass(frozen=True)
class ReferencePreset:
    """The reference's own 3D PDE presets (``harness.py:208-255``): trilinear FEM
    on m^3 cells, kernel-convention sigma0 = sqrt(300), a_min = 0.1, four KL
    modes, S = 4, tau = 1e-3 on the QoI, n_max = 600, initial level 1,
    tol 1e-7, maxit 30000; no level cap (the loop stops on tau / budget)."""

    name: str
    a_hat_mode: str = "constant"
    cells: int = 16
    n_modes: int = 4
    delta: float = 0.25
    sigma0: float = 300.0 ** 0.5
    a_min: float = 0.1
    a_hat_value: float = 1.0
    a_y: float = 1.0
    a_z: float = 1.0
    sigma0_convention: str = "kernel"
    expansion: str = "log"
    ensemble_size: int = 4
    tau: float = 1e-3
    n_max: int = 600
    initial_level: int = 1
    tol: float = 1e-7
    maxit: int = 30000
    max_levels: int = 10_000
    synthetic_samples: int = 0

    def field_kwargs(self) -> dict:
        return dict(delta=self.delta, sigma0=self.sigma0, n_modes=self.n_modes, a_min=self.a_min,
                    a_hat_mode=self.a_hat_mode, a_hat_value=self.a_hat_value, a_y=self.a_y,
                    a_z=self.a_z, sigma0_convention=self.sigma0_convention,
                    expansion=self.expansion, dim=3)

    def to_dict(self) -> dict:
        return asdict(self)

    def make_solver(self, **kw):
        from .field import build_field
        from .solve import EnsembleSolver3D
        return EnsembleSolver3D(build_field(**self.field_kwargs()), self.cells, self.tol,
                                self.maxit, **kw)


PRESETS_3D = {
    "pde_test1": ReferencePreset("pde_test1"),
    "pde_test2": ReferencePreset("pde_test2", a_hat_mode="test2"),
}


CONFIGS = {
    "C1": StudyConfig("C1", cells=64, n_modes=3, delta=0.2, sigma0=1.0, ensemble_size=8,
                      max_total_level=4, tau=1e-5, n_max=10_000),
    "C2": StudyConfig("C2", cells=256, n_modes=4, delta=0.1, sigma0=1.0, ensemble_size=16,
                      max_total_level=5, tau=1e-5, n_max=10_000),
    "C3": StudyConfig("C3", cells=512, n_modes=6, delta=0.1, sigma0=1.5, ensemble_size=32,
                      max_total_level=6, tau=1e-5, n_max=4096),
    "C4": StudyConfig("C4", cells=1024, n_modes=10, delta=0.05, sigma0=2.0, ensemble_size=64,
                      max_total_level=6, tau=1e-5, n_max=2048),
    "C5": StudyConfig("C5", cells=2048, n_modes=20, delta=0.05, sigma0=1.5, ensemble_size=32,
                      max_total_level=5, tau=1e-5, n_max=1024, synthetic_samples=256),
}


def get(name: str):
    if name in PRESETS_3D:
        return PRESETS_3D[name]
    try:
        return CONFIGS[name.upper()]
    except KeyError:
        raise KeyError(f"unknown config {name!r}; choose from "
                       f"{sorted(CONFIGS) + sorted(PRESETS_3D)}") from None
