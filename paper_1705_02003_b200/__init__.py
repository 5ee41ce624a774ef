"""B200-native ensemble solve for surrogate-grouped embedded ensemble propagation.

Drop-in surface for the hot path of the reference package ``uqgroup``
(arXiv 1705.02003): the same entry-point names, arguments and errors, with the
arithmetic in hand-written sm_100a CUDA (``libuqg.so``, C ABI in
``include/uqg.h``) and PyTorch used only for device buffers and streams.

    reference (uqgroup)                      here
    ensemble.EnsembleCsrMatrix/.spmv         ensemble.EnsembleCsrMatrix (device [nnz][S])
    ensemble.ensemble_pcg / jacobi_precond   ensemble.ensemble_pcg (device loop)
    random_field.build_field/eval_a_batch    field.build_field / KLField2D.eval_a_batch
    fem3d.StructuredMesh/assemble/qoi        fv2d.StructuredMesh2D/assemble/qoi (2D 5-point FV)
    grouping.group_by_key/group_natural      grouping.* (device stable sort + chunk)
    harness._PdeProblem.solve_plan           solve.EnsembleSolver2D.solve_plan (level-batched)
    harness.adaptive_run (sur)               driver.adaptive_run
"""

from .errors import (DeviceError, EnsembleError, FemError, FieldError, GroupingError,
                     NumericalBreakdownError)
from .ensemble import (EnsembleCsrMatrix, IdentityPreconditioner, JacobiPreconditioner,
                       LaneSolveResult, ensemble_pcg, jacobi_precond, lane_dot, lane_norms)
from .field import Eigenpair1D, KLField, KLField2D, build_field, eigenpairs_1d
from .fv2d import AssembledEnsembleSystem, StructuredMesh2D, assemble, qoi
from .fem3d import StructuredMesh3D
from .grouping import GroupingPlan, group_by_key, group_natural
from .solve import EnsembleSolver, EnsembleSolver2D, EnsembleSolver3D, LevelSolveResult
from .configs import CONFIGS, PRESETS_3D, ReferencePreset, StudyConfig

__version__ = "0.1.0"

__all__ = [
    "DeviceError", "EnsembleError", "FemError", "FieldError", "GroupingError",
    "NumericalBreakdownError", "EnsembleCsrMatrix", "IdentityPreconditioner",
    "JacobiPreconditioner", "LaneSolveResult", "ensemble_pcg", "jacobi_precond", "lane_dot",
    "lane_norms", "Eigenpair1D", "KLField2D", "build_field", "eigenpairs_1d",
    "AssembledEnsembleSystem", "StructuredMesh2D", "assemble", "qoi", "GroupingPlan",
    "group_by_key", "group_natural", "EnsembleSolver", "EnsembleSolver2D", "EnsembleSolver3D",
    "LevelSolveResult", "CONFIGS", "PRESETS_3D", "ReferencePreset", "StudyConfig", "KLField",
    "StructuredMesh3D", "__version__",
]
