"""pytest plugin (TEST INFRASTRUCTURE): run the reference's own hot-path test
modules unmodified against the drop-ins.

Loaded with ``-p uqgroup_dropin`` before the reference's test modules are
collected.  It imports the reference package ``uqgroup`` (installed into
``baseline/_ref`` by ``tools/stage_reference.py``; its tests are copied next
to it, both git-ignored) and rebinds the hot-path names the tests import -
``from uqgroup import ensemble_pcg, EnsembleCsrMatrix, ...`` - to
``paper_1705_02003_b200``'s device implementations, so the reference's
assertions exercise the CUDA path through the C ABI:

* ``ensemble.py:52-281``: EnsembleCsrMatrix, ensemble_pcg, jacobi_precond,
  IdentityPreconditioner, JacobiPreconditioner, LaneSolveResult, lane_dot,
  lane_norms;
* ``grouping.py:39-122``: GroupingPlan, group_by_key, group_natural;
* ``fem3d.py:57-183`` (the reference's own 3D operator):
  StructuredMesh, assemble (device KL at the Gauss points + device
  assembly), qoi; ``build_field`` -> the drop-in's 3D field.

The reference's own out-of-scope functions (``compute_R``, ``group_oracle``,
``predicted_speedup``) stay the reference's and receive the drop-in's plans.
Exceptions: the exported error names match both the reference's class and
the drop-in's class of the same name (a metaclass ``__instancecheck__``), so
``pytest.raises(X)`` (an isinstance check) catches what either side raises.
"""

from __future__ import annotations

import uqgroup  # the reference (baseline/_ref)
from uqgroup import ensemble as _r_ens
from uqgroup import fem3d as _r_fem
from uqgroup import grouping as _r_grp

import paper_1705_02003_b200 as _uq
from paper_1705_02003_b200 import errors as _err



class _Either(type):
    """Metaclass of the exported error names: an exception matches when it
    is the reference's class or the drop-in's class of the same name."""

    def __instancecheck__(cls, obj):
        return cls.__subclasscheck__(type(obj))

    def __subclasscheck__(cls, sub):
        return any(type.__subclasscheck__(c, sub) for c in cls._either)


for _mod, _name in ((_r_ens, "EnsembleError"), (_r_ens, "NumericalBreakdownError"),
                    (_r_grp, "GroupingError"), (_r_fem, "FemError")):
    _ref = getattr(_mod, _name)
    _both = _Either(_name, (_ref,), {"_either": (_ref, getattr(_err, _name))})
    setattr(_mod, _name, _both)
    setattr(uqgroup, _name, _both)

from paper_1705_02003_b200 import ensemble as _e  # noqa: E402
from paper_1705_02003_b200 import fem3d as _f3  # noqa: E402
from paper_1705_02003_b200 import fv2d as _f2  # noqa: E402
from uqgroup import random_field as _r_rf  # noqa: E402


def _build_field_3d(*args, **kw):
    """The reference's build_field makes the 3D (triple-product) KL field
    its FEM consumes; the drop-in's equivalent is build_field(..., dim=3)."""
    kw.setdefault("dim", 3)
    return _uq.build_field(*args, **kw)


DROPINS = {
    _r_ens: {n: getattr(_e, n) for n in (
        "EnsembleCsrMatrix", "ensemble_pcg", "jacobi_precond", "IdentityPreconditioner",
        "JacobiPreconditioner", "LaneSolveResult", "lane_dot", "lane_norms")},
    _r_grp: {n: getattr(_uq, n) for n in ("GroupingPlan", "group_by_key", "group_natural")},
    # fem3d.py:57-183 on the device: the reference's own operator
    _r_fem: {"StructuredMesh": _f3.StructuredMesh, "assemble": _f3.assemble, "qoi": _f2.qoi,
             "AssembledEnsembleSystem": _f2.AssembledEnsembleSystem},
    _r_rf: {"build_field": _build_field_3d},
}

for _mod, _objs in DROPINS.items():
    for _n, _obj in _objs.items():
        setattr(_mod, _n, _obj)
        if hasattr(uqgroup, _n):
            setattr(uqgroup, _n, _obj)


def pytest_report_header(config):
    return ["uqgroup hot path bound to paper_1705_02003_b200 (device drop-ins): " +
            ", ".join(n for names in DROPINS.values() for n in names)]
