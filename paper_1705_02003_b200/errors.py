"""Exception types of the drop-in surface (same names and bases as uqgroup).

* ``EnsembleError(ValueError)``            <- ensemble.py:44-45
* ``NumericalBreakdownError(RuntimeError)`` <- ensemble.py:48-49
* ``FemError(ValueError)``                 <- fem3d.py:29-30
* ``GroupingError(ValueError)``            <- grouping.py:35-36
* ``FieldError(ValueError)``               <- random_field.py:40-41
"""


class EnsembleError(ValueError):
    """Structural problems: shape mismatches, invalid graphs, bad diagonals."""


class NumericalBreakdownError(RuntimeError):
    """Non-finite values appeared in an active lane during iteration."""


class FemError(ValueError):
    """Invalid mesh or assembly input."""


class GroupingError(ValueError):
    """Invalid grouping input (missing keys, bad ensemble size, unknown S)."""


class FieldError(ValueError):
    """Invalid field configuration or evaluation input."""


class DeviceError(RuntimeError):
    """CUDA failure inside libuqg.so, or no usable CUDA device / extension."""
