"""Exception types of the reference API (same names and bases).

ValidationError  model.py:24-25   (ValueError)
DimensionError   sparse.py:22-23  (ValueError)
ResourceLimitError sparse.py:26-27 (RuntimeError)
"""


class ValidationError(ValueError):
    """Raised when an input violates a documented contract."""


class DimensionError(ValueError):
    """Operand shapes do not line up."""


class ResourceLimitError(RuntimeError):
    """An operation would exceed a configured memory/size cap."""
