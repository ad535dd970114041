"""Exception types of the reference interface, mirrored by name and meaning.

reference: basis.py:26-27 (BasisError), linalg.py:19-28 (SingularMatrixError,
ConvergenceError), system.py:26-27 (CapExceededError).
"""


class BasisError(Exception):
    """A requested basis exceeds what the data supports."""


class SingularMatrixError(Exception):
    """A direct solve hit a pivot too small to trust."""


class ConvergenceError(Exception):
    """An iterative kernel failed to settle within its cap."""


class CapExceededError(Exception):
    """An explicit space-time assembly would exceed the verification cap."""
