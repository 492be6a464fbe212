"""Exception types of the public API (reference: beamnmt/errors.py:4-9).

Both subclass ValueError so callers of the reference keep catching them the
same way.  C-ABI status AMUN_ERR_INVALID is raised as ValueError with the
library's message; every other non-zero status becomes RuntimeError.
"""


class ShapeError(ValueError):
    """Operands have incompatible or unexpected shapes."""


class FormatError(ValueError):
    """A model container, vocabulary, BPE rules file or table is malformed."""
