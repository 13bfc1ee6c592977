"""Exception classes of the reference (/root/reference/pkg/src/sliceattn/core.py:24-29)."""


class ShapeError(ValueError):
    """Dimension mismatch between tensors, masks, or configuration."""


class NumericError(ArithmeticError):
    """Non-finite value produced where the contract requires finite math."""
