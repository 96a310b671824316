"""Shared exception types (mirrors splitfft/errors.py:1-5)."""


class CapacityError(ValueError):
    """Raised when a requested problem size exceeds a configured limit."""
