"""Exception classes, named and typed exactly like the reference's.

pearl_lab/core.py:27-36 defines InvalidDistribution, AllZeroResidual and
ZeroDraftProb as ValueError subclasses; models.py:34-39 adds EmptyCorpus and
InvalidAlpha.  The C ABI returns integer codes that ``_lib.check`` maps back
onto these classes.
"""


class InvalidDistribution(ValueError):
    """Raised when a probability vector fails validation."""


class AllZeroResidual(ValueError):
    """Raised when max(0, p - q) carries no mass (p == q everywhere)."""


class ZeroDraftProb(ValueError):
    """Raised when a drafted token has zero probability under its own draft dist."""


class InvalidAlpha(ValueError):
    """Raised for an acceptance rate outside [0, 1]."""


class DeviceError(RuntimeError):
    """A CUDA / argument failure inside libpearl_b200."""
