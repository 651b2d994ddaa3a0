"""Exception names kept identical to the reference (densify360/errors.py:1-17) so callers
that catch them keep working after the switch."""


class DensifyError(Exception):
    """Root of the package's own exceptions."""


class ConfigError(DensifyError):
    """A configuration value (or combination) is not acceptable."""


class DatasetError(DensifyError):
    """Dataset input is malformed or unreadable."""


class OrderingError(DensifyError):
    """Keyframe ids did not arrive strictly increasing."""


class BackendError(DensifyError):
    """The CUDA library is missing, failed to load, or a kernel call failed.

    There is no CPU fallback: every compute entry point raises this instead."""
