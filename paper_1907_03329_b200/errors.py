"""Exception hierarchy mirroring esrnn::Error (reference errors.hpp:9-67).

The C-ABI returns one status code per class; `_native.NativeApi.check` maps it
back here, so Python callers see the same exception types the reference's C++
callers catch.
"""


class Error(RuntimeError):
    """esrnn::Error (errors.hpp:9)."""


class ParseError(Error):
    """errors.hpp:15"""


class ValidationError(Error):
    """errors.hpp:22"""


class ShapeError(Error):
    """errors.hpp:28"""


class InsufficientLengthError(Error):
    """errors.hpp:34"""


class NumericDomainError(Error):
    """errors.hpp:40"""


class ConfigError(Error):
    """errors.hpp:46"""


class ContractError(Error):
    """errors.hpp:52"""


class EquivalenceError(Error):
    """errors.hpp:58"""


class CheckpointError(Error):
    """errors.hpp:64"""


class CudaError(Error):
    """Device/driver failure or missing CUDA extension (no reference analogue)."""


class NcclError(Error):
    """Collective failure (no reference analogue)."""
