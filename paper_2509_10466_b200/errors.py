"""Exception types of the inpainting path.

Same class names and base classes as the reference (`pkg/src/dimreal/errors.py:4-33`),
so callers that catch the reference's exceptions catch ours.  The C-ABI return codes
(`include/dr_b200.h`, `DR_ERR_*`) map onto them in `_lib.check`.
"""


class ConfigError(ValueError):
    """A configuration value is missing, malformed, or inconsistent."""


class InputError(ValueError):
    """Runtime inputs violate a documented precondition (e.g. dimension mismatch)."""


class DegenerateMaskError(RuntimeError):
    """Mask-area adjustment eroded the mask to empty before reaching bounds."""


class EngineNumericError(RuntimeError):
    """The inpainting engine produced non-finite values or failed numerically."""


class DeviceError(RuntimeError):
    """A CUDA call inside the B200 extension failed (C-ABI code DR_ERR_CUDA)."""


class ProtocolError(ValueError):
    """A transport message failed validation (reference errors.py:21-30); ``field`` names
    the offending field."""

    def __init__(self, field: str, message: str = ""):
        self.field = field
        super().__init__(f"{field}: {message}" if message else field)
