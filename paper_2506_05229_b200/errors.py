"""Error taxonomy of the engine (mirrors ``armt/errors.py:9-24``).

The C-ABI returns integer status codes (``include/armt_b200.h``); the
Python boundary translates every nonzero code into one of these types so
callers see the same exceptions the reference raises.
"""


class EngineError(Exception):
    """Base class for every error the engine raises on purpose."""


class InputError(EngineError):
    """Bad user input: config values, token ids, state compatibility."""


class DimensionError(EngineError):
    """Shapes, dtypes or devices violate an operation's contract."""


class SchedulingError(EngineError):
    """Group/cursor invariants of the wavefront are violated."""


class DeviceError(EngineError):
    """The CUDA extension is missing, or a kernel launch failed."""
