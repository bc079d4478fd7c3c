"""Exception types of the reference API (same names and base classes).

model.py:35-36, kvcache.py:25-30, speculation.py:35-36, verify.py:28-29,
engine.py:72-73, transport.py:30-35.
"""


class ModelError(ValueError):
    """Invalid model configuration or evaluation input."""


class CacheError(ValueError):
    pass


class AllocationExhausted(Exception):
    """No free sequence partition; caller should stall speculation."""


class SpeculationError(RuntimeError):
    pass


class VerifyError(RuntimeError):
    pass


class EngineError(RuntimeError):
    pass


class TransportError(RuntimeError):
    pass


class ProtocolError(TransportError):
    """Ordered-transaction contract violated; always fatal."""


class LibraryMissing(RuntimeError):
    """The sm_100a CUDA library is absent: there is no CPU fallback."""
