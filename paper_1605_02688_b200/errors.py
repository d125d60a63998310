"""Exception vocabulary.

The class names are part of the drop-in surface: user code written against the
reference catches these by name (reference ``pkg/src/texpr/errors.py:4-81``).
The device path raises the same classes for the same conditions, plus
``DeviceError`` for failures reported by the native library (CUDA, NVRTC or
NCCL status codes surfaced through ``tx_last_error``).
"""
from __future__ import annotations

__all__ = [
    "TexprError", "TypeMismatch", "ShapeMismatch", "CycleDetected", "UnknownVariable",
    "UnderdeterminedOutputs", "NotDifferentiable", "DisconnectedInput", "NotSupported",
    "RewriteCycleDetected", "NoImplementationSelected", "AbstractOpRemaining",
    "LengthMismatch", "MissingNonSequence", "MissingTestValue", "NanDetected",
    "BreakpointAbort", "VersionMismatch", "CorruptPayload", "DeviceError",
]


class TexprError(Exception):
    """Root of every deliberate error raised by this package."""


# graph / typing
class TypeMismatch(TexprError): ...
class ShapeMismatch(TexprError): ...
class CycleDetected(TexprError): ...
class UnknownVariable(TexprError): ...
class UnderdeterminedOutputs(TexprError): ...

# differentiation
class NotDifferentiable(TexprError): ...
class DisconnectedInput(TexprError): ...

# rewriting / compilation
class NotSupported(TexprError): ...
class RewriteCycleDetected(TexprError): ...
class NoImplementationSelected(TexprError): ...
class AbstractOpRemaining(TexprError): ...

# loops / diagnostics / serialization (kept for name compatibility)
class LengthMismatch(TexprError): ...
class MissingNonSequence(TexprError): ...
class MissingTestValue(TexprError): ...
class BreakpointAbort(TexprError): ...
class VersionMismatch(TexprError): ...
class CorruptPayload(TexprError): ...


class NanDetected(TexprError):
    """A guard check fired; ``report`` holds the details."""

    def __init__(self, report):
        super().__init__(str(report))
        self.report = report


class DeviceError(TexprError):
    """The native B200 library returned a non-zero status.

    ``code`` is the library's TX_E_* code; the message carries the CUDA /
    NVRTC / NCCL error string captured on the native side.
    """

    def __init__(self, code: int, message: str):
        super().__init__(f"[tx error {code}] {message}")
        self.code = code
