"""Typed errors of the drop-in API, mirroring the reference taxonomy.

Same class names, base classes and machine-greppable ``ident`` strings as the
reference (pkg/src/itq3/errors.py:10-59), so ``except itq3.CorruptionError`` style
code keeps working.  ``from_status`` maps the C ABI status codes of libitq3
(include/itq3.h ``itq3_status``) onto these classes.
"""

from __future__ import annotations


class ItqError(Exception):
    """Root of every error raised by this package."""

    ident = "error"


def _kind(name: str, bases: tuple, ident: str, doc: str):
    return type(name, bases, {"ident": ident, "__doc__": doc, "__module__": __name__})


LengthError = _kind("LengthError", (ItqError, ValueError), "bad-length",
                    "Block or code-stream length not acceptable (power of two, range, multiple of 8).")
DomainError = _kind("DomainError", (ItqError, ValueError), "bad-domain",
                    "Numeric argument outside its valid domain (non-finite, non-positive, out of range).")
ShapeError = _kind("ShapeError", (ItqError, ValueError), "bad-shape", "Operand dimensions do not match.")
CorruptionError = _kind("CorruptionError", (ItqError, ValueError), "corrupt-data",
                        "Serialized data decodes to values a valid encoder cannot produce.")
ContainerError = _kind("ContainerError", (ItqError,), "bad-container", "Container stream error.")
BadMagicError = _kind("BadMagicError", (ContainerError,), "bad-magic", "Container magic is not 'ITQ3'.")
UnsupportedVersionError = _kind("UnsupportedVersionError", (ContainerError,), "bad-version",
                                "Container version is not supported.")
TruncatedStreamError = _kind("TruncatedStreamError", (ContainerError,), "truncated", "Container is truncated.")
SizeMismatchError = _kind("SizeMismatchError", (ContainerError,), "size-mismatch",
                          "Container has trailing bytes.")


class KernelError(ItqError, RuntimeError):
    """libitq3 reported a CUDA launch/runtime failure (status ITQ3_E_CUDA)."""

    ident = "cuda"


_BY_STATUS = {1: LengthError, 2: DomainError, 3: ShapeError, 4: CorruptionError, 16: KernelError}


def from_status(status: int, message: str) -> ItqError:
    return _BY_STATUS.get(status, KernelError)(message)
