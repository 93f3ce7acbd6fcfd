"""Error taxonomy mirroring the reference (core/include/spectree/errors.hpp:12-46).

C-ABI status codes map onto it the way the reference CLI maps exceptions onto
exit codes (tools/main.cpp:703-712): 2 = ArgumentError family, 3 = other
``Error`` (parse / schema / io).  4 and 5 are GPU-only additions.
"""
from __future__ import annotations


class Error(RuntimeError):
    """spectree::Error (errors.hpp:12)."""


class ArgumentError(Error, ValueError):
    """Invalid argument values or geometry (errors.hpp:18)."""


class StructureError(ArgumentError):
    """Malformed linked tree handed to the encoder (errors.hpp:25)."""


class ParseError(Error):
    """Malformed file content (errors.hpp:31)."""


class SchemaError(ParseError):
    """Structurally invalid or wrong-version tree JSON (errors.hpp:37)."""


class IoError(Error):
    """Filesystem-level failure (errors.hpp:43)."""


class CudaError(Error):
    """A CUDA call failed (status 4; no reference analogue)."""


class NoDeviceError(CudaError):
    """No usable CUDA device (status 5).  There is no CPU fallback."""


def raise_for(code: int, message: str) -> None:
    if code == 0:
        return
    if code == 2:
        raise ArgumentError(message)
    if code == 3:
        raise IoError(message)
    if code == 5:
        raise NoDeviceError(message)
    raise CudaError(f"[{code}] {message}")
