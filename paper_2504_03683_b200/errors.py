"""Exception classes raised by the hapigpu analysis path.

Names, base classes and constructor arguments mirror the reference hierarchy
(`/root/reference/pkg/src/hapitrace/errors.py:4-89`) so code that catches the
reference's exceptions keeps working when the GPU engine is swapped in.  Only
the classes that the decode -> pair -> tally/timeline path can raise are
defined here, plus the merge error.
"""

from __future__ import annotations


class HapitraceError(Exception):
    """Root of every error the analysis path raises (errors.py:4-5)."""


class RegistryError(HapitraceError):
    """Schema registry lookup failure (errors.py:37-38)."""


class FingerprintMismatchError(HapitraceError):
    """Tally reports from different API models were merged (errors.py:46-47)."""


class TraceError(HapitraceError):
    """Trace directory / stream file problem (errors.py:50-51)."""


class TraceDirectoryError(TraceError):
    """Missing, unfinalized or incomplete trace directory (errors.py:54-55)."""


class UnknownSchemaError(TraceError):
    """A record names a schema id the registry does not hold (errors.py:62-63)."""


class CorruptRecordError(TraceError):
    """Undecodable record; carries the stream label and byte offset (errors.py:66-72)."""

    def __init__(self, message, stream, offset):
        self.stream = stream
        self.offset = offset
        super().__init__(f"{message} (stream {stream}, byte offset {offset})")


class MuxOrderingError(HapitraceError):
    """A stream's timestamps went backwards (errors.py:75-83)."""

    def __init__(self, stream, index):
        self.stream = stream
        self.index = index
        super().__init__(f"stream {stream} violates timestamp monotonicity at message {index}")


class PipelineError(HapitraceError):
    """Bad pipeline wiring (errors.py:86-87)."""


class EngineError(HapitraceError):
    """The native engine failed (CUDA error, allocation failure, missing library)."""


class UnsupportedTraceError(EngineError):
    """The registry uses a layout the GPU decoder does not implement.

    Raised up front (never silently handled on the CPU): e.g. a host-exit
    ``result`` field of kind string/blob, or device-profiling timestamps that
    are not integer kinds.
    """
