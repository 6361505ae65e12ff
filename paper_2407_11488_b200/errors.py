"""Error taxonomy of the tuner.

Mirrors the reference hierarchy (`pkg/src/tunescape/errors.py:8-98`) so
that callers switching from ``tunescape`` catch the same classes:
domain failures derive from :class:`TunescapeError`; measurement
failures of a configuration are *never* raised, they become
``Observation`` statuses (`SPEC.md:139`, `SPEC.md:181`).

Two classes are new on the B200 side: :class:`DeviceError` (the CUDA
runtime itself is unusable, e.g. the native library is missing) and
:class:`VerificationError` (``run_kernel`` output disagrees with
``answer`` when the caller asked for a hard failure).
"""


class TunescapeError(Exception):
    """Root of every error raised deliberately by this package."""


class ExpressionSyntaxError(TunescapeError):
    """An expression failed to tokenize or parse (ref errors.py:16-22)."""

    def __init__(self, message: str, source: str, position: int):
        self.source = source
        self.position = position
        super().__init__(f"{message} (column {position + 1} in {source!r})")


class ExpressionTypeError(TunescapeError):
    """An expression is ill-typed for the parameter space (ref :25)."""


class EvaluationError(TunescapeError):
    """Evaluating an expression failed, e.g. a zero divisor (ref :29)."""


class SpecSyntaxError(TunescapeError):
    """A space document is not well-formed YAML (ref :33-42)."""

    def __init__(self, message: str, line: int | None = None, column: int | None = None):
        self.line = line
        self.column = column
        where = ""
        if line is not None:
            where = f" (line {line}, column {1 if column is None else column})"
        super().__init__(message + where)


class SpecValidationError(TunescapeError):
    """A space document parsed but is semantically wrong (ref :45)."""


class MissingEntry(TunescapeError):
    """A replay backend has no record for a configuration (ref :49)."""


class ProtocolError(TunescapeError):
    """Bad protocol / backend descriptor / misuse of the API (ref :53)."""


class NoFeasibleData(TunescapeError):
    """An analysis needs at least one successful record (ref :57)."""


class IncompleteCache(TunescapeError):
    """A cache does not cover the whole space (ref :61-69)."""

    def __init__(self, missing: int, total: int):
        self.missing = missing
        self.total = total
        super().__init__(f"cache is missing {missing} of {total} valid configurations")


class SpaceMismatch(TunescapeError):
    """A cache was recorded for a different space (ref :72)."""


class CacheFormatError(TunescapeError):
    """A cache document fails to parse or validate (ref :92)."""


class CacheIOError(TunescapeError):
    """Reading or writing a cache failed at the OS level (ref :96)."""


class DeviceError(TunescapeError):
    """The CUDA runtime (libtsgpu / driver / NVRTC) is unusable.

    Raised on *setup* problems only (library missing, no device); a
    configuration that fails to compile or launch is still an
    ``Observation`` with a failure status.
    """


class VerificationError(TunescapeError):
    """Kernel output does not match the expected answer."""
