"""Errors raised by the tuner, grouped by who has to act on them.

The class *names* are the public contract callers catch (they are the
names SPEC.md uses: ``MissingEntry``, ``IncompleteCache``,
``SpaceMismatch`` ...), so code written against the reference keeps its
``except`` clauses.  Measurement failures of a single configuration are
never raised -- they are ``Observation`` statuses (SPEC.md "Failures are
first-class recorded outcomes").

Intermediate bases group the classes by the stage that raises them, so
a caller can catch "the space definition is wrong" (:class:`SpaceError`)
or "a cache file is unusable" (:class:`CacheError`) in one clause.  The
command line maps every one of them to exit status 1 (SPEC.md ``cli``).

B200-only additions: :class:`DeviceError` (the CUDA runtime is unusable:
library missing, no device) and :class:`VerificationError` (an output
disagrees with ``answer`` and the caller asked for a hard failure).
"""

from __future__ import annotations


class TunescapeError(Exception):
    """Root: every deliberate error of this package derives from it."""


# --- the space (expressions, spec documents) ---------------------------------


class SpaceError(TunescapeError):
    """The definition of a search space is unusable."""


class ExpressionSyntaxError(SpaceError):
    """Text that does not tokenize/parse as an expression.

    ``position`` is the 0-based character offset; the message shows it
    1-based as a column, the form the reference's tests match.
    """

    def __init__(self, message: str, source: str, position: int):
        self.source, self.position = source, position
        Exception.__init__(self, "%s (column %d in %r)" % (message, position + 1, source))


class ExpressionTypeError(SpaceError):
    """Well-formed expression that is ill-typed for its parameter space."""


class SpecSyntaxError(SpaceError):
    """A space document that is not a well-formed YAML mapping."""

    def __init__(self, message: str, line: int | None = None, column: int | None = None):
        self.line, self.column = line, column
        if line is not None:
            message = "%s (line %d, column %d)" % (message, line, column or 1)
        Exception.__init__(self, message)


class SpecValidationError(SpaceError):
    """A space document that parsed but describes an impossible space."""


class EvaluationError(SpaceError):
    """An expression failed on concrete values (zero divisor, ...)."""


# --- measurement and analysis --------------------------------------------------


class ProtocolError(TunescapeError):
    """Misuse of the measurement API: bad protocol, descriptor or call."""


class MissingEntry(TunescapeError):
    """A replay backend holds no record for the requested configuration."""


class NoFeasibleData(TunescapeError):
    """An analysis needs at least one successful record and got none."""


class NonConvergence(TunescapeError):
    """An iterative solver (PageRank) missed its tolerance."""

    def __init__(self, iterations: int, residual: float, tol: float):
        self.iterations, self.residual, self.tol = iterations, residual, tol
        Exception.__init__(self, f"no convergence after {iterations} iterations "
                                 f"(residual {residual:.3e}, tolerance {tol:.3e})")


class NoPortableConfiguration(TunescapeError):
    """No configuration scores above zero on every device of a set."""


class UnknownDevice(TunescapeError):
    """A device subset names a device that has no cache."""


# --- cache files ----------------------------------------------------------------


class CacheError(TunescapeError):
    """A tuning cache cannot be used as given."""


class IncompleteCache(CacheError):
    """A cache that does not cover every valid configuration of its space."""

    def __init__(self, missing: int, total: int):
        self.missing, self.total = missing, total
        Exception.__init__(self, f"cache is missing {missing} of {total} valid configurations")


class SpaceMismatch(CacheError):
    """A cache recorded for a different space than the one supplied."""


class CacheFormatError(CacheError):
    """A cache document that does not parse or violates its schema."""


class CacheIOError(CacheError):
    """The operating system refused to read or write a cache file."""


# --- B200 runtime ------------------------------------------------------------


class DeviceError(TunescapeError):
    """The CUDA runtime (libtsgpu, driver, NVRTC) cannot be used at all.

    Setup problems only; a configuration that fails to compile or launch
    is still an ``Observation`` with a failure status.
    """


class VerificationError(TunescapeError):
    """Kernel output disagrees with the expected answer."""
