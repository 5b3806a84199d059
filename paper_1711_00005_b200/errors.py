"""Error types of the B200 march, named and shaped like the reference's.

Reference: ``pkg/src/pe3d/errors.py:1-77``.  Callers that catch the
reference's exceptions by class name and read their payload fields
(``pivot_index``/``member_index`` on a singular solve, ``range_index``/
``sweep``/``member_index`` on a failed step) see the same fields here.
The C ABI reports failures as a status code plus a ``pe3d_error`` record
(``include/pe3d_b200.h``); :func:`raise_from_record` maps that record back
onto these classes.
"""

from __future__ import annotations


class Pe3dError(Exception):
    """Root of every error this package raises (ref ``errors.py:4``)."""


class ConfigError(Pe3dError):
    """Bad or missing configuration data (ref ``errors.py:8``)."""


class InvariantError(Pe3dError):
    """A named model constraint does not hold.

    The message begins with the constraint text (ref ``errors.py:12-23``)
    so tests can ``match`` on it.
    """

    def __init__(self, constraint, detail=""):
        self.constraint = constraint
        super().__init__(f"{constraint}: {detail}" if detail else constraint)


class DomainError(Pe3dError):
    """Operand outside an operation's domain (ref ``errors.py:26``)."""


class ShapeError(Pe3dError):
    """Inconsistent array shapes (ref ``errors.py:30``)."""


class NativeError(Pe3dError):
    """The CUDA library failed (launch error, bad argument, no device).

    Has no reference counterpart: the reference never leaves the CPU.
    """


class SingularSystemError(Pe3dError):
    """A pivot fell below the 1e-300 floor (ref ``errors.py:33-46``)."""

    def __init__(self, pivot_index, member_index=0, detail=""):
        self.pivot_index = pivot_index
        self.member_index = member_index
        text = f"singular system: pivot {pivot_index}, batch member {member_index}"
        super().__init__(f"{text} ({detail})" if detail else text)


class StepError(Pe3dError):
    """A range step failed in one sweep (ref ``errors.py:49-60``)."""

    def __init__(self, range_index, sweep, member_index, cause=None):
        self.range_index = range_index
        self.sweep = sweep
        self.member_index = member_index
        self.cause = cause
        super().__init__(
            f"range step {range_index} failed in {sweep} sweep at index "
            f"{member_index}: {cause}"
        )


class ColumnTaskError(Pe3dError):
    """Per-column tasks failed (ref ``errors.py:63-77``)."""

    def __init__(self, failures):
        self.column_indices = sorted(failures)
        self.failures = dict(failures)
        shown = ", ".join(f"{i}: {failures[i]}" for i in self.column_indices[:4])
        more = ", ..." if len(self.column_indices) > 4 else ""
        super().__init__(f"task failed on columns {self.column_indices} ({shown}{more})")


# Status codes of the C ABI (include/pe3d_b200.h, enum pe3d_status).
STATUS_OK = 0
STATUS_SINGULAR = 1
STATUS_BAD_ARGUMENT = 2
STATUS_CUDA = 3
SWEEP_NAMES = {0: "depth", 1: "azimuth"}


def raise_from_record(status: int, record) -> None:
    """Turn a non-zero ABI status plus its ``pe3d_error`` record into the
    matching Python exception (no-op on success)."""
    if status == STATUS_OK:
        return
    message = bytes(record.message).split(b"\0", 1)[0].decode(errors="replace")
    if status == STATUS_SINGULAR:
        detail = "singular rank-1 correction" if record.rank1 else ""
        cause = SingularSystemError(record.pivot, record.member, detail)
        if record.range_index >= 0:
            raise StepError(record.range_index, SWEEP_NAMES.get(record.sweep, "?"),
                            record.member, cause) from cause
        raise cause
    if status == STATUS_BAD_ARGUMENT:
        raise InvariantError("native argument check", message)
    raise NativeError(f"CUDA failure (status {status}): {message}")
