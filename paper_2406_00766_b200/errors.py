"""Error taxonomy of the drop-in API.

Mirrors the reference's categories (``pcirc/errors.py:8-40``): every error
maps onto a process exit code (usage 1, validation 2, numeric 3).  The
C-ABI library returns integer status codes; :func:`raise_for_status`
turns them into these exceptions (see ``include/pcirc_b200.h``).
"""


class PcircError(Exception):
    """Root of every error raised by this package."""

    category = "usage"


class UsageError(PcircError):
    """Bad call order or out-of-range knob (``errors.py:15-18``)."""

    category = "usage"


class CircuitValidationError(PcircError):
    """Structural contract violated by a circuit or its data (``errors.py:21-24``)."""

    category = "validation"


class FormatError(CircuitValidationError):
    """Malformed batch / file (``errors.py:27-28``)."""


class NumericError(PcircError):
    """Degenerate numerics: non-finite parameters, dead EM step (``errors.py:31-34``)."""

    category = "numeric"


EXIT_CODES = {"usage": 1, "validation": 2, "numeric": 3}


def exit_code_for(category: str) -> int:
    return EXIT_CODES.get(category, 1)


# status codes returned by the C-ABI (include/pcirc_b200.h: PCB_*)
_STATUS = {
    1: UsageError,
    2: FormatError,
    3: NumericError,
    4: PcircError,  # CUDA launch / runtime failure
}


def raise_for_status(code: int, what: str) -> None:
    if code == 0:
        return
    exc = _STATUS.get(int(code), PcircError)
    raise exc(f"{what} failed with status {code}")
