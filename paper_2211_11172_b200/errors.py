"""Exception types with the reference's names and meaning.

Reference definitions (``pkg/src/schedtune``): ``ScheduleError`` and
``InvalidActionError`` (schedspace.py:23-32), ``RlDivergedError``
(rlcore.py:20-21), ``CostModelError`` (costmodel.py:20-21), ``WorkloadError``
(workload.py:19-20).  ``DeviceError`` is new: a CUDA/ABI failure, or the
native library missing on a GPU box (there is no CPU fallback).
"""


class WorkloadError(ValueError):
    """Unreadable or semantically invalid workload description."""


class ScheduleError(ValueError):
    """Malformed schedule state."""


class InvalidActionError(ValueError):
    """A modification violates its subspace constraints."""

    def __init__(self, subspace: str, detail: str):
        super().__init__(f"invalid {subspace} action: {detail}")
        self.subspace = subspace
        self.detail = detail


class RlDivergedError(RuntimeError):
    """A loss or gradient stopped being finite."""


class CostModelError(ValueError):
    pass


class DeviceError(RuntimeError):
    """The B200 path failed (CUDA error, missing native library, bad call)."""


class SpaceTooLarge(DeviceError):
    """brute_force_best refused a space above its cap (measure.py:30-36)."""

    def __init__(self, size: int, cap: int):
        super().__init__(f"space has {size} states, above the cap of {cap}")
        self.size = size
        self.cap = cap


def to_reference(exc: BaseException):
    """The reference package's own exception for one of ours (the drop-in
    raises these, so ``except schedtune.rlcore.RlDivergedError`` and
    friends catch device failures).  None when ``exc`` has no reference
    counterpart or the reference is not importable."""
    try:
        from schedtune import costmodel, rlcore, schedspace, workload
    except ImportError:
        return None
    if isinstance(exc, InvalidActionError):
        return schedspace.InvalidActionError(exc.subspace,
                                             getattr(exc, "detail", str(exc)))
    table = ((RlDivergedError, rlcore.RlDivergedError),
             (ScheduleError, schedspace.ScheduleError),
             (CostModelError, costmodel.CostModelError),
             (WorkloadError, workload.WorkloadError))
    for ours, theirs in table:
        if isinstance(exc, ours):
            return theirs(*exc.args)
    return None
