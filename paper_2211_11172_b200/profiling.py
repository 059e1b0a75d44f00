"""Launch accounting and optional per-kernel CUDA-event timing.

Every device entry point reports its kernel launches here (always on, an
integer add).  ``timing(True)`` additionally brackets each call with CUDA
events on the launching stream so bench.py can attribute device time to the
dominant kernel (used on an untimed episode, never inside the timed one).
"""

from __future__ import annotations

import contextlib

_launches = 0
_timing = False
_spans = []   # (name, rows, start_event, end_event)


def reset():
    global _launches, _spans
    _launches = 0
    _spans = []


def timing(on: bool):
    global _timing
    _timing = bool(on)


def launch_count() -> int:
    return _launches


def add_launches(n: int):
    """Account kernels executed by a CUDA-graph replay."""
    global _launches
    _launches += n


@contextlib.contextmanager
def span(name: str, rows: int, launches: int = 1):
    global _launches
    _launches += launches
    if not _timing:
        yield
        return
    import torch
    s = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    yield
    e1.record(s)
    _spans.append((name, rows, e0, e1))


def kernel_times() -> dict:
    """{name: {"ms": total, "rows": total rows, "calls": n}}"""
    import torch
    torch.cuda.synchronize()
    out = {}
    for name, rows, e0, e1 in _spans:
        d = out.setdefault(name, {"ms": 0.0, "rows": 0, "calls": 0})
        d["ms"] += e0.elapsed_time(e1)
        d["rows"] += rows
        d["calls"] += 1
    return out
