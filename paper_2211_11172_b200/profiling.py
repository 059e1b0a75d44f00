"""Launch accounting and optional per-kernel CUDA-event timing.

Every device entry point reports its kernel launches here (always on, an
integer add).  ``timing(True)`` additionally brackets each call with CUDA
events on the launching stream so bench.py can attribute device time to the
dominant kernel (used on an untimed episode, never inside the timed one).
"""

from __future__ import annotations

import contextlib

import numpy as np

_launches = 0
_timing = False
_xfer = {"h2d": 0, "d2h": 0}   # host<->device bytes moved by the library
_spans = []   # (name, rows, start_event, end_event)


def reset():
    global _launches, _spans
    _launches = 0
    _spans = []


def xfer(kind: str, *tensors_or_bytes):
    """Account host<->device bytes (``kind`` "h2d" or "d2h") of the copies
    the library issues: tensors (their bytes) or plain byte counts."""
    n = 0
    for t in tensors_or_bytes:
        n += int(t) if isinstance(t, (int, np.integer)) else \
            t.numel() * t.element_size()
    _xfer[kind] += n


def xfer_reset():
    _xfer["h2d"] = _xfer["d2h"] = 0


def xfer_bytes() -> dict:
    return dict(_xfer)


def timing(on: bool):
    global _timing
    _timing = bool(on)


def launch_count() -> int:
    return _launches


def add_launches(n: int):
    """Account kernels executed by a CUDA-graph replay."""
    global _launches
    _launches += n


def _native_count():
    from . import _native as N
    return int(N.load(require_device=False).harl_launch_count())


@contextlib.contextmanager
def span(name: str, rows: int, launches: int | None = 1):
    """``launches=None``: count the library's own launches in the span
    (entry points whose kernel count depends on the path they take)."""
    global _launches
    if launches is None:
        before = _native_count()
        try:
            with span(name, rows, 0):
                yield
        finally:
            _launches += _native_count() - before
        return
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


def native_timing(on: bool, spin_ns: int = 20000):
    """Per-kernel CUDA-event timer inside the native library
    (harl_profile_set): each launch is preceded by a ``spin_ns`` spin kernel
    so its begin event marks the kernel's real start."""
    from . import _native as N
    lib = N.load()
    if on:
        N.check(lib.harl_profile_reset(), "harl_profile_reset")
    N.check(lib.harl_profile_set(1 if on else 0, int(spin_ns)),
            "harl_profile_set")


def native_kernel_times() -> dict:
    """{kernel name: {"ms": summed ms, "launches": n, "units": rows}} from
    the native timer (synchronises the recorded events); ``units`` is the
    rows the launches processed as the library counted them (-1 when a
    launch site does not report them)."""
    import ctypes as C
    import numpy as np
    from . import _native as N
    lib = N.load()
    cap, width = 64, 64
    names = C.create_string_buffer(cap * width)
    ms = np.zeros(cap, dtype=np.float64)
    cnt = np.zeros(cap, dtype=np.int64)
    units = np.zeros(cap, dtype=np.int64)
    n = lib.harl_profile_read(cap, names, width, ms.ctypes.data,
                              cnt.ctypes.data, units.ctypes.data)
    if n < 0:
        N.check(n, "harl_profile_read")
    raw = names.raw
    out = {}
    for k in range(min(n, cap)):
        nm = raw[k * width:(k + 1) * width].split(b"\0", 1)[0].decode()
        out[nm] = {"ms": float(ms[k]), "launches": int(cnt[k]),
                   "units": int(units[k])}
    return out


def native_launch_count() -> int:
    from . import _native as N
    return int(N.load(require_device=False).harl_launch_count())
