"""numpy PCG64 stream bookkeeping for the device-side draws.

The reference draws everything from one ``numpy.random.Generator`` (PCG64,
``tuner.py:250``).  The device kernels reproduce that stream exactly by
jump-ahead (csrc/common.cuh), so host and device share one generator: before
a device call the host hands over ``bit_generator.state``; afterwards it
moves the generator forward by exactly the words the device consumed, while
keeping the buffered 32-bit half (``has_uint32``/``uinteger``) that
``Generator.integers`` relies on — ``PCG64.advance`` would discard it, so
the state arithmetic is done here instead.
"""

from __future__ import annotations

import numpy as np

from . import _native as N

M128 = (1 << 128) - 1
M64 = (1 << 64) - 1
MULT = 0x2360ED051FC65DA44385DF649FCCF645


def _jump(steps: int, inc: int):
    """(A, C) with state_{k+steps} = A*state_k + C (mod 2^128)."""
    acc_a, acc_c = 1, 0
    a, c = MULT, inc
    while steps:
        if steps & 1:
            acc_a = (acc_a * a) & M128
            acc_c = (acc_c * a + c) & M128
        c = ((a + 1) * c) & M128
        a = (a * a) & M128
        steps >>= 1
    return acc_a, acc_c


_JUMPS: dict = {}     # (steps, inc) -> (A, C), shared across episodes


class StreamCursor:
    """The generator's PCG64 state as Python ints, advanced without a
    state-dict round trip per skip (jump constants cached per distinct
    step count); ``sync_to``/``sync_from`` hand it to numpy around calls
    that draw through the Generator itself (``choice``)."""

    def __init__(self, gen: np.random.Generator):
        st = check_pcg64(gen)
        self.gen = gen
        self.s = int(st["state"]["state"])
        self.inc = int(st["state"]["inc"])
        self.has = int(st["has_uint32"])
        self.buf = int(st["uinteger"])

    def skip_u64(self, n: int) -> None:
        if n <= 0:
            return
        j = _JUMPS.get((n, self.inc))
        if j is None:
            if len(_JUMPS) > 4096:
                _JUMPS.clear()
            j = _JUMPS[(n, self.inc)] = _jump(n, self.inc)
        self.s = (j[0] * self.s + j[1]) & M128

    def skip_u32(self, n: int) -> None:
        """``skip_u32`` on the cursor (the buffered half kept the same way)."""
        if n <= 0:
            return
        if self.has:
            n -= 1
            self.has = 0
        if n > 0:
            full, odd = divmod(n, 2)
            self.skip_u64(full + odd)
            self.has, self.buf = odd, output(self.s) >> 32

    def struct(self) -> "N.Pcg64":
        return N.Pcg64(state_hi=self.s >> 64, state_lo=self.s & M64,
                       inc_hi=self.inc >> 64, inc_lo=self.inc & M64,
                       has_uint32=self.has, uinteger=self.buf)

    def sync_to(self) -> None:
        self.gen.bit_generator.state = {
            "bit_generator": "PCG64",
            "state": {"state": self.s, "inc": self.inc},
            "has_uint32": self.has, "uinteger": self.buf}

    def sync_from(self) -> None:
        st = self.gen.bit_generator.state
        self.s = int(st["state"]["state"])
        self.has = int(st["has_uint32"])
        self.buf = int(st["uinteger"])


def advance_state(state: int, inc: int, steps: int) -> int:
    a, c = _jump(steps, inc)
    return (a * state + c) & M128


def output(state: int) -> int:
    hi, lo = state >> 64, state & M64
    x = hi ^ lo
    rot = hi >> 58
    return ((x >> rot) | (x << ((64 - rot) & 63))) & M64


def check_pcg64(gen: np.random.Generator) -> dict:
    st = gen.bit_generator.state
    if st.get("bit_generator") != "PCG64":
        from .errors import DeviceError
        raise DeviceError(
            f"device sampling supports numpy PCG64 generators (the "
            f"reference's default_rng), got {st.get('bit_generator')}")
    return st


def to_struct(gen: np.random.Generator) -> "N.Pcg64":
    st = check_pcg64(gen)
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    return N.Pcg64(state_hi=s >> 64, state_lo=s & M64, inc_hi=inc >> 64,
                   inc_lo=inc & M64, has_uint32=int(st["has_uint32"]),
                   uinteger=int(st["uinteger"]))


def skip_u64(gen: np.random.Generator, n: int) -> None:
    """Consume n 64-bit draws (e.g. ``random`` doubles) without touching
    the buffered 32-bit half, exactly as ``Generator.random`` does."""
    if n <= 0:
        return
    st = check_pcg64(gen)
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    st = dict(st)
    st["state"] = {"state": advance_state(s, inc, n), "inc": inc}
    gen.bit_generator.state = st


def skip_u32(gen: np.random.Generator, n: int) -> None:
    """Consume n 32-bit words of the buffered uint32 stream (what
    ``Generator.integers`` with bounds < 2^32 draws from)."""
    if n <= 0:
        return
    st = dict(check_pcg64(gen))
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    has, buf = int(st["has_uint32"]), int(st["uinteger"])
    if has:
        n -= 1
        has = 0          # numpy keeps the stale `uinteger` value
    if n > 0:
        full, odd = divmod(n, 2)
        s = advance_state(s, inc, full + odd)
        # the last 64-bit draw's high half was buffered; it stays buffered
        # for an odd count and has been consumed for an even one
        has, buf = odd, output(s) >> 32
    st["state"] = {"state": s, "inc": inc}
    st["has_uint32"] = has
    st["uinteger"] = buf
    gen.bit_generator.state = st
