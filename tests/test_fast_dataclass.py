"""space.fast_dataclass_maker: the drop-in's CandidateEntry / ScheduleState
construction without the frozen __init__'s per-field setattr -- equal,
hash-equal, same repr, still frozen; classes it cannot treat that way
(__post_init__, slots, other fields) get their constructor."""

import dataclasses
import os
import sys

import numpy as np
import pytest

from paper_2211_11172_b200.space import fast_dataclass_maker

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@dataclasses.dataclass(frozen=True)
class _S:
    a: str
    b: tuple
    c: int = 0


@dataclasses.dataclass(frozen=True)
class _P:
    a: int

    def __post_init__(self):
        if self.a < 0:
            raise ValueError("negative")


def test_fast_maker_equals_constructor():
    mk = fast_dataclass_maker(_S, ("a", "b", "c"))
    x, y = mk("k", ((1, 2),), 3), _S(a="k", b=((1, 2),), c=3)
    assert x == y and hash(x) == hash(y) and repr(x) == repr(y)
    with pytest.raises(dataclasses.FrozenInstanceError):
        x.c = 4


def test_fast_maker_falls_back_to_the_constructor():
    mk = fast_dataclass_maker(_P, ("a",))
    assert mk(1) == _P(1)
    with pytest.raises(ValueError):
        mk(-1)
    mk2 = fast_dataclass_maker(_S, ("a", "b"))      # not all fields
    assert mk2("k", ()) == _S("k", ())


def test_fast_maker_on_the_reference_classes():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(ref) and ref not in sys.path:
        sys.path.insert(0, ref)
    st = pytest.importorskip("schedtune")
    from schedtune.costmodel import CandidateEntry
    from schedtune.schedspace import ScheduleState
    ms = fast_dataclass_maker(ScheduleState, (
        "sketch_id", "tiles", "compute_at_index", "parallel_fuse_count",
        "unroll_index"))
    s1 = ms("sk", ((4, 2), (8, 1)), 1, 0, 2)
    s2 = ScheduleState(sketch_id="sk", tiles=((4, 2), (8, 1)),
                       compute_at_index=1, parallel_fuse_count=0,
                       unroll_index=2)
    assert s1 == s2 and hash(s1) == hash(s2) and s1.canonical() == s2.canonical()
    me = fast_dataclass_maker(CandidateEntry, ("canonical", "features",
                                               "state", "order"))
    f = np.zeros(3)
    e1 = me(s1.canonical(), f, s1, 7)
    e2 = CandidateEntry(canonical=s2.canonical(), features=f, state=s2, order=7)
    assert repr(e1) == repr(e2) and e1.order == e2.order and e1.state == e2.state
    assert st is not None
