"""Host packing of the GBT ensemble into device node records (no GPU)."""

import numpy as np
import pytest

from paper_2211_11172_b200.device import DeviceForest
from paper_2211_11172_b200.errors import DeviceError


def _chain(depth):
    """A right-leaning chain: `depth` inner nodes then leaves."""
    feat, thr, left, right, val = [], [], [], [], []
    for d in range(depth):
        i = len(feat)
        feat += [0, -1]
        thr += [0.5, 0.0]
        left += [i + 1, -1]
        right += [i + 2, -1]
        val += [0.0, float(d)]
    feat.append(-1); thr.append(0.0); left.append(-1); right.append(-1)
    val.append(-1.0)
    return tuple(np.asarray(a) for a in (feat, thr, left, right, val))


def test_records_offsets_and_leaf_products():
    trees = [_chain(3), _chain(1), _chain(5)]
    rec, firsts = DeviceForest._records(trees, 0.3)
    assert firsts.tolist() == [0, 7, 10]
    assert len(rec) == 7 + 3 + 11
    for (feat, thr, left, right, val), f in zip(trees, firsts):
        r = rec[f:f + len(feat)]
        leaf = feat < 0
        assert np.array_equal(r["feat"], feat.astype(np.int16))
        # leaves: the reference's fp64 product lr * value (costmodel.py:224)
        assert r["v"][leaf].tobytes() == (0.3 * val[leaf]).tobytes()
        assert r["v"][~leaf].tobytes() == thr[~leaf].tobytes()
        assert np.array_equal(r["left"][~leaf], left[~leaf])
        assert np.array_equal(r["right"][~leaf], right[~leaf])
        assert not r["left"][leaf].any() and not r["right"][leaf].any()


def test_records_reject_walks_deeper_than_reference():
    DeviceForest._records([_chain(63)], 0.3)
    with pytest.raises(DeviceError):
        DeviceForest._records([_chain(3), _chain(64)], 0.3)


def test_records_empty():
    rec, firsts = DeviceForest._records([], 0.3)
    assert len(rec) == 0 and len(firsts) == 0
