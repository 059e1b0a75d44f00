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
    rec, firsts, depth = DeviceForest._records(trees, 0.3)
    assert firsts.tolist() == [0, 7, 10]
    assert depth == 5          # internal levels of the deepest tree
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
    assert DeviceForest._records([_chain(63)], 0.3)[2] == 63
    with pytest.raises(DeviceError):
        DeviceForest._records([_chain(3), _chain(64)], 0.3)


def test_records_empty():
    rec, firsts, depth = DeviceForest._records([], 0.3)
    assert len(rec) == 0 and len(firsts) == 0 and depth == 0


def _walk_records(rec, first, x):
    i = first
    while rec["feat"][i] >= 0:
        f = rec["feat"][i]
        i = first + (rec["left"][i] if x[f] <= rec["v"][i] else rec["right"][i])
    return rec["v"][i]


def _walk_perfect(img, T, D, t, x):
    NI, NL = (1 << D) - 1, 1 << D
    b_leaf = (T * NI * 8 + 15) & ~15
    thr = img[:T * NI * 8].view(np.float64).reshape(T, NI)
    leaf = img[b_leaf:b_leaf + T * NL * 8].view(np.float64).reshape(T, NL)
    feat = img[b_leaf + T * NL * 8:b_leaf + T * NL * 8 + T * NI * 2] \
        .view(np.int16).reshape(T, NI)
    i = 0
    for _ in range(D):
        i = 2 * i + (1 if x[feat[t, i]] <= thr[t, i] else 2)
    return leaf[t, i - NI]


def test_perfect_image_walks_to_the_same_leaves():
    """The perfect-tree image (the kernel's layout for forests of depth
    <= 7) gives every row the leaf value of the node-record walk, also for
    NaN features (which go right in both)."""
    rng = np.random.default_rng(0)
    trees = []
    for _ in range(20):
        feat, thr, left, right, val = [], [], [], [], []

        def add(d):
            i = len(feat)
            feat.append(-1); thr.append(0.0); left.append(-1)
            right.append(-1); val.append(0.0)
            if d < 5 and rng.random() < 0.8:
                feat[i] = int(rng.integers(0, 4))
                thr[i] = float(rng.normal())
                left[i] = add(d + 1)
                right[i] = add(d + 1)
            else:
                val[i] = float(rng.normal())
            return i
        add(0)
        trees.append(tuple(np.asarray(a) for a in (feat, thr, left, right,
                                                   val)))
    rec, firsts, depth = DeviceForest._records(trees, 0.3)
    img = DeviceForest.perfect_image(rec, firsts, depth)
    assert len(img) == DeviceForest.perfect_bytes(len(trees), depth)
    X = rng.normal(size=(300, 4))
    X[::7, 1] = np.nan
    for x in X:
        for t, f in enumerate(firsts):
            a = _walk_records(rec, f, x)
            b = _walk_perfect(img, len(trees), depth, t, x)
            assert a.tobytes() == b.tobytes()


def _random_forest(rng, n_trees, max_d, n_feat=4):
    trees = []
    for _ in range(n_trees):
        feat, thr, left, right, val = [], [], [], [], []

        def add(d):
            i = len(feat)
            feat.append(-1); thr.append(0.0); left.append(-1)
            right.append(-1); val.append(0.0)
            if d < max_d and rng.random() < 0.8:
                feat[i] = int(rng.integers(0, n_feat))
                thr[i] = float(rng.normal())
                left[i] = add(d + 1)
                right[i] = add(d + 1)
            else:
                val[i] = float(rng.normal())
            return i
        add(0)
        trees.append(tuple(np.asarray(a) for a in (feat, thr, left, right,
                                                   val)))
    return trees


def _golden_trees():
    import os
    p = os.path.join(os.path.dirname(__file__), "golden", "gbt_fit_large.npz")
    d = np.load(p)
    n = len({k[:7] for k in d.files if k.startswith("tree")})
    return [tuple(d[f"tree{t:03d}_{c}"] for c in
                  ("feature", "threshold", "left", "right", "value"))
            for t in range(n)]


@pytest.mark.parametrize("case", ["golden", "d3", "d6", "d7", "d9", "one"])
def test_native_pack_matches_the_restatement(case):
    """harl_forest_pack (the drop-in's per-episode forest reload) writes
    the numpy restatement's node records, firsts, depth and perfect-tree
    image byte for byte."""
    rng = np.random.default_rng(sum(map(ord, case)))
    trees = {"golden": _golden_trees,
             "d3": lambda: _random_forest(rng, 50, 3),
             "d6": lambda: _random_forest(rng, 50, 6),
             "d7": lambda: _random_forest(rng, 64, 7),
             "d9": lambda: _random_forest(rng, 30, 9),
             "one": lambda: _random_forest(rng, 1, 0)}[case]()
    rec, firsts, depth = DeviceForest._records(trees, 0.3)
    nrec, nfirsts, ndepth, img = DeviceForest.pack_host(trees, 0.3)
    assert ndepth == depth
    assert nrec.tobytes() == rec.tobytes()
    assert nfirsts.tolist() == firsts.tolist()
    if 0 < depth <= DeviceForest.PERFECT_MAX:
        ref = DeviceForest.perfect_image(rec, firsts, depth)
        assert img is not None and img.tobytes() == ref.tobytes()
    else:
        assert img is None


def test_native_pack_errors():
    assert DeviceForest.pack_host([_chain(63)], 0.3)[2] == 63
    with pytest.raises(DeviceError):
        DeviceForest.pack_host([_chain(3), _chain(64)], 0.3)
    nodes, firsts, depth, img = DeviceForest.pack_host([], 0.3)
    assert len(nodes) == 0 and depth == 0 and img is None
    bad = list(_chain(2))
    bad[2] = bad[2].copy()
    bad[2][0] = 99                      # child outside the tree
    with pytest.raises(DeviceError):
        DeviceForest.pack_host([tuple(bad)], 0.3)
    z = np.zeros(0, np.int64)
    with pytest.raises(DeviceError):
        DeviceForest.pack_host([(z, z.astype(float), z, z, z.astype(float))],
                               0.3)
