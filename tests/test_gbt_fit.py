"""GBT refit (SurrogateModel.fit_incremental / _fit_tree, costmodel.py:81-141,
190-212): the oracle restatement and the device refit reproduce the
reference's ensembles bit for bit (node numbering, features, thresholds,
leaf values, base) on recorded training sets."""

import os

import numpy as np
import pytest

from golden_util import GOLDEN, GoldenCase, case_names
from oracle import harl_oracle as O


def _large():
    a = dict(np.load(os.path.join(GOLDEN, "gbt_fit_large.npz")))
    trees = []
    for i in range(int(a["n_trees"][0])):
        p = f"tree{i:03d}_"
        trees.append((a[p + "feature"].astype(np.int64), a[p + "threshold"],
                      a[p + "left"].astype(np.int64),
                      a[p + "right"].astype(np.int64), a[p + "value"]))
    return a["X"], a["y"], float(a["base"][0]), trees, 0.3


def _episode_fit(name):
    gc = GoldenCase(name)
    return (gc.arr["fit_X"], gc.arr["fit_y"], gc.model_base, gc.trees(),
            gc.rec["model_lr"])


CASES = ["large"] + case_names()


def _case(name):
    return _large() if name == "large" else _episode_fit(name)


def _same_trees(got, ref):
    assert len(got) == len(ref)
    for t, (g, r) in enumerate(zip(got, ref)):
        for k, (a, b) in enumerate(zip(g, r)):
            a = np.asarray(a)
            b = np.asarray(b, dtype=a.dtype)
            assert a.shape == b.shape, (t, k)
            assert a.tobytes() == b.tobytes(), (t, k)


@pytest.mark.parametrize("name", CASES)
def test_oracle_refit_matches_reference(name):
    X, y, base, trees, lr = _case(name)
    b, got, _ = O.gbt_fit(X, y, 50, 6, lr, 1)
    assert b == base
    _same_trees(got, trees)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_device_refit_matches_reference(name):
    from paper_2211_11172_b200 import device as D
    X, y, base, trees, lr = _case(name)
    fit = D.gbt_fit(X, y, n_trees=50, max_depth=6, learning_rate=lr,
                    min_leaf=1)
    assert fit.base == base
    _same_trees(fit.trees, trees)
    _, _, pred = O.gbt_fit(X, y, 50, 6, lr, 1)
    assert fit.pred.tobytes() == pred.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("min_leaf,depth,n_trees", [(3, 4, 20), (1, 1, 5),
                                                    (1, 8, 10)])
def test_device_refit_other_configs(min_leaf, depth, n_trees):
    """min_samples_leaf > 1, stumps and deeper trees against the oracle,
    on data with heavy ties (quantised features) and an early stop."""
    from paper_2211_11172_b200 import device as D
    rng = np.random.default_rng(min_leaf * 100 + depth)
    X = np.round(rng.random((700, 12)) * 6) / 6
    y = np.where(rng.random(700) < 0.5, 0.25, 1.0) * (1 + 0 * X[:, 0])
    y[::7] = rng.random(100)[: len(y[::7])]
    base, trees, pred = O.gbt_fit(X, y, n_trees, depth, 0.3, min_leaf)
    fit = D.gbt_fit(X, y, n_trees=n_trees, max_depth=depth,
                    learning_rate=0.3, min_leaf=min_leaf)
    assert fit.base == base
    _same_trees(fit.trees, trees)
    assert fit.pred.tobytes() == pred.tobytes()


@pytest.mark.gpu
def test_device_refit_constant_targets_stop_early():
    from paper_2211_11172_b200 import device as D
    X = np.random.default_rng(0).random((50, 5))
    y = np.full(50, 0.5)
    fit = D.gbt_fit(X, y)
    assert fit.base == 0.5 and fit.trees == []


def _ref_to_heap(tree, K):
    feat, thr, left, right, val = tree
    fh = np.full(K, -2, np.int32)
    th = np.zeros(K)
    vh = np.zeros(K)
    stack = [(0, 0)]
    while stack:
        nid, h = stack.pop()
        fh[h] = feat[nid] if feat[nid] >= 0 else -1
        th[h] = thr[nid] if feat[nid] >= 0 else 0.0
        vh[h] = val[nid]
        if feat[nid] >= 0:
            stack += [(left[nid], 2 * h + 1), (right[nid], 2 * h + 2)]
    return fh, th, vh


@pytest.mark.parametrize("name", CASES[:3])
def test_heap_renumbering_roundtrip(name):
    """heap layout -> the reference's creation-order numbering (no GPU)."""
    from paper_2211_11172_b200.device import heap_tree_to_reference
    _, _, _, trees, _ = _case(name)
    for tr in trees:
        got = heap_tree_to_reference(*_ref_to_heap(tr, 127))
        _same_trees([got], [tr])


def test_native_heap_renumbering_matches_python():
    """harl_heap_to_creation_order == heap_tree_to_reference (no GPU)."""
    from paper_2211_11172_b200.device import (heap_tree_to_reference,
                                              heap_trees_to_reference)
    _, _, _, trees, _ = _case("large")
    heaps = [_ref_to_heap(tr, 127) for tr in trees]
    fh = np.stack([h[0] for h in heaps])
    th = np.stack([h[1] for h in heaps])
    vh = np.stack([h[2] for h in heaps])
    got = heap_trees_to_reference(fh, th, vh)
    _same_trees(got, trees)
    _same_trees(got, [heap_tree_to_reference(*h) for h in heaps])
