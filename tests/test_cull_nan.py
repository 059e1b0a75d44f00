"""TrackSet.cull (stopping.py:68-86) with non-finite advantages.

With a NaN key, Python's tuple comparisons are not a total order, so the
reference's ``sorted(live, key=(adv, -index))`` depends on timsort's
comparison sequence over the index-ordered input -- not "NaN last".  The
host cull (``shard.eliminated``, used by the engine and the sharded path)
must take the reference's exact decision.  Checked against the reference's
own ``TrackSet.cull`` when the package is importable (baseline/_ref), and
against a literal restatement of its sort otherwise."""

import math
import os
import sys

import numpy as np
import pytest

from paper_2211_11172_b200.shard import cull_decision, eliminated

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def _restated(live, adv, n_elim):
    ordered = sorted(zip(live.tolist(), adv.tolist()),
                     key=lambda t: (t[1], -t[0]))
    return sorted(i for i, _ in ordered[:n_elim])


def _cases():
    rng = np.random.default_rng(3)
    for trial in range(60):
        n = int(rng.integers(2, 300))
        live = np.sort(rng.choice(1000, size=n, replace=False))
        adv = rng.standard_normal(n)
        if trial % 3 == 0:
            adv = np.round(adv, 1)                  # ties
        k = int(rng.integers(1, max(2, n // 4)))
        adv[rng.choice(n, size=k, replace=False)] = np.nan
        if trial % 5 == 0:
            adv[rng.integers(n)] = -math.inf
        yield live, adv, int(rng.integers(1, n))


def test_eliminated_matches_reference_sort_with_nan():
    for live, adv, n_elim in _cases():
        got = eliminated(live, adv, n_elim).tolist()
        assert got == _restated(live, adv, n_elim)


def test_eliminated_finite_is_lexsort_order():
    rng = np.random.default_rng(4)
    for _ in range(50):
        n = int(rng.integers(2, 500))
        live = np.sort(rng.choice(5000, size=n, replace=False))
        adv = np.round(rng.standard_normal(n), 1)
        n_elim = int(rng.integers(1, n))
        assert eliminated(live, adv, n_elim).tolist() == \
            _restated(live, adv, n_elim)


def test_against_reference_trackset_cull():
    if os.path.isdir(REF) and REF not in sys.path:
        sys.path.insert(0, REF)
    stopping = pytest.importorskip("schedtune.stopping")
    cfg = stopping.StopConfig(cull_window=1, cull_fraction=0.5, min_tracks=1)
    for live, adv, _ in _cases():
        P = int(live.max()) + 1
        ts = stopping.TrackSet([None] * P, [None] * P, [0.0] * P)
        alive = np.zeros(P, dtype=bool)
        alive[live] = True
        for t in ts.tracks:
            t.alive = bool(alive[t.index])
        ref = ts.cull({int(i): float(a) for i, a in zip(live, adv)}, cfg)
        got = cull_decision(alive, live, adv, 0.5, 1)
        assert got.tolist() == ref
