"""harl_cull_select (host C++, no GPU): TrackSet.cull's decision
(stopping.py:68-86) -- the n_elim lowest (advantage, -index) live tracks go,
NaN advantages last -- against a direct restatement, with the survivor row
list the device gather consumes."""

import ctypes as C
import math

import numpy as np
import pytest

from paper_2211_11172_b200 import _native as N


@pytest.mark.parametrize("seed", range(4))
def test_cull_select_matches_sorted_rule(seed):
    lib = N.load(require_device=False)
    rng = np.random.default_rng(seed)
    for t in range(150):
        P = int(rng.integers(4, 400))
        alive = rng.random(P) < 0.7
        live = np.flatnonzero(alive)
        tracks = live.astype(np.int32).copy()
        rng.shuffle(tracks)
        adv = np.round(rng.random(len(tracks)) * rng.choice([2, 9, 1e6])) / 3
        if t % 5 == 0:
            adv[rng.random(len(adv)) < 0.2] = np.nan
        n = len(live)
        ne = max(0, min(int(math.floor(0.5 * n)), n - int(rng.integers(1, 5))))
        full = {int(tr): a for tr, a in zip(tracks, adv)}

        def key(i):
            a = full[i]
            return (np.isnan(a), 0.0 if np.isnan(a) else a, -i)
        ref = sorted(sorted(live, key=key)[:ne])
        a8 = alive.astype(np.uint8)
        gone = np.zeros(ne, np.int64)
        keep = np.zeros(len(tracks), np.int32)
        nk = C.c_int64(0)
        assert lib.harl_cull_select(
            adv.ctypes.data, tracks.ctypes.data, len(tracks), a8.ctypes.data,
            P, ne, gone.ctypes.data, keep.ctypes.data, C.byref(nk)) == 0
        assert gone.tolist() == [int(x) for x in ref]
        alive2 = alive.copy()
        alive2[ref] = False
        assert np.array_equal(a8.astype(bool), alive2)
        assert keep[:nk.value].tolist() == \
            [r for r in range(len(tracks)) if alive2[tracks[r]]]


def test_cull_select_rejects_dead_rows():
    lib = N.load(require_device=False)
    adv = np.zeros(2)
    tracks = np.asarray([0, 1], np.int32)
    a8 = np.asarray([1, 0], np.uint8)
    gone = np.zeros(1, np.int64)
    keep = np.zeros(2, np.int32)
    nk = C.c_int64(0)
    assert lib.harl_cull_select(adv.ctypes.data, tracks.ctypes.data, 2,
                                a8.ctypes.data, 2, 1, gone.ctypes.data,
                                keep.ctypes.data, C.byref(nk)) != 0
