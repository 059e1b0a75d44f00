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


def test_row_cull_matches_track_cull():
    """engine._cull_rows (the graphed episode's cull on the step's rows)
    makes the same decision as engine._cull, ties and NaNs included."""
    from types import SimpleNamespace
    from paper_2211_11172_b200.engine import EpisodeEngine
    E = EpisodeEngine.__new__(EpisodeEngine)
    rng = np.random.default_rng(2)
    for t in range(300):
        P = int(rng.integers(10, 500))
        alive = rng.random(P) < 0.8
        tracks = np.flatnonzero(alive)
        rng.shuffle(tracks)
        adv = np.round(rng.random(len(tracks)) * rng.choice([3, 50, 1e6])) / 7
        if t % 9 == 0:
            adv[rng.random(len(adv)) < 0.1] = np.nan
        cfg = SimpleNamespace(cull_fraction=0.5,
                              min_tracks=int(rng.integers(1, 10)))
        a1, a2 = alive.copy(), alive.copy()
        g1 = E._cull(tracks, adv, len(tracks), a1, cfg)
        g2, k2 = E._cull_rows(tracks, adv, a2, cfg)
        assert g1.tolist() == g2.tolist() and np.array_equal(a1, a2)
        assert k2.tolist() == np.flatnonzero(a1[tracks]).tolist()


@pytest.mark.parametrize("m", [16384, 65536])
def test_cull_select_full_size_matches_row_cull(m):
    """At bench sizes, the radix-select path makes _cull_rows' decision,
    also with -0.0/+0.0 ties (equal in Python's comparisons), all-equal
    advantages and coarse ties."""
    from types import SimpleNamespace
    from paper_2211_11172_b200.engine import EpisodeEngine
    E = EpisodeEngine.__new__(EpisodeEngine)
    lib = N.load(require_device=False)
    rng = np.random.default_rng(m)
    for case in range(4):
        adv = rng.normal(size=m)
        if case == 1:
            adv = np.round(adv * 3) / 3
        elif case == 2:
            adv[:] = -0.0
            adv[::3] = 0.0
        elif case == 3:
            adv[:] = 1.25
        n_tracks = m + 11
        tracks = rng.permutation(n_tracks)[:m].astype(np.int32)
        alive = np.zeros(n_tracks, bool)
        alive[tracks] = True
        cfg = SimpleNamespace(cull_fraction=0.5, min_tracks=m // 2)
        ne = m // 2
        a8 = alive.astype(np.uint8)
        gone = np.zeros(ne, np.int64)
        keep = np.zeros(m, np.int32)
        nk = C.c_int64(0)
        assert lib.harl_cull_select(
            adv.ctypes.data, tracks.ctypes.data, m, a8.ctypes.data, n_tracks,
            ne, gone.ctypes.data, keep.ctypes.data, C.byref(nk)) == 0
        g, k = E._cull_rows(tracks.astype(np.int64), adv, alive, cfg)
        assert gone.tolist() == g.tolist()
        assert keep[:nk.value].tolist() == k.tolist()
        assert np.array_equal(a8.astype(bool), alive)
