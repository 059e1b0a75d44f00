"""Parity at BASELINE.json's full sizes (C2: conv2d at 16 K tracks; C3:
bmm+softmax at 64 K tracks; C5: GEMM 4096^3 at 1 M tracks), where the oracle cannot replay a whole episode in
seconds, through properties that do not depend on size:

* every visited state is a legal state of the sketch: per tiled dimension
  the level factors multiply to the extent, and the knobs are in range
  (schedspace.py: the walker never leaves the space);
* a random sample of the episode's entry log, re-derived by the oracle --
  features from the logged state (schedspace.py:415-438), score from the
  same forest (costmodel.py:219-230) -- matches the device bit for bit;
* rewards chain along each track: a visit's reward is
  (score - previous score) / previous score of the same track's previous
  visit (tuner.py:389-391), bit for bit.
"""

import numpy as np
import pytest

from gpu_util import needs_gpu

pytestmark = [pytest.mark.gpu, needs_gpu]
torch = pytest.importorskip("torch")


def _episode(config, P):
    import bench
    from paper_2211_11172_b200 import device as D
    from paper_2211_11172_b200.engine import EpisodeEngine
    w = bench.build_workload(config, P)
    tb = w["tables"]
    eng = EpisodeEngine(w["agent"], w["rl"], tb.levels)
    forest = D.DeviceForest(w["trees"], w["base"], w["lr"])
    gen = np.random.default_rng(11)
    res = eng.run_episode(tb, forest, gen, bench.episode_config(P), 0)
    torch.cuda.synchronize()
    return w, tb, res


def _check_legal(tb, res):
    """All visits, on the device (40 M visits at 1 M tracks)."""
    V, L = res.visits, tb.levels
    tiles = res.log_tiles[:tb.local_slots, :V].to(torch.int64)
    assert int(tiles.min()) >= 1
    ext = torch.as_tensor(np.asarray(tb.extents, np.int64), device=tiles.device)
    for d in range(tb.ndims):
        prod = torch.prod(tiles[d * L:(d + 1) * L], dim=0)
        assert bool((prod == ext[d]).all()), f"dim {d}: factors do not multiply to the extent"
    kn = res.log_knobs[:, :V].to(torch.int64)
    assert int(kn[0].max()) < tb.ncas and int(kn[1].max()) <= tb.max_fusible
    assert int(kn[2].max()) < tb.n_unroll and int(kn.min()) >= 0


def _check_sample(w, tb, res, n=2000, seed=0):
    from oracle import harl_oracle as O
    V = res.visits
    idx = np.sort(np.random.default_rng(seed).choice(V, size=min(n, V),
                                                     replace=False))
    it = torch.as_tensor(idx, device=res.log_tiles.device)
    tiles = res.log_tiles[:tb.local_slots].index_select(1, it).cpu().numpy()
    knobs = res.log_knobs.index_select(1, it).cpu().numpy()
    tiles = np.ascontiguousarray(tiles.T).astype(np.uint16)
    knobs = np.ascontiguousarray(knobs.T).astype(np.uint8)
    X = O.featurize(tb, tiles, knobs)
    model = O.GbtModel(base=w["base"], learning_rate=w["lr"], fitted=True,
                       trees=w["trees"])
    ref = model.predict(X)
    got = res.log_score.index_select(0, it).cpu().numpy()
    assert got.tobytes() == ref.tobytes()


def _check_reward_chain(res):
    V = res.visits
    track = res.log_track[:V].cpu().numpy().astype(np.int64)
    score = res.log_score[:V].cpu().numpy()
    reward = res.log_reward[:V].cpu().numpy()
    # visits are logged step by step; the previous visit of a track is its
    # last earlier occurrence
    order = np.argsort(track, kind="stable")
    t_sorted = track[order]
    same = t_sorted[1:] == t_sorted[:-1]
    cur, prev = order[1:][same], order[:-1][same]
    assert len(cur) > 0
    assert reward[cur].tobytes() == \
        ((score[cur] - score[prev]) / score[prev]).tobytes()


def test_c2_full_size_episode_properties():
    w, tb, res = _episode("c2", 16384)
    assert res.visits == 16384 * 40
    _check_legal(tb, res)
    _check_sample(w, tb, res)
    _check_reward_chain(res)


def test_c3_full_size_episode_properties():
    """C3 (bmm + softmax, sketch k3: 2 stages, 7 dims) at 65,536 tracks."""
    w, tb, res = _episode("c3", 65536)
    assert res.visits == 65536 * 40
    assert len(res.train) == 30 and len(res.culls) == 1
    _check_legal(tb, res)
    _check_sample(w, tb, res, seed=2)
    _check_reward_chain(res)


def test_c5_one_million_tracks_properties():
    P = 1 << 20
    w, tb, res = _episode("c5", P)
    assert res.visits == P * 40
    _check_legal(tb, res)
    _check_sample(w, tb, res, n=1000, seed=1)


@pytest.mark.parametrize("P", [1, 3, 129, 1000])
def test_ragged_small_populations(P):
    """Populations that fill no tile, a partial tile or a ragged last tile
    (128-row MMA tiles, 16-row sampler CTAs, 8-lane groups) keep the same
    properties; with one track the cull never fires (min_tracks)."""
    w, tb, res = _episode("c2", P)
    assert res.visits == sum(res.step_rows) > 0
    _check_legal(tb, res)
    _check_sample(w, tb, res, n=min(500, res.visits))
    if P > 1:
        _check_reward_chain(res)
