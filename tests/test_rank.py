"""rank_scores (costmodel.py:266-286) on the device entry log.

CPU: the oracle's restatement reproduces the reference's own rank_scores
answers recorded in tests/golden (several k, with and without an exclude
set of measured states; the fixtures include a repeated state).
GPU: ``device.rank_topk`` selects a superset on which rank_scores returns
exactly the reference's answer, and (no hash collisions) exactly that set.
"""

import numpy as np
import pytest

from golden_util import GoldenCase, case_names
from oracle import harl_oracle as O


def _golden_entries(gc, e_i):
    ep = gc.rec["episodes"][e_i]
    tb = gc.tables(ep["sketch"])
    tiles = gc.arr[f"e{e_i}_entry_tiles"]
    knobs = gc.arr[f"e{e_i}_entry_knobs"]
    scores = gc.arr[f"e{e_i}_entry_score"]
    first = ep["entries_order"][0]
    orders = list(range(first, first + len(knobs)))
    canon = [tb.canonical(t, k) for t, k in zip(tiles, knobs)]
    return tb, tiles, knobs, scores, orders, canon


def _rl_episodes():
    out = []
    for name in case_names():
        gc = GoldenCase(name)
        for e_i, ep in enumerate(gc.rec["episodes"]):
            if "rank" in ep:
                out.append((name, e_i))
    return out


@pytest.mark.parametrize("name,e_i", _rl_episodes())
def test_oracle_rank_scores_matches_reference(name, e_i):
    gc = GoldenCase(name)
    ep = gc.rec["episodes"][e_i]
    tb, tiles, knobs, scores, orders, canon = _golden_entries(gc, e_i)
    import hashlib
    assert hashlib.sha256("\n".join(canon).encode()).hexdigest() == \
        ep["entries_canonical_digest"]
    for r in ep["rank"]:
        pos = O.rank_scores(canon, scores, orders, r["k"], r["exclude"])
        assert [orders[i] for i in pos] == r["chosen"], (r["k"],
                                                         len(r["exclude"]))


def test_arrays_from_canonical_roundtrip():
    gc = GoldenCase("conv2d_l4")
    tb, tiles, knobs, _, _, canon = _golden_entries(gc, 0)
    other = canon[0].replace(tb.sketch_id + "|", "other::k9|")
    t2, k2 = tb.arrays_from_canonical(canon + [other])
    assert np.array_equal(t2, tiles) and np.array_equal(k2, knobs)
    t0, k0 = tb.arrays_from_canonical([])
    assert t0.shape == (0, tb.local_slots) and k0.shape == (0, 3)


# ---------------------------------------------------------------------------
# GPU


def _device_log(tb, tiles, knobs, scores):
    import torch
    from paper_2211_11172_b200 import device as D
    t, k = D.states_to_device(tb, tiles, knobs)
    s = torch.from_numpy(np.ascontiguousarray(scores, np.float64)).cuda()
    return t, k, s


def _check_selection(tb, tiles, knobs, scores, orders, keys, k, exclude_keys,
                     ex_arrays, scratch=None):
    from paper_2211_11172_b200 import device as D
    t, kn, s = _device_log(tb, tiles, knobs, scores)
    idx, st = D.rank_topk(tb, t, kn, s, len(scores), k, ex_arrays, scratch)
    ref = O.rank_scores(keys, scores, orders, k, exclude_keys)
    sub = O.rank_scores([keys[i] for i in idx], scores[idx],
                        [orders[i] for i in idx], k, exclude_keys)
    assert [orders[idx[i]] for i in sub] == [orders[i] for i in ref]
    assert st["selected"] == len(idx) == st["k_target"]
    if st["collisions"] == 0:
        assert sorted(idx.tolist()) == sorted(ref)
    return st


@pytest.mark.gpu
@pytest.mark.parametrize("name,e_i", _rl_episodes())
def test_rank_topk_golden(name, e_i):
    gc = GoldenCase(name)
    ep = gc.rec["episodes"][e_i]
    tb, tiles, knobs, scores, orders, canon = _golden_entries(gc, e_i)
    for r in ep["rank"]:
        ex = tb.arrays_from_canonical(r["exclude"]) if r["exclude"] else None
        _check_selection(tb, tiles, knobs, scores, orders, canon, r["k"],
                         r["exclude"], ex)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [0, 1])
def test_rank_topk_many_duplicates_and_ties(seed):
    """200 K visits drawn from 5 K states (heavy duplication), scores
    quantised to 40 levels (heavy ties: order decides), 300 states
    excluded; k from 0 to beyond the distinct count."""
    from gpu_util import conv_tables
    from paper_2211_11172_b200 import device as D
    tb = conv_tables()
    rng = np.random.default_rng(seed)
    pool_t, pool_k = O.sample_initial(tb, 5000, rng)
    pool_s = np.round(rng.random(5000) * 40) / 40 + 1e-6
    pick = rng.integers(0, 5000, 200_000)
    tiles, knobs, scores = pool_t[pick], pool_k[pick], pool_s[pick]
    # pool entries can coincide as states: key them by content
    content = {}
    keys = [content.setdefault(pool_t[p].tobytes() + pool_k[p].tobytes(), p)
            for p in pick]
    ex_pool = rng.choice(5000, 300, replace=False)
    ex_keys = {content.get(pool_t[p].tobytes() + pool_k[p].tobytes(), -1)
               for p in ex_pool}
    ex_arrays = (pool_t[ex_pool], pool_k[ex_pool])
    orders = list(range(10, 10 + len(pick)))
    sc = D.RankScratch()
    for k in (0, 1, 7, 64, 1000, 4999, 300_000):
        _check_selection(tb, tiles, knobs, scores, orders, keys, k, ex_keys,
                         ex_arrays, sc)
        _check_selection(tb, tiles, knobs, scores, orders, keys, k, set(),
                         None, sc)


@pytest.mark.gpu
def test_rank_topk_empty_and_single():
    from gpu_util import conv_tables
    from paper_2211_11172_b200 import device as D
    tb = conv_tables()
    t, k = O.sample_initial(tb, 1, np.random.default_rng(3))
    s = np.asarray([0.5])
    _check_selection(tb, t, k, s, [0], [0], 5, set(), None)
    dt, dk, ds = _device_log(tb, t, k, s)
    idx, st = D.rank_topk(tb, dt, dk, ds, 0, 5)
    assert len(idx) == 0 and st["selected"] == 0
    # the only state excluded -> nothing left
    idx, st = D.rank_topk(tb, dt, dk, ds, 1, 5, (t, k))
    assert len(idx) == 0 and st["kept"] == 0
