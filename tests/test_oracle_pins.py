"""The reference's own known answers for the hot path,
restated against the host mirror + oracle (CPU) and against the device
kernels (GPU).  Answers come from the reference's tests: tiling counts
(tests/test_schedspace.py:62-80), smallest prime factors (90-93), space
sizes (99-122), the (4,16) -> (2,32) move and its rejections (222-269),
mask boundaries (290-307), head sizes (352-360), decode layout (363-370);
advantage (tests/test_rlcore.py:58-75); untrained / single-example GBT
(tests/test_costmodel.py:40-60)."""

import numpy as np
import pytest

from oracle import harl_oracle as O
from paper_2211_11172_b200 import space as SP
from paper_2211_11172_b200 import workloads as W
from paper_2211_11172_b200.space import SketchTables

GEMM64 = """
subgraphs:
  - id: gemm_64x64x64
    nodes: [{name: mm, kind: matmul, shape: {m: 64, k: 64, n: 64}}]
"""


def _gemm64():
    net = W.loads_network(GEMM64)
    sg = net.subgraphs[0]
    tg = W.TargetConfig(tiling_levels=2)
    ks = W.generate_sketches(sg, tg)
    S = max(k.space.num_tile_slots for k in ks)
    return sg, ks[0], SketchTables(sg, ks[0], tg, S)


def test_tiling_counts_and_order():
    assert SP.enumerate_tilings(1024, 4) == 286
    assert SP.enumerate_tilings(2, 2) == 2
    assert SP.enumerate_tilings(12, 2) == 6
    assert SP.enumerate_tilings(64, 2) == 7
    assert SP.enumerate_tilings(1, 3) == 1
    tl = SP.list_tilings(12, 2)
    assert len(tl) == 6 and all(a * b == 12 for a, b in tl)
    assert list(tl) == sorted(tl)
    assert SP.list_tilings(1024, 4)[0] == (1, 1, 1, 1024)


def test_smallest_prime_factor():
    for n, p in ((4, 2), (15, 3), (7, 7), (4096, 2), (2 * 3 * 7, 2),
                 (49, 7), (3 * 3 * 5, 3)):
        assert SP.smallest_prime_factor(n) == p == O.spf(n)


def test_space_size_gemm64():
    _, sk, _ = _gemm64()
    # 7 two-level tilings per dim, 4 unroll depths, parallel 0..2
    assert SP.space_size(sk) == 7 ** 3 * 4 * 3 * 1 == 4116


def _state(tb, tiles, ca=0, par=0, ur=0):
    t = np.asarray([v for d in tiles for v in d], np.uint16)[None, :]
    k = np.asarray([[ca, par, ur]], np.uint8)
    return t, k


def _act(tb, src, dst, dca=0, dpar=0, dur=0):
    S = tb.num_slots
    a0 = S * S if src < 0 else src * S + dst
    return np.asarray([[a0, dca + 1, dpar + 1, dur + 1]], np.int64)


def test_move_divides_by_smallest_prime():
    _, _, tb = _gemm64()
    t, k = _state(tb, ((4, 16), (2, 32), (4, 16)))
    nt, nk = O.apply_actions(tb, t, k, _act(tb, 0, 1), tb.num_slots)
    assert nt[0].tolist() == [2, 32, 2, 32, 4, 16]
    assert t[0].tolist() == [4, 16, 2, 32, 4, 16]


def test_noop_is_identity():
    _, _, tb = _gemm64()
    t, k = O.sample_initial(tb, 1, np.random.default_rng(1))
    cur_t, cur_k = t, k
    for _ in range(5):
        cur_t, cur_k = O.apply_actions(tb, cur_t, cur_k, _act(tb, -1, -1),
                                       tb.num_slots)
    assert np.array_equal(cur_t, t) and np.array_equal(cur_k, k)


@pytest.mark.parametrize("tiles,ur,act,sub", [
    (((1, 64), (2, 32), (4, 16)), 0, (0, 1, 0, 0, 0), "tiling"),
    (((8, 8), (2, 32), (4, 16)), 3, (-1, -1, -1, 0, 0), "compute_at"),
    (((8, 8), (2, 32), (4, 16)), 3, (-1, -1, 0, 0, 1), "unroll"),
    (((8, 8), (2, 32), (4, 16)), 0, (0, 2, 0, 0, 0), "tiling"),
])
def test_rejections(tiles, ur, act, sub):
    _, _, tb = _gemm64()
    t, k = _state(tb, tiles, ur=ur)
    with pytest.raises(O.OracleInvalidAction) as ei:
        O.apply_actions(tb, t, k, _act(tb, *act), tb.num_slots)
    assert ei.value.subspace == sub


def test_mask_boundaries_and_head_sizes():
    _, _, tb = _gemm64()
    S = tb.num_slots
    t, k = _state(tb, ((1, 64), (2, 32), (4, 16)), ca=0, par=0, ur=3)
    tiling, ca, par, ur = O.action_masks(tb, t, k, S)
    assert tiling.shape == (1, S * S + 1)     # head 0: S^2 + 1 columns
    assert ca.shape == par.shape == ur.shape == (1, 3)
    assert tiling[0, -1]                      # the dummy is always valid
    assert not tiling[0, 0 * S + 1]           # source factor 1
    assert tiling[0, 1 * S + 0]               # 32 can move within dim m
    assert not tiling[0, 1 * S + 2]           # never across dimensions
    assert ca[0].tolist() == [False, True, tb.ncas > 1]  # compute-at at 0
    assert ur[0].tolist() == [True, True, False]    # unroll at the top


def test_decode_layout():
    S = 6
    src, dst, dca, dpar, dur = O.decode(np.asarray([[2 * S + 5, 0, 1, 2],
                                                    [S * S, 2, 2, 0]]), S)
    assert (src.tolist(), dst.tolist()) == ([2, -1], [5, -1])
    assert (dca.tolist(), dpar.tolist(), dur.tolist()) == \
        ([-1, 1], [0, 1], [1, -1])


def test_untrained_and_single_example_gbt():
    X = np.random.default_rng(0).random((4, 7))
    assert O.GbtModel().predict(X).tolist() == [1.0] * 4
    base, trees, pred = O.gbt_fit(X[:1], np.asarray([0.8]))
    m = O.GbtModel(base=base, fitted=True, trees=trees)
    assert m.predict(X).tolist() == [0.8] * 4


# ---------------------------------------------------------------------------
# the same answers through the device kernels


@pytest.mark.gpu
def test_device_move_noop_and_rejections():
    import torch
    from paper_2211_11172_b200 import device as D
    from paper_2211_11172_b200.errors import InvalidActionError
    _, _, tb = _gemm64()
    dsk = D.DeviceSketch(tb)
    t, k = _state(tb, ((4, 16), (2, 32), (4, 16)))
    dt, dk = D.states_to_device(tb, t, k)
    out = D.apply_actions(dsk, dt, dk, 1, _act(tb, 0, 1))
    nt, _ = D.states_to_host(tb, out[0], out[1], 1)
    assert nt[0].tolist() == [2, 32, 2, 32, 4, 16]
    out = D.apply_actions(dsk, dt, dk, 1, _act(tb, -1, -1))
    nt, nk = D.states_to_host(tb, out[0], out[1], 1)
    assert np.array_equal(nt, t) and np.array_equal(nk, k)
    t, k = _state(tb, ((8, 8), (2, 32), (4, 16)), ur=3)
    dt, dk = D.states_to_device(tb, t, k)
    with pytest.raises(InvalidActionError) as ei:
        D.apply_actions(dsk, dt, dk, 1, _act(tb, -1, -1, 0, 0, 1))
    assert ei.value.subspace == "unroll"
    torch.cuda.synchronize()


@pytest.mark.gpu
def test_device_untrained_and_single_example_gbt():
    import torch
    from paper_2211_11172_b200 import device as D
    X = np.random.default_rng(0).random((4, 7))
    Xd = torch.from_numpy(X).cuda()
    f = D.DeviceForest([], 1.0, 0.3, fitted=False)
    assert D.gbt_predict(f, Xd, 4).cpu().numpy().tolist() == [1.0] * 4
    fit = D.gbt_fit(X[:1], np.asarray([0.8]))
    f = D.DeviceForest(fit.trees, fit.base, 0.3)
    assert D.gbt_predict(f, Xd, 4).cpu().numpy().tolist() == [0.8] * 4
