"""Per-operator parity of the CUDA path (through the C ABI) against the
oracle: bit-exact for the integer/fp64 operators (initial sampling, masks,
walker, features, GBT scores, rewards), within the north-star tolerance for
the fp32 networks."""

import math

import numpy as np
import pytest

from gpu_util import (REL_TOL, all_sketch_tables, assert_close_rel,
                      config_tables, needs_gpu, GEMM)
from oracle import harl_oracle as O

pytestmark = [pytest.mark.gpu, needs_gpu]

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def D():
    from paper_2211_11172_b200 import device
    return device


def _random_states(tb, n, seed):
    return O.sample_initial(tb, n, np.random.default_rng(seed))


def _walk(tb, S, tiles, knobs, steps, seed):
    """Random legal walk (oracle) to reach varied, non-uniform states."""
    rng = np.random.default_rng(seed)
    for _ in range(steps):
        masks = O.action_masks(tb, tiles, knobs, S)
        acts = np.zeros((len(tiles), 4), np.int64)
        for h, mk in enumerate(masks):
            for r in range(len(tiles)):
                acts[r, h] = rng.choice(np.flatnonzero(mk[r]))
        tiles, knobs = O.apply_actions(tb, tiles, knobs, acts, S)
    return tiles, knobs


@pytest.mark.parametrize("case", range(len(config_tables())))
def test_init_population_matches_generator_stream(D, case):
    sg, sk, tb = config_tables()[case]
    for seed, n in ((0, 1), (1, 777), (2, 20000)):
        g_ref = np.random.default_rng(seed)
        g_ref.integers(3)  # leave a buffered 32-bit half behind
        g_dev = np.random.default_rng(seed)
        g_dev.integers(3)
        t_ref, k_ref = O.sample_initial(tb, n, g_ref)
        dsk = D.DeviceSketch(tb)
        tiles, knobs = D.init_population(dsk, n, g_dev)
        t_dev, k_dev = D.states_to_host(tb, tiles, knobs, n)
        np.testing.assert_array_equal(t_dev, t_ref)
        np.testing.assert_array_equal(k_dev, k_ref)
        assert g_dev.bit_generator.state == g_ref.bit_generator.state


def test_init_population_rejection_path(D):
    """Seed 7 at 200K tracks of GEMM-4096 hits Lemire's rare rejection
    branch (found by scanning seeds on the host)."""
    sg, sk, tb = all_sketch_tables(GEMM % (4096, 4096, 4096, 4096))[0]
    n = 200_000
    g_ref, g_dev = np.random.default_rng(7), np.random.default_rng(7)
    t_ref, k_ref = O.sample_initial(tb, n, g_ref)
    from paper_2211_11172_b200 import rng as R
    probe = np.random.default_rng(7)
    R.skip_u32(probe, 5 * n)
    assert probe.bit_generator.state != g_ref.bit_generator.state
    dsk = D.DeviceSketch(tb)
    tiles, knobs = D.init_population(dsk, n, g_dev)
    t_dev, k_dev = D.states_to_host(tb, tiles, knobs, n)
    np.testing.assert_array_equal(t_dev, t_ref)
    np.testing.assert_array_equal(k_dev, k_ref)
    assert g_dev.bit_generator.state == g_ref.bit_generator.state


@pytest.mark.parametrize("case", range(len(config_tables())))
def test_featurize_bit_exact(D, case):
    sg, sk, tb = config_tables()[case]
    tiles, knobs = _random_states(tb, 3000, case)
    tiles, knobs = _walk(tb, tb.num_slots, tiles[:200], knobs[:200], 6, case) \
        if case % 2 else (tiles, knobs)
    ref = O.featurize(tb, tiles, knobs)
    dsk = D.DeviceSketch(tb)
    dt, dk = D.states_to_device(tb, tiles, knobs)
    got = D.featurize(dsk, dt, dk, len(tiles)).cpu().numpy()
    assert got.tobytes() == ref.tobytes()


def test_featurize_exhaustive_gemm64(D):
    """All 4116 states of the reference's oracle-scale space
    (tests/test_schedspace.py:137-146)."""
    from paper_2211_11172_b200 import workloads as W
    from paper_2211_11172_b200.space import list_tilings
    import itertools
    sg, sk, tb = all_sketch_tables(GEMM % (64, 64, 64, 64),
                                   W.TargetConfig(tiling_levels=2))[0]
    tl = list_tilings(64, 2)
    rows, kn = [], []
    for combo in itertools.product(tl, tl, tl):
        for par in range(tb.max_fusible + 1):
            for ur in range(tb.n_unroll):
                rows.append([f for t in combo for f in t])
                kn.append([0, par, ur])
    tiles = np.asarray(rows, np.uint16)
    knobs = np.asarray(kn, np.uint8)
    assert len(tiles) == 4116
    dsk = D.DeviceSketch(tb)
    dt, dk = D.states_to_device(tb, tiles, knobs)
    got = D.featurize(dsk, dt, dk, len(tiles)).cpu().numpy()
    assert got.tobytes() == O.featurize(tb, tiles, knobs).tobytes()
    assert len({r.tobytes() for r in got}) == 4116


def test_featurize_log10_sweep(D):
    """glibc-faithful log10 over a wide sweep of footprint values: states
    whose footprints cover 1..10^12 (via a 1-D reduction with a huge
    extent split every way)."""
    from paper_2211_11172_b200 import workloads as W
    text = """
subgraphs:
  - id: red
    nodes: [{name: r, kind: reduction, shape: {a: 60060, b: 55440}}]
"""
    sg, sk, tb = all_sketch_tables(text)[0]
    tiles, knobs = _random_states(tb, 50000, 3)
    ref = O.featurize(tb, tiles, knobs)
    dsk = D.DeviceSketch(tb)
    dt, dk = D.states_to_device(tb, tiles, knobs)
    got = D.featurize(dsk, dt, dk, len(tiles)).cpu().numpy()
    assert got.tobytes() == ref.tobytes()


@pytest.mark.parametrize("case", range(len(config_tables())))
def test_action_masks_match(D, case):
    sg, sk, tb = config_tables()[case]
    tiles, knobs = _random_states(tb, 500, case)
    tiles, knobs = _walk(tb, tb.num_slots, tiles, knobs, 3, case)
    ref = O.action_masks(tb, tiles, knobs, tb.num_slots)
    dsk = D.DeviceSketch(tb)
    dt, dk = D.states_to_device(tb, tiles, knobs)
    got = D.action_masks(dsk, dt, dk, len(tiles))
    for g, r in zip(got, ref):
        np.testing.assert_array_equal(g.cpu().numpy(), r)


@pytest.mark.parametrize("case", range(len(config_tables())))
def test_apply_actions_bit_exact(D, case):
    sg, sk, tb = config_tables()[case]
    S = tb.num_slots
    tiles, knobs = _random_states(tb, 400, case + 100)
    masks = O.action_masks(tb, tiles, knobs, S)
    rng = np.random.default_rng(case)
    acts = np.zeros((len(tiles), 4), np.int64)
    for h, mk in enumerate(masks):
        for r in range(len(tiles)):
            acts[r, h] = rng.choice(np.flatnonzero(mk[r]))
    rt, rk = O.apply_actions(tb, tiles, knobs, acts, S)
    dsk = D.DeviceSketch(tb)
    dt, dk = D.states_to_device(tb, tiles, knobs)
    ot, ok = D.apply_actions(dsk, dt, dk, len(tiles), acts)
    gt, gk = D.states_to_host(tb, ot, ok, len(tiles))
    np.testing.assert_array_equal(gt, rt)
    np.testing.assert_array_equal(gk, rk)


def test_apply_actions_rejections_match_reference_order(D):
    """tests/test_schedspace.py:246-269: unit-factor source, masked deltas;
    the first failing row raises with its subspace."""
    from paper_2211_11172_b200 import workloads as W
    from paper_2211_11172_b200.errors import InvalidActionError
    sg, sk, tb = all_sketch_tables(GEMM % (64, 64, 64, 64),
                                   W.TargetConfig(tiling_levels=2))[0]
    S = tb.num_slots
    tiles = np.asarray([[8, 8, 2, 32, 4, 16], [1, 64, 2, 32, 4, 16],
                        [8, 8, 2, 32, 4, 16]], np.uint16)
    knobs = np.asarray([[0, 0, 3], [0, 0, 0], [0, 0, 3]], np.uint8)
    dsk = D.DeviceSketch(tb)
    dt, dk = D.states_to_device(tb, tiles, knobs)
    noop = S * S
    cases = [
        ([[noop, 1, 1, 1], [0 * S + 1, 1, 1, 1], [noop, 1, 1, 1]], "tiling"),
        ([[noop, 1, 1, 2], [noop, 1, 1, 1], [noop, 1, 1, 1]], "unroll"),
        ([[noop, 1, 1, 1], [noop, 0, 1, 1], [noop, 1, 1, 2]], "compute_at"),
        ([[0 * S + 2, 1, 1, 1], [noop, 1, 1, 1], [noop, 1, 1, 1]], "tiling"),
        ([[noop, 1, 0, 1], [noop, 1, 1, 1], [noop, 1, 1, 1]], "parallel"),
    ]
    for acts, sub in cases:
        with pytest.raises(InvalidActionError) as ei:
            D.apply_actions(dsk, dt, dk, 3, np.asarray(acts))
        assert ei.value.subspace == sub
        with pytest.raises(O.OracleInvalidAction) as eo:
            O.apply_actions(tb, tiles, knobs, np.asarray(acts), S)
        assert eo.value.subspace == sub


def test_apply_move_divides_smallest_prime(D):
    """tests/test_schedspace.py:222-232: (4,16) -> (2,32)."""
    from paper_2211_11172_b200 import workloads as W
    sg, sk, tb = all_sketch_tables(GEMM % (64, 64, 64, 64),
                                   W.TargetConfig(tiling_levels=2))[0]
    S = tb.num_slots
    tiles = np.asarray([[4, 16, 2, 32, 4, 16]], np.uint16)
    knobs = np.zeros((1, 3), np.uint8)
    dsk = D.DeviceSketch(tb)
    dt, dk = D.states_to_device(tb, tiles, knobs)
    ot, ok = D.apply_actions(dsk, dt, dk, 1, np.asarray([[0 * S + 1, 1, 1, 1]]))
    gt, _ = D.states_to_host(tb, ot, ok, 1)
    assert gt.tolist() == [[2, 32, 2, 32, 4, 16]]


def _golden_forest(D, name):
    from golden_util import GoldenCase
    gc = GoldenCase(name)
    model = O.GbtModel(base=gc.model_base, learning_rate=gc.rec["model_lr"],
                       fitted=True, trees=gc.trees())
    forest = D.DeviceForest(gc.trees(), gc.model_base, gc.rec["model_lr"])
    return gc, model, forest


@pytest.mark.parametrize("name", ["gemm64_l2", "conv2d_l4", "bmm_softmax_k3",
                                  "gpu_gemm1024"])
def test_gbt_predict_and_reward_bit_exact(D, name):
    gc, model, forest = _golden_forest(D, name)
    tb = gc.tables(0)
    tiles, knobs = _random_states(tb, 30000, 5)
    X = O.featurize(tb, tiles, knobs)
    ref = model.predict(X)
    old = np.roll(ref, 1)
    Xd = torch.from_numpy(X).cuda()
    got, rew = D.gbt_predict(forest, Xd, len(X),
                             old_score=torch.from_numpy(old).cuda())
    assert got.cpu().numpy().tobytes() == ref.tobytes()
    assert rew.cpu().numpy().tobytes() == ((ref - old) / old).tobytes()


def test_gbt_untrained_and_floor(D):
    """costmodel.py:219-230: untrained -> 1.0; floor at 1e-6
    (tests/test_costmodel.py:40-45,95-103)."""
    X = torch.zeros((10, 49), dtype=torch.float64, device="cuda")
    f0 = D.DeviceForest([], 1.0, 0.3, fitted=False)
    assert D.gbt_predict(f0, X, 10).cpu().numpy().tolist() == [1.0] * 10
    tree = (np.asarray([-1]), np.asarray([0.0]), np.asarray([-1]),
            np.asarray([-1]), np.asarray([-10.0]))
    f1 = D.DeviceForest([tree], 0.5, 0.3)
    ref = O.GbtModel(0.5, 0.3, True, [tree]).predict(np.zeros((10, 49)))
    assert D.gbt_predict(f1, X, 10).cpu().numpy().tolist() == ref.tolist()
    assert ref[0] == 1e-6


# ---------------------------------------------------------------------------
# networks


def _agent(hidden, tb, seed=0):
    from paper_2211_11172_b200.agent import RlConfig, init_session_agents
    cfg = RlConfig(hidden=hidden)
    return init_session_agents([("sg", tb.num_slots)], tb.feature_len, cfg,
                               np.random.default_rng(seed))["sg"], cfg


def _oracle_agent(a):
    return O.Agent.from_param_lists(a.policy, a.value, len(a.hidden))


def _perturb(agent, seed, scale=0.3):
    """Larger head weights than the 0.01 init so softmaxes are not flat."""
    rng = np.random.default_rng(seed)
    for p in agent.policy + agent.value:
        p += scale * rng.standard_normal(p.shape) * (p.std() + 0.05)


@pytest.mark.parametrize("hidden", [(16,), (32, 32), (128, 128)])
@pytest.mark.parametrize("which", ["conv", "bmm3", "gemm"])
def test_policy_logits_logp_and_sampling(D, hidden, which):
    from paper_2211_11172_b200 import workloads as W
    from gpu_util import BMM_SOFTMAX, CONV
    text = {"conv": CONV, "bmm3": BMM_SOFTMAX,
            "gemm": GEMM % (1024, 1024, 1024, 1024)}[which]
    tabs = all_sketch_tables(text)
    sg, sk, tb = tabs[3] if which == "bmm3" else tabs[0]
    agent, _ = _agent(hidden, tb)
    _perturb(agent, 1)
    oa = _oracle_agent(agent)
    tiles, knobs = _random_states(tb, 4096, 11)
    tiles, knobs = _walk(tb, tb.num_slots, tiles[:1500], knobs[:1500], 2, 4)
    n = len(tiles)
    X = O.featurize(tb, tiles, knobs)
    masks = O.action_masks(tb, tiles, knobs, tb.num_slots)
    logits_ref, _ = oa.policy_forward(X)
    dsk = D.DeviceSketch(tb)
    dag = D.DeviceAgent(agent, tb.levels)
    dt, dk = D.states_to_device(tb, tiles, knobs)
    Xd = torch.from_numpy(X).cuda()
    g_ref = np.random.default_rng(99)
    g_dev = np.random.default_rng(99)
    rec = []
    acts_ref, logp_ref = O.select_actions(oa, X, masks, g_ref, record=rec)
    out = D.policy_step(dsk, dag, Xd, dt, dk, n, gen=g_dev, want_logits=True)
    D.raise_status(int(out["status"].item()) & ((1 << 64) - 1))
    assert g_dev.bit_generator.state == g_ref.bit_generator.state
    lg = out["logits"].cpu().numpy()
    cols = dsk.head_cols
    assert_close_rel(lg[:, :len(cols)], logits_ref[0][:, cols], what="head0")
    for h in range(3):
        assert_close_rel(lg[:, len(cols) + 3 * h:len(cols) + 3 * h + 3],
                         logits_ref[h + 1], what=f"head{h + 1}")
    acts = out["actions"][:, :n].cpu().numpy().T
    # every device draw is the oracle's unless u sits within float
    # distance of a CDF boundary
    flips = 0
    for h in range(4):
        p, u = rec[h]["p"], rec[h]["u"]
        c = np.cumsum(p, axis=1)
        for r in np.flatnonzero(acts[:, h] != acts_ref[:, h]):
            flips += 1
            a = acts[r, h]
            lo = c[r, a - 1] if a > 0 else 0.0
            assert p[r, a] > 0
            assert lo - 1e-5 <= u[r] <= c[r, a] + 1e-5
    assert flips <= max(2, n * 4 // 1000)
    # logp of the device's own actions vs the oracle's masked log-softmax
    lp_ref = np.zeros(n)
    for h in range(4):
        lp, _ = O.masked_log_softmax(logits_ref[h], masks[h])
        lp_ref += lp[np.arange(n), acts[:, h]]
    assert_close_rel(out["logp"][:n].cpu().numpy(), lp_ref, what="logp")
    # the walker applied exactly the sampled actions
    rt, rk = O.apply_actions(tb, tiles, knobs, acts, tb.num_slots)
    gt, gk = D.states_to_host(tb, out["tiles"], out["knobs"], n)
    np.testing.assert_array_equal(gt, rt)
    np.testing.assert_array_equal(gk, rk)


@pytest.mark.parametrize("hidden", [(16,), (32, 32), (128, 128)])
def test_policy_injected_actions(D, hidden):
    from gpu_util import CONV
    sg, sk, tb = all_sketch_tables(CONV)[1]
    agent, _ = _agent(hidden, tb, 3)
    _perturb(agent, 2)
    oa = _oracle_agent(agent)
    tiles, knobs = _random_states(tb, 2000, 12)
    X = O.featurize(tb, tiles, knobs)
    masks = O.action_masks(tb, tiles, knobs, tb.num_slots)
    acts, logp = O.select_actions(oa, X, masks, np.random.default_rng(5))
    dsk = D.DeviceSketch(tb)
    dag = D.DeviceAgent(agent, tb.levels)
    dt, dk = D.states_to_device(tb, tiles, knobs)
    out = D.policy_step(dsk, dag, torch.from_numpy(X).cuda(), dt, dk,
                        len(X), inject=acts)
    D.raise_status(int(out["status"].item()) & ((1 << 64) - 1))
    np.testing.assert_array_equal(out["actions"][:, :len(X)].cpu().numpy().T,
                                  acts)
    assert_close_rel(out["logp"][:len(X)].cpu().numpy(), logp, what="logp")
    rt, rk = O.apply_actions(tb, tiles, knobs, acts, tb.num_slots)
    gt, gk = D.states_to_host(tb, out["tiles"], out["knobs"], len(X))
    np.testing.assert_array_equal(gt, rt)
    np.testing.assert_array_equal(gk, rk)


@pytest.mark.parametrize("hidden", [(16,), (32, 32), (128, 128)])
def test_value_estimate(D, hidden):
    from gpu_util import BMM_SOFTMAX
    sg, sk, tb = all_sketch_tables(BMM_SOFTMAX)[3]
    agent, _ = _agent(hidden, tb, 4)
    _perturb(agent, 3)
    oa = _oracle_agent(agent)
    tiles, knobs = _random_states(tb, 5000, 13)
    X = O.featurize(tb, tiles, knobs)
    ref, _ = oa.value(X)
    dag = D.DeviceAgent(agent, tb.levels)
    got = D.value_estimate(dag, torch.from_numpy(X).cuda(), len(X))
    assert_close_rel(got.cpu().numpy(), ref, what="value")
