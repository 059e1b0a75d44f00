"""The CUDA-graph episode path is the eager launch sequence, replayed: on
identical inputs it must produce bit-identical episodes (every kernel is
deterministic), across several consecutive episodes (tables refilled, graphs
reused) and for both kernel families (tcgen05 at hidden (128,128), FFMA
otherwise)."""

import copy

import numpy as np
import pytest

from gpu_util import CONV, BMM_SOFTMAX, all_sketch_tables, needs_gpu

pytestmark = [pytest.mark.gpu, needs_gpu]
torch = pytest.importorskip("torch")


def _setup(hidden, which):
    import bench
    from paper_2211_11172_b200 import device as D
    from paper_2211_11172_b200.agent import RlConfig, init_session_agents
    from paper_2211_11172_b200.engine import EpisodeConfig, EpisodeEngine
    text = CONV if which == "conv" else BMM_SOFTMAX
    tabs = all_sketch_tables(text)
    sg, sk, tb = tabs[0] if which == "conv" else tabs[3]
    rl = RlConfig(hidden=hidden, minibatch=64, buffer_capacity=512)
    agent = init_session_agents([("sg", tb.num_slots)], tb.feature_len, rl,
                                np.random.default_rng(0))["sg"]
    forest = D.DeviceForest(bench.synthetic_forest(tb, 1), 0.5, 0.3)
    cfg = EpisodeConfig(tracks=600, track_len=6, cull_window=3,
                        cull_fraction=0.5, min_tracks=300)
    engines = []
    for graphs in (False, True):
        eng = EpisodeEngine(copy.deepcopy(agent), rl, tb.levels,
                            use_graphs=graphs)
        engines.append(eng)
    return tb, forest, cfg, engines


@pytest.fixture(autouse=True)
def _capture_first_use(monkeypatch):
    """Capture on a plan's first episode so every episode here replays
    graphs (the default runs a plan's first episode eagerly)."""
    from paper_2211_11172_b200 import engine as E
    monkeypatch.setattr(E, "_LAZY_CAPTURE", False)


@pytest.mark.parametrize("hidden,which", [((128, 128), "conv"),
                                          ((32, 32), "bmm")])
@pytest.mark.parametrize("lazy", [False, True])
def test_graph_replay_is_bit_identical(monkeypatch, hidden, which, lazy):
    from paper_2211_11172_b200 import engine as E
    monkeypatch.setattr(E, "_LAZY_CAPTURE", lazy)
    tb, forest, cfg, (eager, graphed) = _setup(hidden, which)
    g1, g2 = np.random.default_rng(5), np.random.default_rng(5)
    for ep in range(4 if lazy else 3):
        r1 = eager.run_episode(tb, forest, g1, cfg, 0)
        out1 = (r1.states(), r1.scores().copy(),
                r1.log_reward[:r1.visits].cpu().numpy().copy(),
                [c[1].copy() for c in r1.culls],
                [t[1].cpu().numpy().copy() for t in r1.train])
        r2 = graphed.run_episode(tb, forest, g2, cfg, 0)
        # graphs are used on the tcgen05 path only; lazily, from a plan's
        # second episode (the first episode's plan differs: empty replay)
        if graphed.dagent.tc and (not lazy or ep >= 2):
            assert any(b.graphs for b in graphed._cache.values())
        np.testing.assert_array_equal(r2.states()[0], out1[0][0])
        np.testing.assert_array_equal(r2.states()[1], out1[0][1])
        assert r2.scores().tobytes() == out1[1].tobytes()
        assert r2.log_reward[:r2.visits].cpu().numpy().tobytes() == \
            out1[2].tobytes()
        for a, b in zip([c[1] for c in r2.culls], out1[3]):
            np.testing.assert_array_equal(a, b)
        for a, b in zip([t[1].cpu().numpy() for t in r2.train], out1[4]):
            assert a.tobytes() == b.tobytes()
        assert g1.bit_generator.state == g2.bit_generator.state
        assert eager.agent.opt_pi.t == graphed.agent.opt_pi.t
        assert eager.replay.wpos == graphed.replay.wpos
        assert torch.equal(eager.dagent.params, graphed.dagent.params)
        assert torch.equal(eager.dagent.m, graphed.dagent.m)
        assert torch.equal(eager.replay.X, graphed.replay.X)


@pytest.mark.parametrize("flag", ["_FUSED_STEP", "_SPLIT_FEATURIZE",
                                  "_SPLIT_FINISH", "_PAR_VALUE",
                                  "_SAMPLE_GBT", "_VALUE_FINISH",
                                  "_OVERLAP_POLICY"])
def test_kernel_fusion_variants_match_default(monkeypatch, flag):
    """Each alternative launch structure produces the default episode bit
    for bit: _FUSED_STEP (k_policy_step_fused: the 3xTF32 policy -> sample/
    apply -> featurize in one kernel, against the 3xTF32 default), _SPLIT_FEATURIZE (k_featurize2 launched after
    the sampler instead of inside it), _SPLIT_FINISH (k_gbt_predict2 +
    k_finish_step instead of the fused k_gbt_finish), _PAR_VALUE (the value
    pass on a forked stream beside the GBT pass, joined by the finish),
    _SAMPLE_GBT (the cost model inside the sampler, k_sample_gbt, then a
    finish-only launch, against the separate k_gbt_finish), _VALUE_FINISH
    (with the sampler-side cost model: the finish in the value kernel's
    epilogue, harl_value_finish_tc, against the finish launch),
    _OVERLAP_POLICY (the next step's policy network on a forked stream
    beside the value and GBT passes, against strictly sequential launches)."""
    from paper_2211_11172_b200 import engine as E
    if flag == "_VALUE_FINISH":   # needs the scores from the sampler
        monkeypatch.setattr(E, "_SAMPLE_GBT", True)
    if flag == "_FUSED_STEP":
        # the fused kernel is the 3xTF32 policy: compare with that default
        monkeypatch.setenv("HARL_TC16", "0")
    tb, forest, cfg, (_, dflt) = _setup((128, 128), "conv")
    _, _, _, (_, alt) = _setup((128, 128), "conv")
    g1, g2 = np.random.default_rng(9), np.random.default_rng(9)
    for ep in range(2):
        monkeypatch.setattr(E, flag, False)
        r1 = dflt.run_episode(tb, forest, g1, cfg, 0)
        s1, sc1 = r1.states(), r1.scores().copy()
        rw1 = r1.log_reward[:r1.visits].cpu().numpy().copy()
        monkeypatch.setattr(E, flag, True)
        r2 = alt.run_episode(tb, forest, g2, cfg, 0)
        np.testing.assert_array_equal(r2.states()[0], s1[0])
        np.testing.assert_array_equal(r2.states()[1], s1[1])
        assert r2.scores().tobytes() == sc1.tobytes()
        assert r2.log_reward[:r2.visits].cpu().numpy().tobytes() == \
            rw1.tobytes()
        assert torch.equal(dflt.dagent.params, alt.dagent.params)
        assert torch.equal(dflt.replay.X, alt.replay.X)
        assert torch.equal(dflt.replay.Xn, alt.replay.Xn)
        assert g1.bit_generator.state == g2.bit_generator.state



@pytest.mark.parametrize("env", [("HARL_PPO_FUSED_ADAM", "1", "0"),
                                 ("HARL_PPO_SPEC", "0", "1")])
def test_fused_wgrad_adam_matches_separate_launches(env):
    """HARL_PPO_FUSED_ADAM=1 (gradients + Adam in one cooperative kernel
    with a grid barrier) and the default speculative single launch
    (k_ppo_wgrad_spec, HARL_PPO_SPEC=0 disables it) leave the same
    parameters, moments, replay ring and scores as the two launches, bit
    for bit."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    script = os.path.join(here, "_episode_digest.py")
    out = []
    name, on, off = env
    for flag in (off, on):
        env_ = dict(os.environ, HARL_PPO_SPEC="0") \
            if name == "HARL_PPO_FUSED_ADAM" else dict(os.environ)
        env_[name] = flag
        r = subprocess.run([sys.executable, script], env=env_, text=True,
                           capture_output=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        out.append(r.stdout.strip().splitlines()[-1])
    assert out[0] == out[1]


def test_graphs_survive_scratch_growth():
    """Captured graphs of one geometry keep working after another geometry
    grows the engine-wide scratch (the policy logits scratch, the PPO
    scratch): the replaced buffers are retired, not freed, so replaying the
    first geometry's graphs again matches the eager engine bit for bit."""
    from paper_2211_11172_b200.engine import EpisodeConfig
    tb, forest, small, (eager, graphed) = _setup((128, 128), "conv")
    big = EpisodeConfig(tracks=2400, track_len=4, cull_window=2,
                        cull_fraction=0.5, min_tracks=1200)
    g1, g2 = np.random.default_rng(3), np.random.default_rng(3)
    for cfg in (small, small, big, big, small, small):
        r1 = eager.run_episode(tb, forest, g1, cfg, 0)
        s1, sc1 = r1.states(), r1.scores().copy()
        r2 = graphed.run_episode(tb, forest, g2, cfg, 0)
        # churn the caching allocator: freed blocks would be handed out now
        junk = [torch.full((1 << 20,), 7.0, device="cuda") for _ in range(8)]
        np.testing.assert_array_equal(r2.states()[0], s1[0])
        assert r2.scores().tobytes() == sc1.tobytes()
        assert torch.equal(eager.dagent.params, graphed.dagent.params)
        del junk
    assert graphed.dagent._retired, "scratch never grew: test is vacuous"
