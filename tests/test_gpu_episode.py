"""Episode-level parity of the B200 engine against the reference.

* Golden replay: the engine runs each recorded reference episode with the
  reference's own action stream injected (and its culls, which depend on
  fp64 advantages); every visited state, feature vector, score and reward
  must be bit-identical to the fixture, the generator must end in the same
  state, networks/advantages/updated parameters within tolerance.
* Shadow replay: the engine samples its own actions on the shared PCG64
  stream; the oracle follows its decisions and checks each sampled index
  against its own fp64 CDF, plus all bit-exact and tolerance quantities.
* PPO: one device update against the oracle's on the same replay batch.
"""

import hashlib

import numpy as np
import pytest

from golden_util import GoldenCase, case_names, digest
from gpu_util import assert_close_rel, needs_gpu, all_sketch_tables, CONV
from oracle import harl_oracle as O

pytestmark = [pytest.mark.gpu, needs_gpu]
torch = pytest.importorskip("torch")

RL_CASES = [n for n in case_names() if GoldenCase(n).is_rl]


def _oracle_from(gc):
    agent = O.Agent.from_param_lists([p.copy() for p in gc.agent.policy],
                                     [p.copy() for p in gc.agent.value],
                                     len(gc.cfg["hidden"]))
    opt_pi = O.Adam.zeros_like(agent.policy_params(), gc.rl.lr_actor)
    opt_v = O.Adam.zeros_like(agent.value_params(), gc.rl.lr_critic)
    model = O.GbtModel(base=gc.model_base, learning_rate=gc.rec["model_lr"],
                       fitted=True, trees=gc.trees())
    rl = O.RlCfg(lr_actor=gc.rl.lr_actor, lr_critic=gc.rl.lr_critic,
                 discount=gc.rl.discount, clip_ratio=gc.rl.clip_ratio,
                 value_loss_weight=gc.rl.value_loss_weight,
                 entropy_weight=gc.rl.entropy_weight,
                 minibatch=gc.rl.minibatch,
                 buffer_capacity=gc.rl.buffer_capacity,
                 train_interval=gc.rl.train_interval)
    cfg = O.EpisodeCfg(tracks=gc.tracks, track_len=gc.track_len,
                       cull_window=gc.cfg["cull_window"] if gc.adaptive
                       else None, cull_fraction=gc.cfg["cull_fraction"],
                       min_tracks=gc.cfg["min_tracks"], rl=gc.is_rl,
                       adaptive=gc.adaptive, rl_cfg=rl)
    return agent, opt_pi, opt_v, model, cfg


def _engine_from(gc):
    from paper_2211_11172_b200 import device as D
    from paper_2211_11172_b200.engine import EpisodeConfig, EpisodeEngine
    eng = EpisodeEngine(gc.agent, gc.rl, gc.target.tiling_levels)
    forest = D.DeviceForest(gc.trees(), gc.model_base, gc.rec["model_lr"])
    cfg = EpisodeConfig.from_tuner(gc.cfg, gc.rec["searcher"])
    return eng, forest, cfg


def _flat(dagent, pol, val):
    return dagent._pack(pol, val)


@pytest.mark.parametrize("name", RL_CASES)
def test_golden_episode_replay(name):
    gc = GoldenCase(name)
    eng, forest, cfg = _engine_from(gc)
    o_agent, o_pi, o_v, model, ocfg = _oracle_from(gc)
    o_replay = O.Replay(gc.rl.buffer_capacity)
    order = 0
    for e_i, ep in enumerate(gc.rec["episodes"]):
        tb = gc.tables(ep["sketch"])
        # oracle run (bit-exact with the reference, tests/test_oracle_golden)
        o_trace = []
        o_entries, _, _ = O.run_episode(tb, gc.slots, ocfg, o_agent, o_pi, o_v,
                                        o_replay, model,
                                        gc.rng_from(ep["rng_state"]), order,
                                        trace=o_trace)
        o_steps = {t["step"]: t for t in o_trace if "step" in t}
        gen = gc.rng_from(ep["rng_state"])
        rec = []
        own_culls = {}

        def cull_override(t, own):
            own_culls[t] = own
            return o_steps[t]["cull"]

        res = eng.run_episode(tb, forest, gen, cfg, order,
                              inject=lambda t: o_steps[t]["actions"],
                              record=rec, cull_override=cull_override)
        # states / scores / rewards of every visit: bit-exact vs reference
        tiles, knobs = res.states()
        key = f"e{e_i}_entry_"
        np.testing.assert_array_equal(tiles, gc.arr[key + "tiles"])
        np.testing.assert_array_equal(knobs, gc.arr[key + "knobs"])
        assert res.scores().tobytes() == gc.arr[key + "score"].tobytes()
        canon = "\n".join(tb.canonical(t, k) for t, k in zip(tiles, knobs))
        assert hashlib.sha256(canon.encode()).hexdigest() == \
            ep["entries_canonical_digest"]
        assert res.visits == ep["entries_order"][2]
        for s_i, (r, st) in enumerate(zip(rec, ep["steps"]), start=1):
            k = f"e{e_i}_s{s_i}_"
            assert digest(r["X"].cpu().numpy()) == st["X"]
            assert r["rewards"].cpu().numpy().tobytes() == \
                gc.arr[k + "rewards"].tobytes()
            assert r["new_feats"].cpu().numpy().tobytes() == \
                o_steps[s_i]["new_feats"].tobytes()
            assert_close_rel(r["logp"].cpu().numpy(), gc.arr[k + "logp"],
                             what="logp")
            assert_close_rel(r["v_cur"].cpu().numpy(), gc.arr[k + "v_cur"],
                             what="v_cur")
            assert_close_rel(r["v_next"].cpu().numpy(), gc.arr[k + "v_next"],
                             what="v_next")
            assert_close_rel(r["adv"].cpu().numpy(), gc.arr[k + "adv"],
                             what="adv")
            if "ppo_idx" in o_steps[s_i]:
                np.testing.assert_array_equal(r["ppo_idx"],
                                              o_steps[s_i]["ppo_idx"])
        # own cull choice equals the reference's unless advantages tie
        for t, own in own_culls.items():
            ref = o_steps[t]["cull"]
            if not np.array_equal(own, ref):
                adv = o_steps[t]["adv"]
                sel = o_steps[t]["sel"]
                a = dict(zip(sel.tolist(), adv.tolist()))
                diff = set(own.tolist()) ^ set(ref.tolist())
                vals = [a[i] for i in diff]
                assert max(vals) - min(vals) < 1e-5, "cull differs, no tie"
        st = gen.bit_generator.state
        assert int(st["state"]["state"]) == \
            int(ep["end_rng_state"]["state"]["state"])
        assert st["has_uint32"] == ep["end_rng_state"]["has_uint32"]
        assert len(eng.replay) == ep["end_buffer_len"]
        # parameters after the episode's PPO updates vs the oracle's
        eng.sync_to_host()
        got = _flat(eng.dagent, gc.agent.policy, gc.agent.value)
        ref = _flat(eng.dagent, o_agent.policy_params(), o_agent.value_params())
        assert_close_rel(got, ref, tol=1e-4, what="params")
        assert gc.agent.opt_pi.t == ep["end_pi_t"]
        order += res.visits


@pytest.mark.parametrize("name", [n for n in case_names()
                                  if not GoldenCase(n).is_rl])
def test_golden_uniform_episode_bit_exact(name):
    """Evolutionary searcher: uniform valid actions drawn on device from the
    session generator (tuner.py:341-348) -- integer work end to end, so the
    whole episode is bit-identical to the reference's, no injection."""
    gc = GoldenCase(name)
    eng, forest, cfg = _engine_from(gc)
    order = 0
    for e_i, ep in enumerate(gc.rec["episodes"]):
        tb = gc.tables(ep["sketch"])
        gen = gc.rng_from(ep["rng_state"])
        rec = []
        res = eng.run_episode(tb, forest, gen, cfg, order, record=rec)
        for s_i, r in enumerate(rec, start=1):
            np.testing.assert_array_equal(
                r["actions"].cpu().numpy().T,
                gc.arr[f"e{e_i}_s{s_i}_actions"].astype(np.int64))
        tiles, knobs = res.states()
        key = f"e{e_i}_entry_"
        np.testing.assert_array_equal(tiles, gc.arr[key + "tiles"])
        np.testing.assert_array_equal(knobs, gc.arr[key + "knobs"])
        assert res.scores().tobytes() == gc.arr[key + "score"].tobytes()
        assert gen.bit_generator.state["state"]["state"] == \
            int(ep["end_rng_state"]["state"]["state"])
        assert gen.bit_generator.state["has_uint32"] == \
            ep["end_rng_state"]["has_uint32"]
        order += res.visits


@pytest.mark.parametrize("name", ["conv2d_l4", "bmm_softmax_k3",
                                  "gemm64_l2"])
def test_sampled_episode_shadow_replay(name):
    """The engine samples on the shared stream; the oracle replays its
    decisions and vouches for every draw."""
    gc = GoldenCase(name)
    eng, forest, cfg = _engine_from(gc)
    o_agent, o_pi, o_v, model, ocfg = _oracle_from(gc)
    o_replay = O.Replay(gc.rl.buffer_capacity)
    ep = gc.rec["episodes"][0]
    tb = gc.tables(ep["sketch"])
    gen = gc.rng_from(ep["rng_state"])
    rec = []
    res = eng.run_episode(tb, forest, gen, cfg, 0, record=rec)
    by_t = {r["t"]: r for r in rec}
    checked = {"draws": 0, "flips": 0}

    def follow(t, info):
        r = by_t[t]
        if info["phase"] == "act":
            return {"actions": r["actions"].cpu().numpy().T.astype(np.int64)}
        return {"cull": r.get("cull")}

    o_trace = []
    O.run_episode(tb, gc.slots, ocfg, o_agent, o_pi, o_v, o_replay, model,
                  gc.rng_from(ep["rng_state"]), 0, trace=o_trace,
                  follow=follow)
    for o in (t for t in o_trace if "step" in t):
        r = by_t[o["step"]]
        np.testing.assert_array_equal(r["sel"].cpu().numpy(), o["sel"])
        acts = o["actions"]
        for h, hd in enumerate(o["heads"]):
            c = np.cumsum(hd["p"], axis=1)
            for row in range(len(acts)):
                checked["draws"] += 1
                a = acts[row, h]
                if a == hd["a"][row]:
                    continue
                checked["flips"] += 1
                lo = c[row, a - 1] if a > 0 else 0.0
                assert hd["p"][row, a] > 0
                assert lo - 1e-5 <= hd["u"][row] <= c[row, a] + 1e-5
        assert r["new_feats"].cpu().numpy().tobytes() == \
            o["new_feats"].tobytes()
        assert r["new_score"].cpu().numpy().tobytes() == \
            o["new_score"].tobytes()
        assert r["rewards"].cpu().numpy().tobytes() == o["rewards"].tobytes()
        assert_close_rel(r["logp"].cpu().numpy(), o["logp"], what="logp")
        assert_close_rel(r["adv"].cpu().numpy(), o["adv"], what="adv")
        if "ppo_idx" in o:
            np.testing.assert_array_equal(r["ppo_idx"], o["ppo_idx"])
    assert checked["flips"] <= max(2, checked["draws"] // 1000)
    eng.sync_to_host()
    got = _flat(eng.dagent, gc.agent.policy, gc.agent.value)
    ref = _flat(eng.dagent, o_agent.policy_params(), o_agent.value_params())
    assert_close_rel(got, ref, tol=1e-4, what="params")


@pytest.mark.parametrize("hidden", [(16,), (32, 32), (128, 128)])
def test_ppo_update_matches_oracle(hidden):
    from paper_2211_11172_b200 import device as D
    from paper_2211_11172_b200.agent import RlConfig, init_session_agents
    sg, sk, tb = all_sketch_tables(CONV)[0]
    cfg = RlConfig(hidden=hidden, minibatch=256, buffer_capacity=1024)
    agent = init_session_agents([("sg", tb.num_slots)], tb.feature_len, cfg,
                                np.random.default_rng(0))["sg"]
    rng = np.random.default_rng(1)
    for p in agent.policy + agent.value:
        p += 0.2 * rng.standard_normal(p.shape) * (p.std() + 0.05)
    oa = O.Agent.from_param_lists([p.copy() for p in agent.policy],
                                  [p.copy() for p in agent.value],
                                  len(hidden))
    # transitions from an oracle rollout of 700 states
    tiles, knobs = O.sample_initial(tb, 700, np.random.default_rng(2))
    X = O.featurize(tb, tiles, knobs)
    masks = O.action_masks(tb, tiles, knobs, tb.num_slots)
    acts, logp = O.select_actions(oa, X, masks, np.random.default_rng(3))
    nt, nk = O.apply_actions(tb, tiles, knobs, acts, tb.num_slots)
    Xn = O.featurize(tb, nt, nk)
    rew = rng.standard_normal(700) * 0.1
    vn, _ = oa.value(Xn)
    vc, _ = oa.value(X)
    adv = rew + 0.9 * vn - vc
    td = rew + 0.9 * vn
    replay = O.Replay(1024)
    replay.push_rows(X, Xn, acts, logp + 1e-3 * rng.standard_normal(700),
                     rew, adv, td, masks)
    ring = D.DeviceReplay(1024, tb.feature_len)
    items = list(replay.items)
    ring.load(np.stack([i[0] for i in items]), np.stack([i[1] for i in items]),
              np.stack([i[2] for i in items]), [i[3] for i in items],
              [i[4] for i in items], [i[5] for i in items],
              [i[6] for i in items],
              [np.stack([i[7][h] for i in items]) for h in range(4)],
              tb.num_slots, tb.levels)
    dag = D.DeviceAgent(agent, tb.levels)
    o_pi = O.Adam.zeros_like(oa.policy_params(), cfg.lr_actor)
    o_v = O.Adam.zeros_like(oa.value_params(), cfg.lr_critic)
    ocfg = O.RlCfg(minibatch=256, buffer_capacity=1024)
    for step in range(1, 4):
        g = np.random.default_rng(10 + step)
        batch, idx = replay.sample(g, 256)
        o_loss = O.ppo_update(oa, o_pi, o_v, batch, ocfg)
        slots = torch.from_numpy(ring.slots_of(idx)).cuda()
        losses = dag.ppo_update(ring, slots, cfg, step, step).cpu().numpy()
        assert int(dag.bad.item()) == 0
        assert_close_rel(losses[:5], [o_loss["actor_loss"],
                                      o_loss["value_loss"],
                                      o_loss["policy_loss"],
                                      o_loss["entropy"],
                                      o_loss["mean_ratio"]], what="losses")
    dag.download()
    got = dag._pack(agent.policy, agent.value)
    ref = dag._pack(oa.policy_params(), oa.value_params())
    assert_close_rel(got, ref, tol=1e-6, what="params")
    gm = dag._pack(agent.opt_pi.m, agent.opt_v.m)
    rm = dag._pack(o_pi.m, o_v.m)
    assert_close_rel(gm, rm, tol=1e-4, what="adam m")
    # the ring round-trips to the reference's transition layout
    exp = ring.export(tb.num_slots, tb.levels)
    np.testing.assert_array_equal(exp["actions"], np.stack([i[2] for i in items]))
    for h in range(4):
        np.testing.assert_array_equal(exp["masks"][h],
                                      np.stack([i[7][h] for i in items]))
