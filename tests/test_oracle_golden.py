"""Pin the oracle to the reference: replay every recorded golden episode and
require bit-identical results (digests of every per-step array, the
entries, the updated parameters and the generator state)."""

import hashlib

import numpy as np
import pytest

from golden_util import GoldenCase, case_names, digest, digest_list
from oracle import harl_oracle as O


def _oracle_setup(gc: GoldenCase):
    agent = O.Agent.from_param_lists(gc.agent.policy, gc.agent.value,
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
                       else None,
                       cull_fraction=gc.cfg["cull_fraction"],
                       min_tracks=gc.cfg["min_tracks"], rl=gc.is_rl,
                       adaptive=gc.adaptive, rl_cfg=rl)
    return agent, opt_pi, opt_v, model, cfg


@pytest.mark.parametrize("name", case_names())
def test_oracle_reproduces_reference_episodes(name):
    gc = GoldenCase(name)
    assert digest_list(gc.agent.policy) == gc.rec["init_policy_digest"]
    assert digest_list(gc.agent.value) == gc.rec["init_value_digest"]
    agent, opt_pi, opt_v, model, cfg = _oracle_setup(gc)
    replay = O.Replay(gc.rl.buffer_capacity)
    order = 0
    for e_i, ep in enumerate(gc.rec["episodes"]):
        assert ep["order_counter"] == order
        assert ep["buffer_len"] == len(replay)
        assert digest_list(agent.policy_params()) == ep["policy_digest"]
        tb = gc.tables(ep["sketch"])
        rng = gc.rng_from(ep["rng_state"])
        trace = []
        entries, order, summary = O.run_episode(
            tb, gc.slots, cfg, agent, opt_pi, opt_v, replay, model, rng,
            order, trace=trace)
        steps = [t for t in trace if "step" in t]
        assert len(steps) == len(ep["steps"])
        for s_i, (mine, ref) in enumerate(zip(steps, ep["steps"]), start=1):
            key = f"e{e_i}_s{s_i}_"
            assert len(mine["sel"]) == ref["m"]
            np.testing.assert_array_equal(
                mine["actions"], gc.arr[key + "actions"].astype(np.int64))
            assert digest_list(mine["masks"]) == ref["masks"]
            if gc.is_rl:
                assert digest(mine["X"]) == ref["X"]
                np.testing.assert_array_equal(mine["logp"],
                                              gc.arr[key + "logp"])
                for k in ("rewards", "v_next", "v_cur", "adv"):
                    np.testing.assert_array_equal(mine[k], gc.arr[key + k])
            if "ppo" in ref:
                assert mine["ppo"] == pytest.approx(ref["ppo"], rel=0, abs=0)
                assert digest_list(mine["ppo_policy"]) == \
                    ref["ppo_policy_digest"]
                assert digest_list(mine["ppo_value"]) == \
                    ref["ppo_value_digest"]
        feats = np.stack([e.features for e in entries])
        assert digest(feats) == ep["entries_features_digest"]
        canon = "\n".join(tb.canonical(e.tiles, e.knobs) for e in entries)
        assert hashlib.sha256(canon.encode()).hexdigest() == \
            ep["entries_canonical_digest"]
        np.testing.assert_array_equal(np.asarray([e.score for e in entries]),
                                      gc.arr[f"e{e_i}_entry_score"])
        assert [entries[0].order, entries[-1].order, len(entries)] == \
            ep["entries_order"]
        st = rng.bit_generator.state
        assert int(st["state"]["state"]) == \
            int(ep["end_rng_state"]["state"]["state"])
        assert st["has_uint32"] == ep["end_rng_state"]["has_uint32"]
        assert digest_list(agent.policy_params()) == ep["end_policy_digest"]
        assert digest_list(agent.value_params()) == ep["end_value_digest"]
        assert digest_list(opt_pi.m + opt_pi.v + opt_v.m + opt_v.v) == \
            ep["end_adam_digest"]
        assert opt_pi.t == ep["end_pi_t"]
        assert len(replay) == ep["end_buffer_len"]
        assert order == ep["end_order_counter"]
