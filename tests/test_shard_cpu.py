"""Multi-rank episode arithmetic (paper_2211_11172_b200.shard) on CPU with
torch.distributed/gloo at world size 2: a population-sharded episode --
interleaved tracks, global-row uniforms, merged culls, replay ownership,
per-shard PPO gradients summed by one all-reduce -- reproduces the
single-device episode (oracle compute on every rank)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2211_11172_b200.shard import (GlobalReplayIndex, ShardLayout,
                                         cull_decision)


def test_global_rows_and_owner():
    P, G = 10, 3
    alive = np.ones(P, dtype=bool)
    alive[[2, 5, 6]] = False
    for r in range(G):
        lay = ShardLayout(P, G, r)
        ids = lay.local_ids[alive[lay.local_ids]]
        rows = lay.global_rows(alive, ids)
        ref = [list(np.flatnonzero(alive)).index(i) for i in ids]
        assert rows.tolist() == ref
    assert ShardLayout.owner([0, 1, 2, 3], 2).tolist() == [0, 1, 0, 1]


def test_replay_index_tracks_the_global_fifo():
    idx = GlobalReplayIndex(cap=5, world=2)
    idx.push_step([0, 1, 0, 1])
    idx.push_step([1, 0, 1])
    assert len(idx) == 5
    ranks, local = idx.locate([0, 1, 4])
    # global order: (0,0)(1,0)(0,1)(1,1)(1,2)(0,2)(1,3) -> last 5
    assert ranks.tolist() == [0, 1, 1] and local.tolist() == [1, 1, 3]


def test_replay_index_matches_a_row_by_row_fifo():
    """The vectorised index against the plain deque of (rank, local push)
    it replaces: random step sizes, some larger than the capacity."""
    from collections import deque
    rng = np.random.default_rng(3)
    for world, cap in ((1, 7), (2, 16), (4, 64), (8, 33)):
        idx = GlobalReplayIndex(cap=cap, world=world)
        ref, counts = deque(maxlen=cap), [0] * world
        for _ in range(40):
            own = rng.integers(0, world, size=int(rng.integers(0, 3 * cap)))
            idx.push_step(own)
            for r in own:
                ref.append((int(r), counts[r]))
                counts[r] += 1
            assert len(idx) == len(ref)
            if len(ref):
                pos = rng.integers(0, len(ref), size=10)
                ranks, local = idx.locate(pos)
                assert ranks.tolist() == [ref[p][0] for p in pos]
                assert local.tolist() == [ref[p][1] for p in pos]


def test_cull_decision_ties_drop_higher_index():
    alive = np.ones(6, dtype=bool)
    gone = cull_decision(alive, np.arange(6), np.array([0, 0, 1, 1, 0, 2.]),
                         0.5, 2)
    assert gone.tolist() == [0, 1, 4]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _setup():
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from golden_util import GoldenCase
    from oracle import harl_oracle as O
    gc = GoldenCase("conv2d_l4")
    return gc, O


def _sharded_episode(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gc, O = _setup()
    ep = gc.rec["episodes"][0]
    tb = gc.tables(ep["sketch"])
    S = gc.slots
    agent = O.Agent.from_param_lists(gc.agent.policy, gc.agent.value,
                                     len(gc.cfg["hidden"]))
    opt_pi = O.Adam.zeros_like(agent.policy_params(), gc.rl.lr_actor)
    opt_v = O.Adam.zeros_like(agent.value_params(), gc.rl.lr_critic)
    model = O.GbtModel(gc.model_base, gc.rec["model_lr"], True, gc.trees())
    rl = O.RlCfg(minibatch=gc.rl.minibatch,
                 buffer_capacity=gc.rl.buffer_capacity)
    rng = gc.rng_from(ep["rng_state"])
    P, L = gc.tracks, gc.track_len
    lay = ShardLayout(P, world, rank)
    # every rank samples the whole population (identical), keeps its own
    tiles_all, knobs_all = O.sample_initial(tb, P, rng)
    tiles = tiles_all.copy()
    knobs = knobs_all.copy()
    feats = O.featurize(tb, tiles, knobs)
    score = model.predict(feats)
    alive = np.ones(P, dtype=bool)
    ring = []                       # this rank's pushes, in push order
    gidx = GlobalReplayIndex(rl.buffer_capacity, world)
    used, t, budget = 0, 0, P * L
    visits = []
    while not (alive.sum() < gc.cfg["min_tracks"] or used >= budget):
        t += 1
        live = np.flatnonzero(alive)
        m = min(len(live), budget - used)
        sel = live[:m]
        mine = sel[sel % world == rank]
        grow = lay.global_rows(alive, mine)
        X = feats[mine]
        masks = O.action_masks(tb, tiles[mine], knobs[mine], S)
        logits, _ = agent.policy_forward(X)
        acts = np.zeros((len(mine), 4), dtype=np.int64)
        logp = np.zeros(len(mine))
        for h, (lg, mk) in enumerate(zip(logits, masks)):
            lp, p = O.masked_log_softmax(lg, mk)
            u = rng.random((m, 1))[:, 0][grow]      # global-row uniforms
            a = O.categorical_from_uniform(p, u)
            acts[:, h] = a
            logp += lp[np.arange(len(mine)), a]
        nt, nk = O.apply_actions(tb, tiles[mine], knobs[mine], acts, S)
        nf = O.featurize(tb, nt, nk)
        new = model.predict(nf)
        rew = (new - score[mine]) / score[mine]
        vc, _ = agent.value(X)
        vn, _ = agent.value(nf)
        adv = rew + rl.discount * vn - vc
        td = rew + rl.discount * vn
        for i in range(len(mine)):
            ring.append((X[i], acts[i], logp[i], adv[i], td[i],
                         tuple(mk[i] for mk in masks)))
        gidx.push_step(sel % world)
        tiles[mine], knobs[mine], feats[mine], score[mine] = nt, nk, nf, new
        visits.append((t, mine, nt, nk, new))
        used += m
        if t % gc.cfg["cull_window"] == 0 and used < budget:
            got = [None] * world
            dist.all_gather_object(got, (mine, adv))
            ids = np.concatenate([g[0] for g in got])
            av = np.concatenate([g[1] for g in got])
            gone = cull_decision(alive, ids, av, gc.cfg["cull_fraction"],
                                 gc.cfg["min_tracks"])
            alive[gone] = False
        if t % rl.train_interval == 0 and len(gidx) >= 2:
            B = min(rl.minibatch, len(gidx))
            pos = rng.choice(len(gidx), size=B, replace=False)
            owners, local = gidx.locate(pos)
            own = [ring[int(k)] for o, k in zip(owners, local) if o == rank]
            grads = [np.zeros_like(p) for p in
                     agent.policy_params() + agent.value_params()]
            if own:
                Xb = np.stack([o[0] for o in own])
                ab = np.stack([o[1] for o in own])
                mb = [np.stack([o[5][h] for o in own]) for h in range(4)]
                _, ga, _, _, gv = O.ppo_grads(
                    agent, Xb, mb, ab, np.asarray([o[2] for o in own]),
                    np.asarray([o[3] for o in own]),
                    np.asarray([o[4] for o in own]), rl, norm=B)
                grads = ga + gv
            flat = torch.from_numpy(np.concatenate([g.ravel() for g in grads]))
            dist.all_reduce(flat)
            off, full = 0, []
            for g in grads:
                full.append(flat[off:off + g.size].numpy().reshape(g.shape))
                off += g.size
            npi = len(agent.policy_params())
            opt_pi.step(agent.policy_params(), full[:npi])
            opt_v.step(agent.value_params(), full[npi:])
    q.put((rank, [(t, ids, nt, nk, new) for t, ids, nt, nk, new in visits],
           [p.copy() for p in agent.policy_params()],
           rng.bit_generator.state["state"]["state"]))
    dist.destroy_process_group()


def test_sharded_oracle_episode_matches_single_device():
    gc, O = _setup()
    ep = gc.rec["episodes"][0]
    tb = gc.tables(ep["sketch"])
    agent = O.Agent.from_param_lists([p.copy() for p in gc.agent.policy],
                                     [p.copy() for p in gc.agent.value],
                                     len(gc.cfg["hidden"]))
    rl = O.RlCfg(minibatch=gc.rl.minibatch,
                 buffer_capacity=gc.rl.buffer_capacity)
    cfg = O.EpisodeCfg(tracks=gc.tracks, track_len=gc.track_len,
                       cull_window=gc.cfg["cull_window"],
                       cull_fraction=gc.cfg["cull_fraction"],
                       min_tracks=gc.cfg["min_tracks"], rl_cfg=rl)
    rng = gc.rng_from(ep["rng_state"])
    trace = []
    O.run_episode(tb, gc.slots, cfg, agent,
                  O.Adam.zeros_like(agent.policy_params(), rl.lr_actor),
                  O.Adam.zeros_like(agent.value_params(), rl.lr_critic),
                  O.Replay(rl.buffer_capacity),
                  O.GbtModel(gc.model_base, gc.rec["model_lr"], True,
                             gc.trees()), rng, 0, trace=trace)
    steps = [s for s in trace if "step" in s]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_episode, args=(r, 2, port, q))
             for r in range(2)]
    for p in procs:
        p.start()
    out = dict((r, rest) for r, *rest in (q.get(timeout=300) for _ in procs))
    for p in procs:
        p.join(timeout=60)
    for k, s in enumerate(steps):
        merged = {}
        for r in (0, 1):
            t, ids, nt, nk, new = out[r][0][k]
            assert t == s["step"]
            for i, tid in enumerate(ids):
                merged[int(tid)] = (nt[i], nk[i], new[i])
        for row, tid in enumerate(s["sel"]):
            nt, nk, new = merged[int(tid)]
            np.testing.assert_array_equal(nt, s["new_tiles"][row])
            np.testing.assert_array_equal(nk, s["new_knobs"][row])
            assert new == s["new_score"][row]
    assert out[0][2] == out[1][2] == int(rng.bit_generator.state["state"]["state"])
    for a, b in zip(out[0][1], agent.policy_params()):
        np.testing.assert_allclose(a, b, rtol=1e-9, atol=1e-12)
    for a, b in zip(out[0][1], out[1][1]):
        np.testing.assert_array_equal(a, b)


def test_shard_tasks_interleaved_partition():
    from paper_2211_11172_b200.shard import shard_tasks
    for world in (1, 2, 4, 8):
        parts = [shard_tasks(24, world, r) for r in range(world)]
        assert sorted(i for p in parts for i in p) == list(range(24))
        assert max(map(len, parts)) - min(map(len, parts)) <= 1
        assert parts[0][:2] == [0, world][:len(parts[0][:2])]
    with pytest.raises(ValueError):
        shard_tasks(24, 2, 2)
