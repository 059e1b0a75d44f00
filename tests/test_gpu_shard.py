"""Population-sharded episodes on the device (world size 2, both ranks on
cuda:0, gloo for the collectives -- the single-box stand-in for NCCL):
the merged shards reproduce the single-device episode (same generator
stream, uniforms at global rows, merged culls, the minibatch rows
all-reduced so every rank runs the single-device PPO update)."""

import os
import socket

import numpy as np
import pytest

from gpu_util import CONV, all_sketch_tables, needs_gpu

pytestmark = [pytest.mark.gpu, needs_gpu]
torch = pytest.importorskip("torch")

P, LEN, CW = 512, 6, 3


def _setup(hidden):
    import bench
    from paper_2211_11172_b200.agent import RlConfig, init_session_agents
    from paper_2211_11172_b200.engine import EpisodeConfig
    sg, sk, tb = all_sketch_tables(CONV)[0]
    rl = RlConfig(hidden=hidden, minibatch=64, buffer_capacity=256)
    agent = init_session_agents([("sg", tb.num_slots)], tb.feature_len, rl,
                                np.random.default_rng(0))["sg"]
    trees = bench.synthetic_forest(tb, 1)
    cfg = EpisodeConfig(tracks=P, track_len=LEN, cull_window=CW,
                        cull_fraction=0.5, min_tracks=P // 2)
    return tb, rl, agent, trees, cfg


def _visits(res, tb):
    tiles, knobs = res.states()
    tr = res.log_track[:res.visits].cpu().numpy()
    sc = res.scores()
    out, p = {}, 0
    for t, m in enumerate(res.step_rows, start=1):
        for i in range(p, p + m):
            out[(t, int(tr[i]))] = (tiles[i].tobytes(), knobs[i].tobytes(),
                                    float(sc[i]))
        p += m
    return out


def _worker(rank, world, port, hidden, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2211_11172_b200 import device as D
    from paper_2211_11172_b200.engine import EpisodeEngine
    tb, rl, agent, trees, cfg = _setup(hidden)
    forest = D.DeviceForest(trees, 0.5, 0.3)
    eng = EpisodeEngine(agent, rl, tb.levels, shard=(world, rank, None))
    gen = np.random.default_rng(11)
    out = []
    for _ in range(2):
        res = eng.run_episode(tb, forest, gen, cfg, 0)
        out.append(_visits(res, tb))
    eng.sync_to_host()
    q.put((rank, out, [p.copy() for p in agent.policy],
           gen.bit_generator.state["state"]["state"]))
    dist.destroy_process_group()


@pytest.mark.parametrize("hidden,mode", [((32, 32), "rows"),
                                         ((128, 128), "rows"),
                                         ((128, 128), "grads")])
def test_sharded_engine_matches_single_device(hidden, mode, monkeypatch):
    """mode "rows" (default): the minibatch rows all-reduced and the
    single-device update run on every rank -- the merged shards equal the
    single-device episode bit for bit, parameters included.  mode "grads"
    (HARL_SHARD_PPO=grads): per-shard gradient sums all-reduced -- equal up
    to the first update, then within fp64 rounding."""
    import torch.multiprocessing as mp
    from paper_2211_11172_b200 import device as D
    from paper_2211_11172_b200.engine import EpisodeEngine
    monkeypatch.setenv("HARL_SHARD_PPO", mode)   # inherited by the ranks
    tb, rl, agent, trees, cfg = _setup(hidden)
    forest = D.DeviceForest(trees, 0.5, 0.3)
    eng = EpisodeEngine(agent, rl, tb.levels, use_graphs=False)
    gen = np.random.default_rng(11)
    ref = []
    for _ in range(2):
        ref.append(_visits(eng.run_episode(tb, forest, gen, cfg, 0), tb))
    eng.sync_to_host()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, hidden, q))
             for r in range(2)]
    for p_ in procs:
        p_.start()
    got = dict((r, rest) for r, *rest in (q.get(timeout=600) for _ in procs))
    for p_ in procs:
        p_.join(timeout=60)
    for ep in range(2):
        merged = dict(got[0][0][ep])
        merged.update(got[1][0][ep])
        assert merged.keys() == ref[ep].keys()
        diff = [k for k in ref[ep] if merged[k] != ref[ep][k]]
        if mode == "rows":
            assert not diff, len(diff)
        else:
            # per-shard gradient sums round differently: a near-boundary
            # draw may flip after the first update; none before
            assert len(diff) <= len(ref[ep]) // 200, len(diff)
    assert got[0][2] == got[1][2] == gen.bit_generator.state["state"]["state"]
    for a, b in zip(got[0][1], got[1][1]):
        np.testing.assert_array_equal(a, b)
    for a, b in zip(got[0][1], agent.policy):
        if mode == "rows":
            np.testing.assert_array_equal(a, b)
        else:
            np.testing.assert_allclose(a, b, rtol=1e-6, atol=1e-9)
