"""Network-output parity at the north-star sizes (>= 64 K candidates).

At these sizes the production tcgen05 kernels run their persistent
multi-tile paths -- ``k_mlp_f16<policy>`` / ``k_mlp_f16<value>`` (3xFP16,
two 128-row tiles in flight per CTA, several tile pairs per CTA above
148 x 128 rows) and, on the 3xTF32 fallback, ``k_policy_tc`` /
``k_value_tc`` -- which the small oracle tests never reach.  Each test compares them with the oracle's fp64
forward chunk by chunk (tests/large_util.py):

* one policy step + V(X)/V(X') at 65,536 rows (C3 sketch k3, 512 tiles)
  and 1,048,576 rows (C5, 8,192 tiles);
* whole recorded episodes: C3 at 65,536 tracks (steps before and after the
  cull and after PPO updates, with the parameters each step ran with) and
  C5 at 1 M tracks (first step and first post-cull step);
* C1 at 1,024 tracks: the full 60-step episode shadow-replayed by the
  oracle (every draw vouched for, states/features/scores/rewards bit-exact,
  logp/advantages within 1e-4; with the device's logp/advantages in the
  oracle's FIFO, the parameters after all 30 PPO updates within 1e-6);
* the golden and shadow replays and the 64 K multi-tile check re-run on
  the 3xTF32 fallback (HARL_TC16=0, with and without HARL_TC64=0).
"""

import os
import subprocess
import sys

import numpy as np
import pytest

from gpu_util import assert_close_rel, needs_gpu
from large_util import (StepCheck, check_advantage, check_policy_rows,
                        check_values, uniforms)
from oracle import harl_oracle as O

pytestmark = [pytest.mark.gpu, needs_gpu]
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _perturb(agent, seed, scale=0.3):
    """Heads larger than the 0.01 init so the softmaxes are not flat."""
    rng = np.random.default_rng(seed)
    for p in agent.policy + agent.value:
        p += scale * rng.standard_normal(p.shape) * (p.std() + 0.05)


def _oracle_agent(agent):
    return O.Agent.from_param_lists([p.copy() for p in agent.policy],
                                    [p.copy() for p in agent.value],
                                    len(agent.hidden))


def _device_states(tb, n, seed):
    """n uniform initial states (device sampler, bit-exact with
    sample_initial_schedules) and their device features."""
    from paper_2211_11172_b200 import device as D
    dsk = D.DeviceSketch(tb)
    tiles, knobs = D.init_population(dsk, n, np.random.default_rng(seed))
    X = D.featurize(dsk, tiles, knobs, n)
    return dsk, tiles, knobs, X


@pytest.mark.parametrize("config,n", [("c3", 65536), ("c5", 1 << 20)])
def test_policy_and_value_multitile_vs_oracle(config, n):
    import bench
    from paper_2211_11172_b200 import device as D
    w = bench.build_workload(config, n)
    tb, agent = w["tables"], w["agent"]
    _perturb(agent, 5)
    oa = _oracle_agent(agent)
    dag = D.DeviceAgent(agent, tb.levels)
    assert dag.tc
    dsk, dt, dk, Xd = _device_states(tb, n, 21)
    tiles, knobs = D.states_to_host(tb, dt, dk, n)
    X = Xd.cpu().numpy()
    # the device features are the oracle's (spot check; bit-exact suites
    # cover the featurizer)
    idx = np.random.default_rng(0).choice(n, 2000, replace=False)
    assert O.featurize(tb, tiles[idx], knobs[idx]).tobytes() == \
        X[idx].tobytes()
    g = np.random.default_rng(77)
    st = g.bit_generator.state
    out = D.policy_step(dsk, dag, Xd, dt, dk, n, gen=g, want_logits=True)
    D.raise_status(int(out["status"].item()) & ((1 << 64) - 1))
    u = uniforms(st, n)
    g_ref = np.random.default_rng()
    g_ref.bit_generator.state = st
    g_ref.random(4 * n)
    assert g.bit_generator.state == g_ref.bit_generator.state
    acts = out["actions"][:, :n].cpu().numpy().T
    nt, nk = D.states_to_host(tb, out["tiles"], out["knobs"], n)
    chk = StepCheck()
    check_policy_rows(chk, tb, oa, X, tiles, knobs, u, acts,
                      out["logp"][:n].cpu().numpy(),
                      out["logits"].cpu().numpy(), dsk.head_cols,
                      new_tiles=nt, new_knobs=nk)
    # V(X) on the states, V(X') on their successors: one k_value_tc launch
    # over both populations
    Xn = D.featurize(dsk, out["tiles"], out["knobs"], n)
    v0 = torch.empty(n, dtype=torch.float32, device="cuda")
    v1 = torch.empty(n, dtype=torch.float32, device="cuda")
    D.value_pair(dag, Xd, n, Xn, n, v0, v1)
    check_values(chk, oa, X, v0.cpu().numpy(), "v_x")
    check_values(chk, oa, Xn.cpu().numpy(), v1.cpu().numpy(), "v_xn")
    chk.assert_ok()
    assert chk.rows == n


class _Rec(list):
    """An engine record that keeps only the named steps."""

    def __init__(self, steps):
        super().__init__()
        self.steps = set(steps)


def _check_recorded(tb, agent, dag, r, chunk=131072):
    """One recorded step of an engine episode against the oracle, with the
    parameters that step ran with."""
    from paper_2211_11172_b200 import device as D
    pol = [p.copy() for p in agent.policy]
    val = [p.copy() for p in agent.value]
    dag._unpack_into(r["params"].cpu().numpy(), pol, val)
    oa = O.Agent.from_param_lists(pol, val, len(agent.hidden))
    m = r["m"]
    tiles, knobs = D.states_to_host(tb, r["tiles"], r["knobs"], m)
    nt, nk = D.states_to_host(tb, r["new_tiles"], r["new_knobs"], m)
    X = r["X"].cpu().numpy()
    Xn = r["new_feats"].cpu().numpy()
    chk = StepCheck()
    check_policy_rows(chk, tb, oa, X, tiles, knobs,
                      uniforms(r["rng_before"], m),
                      r["actions"].cpu().numpy().T,
                      r["logp"].cpu().numpy(), r["logits"].cpu().numpy(),
                      D.DeviceSketch(tb).head_cols, chunk=chunk,
                      new_tiles=nt, new_knobs=nk)
    idx = np.random.default_rng(r["t"]).choice(m, min(m, 4000),
                                               replace=False)
    assert O.featurize(tb, nt[idx], nk[idx]).tobytes() == Xn[idx].tobytes()
    check_values(chk, oa, X, r["v_cur"].cpu().numpy(), "v_cur")
    check_values(chk, oa, Xn, r["v_next"].cpu().numpy(), "v_next")
    check_advantage(chk, oa, X, Xn, r["rewards"].cpu().numpy(),
                    r["adv"].cpu().numpy())
    chk.assert_ok()
    return chk


@pytest.mark.parametrize("config,P,steps", [
    ("c3", 65536, (1, 2, 3, 20, 21, 22, 41, 60)),
    ("c5", 1 << 20, (1, 21)),
])
def test_episode_steps_at_full_size(config, P, steps):
    """Recorded steps of a whole engine episode at the configs' sizes: the
    first steps (512 / 8,192 tiles), the cull step, the first post-cull
    steps (half the rows; M=128 multi-tile still) and steps after several
    PPO updates, each with the parameters it ran with."""
    import bench
    from paper_2211_11172_b200 import device as D
    from paper_2211_11172_b200.engine import EpisodeEngine
    w = bench.build_workload(config, P)
    tb, agent = w["tables"], w["agent"]
    eng = EpisodeEngine(agent, w["rl"], tb.levels)
    forest = D.DeviceForest(w["trees"], w["base"], w["lr"])
    rec = _Rec(steps)
    res = eng.run_episode(tb, forest, np.random.default_rng(5),
                          bench.episode_config(P), 0, record=rec)
    assert res.visits == 40 * P
    assert [r["t"] for r in rec] == list(steps)
    for r in rec:
        assert r["m"] == (P if r["t"] <= 20 else P // 2)
        _check_recorded(tb, agent, eng.dagent, r)
    assert len(res.train) == 30


def test_c1_full_episode_shadow_replay():
    """C1 (GEMM 1024^3, 1,024 tracks): the whole 60-step episode -- 2 K
    ... 40 K visits, a cull, 30 PPO updates -- replayed by the oracle on the
    device's decisions."""
    import bench
    from paper_2211_11172_b200 import device as D
    from paper_2211_11172_b200.engine import EpisodeEngine
    P = 1024
    w = bench.build_workload("c1", P)
    tb, agent = w["tables"], w["agent"]
    oa = _oracle_agent(agent)
    eng = EpisodeEngine(agent, w["rl"], tb.levels)
    forest = D.DeviceForest(w["trees"], w["base"], w["lr"])
    rec = []
    res = eng.run_episode(tb, forest, np.random.default_rng(9),
                          bench.episode_config(P), 0, record=rec)
    by_t = {r["t"]: r for r in rec}

    def follow(t, info):
        r = by_t[t]
        if info["phase"] == "act":
            return {"actions": r["actions"].cpu().numpy().T.astype(np.int64)}
        if info["phase"] == "push":
            # the FIFO gets the device's fp32-network outputs, so every PPO
            # update below sees the device's inputs (its own outputs are
            # compared at 1e-4 per step; the update arithmetic at 1e-6)
            rw = r["rewards"].cpu().numpy()
            vn = r["v_next"].cpu().numpy().astype(np.float64)
            return {"logp": r["logp"].cpu().numpy(),
                    "adv": r["adv"].cpu().numpy(), "td": rw + 0.9 * vn}
        return {"cull": r.get("cull")}

    rl = w["rl"]
    ocfg = O.EpisodeCfg(tracks=P, track_len=40, cull_window=20,
                        cull_fraction=0.5, min_tracks=P // 2,
                        rl_cfg=O.RlCfg(minibatch=rl.minibatch,
                                       buffer_capacity=rl.buffer_capacity))
    o_pi = O.Adam.zeros_like(oa.policy_params(), rl.lr_actor)
    o_v = O.Adam.zeros_like(oa.value_params(), rl.lr_critic)
    trace = []
    entries, _, _ = O.run_episode(
        tb, tb.num_slots, ocfg, oa, o_pi, o_v, O.Replay(rl.buffer_capacity),
        O.GbtModel(w["base"], w["lr"], True, w["trees"]),
        np.random.default_rng(9), 0, trace=trace, follow=follow)
    tiles, knobs = res.states()
    assert np.array_equal(tiles, np.stack([e.tiles for e in entries]))
    assert np.array_equal(knobs, np.stack([e.knobs for e in entries]))
    assert res.scores().tobytes() == \
        np.asarray([e.score for e in entries]).tobytes()
    draws = flips = 0
    o_steps = [t for t in trace if "step" in t]
    assert len(o_steps) == 60
    for o in o_steps:
        r = by_t[o["step"]]
        np.testing.assert_array_equal(r["sel"].cpu().numpy(), o["sel"])
        acts = o["actions"]
        for h, hd in enumerate(o["heads"]):
            draws += len(acts)
            diff = np.flatnonzero(acts[:, h] != hd["a"])
            flips += len(diff)
            for row in diff:
                c = np.cumsum(hd["p"][row])
                a = acts[row, h]
                lo = c[a - 1] if a > 0 else 0.0
                assert hd["p"][row, a] > 0
                assert lo - 1e-5 <= hd["u"][row] <= c[a] + 1e-5
        assert r["new_feats"].cpu().numpy().tobytes() == \
            o["new_feats"].tobytes()
        assert r["rewards"].cpu().numpy().tobytes() == o["rewards"].tobytes()
        assert_close_rel(r["logp"].cpu().numpy(), o["logp"], what="logp")
        assert_close_rel(r["adv"].cpu().numpy(), o["adv"], what="adv")
        if "ppo_idx" in o:
            np.testing.assert_array_equal(r["ppo_idx"], o["ppo_idx"])
    assert flips <= max(2, draws // 1000)
    eng.sync_to_host()
    got = eng.dagent._pack(agent.policy, agent.value)
    ref = eng.dagent._pack(oa.policy_params(), oa.value_params())
    # 30 chained PPO updates (B = 256 of a 4,096-row FIFO) on identical
    # inputs: fp64 arithmetic, so the PPO kernels' tolerance (1e-6)
    assert_close_rel(got, ref, tol=1e-6, what="params after 30 updates")


@pytest.mark.parametrize("env", [{"HARL_TC16": "0"},
                                 {"HARL_TC16": "0", "HARL_TC64": "0"}],
                         ids=["tf32", "tf32-m128"])
def test_replays_on_the_tf32_fallback(env):
    """The 3xTF32 kernels (the fallback where the 3xFP16 image does not fit:
    more than 128 padded head columns, F > 64 staging) stay verified: the
    golden and shadow replays and the 64 K multi-tile oracle check re-run
    with HARL_TC16=0, and with HARL_TC64=0 as well (k_policy_tc's M=128
    tiles on every launch), in a child process."""
    p = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-x", "-p",
         "no:cacheprovider",
         os.path.join(ROOT, "tests", "test_gpu_episode.py"),
         os.path.join(ROOT, "tests", "test_gpu_large.py"),
         "-k", "golden_episode_replay or shadow_replay or "
               "multitile_vs_oracle and c3"],
        cwd=ROOT, env=dict(os.environ, **env), capture_output=True,
        text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-2000:]
    assert " passed" in p.stdout


def test_cluster_ppo_kernel_parity():
    """HARL_PPO_CL=1 (k_ppo_rows_cl: the per-row PPO work on 8-CTA
    clusters, DMMA layers, distributed-shared-memory exchanges) keeps the
    PPO parity: the update vs the oracle, the golden and shadow replays and
    the C1 60-step shadow replay with 30 chained updates, in a child
    process."""
    p = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-x", "-p",
         "no:cacheprovider",
         os.path.join(ROOT, "tests", "test_gpu_episode.py"),
         os.path.join(ROOT, "tests", "test_gpu_large.py"),
         "-k", "ppo_update_matches_oracle or golden_episode_replay or "
               "shadow_replay"],
        cwd=ROOT, env=dict(os.environ, HARL_PPO_CL="1"), capture_output=True,
        text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-2000:]
    assert " passed" in p.stdout
