"""The cost model fused into the sampler (k_sample_gbt, harl_policy_step_tc_gbt)
scores the successor rows exactly as the separate GBT launch does
(SurrogateModel.predict + reward, costmodel.py:219-230, tuner.py:389-391):
bit-identical scores and rewards for forests staged in shared memory
(perfect-tree image, depth <= 6), forests the launch's region cannot hold
after a reload (deeper: the in-kernel walk over the global node records),
an unfitted model (constant 1.0), and the host-side fallback for forests
beyond the fused kernel's 64 trees (nothing launched, the caller scores)."""

import numpy as np
import pytest

from gpu_util import CONV, all_sketch_tables, needs_gpu

pytestmark = [pytest.mark.gpu, needs_gpu]
torch = pytest.importorskip("torch")


def _step(tb, agent_np, n, forest, fuse, seed=3):
    from paper_2211_11172_b200 import device as D
    from paper_2211_11172_b200.agent import RlConfig  # noqa: F401
    dsk = D.DeviceSketch(tb)
    dag = D.DeviceAgent(agent_np, tb.levels)
    assert dag.tc
    tiles, knobs = D.init_population(dsk, n, np.random.default_rng(seed))
    X = D.featurize(dsk, tiles, knobs, n)
    old = D.gbt_predict(forest, X, n)
    old = old[0] if isinstance(old, tuple) else old
    feat_out = torch.empty((n, tb.feature_len), dtype=torch.float64,
                           device=X.device)
    score = torch.full((n,), np.nan, dtype=torch.float64, device=X.device)
    reward = torch.full((n,), np.nan, dtype=torch.float64, device=X.device)
    out = D.policy_step(dsk, dag, X, tiles, knobs, n,
                        gen=np.random.default_rng(seed + 1), feat_out=feat_out,
                        gbt=(forest, old, score, reward) if fuse else None)
    D.raise_status(int(out["status"].item()) & ((1 << 64) - 1))
    torch.cuda.synchronize()
    return out, feat_out, old, score, reward


def _agent(tb):
    from paper_2211_11172_b200.agent import RlConfig, init_session_agents
    rl = RlConfig(hidden=(128, 128), minibatch=64, buffer_capacity=512)
    return init_session_agents([("sg", tb.num_slots)], tb.feature_len, rl,
                               np.random.default_rng(0))["sg"]


@pytest.mark.parametrize("n_trees,depth,fused", [(50, 6, True), (17, 3, True),
                                                 (56, 6, True), (50, 7, True),
                                                 (70, 6, False)])
@pytest.mark.parametrize("n", [1000, 16384])
def test_fused_cost_model_matches_separate_launch(n_trees, depth, fused, n):
    import bench
    from paper_2211_11172_b200 import device as D
    _, _, tb = all_sketch_tables(CONV)[0]
    agent = _agent(tb)
    forest = D.DeviceForest(bench.synthetic_forest(tb, 2, n_trees, depth),
                            0.5, 0.3)
    out, feat, old, score, reward = _step(tb, agent, n, forest, True)
    assert out["gbt_fused"] is fused
    _, feat_ref, _, _, _ = _step(tb, agent, n, forest, False)
    assert feat.cpu().numpy().tobytes() == feat_ref.cpu().numpy().tobytes()
    ref_reward = torch.empty_like(reward)
    ref = D.gbt_predict(forest, feat_ref, n, old_score=old, reward=ref_reward)
    ref = ref[0] if isinstance(ref, tuple) else ref
    if not fused:
        return
    assert score.cpu().numpy().tobytes() == ref[:n].cpu().numpy().tobytes()
    assert reward.cpu().numpy().tobytes() == \
        ref_reward[:n].cpu().numpy().tobytes()


def test_fused_cost_model_after_reloads():
    """One forest's buffers, reloaded: depth 6 (staged), depth 7 (the
    launch-time region holds depth <= 6: global node walk), unfitted
    (score 1.0), depth 4 again -- each bit-identical to the separate launch."""
    import bench
    from paper_2211_11172_b200 import device as D
    _, _, tb = all_sketch_tables(CONV)[0]
    agent = _agent(tb)
    n = 4096
    forest = D.DeviceForest(bench.synthetic_forest(tb, 4, 50, 6), 0.5, 0.3,
                            node_capacity=50 * 255, tree_capacity=50)
    for seed, depth, fitted in ((5, 7, True), (6, 6, False), (7, 4, True)):
        assert forest.load(bench.synthetic_forest(tb, seed, 48, depth), 0.25,
                           0.3, fitted=fitted)
        out, feat, old, score, reward = _step(tb, agent, n, forest, True,
                                              seed=seed)
        assert out["gbt_fused"]
        ref_reward = torch.empty_like(reward)
        ref = D.gbt_predict(forest, feat, n, old_score=old, reward=ref_reward)
        ref = ref[0] if isinstance(ref, tuple) else ref
        assert score.cpu().numpy().tobytes() == ref[:n].cpu().numpy().tobytes()
        assert reward.cpu().numpy().tobytes() == \
            ref_reward[:n].cpu().numpy().tobytes()
        if not fitted:
            assert (score.cpu().numpy() == 1.0).all()


def test_native_agent_copy_matches_numpy_pack():
    """DeviceAgent's native pack/unpack (harl_agent_copy) writes the same
    flat block and the same numpy arrays as the numpy restatement
    (_pack / _unpack_into), for parameters and both Adam moments."""
    from paper_2211_11172_b200 import device as D
    _, _, tb = all_sketch_tables(CONV)[0]
    agent = _agent(tb)
    rng = np.random.default_rng(4)
    for lst in (agent.policy, agent.value, agent.opt_pi.m, agent.opt_v.m,
                agent.opt_pi.v, agent.opt_v.v):
        for a in lst:
            a[...] = rng.normal(size=a.shape)
    dag = D.DeviceAgent(agent, tb.levels)
    for pol, val in ((agent.policy, agent.value),
                     (agent.opt_pi.m, agent.opt_v.m),
                     (agent.opt_pi.v, agent.opt_v.v)):
        ref = dag._pack(pol, val)
        got = np.full(dag.n_params, np.nan)
        got[:] = ref          # untouched padding (if any) equal on both sides
        got_n = got.copy()
        assert dag._native_copy(got_n, pol, val, False)
        assert got_n.tobytes() == ref.tobytes()
        flat = rng.normal(size=dag.n_params)
        a1 = [x.copy() for x in pol], [x.copy() for x in val]
        a2 = [x.copy() for x in pol], [x.copy() for x in val]
        dag._unpack_into(flat, *a1)
        assert dag._native_copy(flat, *a2, True)
        for x, y in zip(a1[0] + a1[1], a2[0] + a2[1]):
            assert x.tobytes() == y.tobytes()


def test_upload_skipped_only_while_the_host_lists_are_unchanged():
    """DeviceAgent.upload skips the copy when the numpy lists still hold,
    bit for bit, what the last download wrote; any change (one element of
    one Adam moment) is uploaded; an episode always invalidates."""
    import torch
    from paper_2211_11172_b200 import device as D
    _, _, tb = all_sketch_tables(CONV)[0]
    agent = _agent(tb)
    dag = D.DeviceAgent(agent, tb.levels)
    calls = []
    orig = dag.refresh_derived
    dag.refresh_derived = lambda: (calls.append(1), orig())[1]
    dag.upload()
    dag.download()
    n0 = len(calls)
    dag.upload()                       # unchanged: skipped
    assert len(calls) == n0
    agent.opt_v.m[1].reshape(-1)[3] += 0.5
    dag.upload()                       # changed: uploaded
    assert len(calls) == n0 + 1
    torch.cuda.synchronize()
    dag.download()
    assert agent.opt_v.m[1].reshape(-1)[3] == dag._pin_np[1][
        dag.val_layout.off_b[0] + 3]
    dag._device_is_pin = False         # what run_episode does
    dag.upload()
    assert len(calls) == n0 + 2
