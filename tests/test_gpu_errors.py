"""Error-path parity: the reference's exceptions, raised where it raises.

* a non-finite row in a PPO minibatch: ``ppo_update`` raises
  RlDivergedError and takes no Adam step (rlcore.py:368-373), pinned by the
  reference's ``test_nan_batch_raises`` (tests/test_rlcore.py:346-362);
* the drop-in session raises ``schedtune``'s own classes (so
  ``except schedtune.rlcore.RlDivergedError`` catches a device
  divergence);
* shapes beyond the device tables run on the reference's own path, with the
  session advancing exactly as the reference session does."""

import os
import sys

import numpy as np
import pytest

from gpu_util import CONV, all_sketch_tables, needs_gpu
from oracle import harl_oracle as O

pytestmark = [pytest.mark.gpu, needs_gpu]
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def _ring_with_nan(tb, agent, n=64):
    from paper_2211_11172_b200 import device as D
    oa = O.Agent.from_param_lists(agent.policy, agent.value, len(agent.hidden))
    tiles, knobs = O.sample_initial(tb, n, np.random.default_rng(2))
    X = O.featurize(tb, tiles, knobs)
    masks = O.action_masks(tb, tiles, knobs, tb.num_slots)
    acts, logp = O.select_actions(oa, X, masks, np.random.default_rng(3))
    nt, nk = O.apply_actions(tb, tiles, knobs, acts, tb.num_slots)
    Xn = O.featurize(tb, nt, nk)
    X = X.copy()
    X[0, 0] = np.nan                       # the reference test's bad row
    z = np.zeros(n)
    ring = D.DeviceReplay(n, tb.feature_len)
    ring.load(X, Xn, acts, logp, z, z + 0.1, z, masks, tb.num_slots,
              tb.levels)
    return ring


@pytest.mark.parametrize("spec", [True, False])
@pytest.mark.parametrize("hidden", [(16,), (128, 128)])
def test_ppo_nan_row_diverges_without_a_step(hidden, spec, monkeypatch):
    """A NaN minibatch row: RlDivergedError and no Adam step (rlcore.py:
    368-375), also when the update ran speculatively (gradients + Adam in
    one launch, restored from the backup) and a later update of the same
    episode ran before the check (it skips)."""
    from paper_2211_11172_b200 import device as D
    monkeypatch.setattr(D, "_PPO_SPEC", spec)
    from paper_2211_11172_b200.agent import RlConfig, init_session_agents
    from paper_2211_11172_b200.errors import RlDivergedError
    sg, sk, tb = all_sketch_tables(CONV)[0]
    cfg = RlConfig(hidden=hidden, minibatch=64, buffer_capacity=64)
    agent = init_session_agents([("sg", tb.num_slots)], tb.feature_len, cfg,
                                np.random.default_rng(0))["sg"]
    ring = _ring_with_nan(tb, agent)
    dag = D.DeviceAgent(agent, tb.levels)
    before = dag.params.clone()
    m_before = dag.m.clone()
    v_before = dag.v.clone()
    p32_before = dag.params32.clone()
    slots = torch.arange(64, dtype=torch.int32, device="cuda")
    dag.ppo_update(ring, slots, cfg, 1, 1)
    dag.ppo_update(ring, slots[1:], cfg, 2, 2)   # clean, but after the flag
    torch.cuda.synchronize()
    assert int(dag.bad.item()) != 0
    with pytest.raises(RlDivergedError):
        dag.raise_if_diverged()
    # no Adam step: the reference raises before opt.step
    assert torch.equal(dag.params, before)
    assert torch.equal(dag.m, m_before)
    assert torch.equal(dag.v, v_before)
    assert torch.equal(dag.params32, p32_before)
    # a clean minibatch (row 0 left out) updates normally
    dag.bad.zero_()
    dag.ppo_update(ring, slots[1:], cfg, 1, 1)
    dag.raise_if_diverged()
    assert not torch.equal(dag.params, before)


def _ref_modules():
    if os.path.isdir(REF) and REF not in sys.path:
        sys.path.insert(0, REF)
    return pytest.importorskip("schedtune")


def _session_pair(tmp_path, yaml_text, tgt_levels=2, **over):
    _ref_modules()
    from schedtune.measure import SimulatedBackend
    from schedtune.tuner import TunerConfig, TuningSession
    from schedtune.workload import TargetConfig, load_network
    from paper_2211_11172_b200.compat import b200_session_class
    p = tmp_path / "w.yaml"
    p.write_text(yaml_text)
    net = load_network(str(p))
    kw = dict(total_trials=24, top_k=8, min_tracks=8, initial_tracks=16,
              cull_window=3, episode_len=6, hidden=(16,), minibatch=32,
              buffer_capacity=64)
    kw.update(over)
    cfg = TunerConfig(**kw)
    tgt = TargetConfig(tiling_levels=tgt_levels)
    B200 = b200_session_class(TuningSession)
    ref = TuningSession(net, tgt, cfg, SimulatedBackend(), "rl",
                        out_dir=str(tmp_path / "ref"), workload_path=str(p))
    dev = B200(net, tgt, cfg, SimulatedBackend(), "rl",
               out_dir=str(tmp_path / "dev"), workload_path=str(p))
    return ref, dev


GEMM64 = """
name: gemm-64
subgraphs:
  - id: gemm_64x64x64
    weight: 1
    nodes:
      - name: mm
        kind: matmul
        shape: {m: 64, k: 64, n: 64}
"""


@pytest.mark.parametrize("hidden", [(16,), (128, 128)])
def test_drop_in_divergence_is_the_reference_exception(tmp_path, hidden):
    """A NaN in the value network: V(X), advantages and the critic loss go
    non-finite; both sessions raise schedtune.rlcore.RlDivergedError."""
    st = _ref_modules()
    ref, dev = _session_pair(tmp_path, GEMM64, hidden=hidden)
    for s in (ref, dev):
        sg = s.net.subgraphs[0].id
        s.agents[sg].value.params()[0][0, 0] = np.nan
    with pytest.raises(st.rlcore.RlDivergedError):
        ref.run_round()
    with pytest.raises(st.rlcore.RlDivergedError):
        dev.run_round()


def test_drop_in_invalid_action_is_the_reference_exception():
    """The device walker's InvalidActionError maps to the reference class
    with the same subspace and message."""
    st = _ref_modules()
    from paper_2211_11172_b200 import errors as E
    e = E.to_reference(E.InvalidActionError("unroll", "row 3"))
    assert isinstance(e, st.schedspace.InvalidActionError)
    assert e.subspace == "unroll" and str(e) == "invalid unroll action: row 3"
    assert isinstance(E.to_reference(E.ScheduleError("x")),
                      st.schedspace.ScheduleError)
    assert isinstance(E.to_reference(E.CostModelError("x")),
                      st.costmodel.CostModelError)


BIG = """
name: big-matmul
subgraphs:
  - id: mm_big
    weight: 1
    nodes: [{name: mm, kind: matmul, shape: {m: 131072, k: 64, n: 64}}]
"""


def test_drop_in_falls_back_beyond_device_tables(tmp_path):
    """An extent above the u16 tile factors (131072): SketchTables refuses
    it, the drop-in runs that sketch on the reference's path, and the
    session is the reference session bit for bit (same generator state,
    same visits, same measured set)."""
    _ref_modules()
    ref, dev = _session_pair(tmp_path, BIG, tgt_levels=2)
    for _ in range(2):
        ref.run_round()
        dev.run_round()
        assert dev.rng.bit_generator.state == ref.rng.bit_generator.state
        assert dev.order_counter == ref.order_counter
        assert sorted(dev.measured) == sorted(ref.measured)
    assert dev._b200_host_sketches
