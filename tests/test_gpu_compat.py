"""The drop-in: the reference's own TuningSession with ``_run_episode``
replaced by the B200 engine.  Needs the unmodified reference package
importable (installed into baseline/_ref); skipped otherwise.

Checks that hold exactly even though device sampling may flip a
near-boundary draw: the generator ends each round in the reference's state
(RNG consumption is data-independent), the same number of entries/visits,
the same trajectory-event skeleton, checkpoints round-trip."""

import json
import os
import sys

import numpy as np
import pytest

from gpu_util import needs_gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
if os.path.isdir(REF) and REF not in sys.path:
    sys.path.insert(0, REF)
schedtune = pytest.importorskip("schedtune")

pytestmark = [pytest.mark.gpu, needs_gpu]

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


def _sessions(tmp_path, hidden, searcher="rl"):
    from schedtune.measure import SimulatedBackend
    from schedtune.tuner import TunerConfig, TuningSession
    from schedtune.workload import TargetConfig, load_network
    from paper_2211_11172_b200.compat import b200_session_class
    p = tmp_path / "w.yaml"
    p.write_text(GEMM64)
    net = load_network(str(p))
    cfg = TunerConfig(total_trials=24, top_k=8, min_tracks=8,
                      initial_tracks=16, cull_window=3, episode_len=6,
                      hidden=hidden, minibatch=32, buffer_capacity=64)
    tgt = TargetConfig(tiling_levels=2)
    B200 = b200_session_class(TuningSession)
    ref = TuningSession(net, tgt, cfg, SimulatedBackend(), searcher,
                        out_dir=str(tmp_path / "ref"), workload_path=str(p))
    dev = B200(net, tgt, cfg, SimulatedBackend(), searcher,
               out_dir=str(tmp_path / "dev"), workload_path=str(p))
    return ref, dev


@pytest.mark.parametrize("hidden", [(16,), (128, 128)])
def test_drop_in_rounds_match_reference_structure(tmp_path, hidden):
    ref, dev = _sessions(tmp_path, hidden)
    for _ in range(3):
        ref.run_round()
        dev.run_round()
        assert dev.rng.bit_generator.state == ref.rng.bit_generator.state
        assert dev.order_counter == ref.order_counter
        assert dev.trials_used == ref.trials_used
        sg = ref.net.subgraphs[0].id
        assert len(dev.buffers[sg]) == len(ref.buffers[sg])
        assert dev.agents[sg].opt_pi.t == ref.agents[sg].opt_pi.t

    def skeleton(path):
        ev = [json.loads(l) for l in open(path)]
        return [(e["event"], e.get("step"), e.get("alive"),
                 len(e.get("rewards", [])), len(e.get("eliminated", [])))
                for e in ev if e["event"] in ("episode_step", "cull", "train",
                                              "episode_end")]
    assert skeleton(tmp_path / "dev" / "trajectory.jsonl") == \
        skeleton(tmp_path / "ref" / "trajectory.jsonl")


def test_drop_in_checkpoint_round_trip(tmp_path):
    from schedtune.tuner import read_checkpoint
    ref, dev = _sessions(tmp_path, (16,))
    dev.run_round()
    path = str(tmp_path / "ck.bin")
    dev.save(path)
    meta, arrays = read_checkpoint(path)
    sg = dev.net.subgraphs[0].id
    assert meta["buffers"][sg] == len(dev.buffers[sg])
    assert arrays[f"buffer/{sg}/mask0"].dtype == bool
    for i, p in enumerate(dev.agents[sg].policy.params()):
        np.testing.assert_array_equal(arrays[f"agent/{sg}/pi/{i}"], p)
