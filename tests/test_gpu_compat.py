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


def _sessions(tmp_path, hidden, searcher="rl", total_trials=24):
    from schedtune.measure import SimulatedBackend
    from schedtune.tuner import TunerConfig, TuningSession
    from schedtune.workload import TargetConfig, load_network
    from paper_2211_11172_b200.compat import b200_session_class
    p = tmp_path / "w.yaml"
    p.write_text(GEMM64)
    net = load_network(str(p))
    cfg = TunerConfig(total_trials=total_trials, top_k=8, min_tracks=8,
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


@pytest.mark.parametrize("searcher", ["rl", "evolutionary"])
def test_drop_in_topk_entries_rank_like_full_list(tmp_path, searcher):
    """The default entry list (device top-k' superset) and the full visit
    list give run_round the same rank_scores answer, round after round
    (the measured set grows, so exclusions are exercised)."""
    from schedtune.costmodel import rank_scores
    _, dev = _sessions(tmp_path, (16,), searcher, total_trials=64)
    orig = dev._b200_entries
    seen = []

    def spy(res, tables, sketch, pending=None):
        top = orig(res, tables, sketch, pending)
        dev.b200_all_entries = True
        try:
            full = orig(res, tables, sketch)
        finally:
            dev.b200_all_entries = False
        k_hat = min(dev.cfg.top_k, dev.cfg.total_trials - dev.trials_used)
        a = rank_scores(dev.model, top, k_hat, exclude=dev.measured)
        b = rank_scores(dev.model, full, k_hat, exclude=dev.measured)
        assert [(e.order, e.canonical) for e in a] == \
            [(e.order, e.canonical) for e in b]
        for x, y in zip(a, b):
            assert x.features.tobytes() == y.features.tobytes()
        assert len(top) <= len(full) == res.visits
        seen.append((len(top), len(full), len(dev.measured)))
        return top

    dev._b200_entries = spy
    while dev.trials_used < dev.cfg.total_trials:
        dev.run_round()
    assert len(seen) >= 4 and seen[-1][2] > 0


def test_drop_in_device_refit_matches_host_refit(tmp_path):
    """After real rounds (device refits inside run_round), the session
    model's next refit on the device equals the reference's own host
    fit_incremental from the same state: trees, base and FitReport."""
    from schedtune.costmodel import SurrogateModel
    _, dev = _sessions(tmp_path, (16,), total_trials=64)
    for _ in range(4):
        dev.run_round()
    m = dev.model
    assert getattr(m, "_b200_refit_of", None) is m
    host = SurrogateModel(m.cfg)
    host._feat, host._thr, host._sg = list(m._feat), list(m._thr), list(m._sg)
    host._best_thr = dict(m._best_thr)
    host.base, host.fitted, host.trees = m.base, m.fitted, list(m.trees)
    ex = m.training_examples()
    rep_h = SurrogateModel.fit_incremental(host, ex)
    rep_d = m.fit_incremental(ex)
    assert (rep_d.n_examples, rep_d.loss_before, rep_d.loss_after) == \
        (rep_h.n_examples, rep_h.loss_before, rep_h.loss_after)
    assert m.base == host.base and len(m.trees) == len(host.trees)
    assert m.dump_text() == host.dump_text()


def test_drop_in_log_lines_are_json_dumps_bytes(tmp_path):
    """The fast-path trajectory lines (reward lists through
    harl_format_floats, episode_end by f-string) are byte-identical to
    json.dumps(sort_keys=True) of the same objects, as TrajectoryLogger
    writes them (tuner.py:162-164)."""
    _, dev = _sessions(tmp_path, (16,))
    for _ in range(2):
        dev.run_round()
    n = 0
    for line in open(tmp_path / "dev" / "trajectory.jsonl"):
        obj = json.loads(line)
        assert json.dumps(obj, sort_keys=True) + "\n" == line
        n += obj["event"] in ("episode_step", "episode_end")
    assert n > 0


def test_drop_in_checkpoint_from_device_rings_equals_transitions(tmp_path):
    """Checkpoints written while the replay FIFO lives on the device export
    the same buffer arrays the reference builds from Transition objects."""
    from schedtune.tuner import read_checkpoint
    _, dev = _sessions(tmp_path, (16,))
    dev.run_round()
    sg = dev.net.subgraphs[0].id
    assert dev.buffers[sg]._on_device
    p1 = str(tmp_path / "a.bin")
    dev.save(p1)
    assert dev.buffers[sg]._on_device          # no materialisation
    items = list(dev.buffers[sg].buf)           # materialise the deque
    assert not dev.buffers[sg]._on_device
    p2 = str(tmp_path / "b.bin")
    dev.save(p2)                                # the reference's own path
    assert open(p1, "rb").read() == open(p2, "rb").read()
    assert len(items) == len(dev.buffers[sg])
    dev.run_round()                             # reloads the ring from the deque
    meta, arrays = read_checkpoint(p2)
    assert meta["buffers"][sg] == len(items)
