"""bench.py's measurement bookkeeping (CPU) and its cost-model warm start
(GPU) -- the numbers the bench line reports must be derived the way
DESIGN.md §5 says."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _tables(cfg="c2"):
    return bench.build_workload(cfg, 1024, synthetic=False)["tables"]


def test_kernel_work_matches_survey_8d():
    """160,512 flop per C2 schedule (policy + 2 value
    passes), 515 B of walker+featurize bytes per C2 schedule."""
    tb = _tables("c2")
    w = bench.kernel_work(tb, 128, 16384)
    assert w["k_policy_tc"][1] + 2 * w["k_value_tc"][1] == 160512
    assert w["k_mlp_f16<policy>"] == w["k_policy_tc"]
    assert w["k_mlp_f16<value>"] == w["k_value_tc"]
    assert w["k_sample_rows"] == ("hbm", 515)        # featurizes in-kernel
    w64 = bench.kernel_work(tb, 128, 65536)
    assert w64["k_sample_rows"][1] + w64["k_featurize2"][1] - \
        (2 * tb.local_slots + 3) == 515
    tb1 = _tables("c1")
    w1 = bench.kernel_work(tb1, 128, 1024)
    assert w1["k_policy_tc"][1] + 2 * w1["k_value_tc"][1] == 148224
    assert w1["k_sample_rows"][1] == 451


def test_roofline_uses_library_rows_per_launch():
    """Rows come from the library's per-launch counts, never from a host
    span: two policy kernels sharing an episode each get only their own
    rows, and the dominant kernel is the one with the most device time."""
    tb = _tables("c2")
    peaks = {"tf32_tflops": 1000.0, "fp64_tflops": 40.0, "hbm_gbs": 6500.0}
    native = {
        "k_policy_tc": {"ms": 0.4, "launches": 20, "units": 20 * 16384},
        "k_policy_tc64": {"ms": 0.3, "launches": 40, "units": 40 * 8192},
        "k_sample_rows": {"ms": 1.0, "launches": 60,
                          "units": 20 * 16384 + 40 * 8192},
        "k_pack_heads": {"ms": 0.01, "launches": 1, "units": -1},
    }
    roof, table = bench.roofline_table(native, tb, 128, 16384, peaks, 1000)
    assert roof["kernel"] == "k_sample_rows"
    assert roof["rows_per_launch"] == pytest.approx((20 * 16384 + 40 * 8192)
                                                    / 60, rel=1e-3)
    pol = bench.kernel_work(tb, 128, 16384)["k_policy_tc"][1]
    want = pol * 20 * 16384 / 0.4e-3 / 1e12
    assert table["k_policy_tc"]["achieved"] == pytest.approx(want, rel=1e-3)
    assert table["k_policy_tc"]["frac"] == pytest.approx(want / 1000.0,
                                                         rel=1e-3)
    assert "bound" not in table["k_pack_heads"]      # no units: time only
    for ent in table.values():
        assert ent.get("frac", 0.0) < 1.0


@pytest.mark.gpu
def test_device_warm_start_matches_reference():
    """The bench's device warm start (harl_sim_time + harl_gbt_fit over 512
    uniform states) grows the reference's trees bit for bit: the same
    states from the same generator, SimulatedBackend throughputs,
    SurrogateModel.observe + fit_round."""
    try:
        bench._ref_import()
    except ImportError:
        pytest.skip("baseline/_ref not installed")
    import torch
    from schedtune.costmodel import SurrogateModel
    from schedtune.measure import MeasureRequest, SimulatedBackend
    from schedtune.schedspace import SketchContext, sample_initial_schedules
    from schedtune.workload import TargetConfig, generate_sketches
    for cfg in ("c1", "c2", "c3"):
        w = bench.build_workload(cfg, 1024, synthetic=False)
        tb = w["tables"]
        trees, base = bench.device_warm_start(
            tb, w["sg"].flops, np.random.default_rng(7),
            torch.device("cuda"))
        net = bench.ref_network(cfg)
        sg = net.subgraphs[0]
        sketch = generate_sketches(sg, TargetConfig())[
            bench.CONFIGS[cfg]["sketch"]]
        ctx = SketchContext(sg, sketch, TargetConfig())
        states = sample_initial_schedules(sketch, 512,
                                          np.random.default_rng(7))
        res = SimulatedBackend().measure_batch(
            [MeasureRequest(state=s, ctx=ctx) for s in states])
        m = SurrogateModel()
        for s, r in zip(states, res):
            m.observe(ctx.featurize(s), r.throughput, sg.id)
        m.fit_round()
        assert base == m.base
        assert len(trees) == len(m.trees) == 50
        for got, ref in zip(trees, m.trees):
            for g, r_ in zip(got, (ref.feature, ref.threshold, ref.left,
                                   ref.right, ref.value)):
                assert np.asarray(g).tobytes() == \
                    np.asarray(r_, dtype=np.asarray(g).dtype).tobytes()
