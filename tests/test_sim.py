"""The analytic measurement model (measure.py:78-167): the oracle's
simulate_time / brute_force_best restatement and the device kernels against
the reference's own values (tests/golden/sim_golden.json, recorded by
make_golden.py with the workload texts it used: 27 sketches x 40 states
under default and custom SimHwParams, and the GEMM-64 optima)."""

import json
import os

import pytest

from golden_util import GOLDEN
from oracle import harl_oracle as O
from paper_2211_11172_b200 import workloads as W
from paper_2211_11172_b200.space import SketchTables


def _golden():
    with open(os.path.join(GOLDEN, "sim_golden.json")) as fh:
        return json.load(fh)


def _tables(g, case):
    net = W.loads_network(g["yaml"][case["workload"]])
    target = W.TargetConfig(**{k: (tuple(v) if isinstance(v, list) else v)
                               for k, v in case["target"].items()})
    sg = net.subgraphs[case["sg"]]
    ks = W.generate_sketches(sg, target)
    S = max(k.space.num_tile_slots for k in ks)
    return SketchTables(sg, ks[case["sketch"]], target, S)


def _params(g, name):
    p = dict(g["params"][name])
    if "unroll_factors" in p:
        p["unroll_factors"] = tuple(tuple(x) for x in p["unroll_factors"])
    return p


@pytest.mark.parametrize("pname", ["default", "custom"])
def test_oracle_simulate_time_matches_reference(pname):
    g = _golden()
    prm = _params(g, pname)
    assert len(g["cases"]) >= 20
    for case in g["cases"]:
        tb = _tables(g, case)
        tiles, knobs = tb.arrays_from_canonical(case["states"])
        for t, k, want in zip(tiles, knobs, case[pname]):
            assert repr(O.sim_time(tb, t, k, prm)) == want, \
                (case["workload"], case["sketch"])


def test_oracle_brute_force_matches_reference():
    g = _golden()
    for rec in g["brute"]:
        tb = _tables(g, rec)
        t, k, tm = O.brute_force_best(tb, _params(g, rec["params"]))
        assert tb.canonical(t, k) == rec["state"] and repr(tm) == rec["time"]


@pytest.mark.gpu
@pytest.mark.parametrize("pname", ["default", "custom"])
def test_device_simulate_time_bit_exact(pname):
    from paper_2211_11172_b200 import device as D
    g = _golden()
    prm = _params(g, pname)
    for case in g["cases"]:
        tb = _tables(g, case)
        tiles, knobs = tb.arrays_from_canonical(case["states"])
        dt, dk = D.states_to_device(tb, tiles, knobs)
        out = D.simulate_time(D.DeviceSketch(tb), dt, dk, len(knobs), prm)
        got = [repr(float(x)) for x in out.cpu().numpy()]
        assert got == case[pname], (case["workload"], case["sketch"])


@pytest.mark.gpu
def test_device_brute_force_matches_reference():
    from paper_2211_11172_b200 import device as D
    g = _golden()
    for rec in g["brute"]:
        tb = _tables(g, rec)
        t, k, tm = D.brute_force_best(tb, _params(g, rec["params"]))
        assert tb.canonical(t, k) == rec["state"] and repr(tm) == rec["time"]


@pytest.mark.gpu
def test_device_brute_force_refuses_large_spaces():
    from paper_2211_11172_b200 import device as D
    from paper_2211_11172_b200.errors import SpaceTooLarge
    g = _golden()
    tb = _tables(g, g["brute"][0])
    with pytest.raises(SpaceTooLarge):
        D.brute_force_best(tb, cap=100)
