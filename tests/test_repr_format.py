"""harl_format_floats (host C++, no GPU): json.dumps' float rendering
(float.__repr__, NaN / Infinity) byte for byte, on edge cases and on a
million random bit patterns."""

import json

import numpy as np

from paper_2211_11172_b200 import device as D


def _ref(v):
    return json.dumps([float(x) for x in v])[1:-1]


def test_edge_cases():
    v = np.asarray([0.0, -0.0, 1.0, -1.0, 0.1, 1e16, 1e15, 9999999999999998.0,
                    1e17, 1e-4, 1e-5, 0.00011, 123456789012345678.0, 5e-324,
                    2.2250738585072014e-308, 1.7976931348623157e308,
                    float("nan"), float("inf"), -float("inf"), 1e22, 1e23,
                    0.5, 100.0, 1e100, 1.5e-7, 3.0000000000000004, 2.0 ** 53,
                    2.0 ** 60, -123.456, 1e-300])
    assert D.format_floats(v) == _ref(v)
    assert D.format_floats(np.zeros(0)) == ""


def test_random_bit_patterns_and_rewards():
    rng = np.random.default_rng(0)
    bits = rng.integers(0, 2 ** 63, 400_000, dtype=np.uint64) | \
        (rng.integers(0, 2, 400_000, dtype=np.uint64) << np.uint64(63))
    for v in (bits.view(np.float64), rng.standard_normal(100_000) * 0.01,
              np.ldexp(1.0, rng.integers(-1074, 1023, 50_000)),
              np.round(rng.random(50_000) * 1e6) / 1e3):
        assert D.format_floats(v) == _ref(v)
        assert D.format_floats(v, threads=1) == _ref(v)
