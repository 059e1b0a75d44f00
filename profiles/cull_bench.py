"""harl_cull_select alone on a C2-sized cull (16 K rows of a 16 K-track
population, half eliminated): microseconds per call, plus the engine's
surrounding host work (NaN scan, alive view).

    python profiles/cull_bench.py
"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_11172_b200 import _native as N  # noqa: E402


def main():
    lib = N.load(require_device=False)
    m = 16384
    rng = np.random.default_rng(0)
    adv = (rng.standard_normal(m) * 0.01).astype(np.float32).astype(np.float64)
    tracks = rng.permutation(m).astype(np.int32)
    gone = np.zeros(m // 2, np.int64)
    keep = np.zeros(m, np.int32)
    nk = C.c_int64(0)
    ts = []
    for _ in range(50):
        alive = np.ones(m, bool)
        t = time.perf_counter()
        np.isnan(adv).any()
        a8 = alive.view(np.uint8)
        lib.harl_cull_select(adv.ctypes.data, tracks.ctypes.data, m,
                             a8.ctypes.data, m, m // 2, gone.ctypes.data,
                             keep.ctypes.data, C.byref(nk))
        ts.append((time.perf_counter() - t) * 1e6)
    print(json.dumps({"us_median": round(float(np.median(ts)), 1),
                      "us_min": round(float(np.min(ts)), 1)}))


if __name__ == "__main__":
    main()
