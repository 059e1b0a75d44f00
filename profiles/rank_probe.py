"""Time the device rank_scores path of one C2 episode: the rank kernels,
the gather + featurize of the selection and the host copies.

    python profiles/rank_probe.py
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2211_11172_b200 import device as D  # noqa: E402
from paper_2211_11172_b200 import profiling  # noqa: E402
from paper_2211_11172_b200.engine import EpisodeEngine  # noqa: E402


def main():
    w = bench.build_workload("c2", None)
    tb, P = w["tables"], w["P"]
    eng = EpisodeEngine(w["agent"], w["rl"], tb.levels)
    forest = D.DeviceForest(w["trees"], w["base"], w["lr"])
    gen = np.random.default_rng(5)
    res = eng.run_episode(tb, forest, gen, bench.episode_config(P), 0)
    sc = D.RankScratch()
    for _ in range(3):
        res.top_entries(64, None, sc)
    torch.cuda.synchronize()
    out = {}
    t = time.perf_counter()
    for _ in range(10):
        D.rank_topk(tb, res.log_tiles, res.log_knobs, res.log_score,
                    res.visits, 64, None, sc, sort=False)
    torch.cuda.synchronize()
    out["rank_topk_ms"] = (time.perf_counter() - t) * 100
    t = time.perf_counter()
    for _ in range(10):
        res.top_entries(64, None, sc)
    torch.cuda.synchronize()
    out["top_entries_ms"] = (time.perf_counter() - t) * 100
    profiling.reset()
    profiling.native_timing(True)
    res.top_entries(64, None, sc)
    torch.cuda.synchronize()
    kt = profiling.native_kernel_times()
    profiling.native_timing(False)
    out["kernels_us"] = {k: round(v["ms"] * 1e3, 1) for k, v in kt.items()}
    out["visits"] = res.visits
    print(json.dumps(out))


if __name__ == "__main__":
    main()
