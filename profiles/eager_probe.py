"""Device time of a C2 episode with eager launches (use_graphs=False, the
sharded engine's launch mode) against the graphed default.

    python profiles/eager_probe.py
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2211_11172_b200 import device as D  # noqa: E402
from paper_2211_11172_b200.engine import EpisodeEngine  # noqa: E402


def main():
    w = bench.build_workload("c2", None)
    tb, P = w["tables"], w["P"]
    cfg = bench.episode_config(P)
    forest = D.DeviceForest(w["trees"], w["base"], w["lr"])
    out = {}
    for graphs in (True, False):
        eng = EpisodeEngine(w["agent"], w["rl"], tb.levels, use_graphs=graphs)
        gen = np.random.default_rng(5)
        for _ in range(3):
            eng.run_episode(tb, forest, gen, cfg, 0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            eng.run_episode(tb, forest, gen, cfg, 0)
        e1.record()
        torch.cuda.synchronize()
        out["graphs" if graphs else "eager"] = round(e0.elapsed_time(e1) / 5, 3)
    print(json.dumps({"ms_per_episode": out}))


if __name__ == "__main__":
    main()
