"""cProfile of one eager C2 episode (use_graphs=False: the sharded mode's
launch path): the host-side cost per launch.

    python profiles/eager_cprofile.py
"""
import cProfile
import io
import os
import pstats
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
    eng = EpisodeEngine(w["agent"], w["rl"], tb.levels, use_graphs=False)
    gen = np.random.default_rng(5)
    for _ in range(3):
        eng.run_episode(tb, forest, gen, cfg, 0)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    eng.run_episode(tb, forest, gen, cfg, 0)
    torch.cuda.synchronize()
    pr.disable()
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
    print(s.getvalue())


if __name__ == "__main__":
    main()
