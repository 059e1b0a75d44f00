"""Host-side phases of one graphed C2 episode (perf_counter around the
engine's host steps), to size the GPU-idle bubbles the segment probe sees.

    python profiles/host_probe.py
"""
import json
import os
import sys
import time
from collections import defaultdict

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2211_11172_b200 import device as D  # noqa: E402
from paper_2211_11172_b200 import engine as E  # noqa: E402


def main():
    w = bench.build_workload("c2", None)
    tb, P = w["tables"], w["P"]
    eng = E.EpisodeEngine(w["agent"], w["rl"], tb.levels)
    forest = D.DeviceForest(w["trees"], w["base"], w["lr"])
    gen = np.random.default_rng(5)
    cfg = bench.episode_config(P)
    for _ in range(3):
        eng.run_episode(tb, forest, gen, cfg, 0)
    torch.cuda.synchronize()
    acc = defaultdict(float)

    def wrap(obj, name, label):
        f = getattr(obj, name)

        def g(*a, **k):
            t = time.perf_counter()
            r = f(*a, **k)
            acc[label] += (time.perf_counter() - t) * 1e3
            return r
        setattr(obj, name, g)
    wrap(D, "init_population", "init_population (incl. sync)")
    wrap(D, "featurize", "featurize launch")
    wrap(D, "gbt_predict", "gbt launch")
    wrap(eng, "_cull_inputs", "cull D2H (incl. wait for segment)")
    wrap(eng, "_cull", "cull host")
    wrap(torch.cuda.CUDAGraph, "replay", "graph replay calls")
    E._HOST_TRACE = trace = []
    torch.cuda.synchronize()
    t = time.perf_counter()
    eng.run_episode(tb, forest, gen, cfg, 0)
    torch.cuda.synchronize()
    acc["episode total"] = (time.perf_counter() - t) * 1e3
    E._HOST_TRACE = None
    print(json.dumps({k: round(v, 3) for k, v in acc.items()}))
    print(json.dumps([(a, k0, k1, round((tt - t) * 1e3, 3))
                      for a, k0, k1, tt in trace]))


if __name__ == "__main__":
    main()
