"""Host-side cost of the e2e leg's per-episode input phase (bench.py
E2EHost.episode before the episode): enqueueing the agent copies, the fp32
rollout copy, the tcgen05 image/transposition refresh and the forest
reload, each timed on the host (perf_counter, median of 20).

    python profiles/e2e_host_probe.py
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
from paper_2211_11172_b200.engine import EpisodeEngine  # noqa: E402


def main():
    w = bench.build_workload("c2", 16384)
    tb = w["tables"]
    eng = EpisodeEngine(w["agent"], w["rl"], tb.levels)
    forest = D.DeviceForest(w["trees"], w["base"], w["lr"])
    host = bench.E2EHost(eng, w, torch.device("cuda"), 16384 * 40)
    da = eng.dagent
    parts = {"copies": [], "params32": [], "refresh": [], "forest": []}
    for _ in range(20):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k, t in host.agent_in.items():
            getattr(da, k).copy_(t, non_blocking=True)
        t1 = time.perf_counter()
        da.params32.copy_(da.params)
        t2 = time.perf_counter()
        da.refresh_derived()
        t3 = time.perf_counter()
        forest.load(w["trees"], w["base"], w["lr"])
        t4 = time.perf_counter()
        for k, a, b in (("copies", t0, t1), ("params32", t1, t2),
                        ("refresh", t2, t3), ("forest", t3, t4)):
            parts[k].append((b - a) * 1e3)
    print(json.dumps({k: round(float(np.median(v)), 4) for k, v in parts.items()}))


if __name__ == "__main__":
    main()
