"""Where an episode's wall time goes: CUDA events around every graph-segment
replay (the steps between host cull decisions) versus the episode total.

    python profiles/segment_probe.py [config] [P]
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
    cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    P = int(sys.argv[2]) if len(sys.argv) > 2 else None
    w = bench.build_workload(cfg_name, P)
    tb, P = w["tables"], w["P"]
    ecfg = bench.episode_config(P)
    eng = EpisodeEngine(w["agent"], w["rl"], tb.levels)
    forest = D.DeviceForest(w["trees"], w["base"], w["lr"])
    gen = np.random.default_rng(5)
    for _ in range(3):
        eng.run_episode(tb, forest, gen, ecfg, 0)
    torch.cuda.synchronize()
    orig = torch.cuda.CUDAGraph.replay
    marks = []

    def replay(self):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        orig(self)
        e1.record()
        marks.append((e0, e1, time.perf_counter()))
    torch.cuda.CUDAGraph.replay = replay
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    s0.record()
    t0 = time.perf_counter()
    eng.run_episode(tb, forest, gen, ecfg, 0)
    s1.record()
    s1.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    torch.cuda.CUDAGraph.replay = orig
    segs = [a.elapsed_time(b) for a, b, _ in marks]
    gaps = [marks[i][1].elapsed_time(marks[i + 1][0])
            for i in range(len(marks) - 1)]
    print(json.dumps({"config": cfg_name, "P": P,
                      "episode_ms_device": round(s0.elapsed_time(s1), 3),
                      "episode_ms_wall": round(wall, 3),
                      "segment_ms": [round(x, 3) for x in segs],
                      "between_segments_ms": [round(x, 3) for x in gaps],
                      "before_first_ms": round(s0.elapsed_time(marks[0][0]), 3),
                      "after_last_ms": round(marks[-1][1].elapsed_time(s1), 3)}))


if __name__ == "__main__":
    main()
