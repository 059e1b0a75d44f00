"""Helper for tests/test_gpu_graphs.py: run two graphed C2-style episodes at
a small population and print a digest of everything they leave behind
(agent parameters, Adam moments, replay ring, visited scores).  Run in a
subprocess so library switches read once per process (HARL_PPO_FUSED_ADAM)
can be compared."""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import bench
    from paper_2211_11172_b200 import device as D
    from paper_2211_11172_b200.engine import EpisodeEngine
    w = bench.build_workload("c2", 1024)
    tb = w["tables"]
    eng = EpisodeEngine(w["agent"], w["rl"], tb.levels)
    forest = D.DeviceForest(w["trees"], w["base"], w["lr"])
    gen = np.random.default_rng(3)
    cfg = bench.episode_config(1024)
    h = hashlib.sha256()
    for _ in range(3):
        r = eng.run_episode(tb, forest, gen, cfg, 0)
        h.update(r.scores().tobytes())
    torch.cuda.synchronize()
    for t in (eng.dagent.params, eng.dagent.m, eng.dagent.v, eng.replay.X,
              eng.replay.scalars):
        h.update(t.cpu().numpy().tobytes())
    print(h.hexdigest())


if __name__ == "__main__":
    main()
