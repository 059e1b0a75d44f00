"""Phase timeline of CTA 0 of the wide tcgen05 policy kernel (globaltimer
timestamps, harl_debug_timestamps) for one rollout step at P rows.

    python profiles/phase_probe.py [P]
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2211_11172_b200 import _native as N  # noqa: E402
from paper_2211_11172_b200 import device as D  # noqa: E402
from paper_2211_11172_b200.engine import EpisodeConfig, EpisodeEngine  # noqa: E402

NAMES = ["start", "init", "x_staged", "bias_ready", "mma_weights_ready",
         "first_issue", "first_done", "-", "-", "loop_end", "end"]
SNAMES = ["start", "rng", "state", "softmax", "cdf", "shift_heads", "decided", "end"]
GNAMES = ["start", "x0", "walk0", "sum0", "x1", "walk1", "sum1"]
FNAMES = ["start", "staged", "rows", "end"]
ANAMES = ["start", "bad_checked", "updated", "end"]
WNAMES = ["start", "staged0", "summed"]
PNAMES = ["start", "gather", "pol_fwd", "heads", "val_fwd", "terms", "pol_bwd", "val_bwd", "end"]


def main():
    P = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    w = bench.build_workload("c2", P)
    tb = w["tables"]
    forest = D.DeviceForest(w["trees"], w["base"], w["lr"])
    graphs = len(sys.argv) > 2 and sys.argv[2] == "graph"
    eng = EpisodeEngine(w["agent"], w["rl"], tb.levels, use_graphs=graphs)
    cfg = EpisodeConfig(tracks=P, track_len=2, cull_window=20,
                        cull_fraction=0.5, min_tracks=P // 2)
    cfg1 = EpisodeConfig(tracks=P, track_len=1, cull_window=20,
                         cull_fraction=0.5, min_tracks=P // 2)
    lib = N.load()
    gen = np.random.default_rng(0)
    for rep in range(3):
        N.check(lib.harl_debug_timestamps(2 if rep == 2 else 1, None, 0), "dbg")
        eng.run_episode(tb, forest, gen, cfg1 if graphs else cfg, 0)
        torch.cuda.synchronize()
        ts = np.zeros(64, dtype=np.uint64)
        N.check(lib.harl_debug_timestamps(0, ts.ctypes.data_as(C.c_void_p), 64), "dbg")
        for nm, lo, names in (("policy", 0, NAMES), ("sample", 16, SNAMES),
                              ("gbt", 24, GNAMES), ("featurize", 32, FNAMES),
                              ("ppo_rows", 40, PNAMES), ("adam", 50, ANAMES),
                              ("wgrad", 54, WNAMES)):
            t = ts[lo:lo + len(names)].astype(np.int64)
            rel = (t - t[0]) / 1e3
            print(f"rep {rep} {nm}: " + " ".join(f"{n}={r:.2f}" for n, r in zip(names, rel)))
            if nm == "sample":   # featurize inside the sampler ends at 31
                print(f"rep {rep} sample " + " ".join(
                    f"{n}={(int(ts[i]) - int(ts[16])) / 1e3:.2f}" for n, i in
                    (("fill_start", 38), ("fill_done", 39), ("fill_synced", 36),
                     ("feat_zeroed", 32), ("feat_lut", 33), ("feat_row", 34),
                     ("feat_barrier", 35), ("featurized", 31))))
        t = ts[57:60].astype(np.int64)
        print(f"rep {rep} ppo_cl exchange: push={(t[1]-t[0])/1e3:.2f} sync={(t[2]-t[1])/1e3:.2f}")
        if rep == 2:
            a0, a1, b0, b1 = (int(x) for x in ts[60:64])
            print(f"sampler grid {(a1 - a0) / 1e3:.2f} us, gap to featurize "
                  f"{(b0 - a1) / 1e3:.2f} us, featurize grid {(b1 - b0) / 1e3:.2f} us")


if __name__ == "__main__":
    main()
