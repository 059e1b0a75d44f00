"""Do the value pass and the next step's policy network overlap when the
policy runs on a forked stream?  Replays three captured graphs at P rows
(value alone, value then policy on one stream, value || policy on two
streams) and prints the per-replay device time of each.

    python profiles/overlap_probe.py [P]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2211_11172_b200 import device as D  # noqa: E402


def main():
    P = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    w = bench.build_workload("c2", P)
    tb = w["tables"]
    dsk = D.DeviceSketch(tb)
    dag = D.DeviceAgent(w["agent"], tb.levels)
    tiles, knobs = D.init_population(dsk, P, np.random.default_rng(1))
    X = D.featurize(dsk, tiles, knobs, P)
    v0 = torch.empty(P, dtype=torch.float32, device="cuda")
    v1 = torch.empty(P, dtype=torch.float32, device="cuda")
    side = torch.cuda.Stream()

    def value():
        D.value_pair(dag, X, 0, X, P, v0, v1, settled=True)

    def policy():
        D.policy_mlp(dsk, dag, X, P)

    def value2():
        D.value_pair(dag, X, P, X, P, v0, v1, settled=True)

    def value2p():
        D.value_pair(dag, X, P, X, P, v0, v1, settled=True, paired=True)

    def par2p():
        main = torch.cuda.current_stream()
        side.wait_stream(main)
        with torch.cuda.stream(side):
            policy()
        value2p()
        main.wait_stream(side)

    def par2():
        main = torch.cuda.current_stream()
        side.wait_stream(main)
        with torch.cuda.stream(side):
            policy()
        value2()
        main.wait_stream(side)

    def seq():
        value()
        policy()

    def par():
        main = torch.cuda.current_stream()
        side.wait_stream(main)
        with torch.cuda.stream(side):
            policy()
        value()
        main.wait_stream(side)

    out = {}
    for name, fn in (("value", value), ("policy", policy), ("seq", seq),
                     ("par", par), ("value2", value2), ("value2p", value2p),
                     ("par2", par2), ("par2p", par2p)):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            fn()
            fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(20):
                fn()
        torch.cuda.synchronize()
        for _ in range(3):
            g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        out[name] = round(e0.elapsed_time(e1) / 200 * 1e3, 2)   # us per call
    print(json.dumps({"P": P, "us_per_call": out}))


if __name__ == "__main__":
    main()
