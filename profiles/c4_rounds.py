"""Per-round timeline of the C4 drop-in session (one GPU): which subgraph
each round picked, the episode's device-synchronised time, the round's
wall time, and whether the episode replayed captured graphs.

    python profiles/c4_rounds.py [rounds] [P]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 13
    P = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    bench._ref_import()
    import torch
    sess, _ = bench.taskset_session("b200", P, 0, 1, rounds + 1)
    orig = sess._run_episode
    info = {}

    def timed(sg, sketch, rnd):
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = orig(sg, sketch, rnd)
        torch.cuda.synchronize()
        info["ep_ms"] = (time.perf_counter() - t) * 1e3
        info["sg"] = sg.id
        eng = sess._b200_engines.get(sg.id)
        if eng is not None:
            info["graphed"] = [bool(b.graphs) for b in eng._cache.values()]
            info["uses"] = [getattr(b, "uses", 0) for b in eng._cache.values()]
        return out
    sess._run_episode = timed
    for r in range(rounds):
        info.clear()
        t = time.perf_counter()
        sess.run_round()
        torch.cuda.synchronize()
        info["round_ms"] = round((time.perf_counter() - t) * 1e3, 2)
        info["ep_ms"] = round(info.get("ep_ms", 0.0), 2)
        info["round"] = r
        print(json.dumps(info), flush=True)


if __name__ == "__main__":
    main()
