"""Host timeline of one drop-in call (B200TuningSession._run_episode) with
no added synchronisation: perf_counter stamps at the call's phase
boundaries, to see which host phases sit on the critical path.

    python profiles/e2e_timeline.py [--config c2] [--calls 5]
"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--calls", type=int, default=5)
    args = ap.parse_args()
    P = bench.CONFIGS[args.config]["population"]
    bench._ref_import()
    sess, sg, sketch = bench.ref_session(args.config, P, seed=0, b200=True)
    rnd = 0
    for _ in range(3):
        rnd += 1
        sess._run_episode(sg, sketch, rnd)
    torch.cuda.synchronize()
    eng = sess._b200_engines[sg.id]
    marks = []

    def wrap(obj, name):
        f = getattr(obj, name)

        def g(*a, **k):
            marks.append((name + ">", time.perf_counter()))
            r = f(*a, **k)
            marks.append(("<" + name, time.perf_counter()))
            return r
        setattr(obj, name, g)
    for o, n in ((eng.dagent, "upload"), (eng, "run_episode"),
                 (eng.dagent, "download_async"), (sess, "_b200_entries_launch"),
                 (sess, "_b200_entries"), (eng, "sync_to_host"),
                 (sess, "_b200_prepare")):
        wrap(o, n)
    out = []
    for _ in range(args.calls):
        rnd += 1
        bench.l2_flush(torch, torch.device("cuda"))
        torch.cuda.synchronize()
        marks.clear()
        t0 = time.perf_counter()
        sess._run_episode(sg, sketch, rnd)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        out.append([(n, round((t - t0) * 1e3, 3)) for n, t in marks] +
                   [("end", round((t1 - t0) * 1e3, 3))])
    print(json.dumps(out[-1]))


if __name__ == "__main__":
    main()
