"""brute_force_best (measure.py:135-167) on the device vs the reference's
host loop: states/s, and the identical optimum where the reference can run.

    python profiles/brute_bench.py
"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))

from paper_2211_11172_b200 import device as D  # noqa: E402
from paper_2211_11172_b200 import workloads as W  # noqa: E402
from paper_2211_11172_b200.space import SketchTables  # noqa: E402

CASES = [
    ("gemm_64", "subgraphs:\n  - id: gemm_64x64x64\n    nodes: [{name: mm, "
     "kind: matmul, shape: {m: 64, k: 64, n: 64}}]\n", 2),
    ("gemm_256_l3", "subgraphs:\n  - id: gemm_256\n    nodes: [{name: mm, "
     "kind: matmul, shape: {m: 256, k: 256, n: 256}}]\n", 3),
    ("gemm_1024_l4", "subgraphs:\n  - id: gemm_1024\n    nodes: [{name: mm, "
     "kind: matmul, shape: {m: 1024, k: 1024, n: 1024}}]\n", 4),
]


def main():
    out = []
    for name, yaml, L in CASES:
        net = W.loads_network(yaml)
        tg = W.TargetConfig(tiling_levels=L)
        sg = net.subgraphs[0]
        sk = W.generate_sketches(sg, tg)[0]
        tb = SketchTables(sg, sk, tg)
        size = D.space_states(tb)
        D.brute_force_best(tb, cap=1 << 62)            # warm-up
        torch.cuda.synchronize()
        t = time.perf_counter()
        tl, kn, tm = D.brute_force_best(tb, cap=1 << 62)
        dev_s = time.perf_counter() - t
        rec = {"space": name, "states": size,
               "device_s": round(dev_s, 4),
               "device_states_per_s": round(size / dev_s),
               "optimum": tb.canonical(tl, kn), "time": repr(tm)}
        if size <= 1_000_000:
            from schedtune.measure import SimHwParams, brute_force_best
            from schedtune.schedspace import SketchContext
            from schedtune.workload import TargetConfig, generate_sketches
            from schedtune.workload import load_network
            p = "/tmp/brute_%s.yaml" % name
            open(p, "w").write(yaml)
            rnet = load_network(p)
            rtg = TargetConfig(tiling_levels=L)
            rsk = generate_sketches(rnet.subgraphs[0], rtg)[0]
            ctx = SketchContext(rnet.subgraphs[0], rsk, rtg)
            t = time.perf_counter()
            st, rt = brute_force_best(ctx, SimHwParams(), cap=1_000_000)
            ref_s = time.perf_counter() - t
            rec.update(reference_s=round(ref_s, 3),
                       reference_states_per_s=round(size / ref_s),
                       identical=st.canonical() == rec["optimum"]
                       and repr(rt) == rec["time"])
        out.append(rec)
        print(json.dumps(rec))


if __name__ == "__main__":
    main()
