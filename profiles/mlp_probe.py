"""Isolated rollout-network launches for ncu captures and CUDA-event timing
of the tensor-core kernels at a chosen population.

    python profiles/mlp_probe.py [--config c3] [--rows 65536] [--reps 5]

Builds the config's tables and a random-init agent (the bench's), a
uniform population of ``rows`` states and its features, then launches
``reps`` x (policy step [k_mlp_f16<policy> + sampler + featurize], V(X)/V(X')
[k_mlp_f16<value>] and the warm-started GBT over X' [k_gbt_predict2]) --
the launch list ncu filters with -k.  Prints per-kernel
CUDA-event times (library timer) and the algorithmic TF/s of the MLPs."""

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--rows", type=int, default=65536)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--time", action="store_true")
    ap.add_argument("--phases", action="store_true",
                    help="CTA 0 cycle accounting of the f16 kernels")
    args = ap.parse_args()
    import torch
    import bench
    from paper_2211_11172_b200 import device as D
    from paper_2211_11172_b200 import profiling
    w = bench.build_workload(args.config, args.rows, synthetic=False)
    tb = w["tables"]
    n = args.rows
    dsk = D.DeviceSketch(tb)
    dag = D.DeviceAgent(w["agent"], tb.levels)
    gen = np.random.default_rng(3)
    t, k = D.init_population(dsk, n, gen)
    X = D.featurize(dsk, t, k, n)
    Xn = torch.empty_like(X)
    v0 = torch.empty(n, dtype=torch.float32, device="cuda")
    v1 = torch.empty(n, dtype=torch.float32, device="cuda")
    out = None
    trees, base = bench.device_warm_start(tb, w["sg"].flops,
                                          np.random.default_rng(1),
                                          torch.device("cuda"))
    forest = D.DeviceForest(trees, base, 0.3)
    score = torch.empty(n, dtype=torch.float64, device="cuda")
    if args.time:
        profiling.native_timing(True)
    for _ in range(args.reps):
        out = D.policy_step(dsk, dag, X, t, k, n, gen=gen, out=out,
                            feat_out=Xn)
        D.value_pair(dag, X, n, Xn, n, v0, v1)
        D.gbt_predict(forest, Xn, n, out=score)
    torch.cuda.synchronize()
    D.raise_status(int(out["status"].item()) & ((1 << 64) - 1))
    if args.phases:
        import ctypes as C
        from paper_2211_11172_b200 import _native as N
        lib = N.load()
        buf = (C.c_ulonglong * 64)()
        out = {}
        for name, fn in (("policy", lambda: D.policy_step(
                dsk, dag, X, t, k, n, gen=gen, out=None, feat_out=Xn)),
                         ("value", lambda: D.value_pair(dag, X, n, Xn, n,
                                                        v0, v1))):
            N.check(lib.harl_debug_timestamps(3, None, 0), "dbg")
            fn()
            torch.cuda.synchronize()
            N.check(lib.harl_debug_timestamps(0, buf, 64), "dbg")
            v = list(buf)
            out[name] = {"epi_wait": v[32], "epi_hidden": v[33],
                         "epi_out_stage": v[34], "events": v[35],
                         "mma_wait": v[36], "mma_issue": v[37],
                         "epi_total": v[38]}
        print(json.dumps({"phases_cycles_cta0": out}))
    if args.time:
        kt = profiling.native_kernel_times()
        profiling.native_timing(False)
        work = bench.kernel_work(tb, 128, n)
        rep = {}
        for name, st in kt.items():
            e = {"us_per_launch": 1e3 * st["ms"] / st["launches"]}
            if name in work and work[name][0] == "tensor" and st["units"] > 0:
                e["tflops"] = work[name][1] * st["units"] / (st["ms"] * 1e-3) / 1e12
            rep[name] = e
        print(json.dumps({"config": args.config, "rows": n, "kernels": rep}))


if __name__ == "__main__":
    main()
