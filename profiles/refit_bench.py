"""GBT refit timing: device harl_gbt_fit vs the reference's host
fit_incremental (baseline/_ref) on the same realistic training sets
(featurized uniform conv2d/GEMM states, SimulatedBackend targets).

    python profiles/refit_bench.py [n ...]

Prints one JSON line per n: device ms (CUDA events, after a warm-up fit),
host ms (time.perf_counter around SurrogateModel.fit_incremental), whether
the trees are identical, and the top device kernels by time."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")


def training_set(n, seed=0):
    from schedtune.measure import MeasureRequest, SimulatedBackend
    from schedtune.schedspace import SketchContext, sample_initial_schedules
    from schedtune.workload import TargetConfig, generate_sketches
    from schedtune.workload import load_network
    from schedtune.costmodel import GbtConfig, SurrogateModel
    import bench
    rng = np.random.default_rng(seed)
    model = SurrogateModel(GbtConfig(dataset_cap=max(n, 1)))
    backend = SimulatedBackend()
    tg = TargetConfig()
    p = os.path.join(ROOT, "workloads", "resnet50.yaml")
    net = load_network(p)
    sgs = net.subgraphs[:6]
    per = n // (3 * len(sgs)) + 1
    for sg in sgs:
        for sk in generate_sketches(sg, tg):
            ctx = SketchContext(sg, sk, tg)
            states = sample_initial_schedules(sk, per, rng)
            for s, r in zip(states, backend.measure_batch(
                    [MeasureRequest(s, ctx) for s in states])):
                if r.valid:
                    model.observe(ctx.featurize(s), r.throughput, sg.id)
    ex = model.training_examples()[:n]
    return model, ex


def main():
    import torch
    from paper_2211_11172_b200 import device as D
    from paper_2211_11172_b200 import profiling
    from schedtune.costmodel import SurrogateModel
    ns = [int(a) for a in sys.argv[1:]] or [1024, 4096, 10000]
    for n in ns:
        model, ex = training_set(n)
        X = np.stack([e.features for e in ex])
        y = np.asarray([e.target for e in ex])
        Xd = torch.from_numpy(X).cuda()
        D.gbt_fit(Xd, y)                       # warm-up (allocations)
        torch.cuda.synchronize()
        profiling.reset()
        profiling.native_timing(True)
        D.gbt_fit(Xd, y)
        torch.cuda.synchronize()
        kt = profiling.native_kernel_times()
        profiling.native_timing(False)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fit = D.gbt_fit(Xd, y)
        e1.record()
        e1.synchronize()
        dev_ms = e0.elapsed_time(e1)
        host = SurrogateModel(model.cfg)
        t = time.perf_counter()
        SurrogateModel.fit_incremental(host, ex)
        host_ms = (time.perf_counter() - t) * 1e3
        same = len(host.trees) == len(fit.trees) and all(
            all(np.asarray(a).tobytes() == np.asarray(b, np.asarray(a).dtype).tobytes()
                for a, b in zip(ft, (ht.feature, ht.threshold, ht.left,
                                     ht.right, ht.value)))
            for ft, ht in zip(fit.trees, host.trees)) and fit.base == host.base
        top = sorted(kt.items(), key=lambda kv: -kv[1]["ms"])[:6]
        print(json.dumps({"n": len(y), "features": X.shape[1],
                          "trees": len(fit.trees), "device_ms": round(dev_ms, 2),
                          "host_ms": round(host_ms, 1),
                          "speedup": round(host_ms / dev_ms, 1),
                          "identical": bool(same),
                          "device_kernels_ms (timed pass, incl. per-launch spin)":
                              {k: round(v["ms"], 3) for k, v in top}}))


if __name__ == "__main__":
    main()
