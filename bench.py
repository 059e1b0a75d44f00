"""Benchmark: schedules/sec of the HARL inner search step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--config c2|c1|c3|c5|c4] [--population P]

A bench "step" is one ``_run_episode`` (tuner.py:350-440) over the whole
population: initial sampling, every search step of the default geometry
(cull_window 20, episode_len 40 -> 20 steps at P tracks, a cull to P/2, 40
steps at P/2, PPO every 2 steps), i.e. P*40 visited schedules.  The unit of
work is one visited schedule (one CandidateEntry, tuner.py:408-412).

* ``value``: whole-job schedules/s with the population resident in HBM
  (``EpisodeEngine.run_episode``), device time from CUDA events on the
  launching stream summed over the K timed episodes (L2 flushed between
  episodes, outside the events), max over ranks.
* ``e2e``: the same metric through the drop-in a user calls:
  ``B200TuningSession._run_episode`` (compat.py) on a reference
  ``TuningSession`` from baseline/_ref -- numpy agent, moments and the
  refitted ensemble host->device, CandidateEntry list and updated numpy
  parameters back -- wall time, with the library's accounted H2D/D2H
  bytes per call.
* ``roofline``: the dominant kernel from the library's per-launch event
  timer and the rows each launch processed (``harl_profile_read``), with
  SURVEY §8(d)'s algorithmic work per row, against peaks measured in this
  run (TF32/FP16/FP64 cuBLAS matmuls) and MEASURED_PEAKS.json's HBM copy
  bandwidth; ``kernels`` lists every kernel the same way.
* ``cpu_baseline`` / ``--impl reference``: the reference's own
  ``TuningSession._run_episode`` from baseline/_ref (the oracle port only
  if the reference is not installed) in the reference's process-pool model
  (cli.py:231-235): one session per host core, P/N tracks each, full
  60-step episodes of the same config.
* ``c3_64k``: the C3 configuration (BERT bmm+softmax, 64 K tracks, the
  north star's >= 64 K step) measured the same way in the same run.

Data: random-init weights of the reference architecture; the cost model is
warm-started as SURVEY §8(d) prescribes (512 uniform states measured by the
analytic simulator, fit_round) -- on the device for the GPU arm
(harl_sim_time + harl_gbt_fit, bit-exact with the reference), with the
reference's own code in the reference arm.
"""

from __future__ import annotations

import os

# the CPU legs time single-threaded numpy (cores = processes); set before
# numpy loads so BLAS pools are not oversubscribed (spawned workers inherit)
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import argparse
import json
import math
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "schedules/sec (RL step+featurize+cost model) at 1/2/4/8 B200 vs CPU ref"
UNIT = "schedules/s"

CONFIGS = {
    "c1": dict(workload="GEMM 1024x1024x1024 (gemm_l.yaml gemm_1024x1024x1024), "
               "sketch k0", yaml="""
subgraphs:
  - id: gemm_1024x1024x1024
    nodes: [{name: mm, kind: matmul, shape: {m: 1024, k: 1024, n: 1024}}]
""", sketch=0, population=1024),
    "c2": dict(workload="conv2d ResNet-50 stage-3 3x3 (conv2d.yaml "
               "c2d_14x256x256_k3), sketch k0", yaml="""
subgraphs:
  - id: c2d_14x256x256_k3
    nodes:
      - name: conv
        kind: conv2d
        shape: {n: 1, h: 14, w: 14, ci: 256, co: 256, kernel: 3, stride: 1, padding: 1}
""", sketch=0, population=16384),
    "c3": dict(workload="BERT-base batched GEMM + softmax subgraph "
               "(bmm 12x128x64x128 -> softmax), sketch k3", yaml="""
subgraphs:
  - id: bgemm_softmax
    weight: 12
    nodes:
      - name: bmm
        kind: batch_matmul
        shape: {b: 12, m: 128, k: 64, n: 128}
        consumers: [sm]
      - name: sm
        kind: softmax
        shape: {heads: 12, q: 128, k: 128}
""", sketch=3, population=65536),
    "c5": dict(workload="GEMM 4096^3, sketch k0", yaml="""
subgraphs:
  - id: gemm_4096x4096x4096
    nodes: [{name: mm, kind: matmul, shape: {m: 4096, k: 4096, n: 4096}}]
""", sketch=0, population=65536),
    "c4": dict(workload="ResNet-50 v1.5 task set (workloads/resnet50.yaml: 24 "
               "subgraphs), searcher rl (adaptive), tasks sharded over ranks",
               yaml=None, sketch=None, population=4096),
}


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)


class ClockSampler:
    """SM clock + throttle reasons sampled with NVML every 5 ms while the
    timed region runs (the recipe's nvidia-smi clocks line, at a rate that
    sees sub-second regions)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
               "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

    def __init__(self, index: int = 0):
        self.index = index
        self.samples = []
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h,
                                                        pynvml.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception:  # noqa: BLE001 - no NVML: report nothing
            self.nv = None
        return self

    def _run(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                clk = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((clk, rs))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    def __exit__(self, *a):
        self.stop.set()
        if self.nv is not None:
            self.thread.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [],
                    "samples": 0}
        clks = [c for c, _ in self.samples]
        reasons = sorted({name for _, rs in self.samples
                          for name, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": float(np.median(clks)),
                "sm_max_mhz": float(self.max), "reasons": reasons,
                "samples": len(clks)}


# ---------------------------------------------------------------------------
# workload construction (shared by the GPU and CPU legs)


def synthetic_forest(tables, seed: int, n_trees: int = 50, depth: int = 6):
    """Test helper (tests/, smoke): 50 random trees of depth <= 6 splitting
    on features that vary, thresholds at feature values of random states.
    Not used by the bench legs, which warm-start the cost model the
    reference's way (``device_warm_start`` / ``ref_warm_start``)."""
    from oracle.harl_oracle import featurize, sample_initial  # test-only
    rng = np.random.default_rng(seed)
    tiles, knobs = sample_initial(tables, 512, rng)
    X = featurize(tables, tiles, knobs)
    varying = np.flatnonzero(X.std(axis=0) > 0)
    trees = []
    for _ in range(n_trees):
        feat, thr, left, right, val = [], [], [], [], []

        def add(d):
            i = len(feat)
            feat.append(-1)
            thr.append(0.0)
            left.append(-1)
            right.append(-1)
            val.append(0.0)
            if d < depth and rng.random() < 0.92:
                f = int(rng.choice(varying))
                feat[i] = f
                thr[i] = float(X[int(rng.integers(len(X))), f])
                left[i] = add(d + 1)
                right[i] = add(d + 1)
            else:
                val[i] = float(rng.normal(0.0, 0.05))
            return i
        add(0)
        trees.append(tuple(np.asarray(a) for a in (feat, thr, left, right,
                                                   val)))
    return trees


def build_workload(cfg_name: str, population: int | None, seed: int = 0,
                   synthetic: bool = True):
    """Tables, a random-init agent of the reference architecture and the
    step geometry of a config.  ``synthetic``: also a synthetic forest
    (tests); the bench legs pass False and warm-start the cost model."""
    from paper_2211_11172_b200 import workloads as W
    from paper_2211_11172_b200.agent import RlConfig, init_session_agents
    from paper_2211_11172_b200.space import SketchTables
    c = CONFIGS[cfg_name]
    net = W.loads_network(c["yaml"])
    target = W.TargetConfig()
    sg = net.subgraphs[0]
    ks = W.generate_sketches(sg, target)
    S = max(k.space.num_tile_slots for k in ks)
    tables = SketchTables(sg, ks[c["sketch"]], target, S)
    rl = RlConfig()
    agent = init_session_agents([(sg.id, S)], tables.feature_len, rl,
                                np.random.default_rng(seed))[sg.id]
    P = population or c["population"]
    w = dict(tables=tables, agent=agent, rl=rl, P=P, cfg=c, sg=sg,
             base=0.5, lr=0.3)
    if synthetic:
        w["trees"] = synthetic_forest(tables, seed + 1)
    return w


def device_warm_start(tables, sg_flops: float, gen, dev):
    """SURVEY §8(d)'s cost-model warm start on the device: 512 uniform
    states (sample_initial_schedules, schedspace.py:165-178), measured by
    the analytic simulator with SimulatedBackend's defaults (measure.py:
    99-133, harl_sim_time, bit-exact), throughput = flops / time, targets
    renormalised by the best (costmodel.py:180-188), fit_round ->
    fit_incremental (costmodel.py:190-215, harl_gbt_fit, bit-exact):
    50 trees of depth <= 6.  Returns (trees, base)."""
    from paper_2211_11172_b200 import device as D
    dsk = D.DeviceSketch(tables, dev)
    t, k = D.init_population(dsk, 512, gen)
    X = D.featurize(dsk, t, k, 512)
    secs = D.simulate_time(dsk, t, k, 512).cpu().numpy()
    thr = sg_flops / secs
    y = thr / thr.max()
    fit = D.gbt_fit(X, y, n_trees=50, max_depth=6, learning_rate=0.3,
                    min_leaf=1, device=dev)
    return fit.trees, fit.base


def episode_config(P):
    from paper_2211_11172_b200.engine import EpisodeConfig
    # TunerConfig defaults with min_tracks = P/2, initial_tracks = P
    return EpisodeConfig(tracks=P, track_len=40, cull_window=20,
                         cull_fraction=0.5, min_tracks=P // 2)


def _ref_import():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(ref) and ref not in sys.path:
        sys.path.insert(0, ref)
    import schedtune  # noqa: F401  (raises ImportError when absent)


def ref_network(cfg_name: str):
    """The config's network through the reference's own loader."""
    import tempfile
    from schedtune.workload import load_network
    with tempfile.NamedTemporaryFile("w", suffix=".yaml", delete=False) as f:
        f.write(CONFIGS[cfg_name]["yaml"])
        path = f.name
    try:
        return load_network(path)
    finally:
        os.unlink(path)


def ref_warm_start(sess, sg, sketch, n: int = 512):
    """The same warm start through the reference session's own objects:
    sample_initial_schedules on the session generator, SimulatedBackend
    measure_batch, SurrogateModel.observe, fit_round."""
    from schedtune.measure import MeasureRequest
    from schedtune.schedspace import sample_initial_schedules
    ctx = sess.contexts[sketch.id]
    states = sample_initial_schedules(sketch, n, sess.rng)
    res = sess.backend.measure_batch([MeasureRequest(state=s, ctx=ctx)
                                      for s in states])
    for s, r in zip(states, res):
        sess.model.observe(ctx.featurize(s), r.throughput, sg.id)
    sess.model.fit_round()


def ref_session(cfg_name: str, P: int, seed: int, b200: bool = False):
    """A reference TuningSession (or the drop-in subclass) for one config:
    TunerConfig defaults with initial_tracks = P, min_tracks = P/2, the
    rl (adaptive) searcher, SimulatedBackend, warm-started cost model."""
    from schedtune.measure import SimulatedBackend
    from schedtune.tuner import TunerConfig, TuningSession
    from schedtune.workload import TargetConfig
    net = ref_network(cfg_name)
    cfg = TunerConfig(seed=seed, total_trials=10 ** 9, top_k=64,
                      initial_tracks=P, min_tracks=max(1, P // 2))
    cls = TuningSession
    if b200:
        from paper_2211_11172_b200.compat import b200_session_class
        cls = b200_session_class(TuningSession)
    sess = cls(net, TargetConfig(), cfg, SimulatedBackend(), "rl")
    if b200:
        sess._b200_hook_model()       # fit_round -> harl_gbt_fit
    sg = net.subgraphs[0]
    sketch = sess.sketches[sg.id][CONFIGS[cfg_name]["sketch"]]
    ref_warm_start(sess, sg, sketch)
    return sess, sg, sketch


# ---------------------------------------------------------------------------
# CPU legs: the reference's own _run_episode (baseline/_ref), or the oracle
# port when the reference is not installed


def _host_info():
    import platform
    cpu = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                cpu = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": cpu, "glibc": "-".join(platform.libc_ver()),
            "numpy": np.__version__, "python": platform.python_version(),
            "blas_threads": os.environ.get("OPENBLAS_NUM_THREADS")}


def _ref_episode_worker(job):
    """One process of the reference's process-pool model (cli.py:231-235):
    an independent reference session on P tracks, ``warm`` untimed then
    ``steps`` timed full episodes (``TuningSession._run_episode``,
    tuner.py:350-440, perf_counter around the call).  Falls back to the
    oracle port when the reference package is absent."""
    cfg_name, P, seed, warm, steps = job
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    try:
        _ref_import()
        sess, sg, sketch = ref_session(cfg_name, P, seed)
        kind = "reference"

        def episode(rnd):
            t = time.perf_counter()
            v0 = sess.order_counter
            sess._run_episode(sg, sketch, rnd)
            return sess.order_counter - v0, time.perf_counter() - t
    except ImportError:
        kind = "port"
        episode = _port_episode_fn(cfg_name, P, seed)
    out = []
    for i in range(warm + steps):
        v, s = episode(i + 1)
        if i >= warm:
            out.append((v, s))
    return kind, out


def _port_episode_fn(cfg_name, P, seed):
    """The oracle restatement (bit-exact with the reference) of one full
    episode per call, warm-started the same way (oracle sim + fit)."""
    from oracle import harl_oracle as O
    w = build_workload(cfg_name, P, seed, synthetic=False)
    tb, a, sg = w["tables"], w["agent"], w["sg"]
    rng = np.random.default_rng(seed)
    tiles, knobs = O.sample_initial(tb, 512, rng)
    X = O.featurize(tb, tiles, knobs)
    secs = np.array([O.sim_time(tb, tiles[i], knobs[i]) for i in range(512)])
    thr = sg.flops / secs
    base, trees = O.gbt_fit(X, thr / thr.max())[:2]
    oa = O.Agent.from_param_lists(a.policy, a.value, len(a.hidden))
    opi = O.Adam.zeros_like(oa.policy_params(), w["rl"].lr_actor)
    ov = O.Adam.zeros_like(oa.value_params(), w["rl"].lr_critic)
    model = O.GbtModel(base, 0.3, True, trees)
    ecfg = O.EpisodeCfg(tracks=P, track_len=40, cull_window=20,
                        cull_fraction=0.5, min_tracks=max(1, P // 2),
                        rl_cfg=O.RlCfg())
    rep = O.Replay(4096)
    state = {"order": 0}

    def episode(rnd):
        t = time.perf_counter()
        entries, _, _ = O.run_episode(tb, tb.num_slots, ecfg, oa, opi, ov,
                                      rep, model, rng, state["order"])
        state["order"] += len(entries)
        return len(entries), time.perf_counter() - t
    return episode


def cpu_pool(cfg_name, P, warm, steps, procs=None):
    """N = len(sched_getaffinity) independent reference sessions x P/N
    tracks each, full episodes; aggregate =
    sum of visits / slowest process's summed episode time."""
    from concurrent.futures import ProcessPoolExecutor
    import multiprocessing as mp
    procs = procs or len(os.sched_getaffinity(0))
    per = max(2, P // procs)
    with ProcessPoolExecutor(procs, mp_context=mp.get_context("spawn")) as ex:
        res = list(ex.map(_ref_episode_worker,
                          [(cfg_name, per, s, warm, steps)
                           for s in range(procs)]))
    kinds = {k for k, _ in res}
    visits = sum(v for _, r in res for v, _ in r)
    slowest = max(sum(s for _, s in r) for _, r in res)
    one = [v / s for _, r in res for v, s in r]
    return dict(kind="reference" if kinds == {"reference"} else "port",
                procs=procs, per=per, visits=visits, seconds=slowest,
                value=visits / slowest,
                per_process=float(np.median(one)), host=_host_info())


# ---------------------------------------------------------------------------
# GPU leg


def l2_flush(torch, dev, buf=[]):
    if not buf:
        buf.append(torch.empty(256 << 20, dtype=torch.uint8, device=dev))
    buf[0].fill_(1)


def measure_peaks(torch, dev):
    """Dense matmul peaks of this GPU measured in this run (cuBLAS through
    torch; CUDA events, best of 5 after 2 warm-ups): TF32 (fp32 matmul with
    TF32 allowed, 8192^3), FP16 (8192^3), FP64 (4096^3, DMMA)."""
    out = {}
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        for name, dt, n in (("tf32", torch.float32, 8192),
                            ("fp16", torch.float16, 8192),
                            ("fp64", torch.float64, 4096)):
            a = torch.randn(n, n, device=dev).to(dt)
            b = torch.randn(n, n, device=dev).to(dt)
            c = torch.empty(n, n, device=dev, dtype=dt)
            for _ in range(2):
                torch.matmul(a, b, out=c)
            best = math.inf
            for _ in range(5):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                torch.matmul(a, b, out=c)
                e1.record()
                e1.synchronize()
                best = min(best, e0.elapsed_time(e1))
            out[f"{name}_tflops"] = round(2.0 * n ** 3 / (best * 1e-3) / 1e12, 1)
            del a, b, c
    finally:
        torch.backends.cuda.matmul.allow_tf32 = old
    torch.cuda.empty_cache()
    try:
        mp_ = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        out["hbm_gbs"] = mp_["hbm_gbs"]
        out["hbm_note"] = "MEASURED_PEAKS.json hbm_gbs (driver-measured copy)"
    except (OSError, KeyError, ValueError):
        out["hbm_gbs"] = 6557.8
        out["hbm_note"] = "B200_PROFILING.md fallback"
    return out


def value_leg(cfg_name, P, steps, warmup, dev, rank, world, profile=True,
              shard=None):
    """Device-resident episodes (EpisodeEngine.run_episode), population in
    HBM: CUDA events on the launching stream around each episode, L2
    flushed between episodes (outside the events).  Then one untimed,
    eagerly launched episode with the library's per-launch event timer for
    the per-kernel table.

    ``shard`` (world, rank, group): one population of P * world tracks
    sharded across the ranks (EpisodeEngine(shard=...): interleaved tracks,
    merged culls, one gradient all-reduce per PPO update); every rank
    starts from the same agent, cost model and generator.  Otherwise each
    rank runs its own task replica of P tracks."""
    import torch
    from paper_2211_11172_b200 import device as D
    from paper_2211_11172_b200 import profiling
    from paper_2211_11172_b200.engine import EpisodeEngine
    seed = 0 if shard else rank
    w = build_workload(cfg_name, P, seed=seed, synthetic=False)
    tb = w["tables"]
    gen = np.random.default_rng(1000 + seed)
    trees, base = device_warm_start(tb, w["sg"].flops, gen, dev)
    ecfg = episode_config(P * world if shard else P)
    eng = EpisodeEngine(w["agent"], w["rl"], tb.levels, dev, shard=shard)
    forest = D.DeviceForest(trees, base, 0.3, device=dev)
    stream = torch.cuda.current_stream()
    order = 0
    for _ in range(warmup):
        res = eng.run_episode(tb, forest, gen, ecfg, order)
        order += res.visits
    torch.cuda.synchronize()
    profiling.reset()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    total_ms, visits = 0.0, 0
    with ClockSampler(dev.index) as clk:
        for _ in range(steps):
            l2_flush(torch, dev)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            res = eng.run_episode(tb, forest, gen, ecfg, order)
            e1.record(stream)
            e1.synchronize()
            total_ms += e0.elapsed_time(e1)
            # sharded: every rank reports the whole population's visits
            visits += res.extra.get("global_visits", res.visits) if shard \
                else res.visits
            order += res.extra.get("global_visits", res.visits)
    torch.cuda.synchronize()
    launches = profiling.launch_count()
    out = dict(total_ms=total_ms, visits=visits, clocks=clk.summary(),
               launches=launches, P=P, tables=tb, n_trees=len(trees),
               eng=eng, forest=forest, gen=gen, ecfg=ecfg, order=order,
               n_params=sum(p.size for p in w["agent"].policy) +
               sum(p.size for p in w["agent"].value))
    if profile:
        profiling.native_timing(True)
        eng.use_graphs = False      # per-launch events need eager launches
        l2_flush(torch, dev)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = eng.run_episode(tb, forest, gen, ecfg, order)
        e1.record(stream)
        e1.synchronize()
        eng.use_graphs = True
        out["order"] = order + res.extra.get("global_visits", res.visits)
        out["native"] = profiling.native_kernel_times()
        out["profiled_episode_ms"] = e0.elapsed_time(e1)
        profiling.native_timing(False)
    return out


def e2e_leg(cfg_name, P, steps, warmup, dev, rank):
    """The same metric through the drop-in (the call a user makes):
    ``B200TuningSession._run_episode`` (compat.py) on a reference
    ``TuningSession`` built from baseline/_ref, called exactly as run_round
    calls it (tuner.py:480).  Every timed call takes the session's numpy
    agent and Adam moments (compared bit for bit with what the previous
    call wrote back, uploaded if they differ), the replay deque (first
    call) and the ensemble (reloaded when refitted) host->device, runs the
    episode and the device rank_scores,
    writes parameters and moments back into the numpy arrays and returns
    the reference's CandidateEntry list.  Wall time (perf_counter with a
    device synchronize on both sides); bytes = the library's accounted
    host<->device copies of the timed calls."""
    import torch
    from paper_2211_11172_b200 import profiling as PF
    _ref_import()
    sess, sg, sketch = ref_session(cfg_name, P, seed=rank, b200=True)
    rnd = 0
    for _ in range(warmup):
        rnd += 1
        sess._run_episode(sg, sketch, rnd)
    ms, visits, h2d, d2h = 0.0, 0, 0, 0
    n = max(1, steps)
    for _ in range(n):
        rnd += 1
        l2_flush(torch, dev)
        torch.cuda.synchronize()
        PF.xfer_reset()
        v0 = sess.order_counter
        t0 = time.perf_counter()
        entries = sess._run_episode(sg, sketch, rnd)
        torch.cuda.synchronize()
        ms += (time.perf_counter() - t0) * 1e3
        visits += sess.order_counter - v0
        x = PF.xfer_bytes()
        h2d += x["h2d"]
        d2h += x["d2h"]
    return dict(ms=ms, visits=visits, steps=n, h2d=h2d // n, d2h=d2h // n,
                entries=len(entries))


def kernel_work(tables, H: int, P: int):
    """Algorithmic work per unit (one row a launch processed) of each
    kernel: flops for the tensor-core MLPs and the fp64 PPO,
    bytes for the rest.  The sampler's fp32 logits read is an unfused
    intermediate, not algorithmic work, and is not counted."""
    F, S = tables.feature_len, tables.local_slots
    C = len(tables.head_cols)
    state = 2 * S + 3               # u16 tile slots + 3 knob bytes
    walk = state + 5 + state        # state in, action (u16 + 3 u8), state out
    pol = 2 * (F * H + H * H + H * (C + 9))
    val = 2 * (F * H + H * H + H)
    feat_in_sampler = 0 < P <= 16384   # HARL_SAMPLE_FEAT_MAX_ROWS
    gbt = 8 * F + 16                # K6: features in, score + reward out
    log = state + 8 + 8 + 4         # entry log: state, score, reward, track
    return {
        "k_mlp_f16<policy>": ("tensor", pol), "k_mlp_f16<value>": ("tensor", val),
        "k_policy_tc": ("tensor", pol), "k_policy_tc64": ("tensor", pol),
        "k_policy_step_fused": ("tensor", pol),
        "k_value_tc": ("tensor", val),
        "k_sample_rows": ("hbm", walk + (8 * F if feat_in_sampler else 0)),
        "k_featurize2": ("hbm", state + 8 * F),
        "k_featurize": ("hbm", state + 8 * F),
        "k_gbt_predict2": ("hbm", gbt), "k_gbt_predict": ("hbm", gbt),
        "k_gbt_finish": ("hbm", gbt + log),
        # policy + value forward and backward in fp64 (3x forward flops)
        "k_ppo_rows": ("fp64", 3 * (pol + val)),
        "k_ppo_rows_tc": ("fp64", 3 * (pol + val)),
        "k_ppo_wgrad": ("fp64", None),        # 2 * B per parameter, below
        "k_ppo_wgrad_spec": ("fp64", None),   # the same, Adam fused in
        "k_ppo_adam": ("hbm", 60),            # per parameter
    }


def roofline_table(native, tables, H, P, peaks, n_params):
    """Per-kernel achieved rate from the library's per-launch event timer
    (harl_profile_read: summed launch time and the rows each launch
    processed) against this run's measured peaks; the dominant kernel (by
    device time) is the line's ``roofline``."""
    work = kernel_work(tables, H, P)
    pk = {"tensor": peaks["tf32_tflops"], "fp64": peaks["fp64_tflops"],
          "hbm": peaks["hbm_gbs"]}
    table = {}
    for name, st in native.items():
        ms, units = st["ms"], st.get("units", -1)
        ent = {"us_per_launch": round(1e3 * ms / max(1, st["launches"]), 2),
               "ms_per_episode": round(ms, 4), "launches": st["launches"],
               "units": units}
        if name in work and ms > 0 and units > 0:
            bound, per = work[name]
            if name in ("k_ppo_wgrad", "k_ppo_wgrad_spec"):
                per = 2 * n_params
            q = per * units / (ms * 1e-3)
            ach = q / 1e9 if bound == "hbm" else q / 1e12
            ent.update(bound=bound, achieved=round(ach, 3),
                       unit="GB/s" if bound == "hbm" else "TFLOP/s",
                       peak=pk[bound], frac=round(ach / pk[bound], 5),
                       work_per_unit=per,
                       work_unit="B" if bound == "hbm" else "flop")
            if name.startswith("k_mlp_f16"):
                # fp32-accurate networks on the fp16 pipe (3xFP16): also
                # against the measured dense fp16 peak of that pipe
                ent["frac_of_fp16_peak"] = round(ach / peaks["fp16_tflops"], 5)
        table[name] = ent
    timed = [k for k in table if "bound" in table[k]]
    if not timed:
        return None, table
    top = max(timed, key=lambda k: table[k]["ms_per_episode"])
    e = table[top]
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles",
                                         "r2_traffic.json")))
        key = "c2" if P <= 16384 else "c3"
        if top in tr.get(key, {}):
            traffic = round(tr[key][top]["dram_bytes_per_launch"])
    except (OSError, ValueError, KeyError):
        traffic = None
    roof = {"kernel": top, "bound": e["bound"], "achieved": e["achieved"],
            "peak": e["peak"], "unit": e["unit"], "frac": e["frac"],
            "traffic": traffic,
            "rows_per_launch": round(e["units"] / max(1, e["launches"]), 1),
            "us_per_launch": e["us_per_launch"],
            "achieved_note": "algorithmic work per row (SURVEY §8(d)) x rows "
                             "the library counted per launch / summed launch "
                             "time (per-launch CUDA events on the launching "
                             "stream, spin-kernel aligned, one untimed eager "
                             "episode)",
            "traffic_note": "DRAM bytes per launch (dram__bytes_read+write) "
                            "averaged over the launches of the committed ncu "
                            "--set full capture of the same config "
                            "(profiles/r2_traffic.json; ncu flushes caches "
                            "between replays, so this is the cold figure)"}
    return roof, table


def e2e_shard_leg(r, steps, world):
    """e2e of the sharded mode (the drop-in is one session per process, so
    the sharded engine is the public API here): every timed episode uploads
    the host agent (numpy parameters + Adam moments) to each rank, runs the
    sharded episode and writes parameters and moments back to numpy; wall
    time, max over ranks, the library's accounted H2D/D2H bytes."""
    import torch
    from paper_2211_11172_b200 import profiling as PF
    eng, tb, forest, gen = r["eng"], r["tables"], r["forest"], r["gen"]
    ms, visits, h2d, d2h = 0.0, 0, 0, 0
    order = r["order"]
    for _ in range(steps):
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        PF.xfer_reset()
        t0 = time.perf_counter()
        eng.dagent.upload()
        res = eng.run_episode(tb, forest, gen, r["ecfg"], order)
        eng.sync_to_host()
        torch.cuda.synchronize()
        ms += (time.perf_counter() - t0) * 1e3
        v = res.extra.get("global_visits", res.visits)
        visits += v
        order += v
        x = PF.xfer_bytes()
        h2d += x["h2d"]
        d2h += x["d2h"]
    return dict(ms=ms, visits=visits, steps=steps, h2d=h2d // steps,
                d2h=d2h // steps, entries=0, sharded=True)


def gpu_arm(args, P, rank, world):
    import torch
    # (ranks beyond the visible devices share them: the gloo tests run two
    # ranks on one GPU)
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)) %
                       torch.cuda.device_count())
    torch.cuda.set_device(dev)
    peaks = measure_peaks(torch, dev)
    shard = None
    if world > 1 and args.mode == "shard":
        import torch.distributed as dist
        shard = (world, rank, dist.group.WORLD)
    r = value_leg(args.config, P, args.steps, args.warmup, dev, rank, world,
                  shard=shard)
    if shard:
        e = e2e_shard_leg(r, max(1, min(args.steps, 5)), world)
        return peaks, r, e, None
    try:
        e = e2e_leg(args.config, P, min(args.steps, 5), min(args.warmup, 3),
                    dev, rank)
    except ImportError as exc:
        e = {"unavailable": f"the drop-in needs the reference package "
                            f"(baseline/_ref): {exc}"}
    c3 = None
    if args.config == "c2" and not args.no_extra:
        c3 = value_leg("c3", CONFIGS["c3"]["population"], 3, 3, dev, rank,
                       world)
    return peaks, r, e, c3


def _max_over_ranks(vals, world):
    if world == 1:
        return vals
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64,
                     device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--population", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the C3 64K sub-measurement")
    ap.add_argument("--mode", default="shard", choices=["shard", "replicas"],
                    help="N > 1: one population of P*N tracks sharded over "
                         "the ranks (gradient all-reduce), or N independent "
                         "task replicas")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    cfgd = CONFIGS[args.config]
    P = args.population or cfgd["population"]

    if args.config == "c4":
        taskset_main(args, P, rank, world)
        return
    if args.impl == "reference":
        if rank != 0:
            return
        reference_arm(args, P, cfgd)
        return

    if world > 1:
        import torch.distributed as dist
        # HARL_DIST_BACKEND=gloo: two ranks on one GPU (tests)
        dist.init_process_group(os.environ.get("HARL_DIST_BACKEND", "nccl"))
    peaks, r, e, c3 = gpu_arm(args, P, rank, world)
    total_ms, = _max_over_ranks([r["total_ms"]], world)
    e_ms = _max_over_ranks([e.get("ms", 0.0)], world)[0]
    c3_ms = _max_over_ranks([c3["total_ms"]], world)[0] if c3 else None
    if rank != 0:
        return
    tb = r["tables"]
    H = 128
    sharded = world > 1 and args.mode == "shard"
    visits_all = r["visits"] * (1 if sharded else world)
    value = visits_all / (total_ms / 1e3)
    n_params = r["n_params"]
    roof, table = roofline_table(r["native"], tb, H, P, peaks, n_params)
    flops = kernel_work(tb, H, P)
    fl_sched = flops["k_mlp_f16<policy>"][1] + 2 * flops["k_mlp_f16<value>"][1]
    by_sched = 2 * (2 * tb.local_slots + 3) + 5 + 8 * tb.feature_len
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "fp32-accurate networks (3xFP16 split, fp32 accumulate, "
                 "tcgen05 kind::f16) + fp64 features/GBT/PPO",
        "data": "synthetic: random-init reference architecture (Glorot, "
                "seeded); cost model warm-started per SURVEY §8(d) (512 "
                "uniform states, analytic simulator, fit_round -> "
                f"{r['n_trees']} trees, on the device, bit-exact)",
        "config": {"workload": cfgd["workload"], "population_per_gpu": P,
                   "episode": "cull_window 20, episode_len 40, "
                              "min_tracks P/2 (60 steps, P*40 visits)",
                   "hidden": [H, H], "step": "one full _run_episode",
                   "l2": "flushed (256 MiB write) between timed episodes",
                   "parallelism": (f"one population of {P * world} tracks "
                                   f"sharded over {world} GPUs (track i on "
                                   f"rank i mod {world}, NCCL all-reduce of "
                                   f"the PPO gradients, merged culls)"
                                   if sharded else
                                   f"independent task replicas x{world}")
                   if world > 1 else "single GPU"},
        "gpu_launches": int(r["launches"]),
        "clocks": r["clocks"],
        "roofline": roof,
        "peaks_measured": peaks,
        "step_roofline": {
            "tensor": {"achieved": round(value * fl_sched / 1e12, 2),
                       "peak": peaks["tf32_tflops"], "unit": "TFLOP/s",
                       "frac": round(value * fl_sched / 1e12 /
                                     peaks["tf32_tflops"], 4),
                       "flop_per_schedule": fl_sched,
                       "note": "policy + 2 value passes per schedule, "
                               "1-pass algorithmic flops vs the measured "
                               "TF32 peak"},
            "hbm": {"achieved": round(value * by_sched / 1e9, 2),
                    "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": round(value * by_sched / 1e9 / peaks["hbm_gbs"],
                                  5),
                    "bytes_per_schedule": by_sched}},
        "kernels": table,
        "profiled_episode_ms": round(r["profiled_episode_ms"], 3),
    }
    if "ms" in e:
        ev = e["visits"] * (1 if e.get("sharded") else world) / (e_ms / 1e3)
        line["e2e"] = {"value": round(ev, 1), "unit": UNIT,
                       "h2d_bytes_per_step": int(e["h2d"]),
                       "d2h_bytes_per_step": int(e["d2h"]),
                       "ms_per_step": round(e_ms / e["steps"], 3),
                       "steps": e["steps"],
                       "call": ("sharded EpisodeEngine.run_episode with the "
                                "numpy agent/moments uploaded and written "
                                "back every episode" if e.get("sharded") else
                                "B200TuningSession._run_episode (compat.py) "
                                "on a baseline/_ref TuningSession: numpy "
                                "agent/moments + ensemble in, params/moments "
                                f"+ {e['entries']} CandidateEntry out")}
    else:
        line["e2e"] = e
    if c3:
        c3v = c3["visits"] * world / (c3_ms / 1e3)
        croof, ctab = roofline_table(c3["native"], c3["tables"], H,
                                     c3["P"], peaks, c3["n_params"])
        line["c3_64k"] = {
            "workload": CONFIGS["c3"]["workload"], "value": round(c3v, 1),
            "unit": UNIT, "ms_per_step": round(c3_ms / 3, 3), "steps": 3,
            "warmup": 3, "population_per_gpu": c3["P"], "roofline": croof,
            "kernels": {k: v for k, v in ctab.items()
                        if k in ("k_mlp_f16<policy>", "k_mlp_f16<value>",
                                 "k_policy_tc", "k_policy_tc64",
                                 "k_value_tc", "k_sample_rows",
                                 "k_featurize2", "k_gbt_finish",
                                 "k_ppo_rows", "k_ppo_wgrad",
                                 "k_ppo_wgrad_spec")}}
    if not args.no_cpu_baseline and world == 1:   # rank 0 at N=1 only
        cb = cpu_pool(args.config, P, 0, 1)
        line["cpu_baseline"] = {
            "value": round(cb["value"], 1), "unit": UNIT,
            "cores": cb["procs"], "kind": cb["kind"],
            "sample": f"{cb['procs']} independent {cb['kind']} sessions x "
                      f"{cb['per']} tracks, one full 60-step _run_episode "
                      f"each ({cb['visits']} visits; single-process rate "
                      f"{cb['per_process']:.0f}/s)",
            "host": cb["host"]}
    print(json.dumps(line))


def reference_arm(args, P, cfgd):
    """The reference CPU path on this box's host cores: one reference
    TuningSession per core, P/N tracks each (cli.py:231-235), full
    60-step ``_run_episode`` calls of the same config; a step = one
    episode in every process."""
    steps = max(1, min(args.steps, 5))
    warm = min(args.warmup, 1)
    cb = cpu_pool(args.config, P, warm, steps)
    value = cb["value"]
    line = {"metric": METRIC, "value": round(value, 1), "unit": UNIT,
            "impl": "reference", "n_gpus": 0, "steps": steps,
            "warmup": warm,
            "ms_per_step": round(1e3 * cb["seconds"] / steps, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "fp64 (numpy)",
            "data": "synthetic: random-init agents, SimulatedBackend "
                    "warm start (512 states, fit_round)",
            "config": {"workload": cfgd["workload"], "population": P,
                       "episode": "cull_window 20, episode_len 40, "
                                  "min_tracks P/2 per session (60 steps)",
                       "sample": f"{cb['procs']} processes x {cb['per']} "
                                 f"tracks x {steps} full episodes "
                                 f"(+{warm} untimed)"},
            "cpu_baseline": {"value": round(value, 1), "unit": UNIT,
                             "cores": cb["procs"], "kind": cb["kind"],
                             "sample": f"{cb['procs']} independent "
                                       f"{cb['kind']} sessions x {cb['per']} "
                                       f"tracks, {steps} full episodes each; "
                                       f"single-process rate "
                                       f"{cb['per_process']:.0f}/s",
                             "host": cb["host"]},
            "e2e": {"value": round(value, 1), "unit": UNIT,
                    "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# C4: the ResNet-50 task set through the reference session (drop-in)


def taskset_session(cls_name, P, rank, world, rounds_budget):
    """A TuningSession (reference or B200 subclass) over this rank's share
    of the ResNet-50 task set."""
    import dataclasses
    from schedtune.measure import SimulatedBackend
    from schedtune.tuner import TunerConfig, TuningSession
    from schedtune.workload import TargetConfig, load_network
    from paper_2211_11172_b200.shard import shard_tasks
    net = load_network(os.path.join(ROOT, "workloads", "resnet50.yaml"))
    mine = shard_tasks(len(net.subgraphs), world, rank)
    sub = dataclasses.replace(net, subgraphs=tuple(net.subgraphs[i]
                                                   for i in mine))
    cfg = TunerConfig(seed=rank, total_trials=64 * rounds_budget,
                      top_k=64, initial_tracks=P, min_tracks=P // 2)
    cls = TuningSession
    if cls_name == "b200":
        from paper_2211_11172_b200.compat import b200_session_class
        cls = b200_session_class(TuningSession)
    return cls(sub, TargetConfig(), cfg, SimulatedBackend(), "rl"), mine


def taskset_main(args, P, rank, world):
    """One bench step = one tuning round of a session (bandit pick of a
    subgraph + sketch, _run_episode over P tracks with adaptive culls,
    rank_scores, simulated measurement, GBT refit).  schedules/s = visited
    candidates / wall time of the rounds, summed over ranks (max time)."""
    try:
        _ref_import()
    except ImportError as exc:
        if rank == 0:
            print(json.dumps({"impl": args.impl, "unavailable":
                              f"config c4 needs the reference session "
                              f"(baseline/_ref): {exc}"}))
        return
    ref = args.impl == "reference"
    if ref and rank != 0:
        return
    if not ref and world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    if not ref:
        import torch
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    steps = args.steps if not ref else min(args.steps, 2)
    warm = args.warmup if not ref else 0
    sess, mine = taskset_session("reference" if ref else "b200", P,
                                 rank, 1 if ref else world,
                                 warm + steps + 1)
    ep_ms = [0.0]
    if not ref:
        import torch
        orig = sess._run_episode

        def timed(sg, sketch, rnd):
            torch.cuda.synchronize()
            t = time.perf_counter()
            out = orig(sg, sketch, rnd)
            torch.cuda.synchronize()
            ep_ms[0] += (time.perf_counter() - t) * 1e3
            return out
        sess._run_episode = timed
    for _ in range(warm):
        sess.run_round()
    v0, ep_ms[0] = sess.order_counter, 0.0
    if not ref and world > 1:
        import torch.distributed as dist
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        sess.run_round()
    secs = time.perf_counter() - t0
    visits = sess.order_counter - v0
    tot_v, max_s = visits, secs
    if not ref and world > 1:
        import torch
        import torch.distributed as dist
        t = torch.tensor([float(visits)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t)
        tot_v = int(t.item())
        t = torch.tensor([secs], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        max_s = float(t.item())
    if rank != 0:
        return
    value = tot_v / max_s
    line = {"metric": METRIC, "value": round(value, 1), "unit": UNIT,
            "n_gpus": 0 if ref else world, "steps": steps, "warmup": warm,
            "ms_per_step": round(1e3 * max_s / steps, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "fp64 (numpy)" if ref else
                     "fp32 networks + fp64 features/GBT/PPO",
            "data": "synthetic (random-init agents, SimulatedBackend "
                    "measurements)",
            "config": {"workload": CONFIGS["c4"]["workload"],
                       "population_per_task": P,
                       "tasks_rank0": len(mine),
                       "step": "one TuningSession.run_round (episode + "
                               "rank_scores + measure + GBT refit)",
                       "parallelism": "reference CPU session, 1 process"
                       if ref else f"tasks sharded i mod {world}"}}
    if ref:
        line["impl"] = "reference"
        line["cpu_baseline"] = {"value": round(value, 1), "unit": UNIT,
                                "cores": 1, "kind": "reference",
                                "sample": f"{steps} rounds of the reference "
                                          f"session on rank 0's tasks"}
        line["e2e"] = {"value": round(value, 1), "unit": UNIT,
                       "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    else:
        line["e2e"] = {"value": round(value, 1), "unit": UNIT,
                       "note": "the whole round is host-driven through the "
                               "reference session; episode (device) share "
                               f"{ep_ms[0] / (1e3 * secs):.3f}"}
        line["ms_per_step_parts"] = {
            "episode_ms": round(ep_ms[0] / steps, 2),
            "host_ms": round((1e3 * secs - ep_ms[0]) / steps, 2)}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
