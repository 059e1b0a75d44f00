"""Benchmark: schedules/sec of the HARL inner search step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--config c2|c1|c3|c5] [--population P]

A bench "step" is one ``_run_episode`` (tuner.py:350-440) over the whole
population: initial sampling, every search step of the default geometry
(cull_window 20, episode_len 40 -> 20 steps at P tracks, a cull to P/2, 40
steps at P/2, PPO every 2 steps), i.e. P*40 visited schedules.  The unit of
work is one visited schedule (one CandidateEntry, tuner.py:408-412).

* ``value``: whole-job schedules/s with the population resident in HBM,
  device time via CUDA events on the launching stream, summed over the K
  timed episodes (L2 flushed between episodes, outside the events), max over
  ranks.
* ``e2e``: the same metric through the host-buffer call a drop-in makes per
  episode: agent parameters/moments, replay ring, forest and generator state
  go host->device before; after the episode the device rank_scores
  (costmodel.py:266-286) selects the top-k' distinct unmeasured entries and
  those (states, features, scores), the per-visit rewards and the updated
  agent/ring come back device->host, every episode.
* ``cpu_baseline``: the oracle (numpy restatement of the reference, bit-exact
  with it) timed on this host on a bounded sample of the same workload.
* ``--impl reference``: the reference CPU path (the oracle port) with all
  host cores, one independent session per core (the reference's own
  process-pool model, cli.py:231-235), same metric.

Synthetic data: random-init weights of the reference architecture, a
synthetic depth-6 50-tree GBT forest with thresholds drawn from real feature
values (no measurements are available offline).
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
# workload construction (shared by the GPU and CPU legs)


def synthetic_forest(tables, seed: int, n_trees: int = 50, depth: int = 6):
    """50 trees of depth <= 6 (the reference's GbtConfig defaults,
    costmodel.py:24-31) splitting on features that actually vary, with
    thresholds at feature values of random states so walks branch."""
    from oracle.harl_oracle import featurize, sample_initial  # host-only
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


def build_workload(cfg_name: str, population: int | None, seed: int = 0):
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
    return dict(tables=tables, agent=agent, rl=rl, P=P, cfg=c,
                trees=synthetic_forest(tables, seed + 1), base=0.5, lr=0.3)


def episode_config(P):
    from paper_2211_11172_b200.engine import EpisodeConfig
    # TunerConfig defaults with min_tracks = P/2, initial_tracks = P
    return EpisodeConfig(tracks=P, track_len=40, cull_window=20,
                         cull_fraction=0.5, min_tracks=P // 2)


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
# CPU legs


def cpu_episode_sample(cfg_name, P, steps, seed=0):
    """Oracle episode on P tracks for `steps` search steps; returns
    (visits, seconds)."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle import harl_oracle as O
    w = build_workload(cfg_name, P, seed)
    a = w["agent"]
    oa = O.Agent.from_param_lists(a.policy, a.value, len(a.hidden))
    opi = O.Adam.zeros_like(oa.policy_params(), w["rl"].lr_actor)
    ov = O.Adam.zeros_like(oa.value_params(), w["rl"].lr_critic)
    model = O.GbtModel(w["base"], w["lr"], True, w["trees"])
    ecfg = O.EpisodeCfg(tracks=P, track_len=steps, cull_window=20,
                        cull_fraction=0.5, min_tracks=P // 2,
                        rl_cfg=O.RlCfg())
    t = time.perf_counter()
    entries, _, _ = O.run_episode(w["tables"], w["tables"].num_slots, ecfg,
                                  oa, opi, ov, O.Replay(4096), model,
                                  np.random.default_rng(seed + 7), 0)
    return len(entries), time.perf_counter() - t


def _cpu_worker(args):
    cfg_name, P, steps, seed = args
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    return cpu_episode_sample(cfg_name, P, steps, seed)


def cpu_parallel(cfg_name, P, steps, procs):
    """The reference's own parallelism model: independent sessions in a
    process pool (cli.py:231-235), P/procs tracks each."""
    from concurrent.futures import ProcessPoolExecutor
    import multiprocessing as mp
    per = max(2, P // procs)
    t = time.perf_counter()
    with ProcessPoolExecutor(procs, mp_context=mp.get_context("spawn")) as ex:
        res = list(ex.map(_cpu_worker, [(cfg_name, per, steps, s)
                                        for s in range(procs)]))
    wall = time.perf_counter() - t
    visits = sum(v for v, _ in res)
    slowest = max(s for _, s in res)
    return visits, slowest, wall


# ---------------------------------------------------------------------------
# GPU leg


def l2_flush(torch, dev, buf=[]):
    if not buf:
        buf.append(torch.empty(256 << 20, dtype=torch.uint8, device=dev))
    buf[0].fill_(1)


def run_gpu(args, rank, world):
    import torch
    from paper_2211_11172_b200 import device as D
    from paper_2211_11172_b200 import profiling
    from paper_2211_11172_b200.engine import EpisodeEngine
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    w = build_workload(args.config, args.population, seed=rank)
    P = w["P"]
    tb = w["tables"]
    ecfg = episode_config(P)
    eng = EpisodeEngine(w["agent"], w["rl"], tb.levels, dev)
    forest = D.DeviceForest(w["trees"], w["base"], w["lr"], device=dev)
    gen = np.random.default_rng(1000 + rank)
    stream = torch.cuda.current_stream()
    order = 0
    for _ in range(args.warmup):
        res = eng.run_episode(tb, forest, gen, ecfg, order)
        order += res.visits
    torch.cuda.synchronize()
    profiling.reset()
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = 0.0
    visits = 0
    with ClockSampler(dev.index) as clk:
        for _ in range(args.steps):
            l2_flush(torch, dev)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            res = eng.run_episode(tb, forest, gen, ecfg, order)
            e1.record(stream)
            e1.synchronize()
            total_ms += e0.elapsed_time(e1)
            visits += res.visits
            order += res.visits
    torch.cuda.synchronize()
    launches = profiling.launch_count()
    # one extra, untimed episode with per-call CUDA events: kernel shares
    profiling.reset()
    profiling.timing(True)
    profiling.native_timing(True)
    eng.use_graphs = False          # per-launch events need eager launches
    res = eng.run_episode(tb, forest, gen, ecfg, order)
    eng.use_graphs = True
    order += res.visits
    kstats = profiling.kernel_times()
    native = profiling.native_kernel_times()
    profiling.native_timing(False)
    profiling.timing(False)
    if world > 1:
        dist.barrier()
    # ---- e2e: host buffers in and out every episode ------------------------
    host = E2EHost(eng, w, dev, ecfg.budget)
    e2e_ms, h2d, d2h, e2e_visits = 0.0, 0, 0, 0
    e2e_parts = {}
    for _ in range(max(1, min(args.steps, 3))):
        l2_flush(torch, dev)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        b_in, b_out, v, parts = host.episode(forest, gen, ecfg, order)
        torch.cuda.synchronize()
        e2e_ms += (time.perf_counter() - t0) * 1e3
        h2d, d2h = b_in, b_out
        e2e_visits += v
        order += v
        for k_, t_ in parts.items():
            e2e_parts[k_] = e2e_parts.get(k_, 0.0) + t_
    return dict(total_ms=total_ms, visits=visits, clocks=clk.summary(),
                launches=launches, kstats=kstats, native=native, e2e_ms=e2e_ms,
                e2e_visits=e2e_visits, h2d=h2d, d2h=d2h, P=P,
                e2e_parts=e2e_parts)


class E2EHost:
    """The drop-in's host side for the e2e number: pinned host buffers for
    every per-episode input (agent parameters + Adam moments, replay ring,
    GBT ensemble; the replay ring stays resident like the drop-in's) and
    output (the rank_scores selection -- top-k' distinct
    unmeasured entries with states, features, scores -- the per-visit
    rewards of the trajectory log, the updated agent and ring), allocated
    once.  Each timed episode copies the inputs host->device, runs
    ``_run_episode`` + the device rank_scores and copies the outputs back
    (what ``compat.B200TuningSession._run_episode`` moves per round, without
    the reference's Python object construction).  The selected states
    accumulate as the "measured" exclusion set, as in a session."""

    def __init__(self, eng, w, dev, visits):
        import torch
        self.eng, self.w, self.dev = eng, w, dev
        self.tb = w["tables"]
        da, ring = eng.dagent, eng.replay
        pin = lambda t: torch.empty(t.shape, dtype=t.dtype).pin_memory()
        self.agent_in = {k: pin(getattr(da, k)) for k in ("params", "m", "v")}
        for k, t in self.agent_in.items():
            t.copy_(getattr(da, k))
        self.agent_out = {k: pin(getattr(da, k)) for k in ("params", "m", "v")}
        keys = ("X", "Xn", "actions", "scalars", "move_bits", "shift_bits")
        self.ring_out = {k: pin(getattr(ring, k)) for k in keys}
        self.V = (visits, torch.empty(visits, dtype=torch.float64).pin_memory())
        from paper_2211_11172_b200 import device as D
        self.rank_scratch = D.RankScratch(dev)
        self.top_k = 64                 # TunerConfig.top_k default
        # allocations a session makes once, outside the per-round path
        self.rank_scratch.ensure(visits, 64 * 16, self.top_k)
        self.rank_scratch.host_pins(4 * self.top_k, w["tables"])
        self.measured = None

    def episode(self, forest, gen, ecfg, order):
        import torch
        eng, tb = self.eng, self.tb
        da, ring = eng.dagent, eng.replay
        parts = {}
        t0 = time.perf_counter()
        nin = 0
        for k, t in self.agent_in.items():
            getattr(da, k).copy_(t, non_blocking=True)
            nin += t.numel() * t.element_size()
        da.params32.copy_(da.params)            # fp32 rollout copy
        da.refresh_derived()                    # tcgen05 images + transposes
        # the replay ring is not uploaded: between episodes the drop-in keeps
        # it in device memory (compat._RingBuffer); it is still exported
        # below, as the per-round checkpoint does
        w = self.w
        forest.load(w["trees"], w["base"], w["lr"])
        nin += forest.n_nodes * 16 + forest.n_trees * 4 + forest.HDR.itemsize
        t1 = time.perf_counter()
        res = eng.run_episode(tb, forest, gen, ecfg, order)
        t2 = time.perf_counter()
        V = res.visits
        if self.V is None or self.V[0] < V:
            self.V = (V, torch.empty(V, dtype=torch.float64).pin_memory())
        # rank_scores on the device (what run_round consumes): the top-k'
        # distinct unmeasured entries come back with their features; the
        # per-visit rewards come back for the trajectory log
        idx, tiles, knobs, feats, scores, _ = res.top_entries(
            self.top_k, self.measured, self.rank_scratch)
        self.V[1][:V].copy_(res.log_reward[:V], non_blocking=True)
        nout = len(idx) * (2 * tb.local_slots + 3 + 8 * tb.feature_len + 8 + 8) \
            + V * 8
        # the chosen states become "measured" for the next episodes
        mt = tiles if self.measured is None else \
            np.concatenate([self.measured[0], tiles])
        mk = knobs if self.measured is None else \
            np.concatenate([self.measured[1], knobs])
        self.measured = (mt, mk)
        t2b = time.perf_counter()
        for k, t in self.agent_out.items():
            t.copy_(getattr(da, k), non_blocking=True)
            nout += t.numel() * t.element_size()
        for k, t in self.ring_out.items():
            t.copy_(getattr(ring, k), non_blocking=True)
            nout += t.numel() * t.element_size()
        torch.cuda.current_stream().synchronize()
        t3 = time.perf_counter()
        parts.update(h2d_ms=(t1 - t0) * 1e3, episode_ms=(t2 - t1) * 1e3,
                     rank_ms=(t2b - t2) * 1e3, d2h_ms=(t3 - t2b) * 1e3)
        return nin, nout, V, parts


# kernel -> (profiling span whose rows it processes, bound)
KERNEL_SPAN = {
    "k_trunk_tc<policy>": ("policy_tc", "tensor"),
    "k_heads_tc": ("policy_tc", "tensor"),
    "k_sample_rows": ("policy_tc", "hbm"),
    "k_trunk_tc<value>": ("value_tc", "tensor"),
    "k_policy_tc": ("policy_tc", "tensor"),
    "k_policy_tc64": ("policy_tc", "tensor"),
    "k_policy_step_fused": ("policy_tc", "tensor"),
    "k_value_tc": ("value_tc", "tensor"),
    "k_featurize": ("featurize", "hbm"),
    "k_featurize2": ("featurize", "hbm"),
    "k_gbt_predict": ("gbt", "hbm"),
    "k_gbt_predict2": ("gbt", "hbm"),
    "k_finish_step": ("finish", "hbm"),
    "k_gbt_finish": ("gbt", "hbm"),
    "k_ring_rows": ("finish", "hbm"),
    "k_ppo_rows": ("ppo", "fp64"),
    "k_ppo_rows_tc": ("ppo", "fp64"),
}


def per_row_work(tables, H, feat_in_sampler=False):
    """Algorithmic work per row (one schedule / one minibatch row) of each
    kernel: flops for the MLP kernels, HBM bytes for the rest (DESIGN.md
    "Kernels and their rooflines" states the same figures)."""
    F, S = tables.feature_len, tables.num_slots
    C = len(tables.head_cols)
    NH = C + 9                      # tiling columns + 3 + 3 + 3 knob heads
    state = 2 * S + 3               # int16 tile slots + 3 knob bytes
    return {
        "k_trunk_tc<policy>": 2 * (F * H + H * H),
        "k_heads_tc": 2 * H * NH,
        "k_trunk_tc<value>": 2 * (F * H + H * H + H),   # per evaluated row
        "k_policy_tc": 2 * (F * H + H * H + H * NH),
        "k_policy_tc64": 2 * (F * H + H * H + H * NH),
        # + the sampler/walker and the featurizer of the same rows
        "k_policy_step_fused": 2 * (F * H + H * H + H * NH),
        "k_value_tc": 2 * (F * H + H * H + H),
        # logits in; actions, logp, successor state out (+ its feature row
        # when the sampler featurizes, <= 16 K rows per launch)
        "k_sample_rows": 4 * NH + state + 16 + 8 + state +
                         (8 * F if feat_in_sampler else 0),
        "k_featurize": state + 8 * F,
        "k_featurize2": state + 8 * F,
        "k_gbt_predict": 8 * F + 8,
        "k_gbt_predict2": 8 * F + 8,
        # reward/score/v/adv/log entry (state + score + track) + ring scalars
        "k_finish_step": 8 * 6 + state + 8 + 4 + 8 * 4 + 16 + 4,
        # GBT (features in, score + reward out) + the finish row work
        "k_gbt_finish": 8 * F + 8 + 8 * 6 + state + 8 + 4 + 8 * 4 + 16 + 4,
        "k_ring_rows": 2 * 8 * F * 2,               # X and X' read + written
        # policy + value forward and backward in fp64 (3x forward flops)
        "k_ppo_rows": 3 * 2 * (2 * (F * H + H * H) + H * NH + H),
        "k_ppo_rows_tc": 3 * 2 * (2 * (F * H + H * H) + H * NH + H),
    }


def roofline_entry(native, spans, tables, hidden, P=0):
    """Dominant kernel's achieved rate vs the measured peak, from the native
    per-kernel event timer (harl_profile_*) of the untimed profiled episode;
    rows per kernel come from the matching host span."""
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    if not native:
        return None
    # the sampler featurizes in-kernel up to 16 K rows per launch
    # (HARL_SAMPLE_FEAT_MAX_ROWS, harl_b200.cu)
    work = per_row_work(tables, hidden, feat_in_sampler=0 < P <= 16384)
    hbm = peaks.get("hbm_gbs", 6650.0)
    bf16 = peaks.get("bf16_tflops", 1590.0)
    tf32 = bf16 * 1.1 / 2.25        # dense tf32 : bf16 nominal ratio
    fp64 = 37.0                     # B200 nominal fp64 (no measured figure)
    table = {}
    for name, st in native.items():
        if st["ms"] <= 0:
            continue
        if name not in KERNEL_SPAN:     # listed with its time only
            table[name] = {"bound": None, "achieved": 0.0, "peak": None,
                           "unit": None, "frac": 0.0,
                           "us_per_launch": 1e3 * st["ms"] / max(1, st["launches"]),
                           "ms_per_episode": st["ms"]}
            continue
        span, bound = KERNEL_SPAN[name]
        rows = spans.get(span, {}).get("rows", 0)
        q = work[name] * rows
        if bound == "hbm":
            ach = q / (st["ms"] * 1e-3) / 1e9
            ent = {"bound": "hbm", "achieved": ach, "peak": hbm,
                   "unit": "GB/s"}
        else:
            ach = q / (st["ms"] * 1e-3) / 1e12
            pk = tf32 if bound == "tensor" else fp64
            ent = {"bound": "tensor" if bound == "tensor" else "fp64",
                   "achieved": ach, "peak": round(pk, 1), "unit": "TFLOP/s"}
        ent["frac"] = ent["achieved"] / ent["peak"]
        ent["us_per_launch"] = 1e3 * st["ms"] / max(1, st["launches"])
        ent["ms_per_episode"] = st["ms"]
        table[name] = ent
    if not table:
        return None
    top = max((k for k in table if table[k]["bound"]),
              key=lambda k: table[k]["ms_per_episode"])
    e = table[top]
    # DRAM bytes per launch of that kernel from the committed ncu --set full
    # capture (per row there, scaled to this run's average rows per launch)
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "r1_traffic.json")))
        if top in tr:
            span = KERNEL_SPAN[top][0]
            rows = spans.get(span, {}).get("rows", 0)
            launches = native[top]["launches"] or 1
            per_row = tr[top]["dram_bytes_per_launch"] / tr[top]["rows_per_launch"]
            traffic = round(per_row * rows / launches)
    except (OSError, ValueError, KeyError):
        traffic = None
    out = {"kernel": top, "bound": e["bound"],
           "achieved": round(e["achieved"], 3), "peak": e["peak"],
           "unit": e["unit"], "frac": round(e["frac"], 5), "traffic": traffic,
           "traffic_note": "DRAM bytes/launch (dram__bytes_read+write) from "
                           "profiles/r1_traffic.json (ncu --set full), scaled "
                           "to this run's rows/launch; population data is "
                           "L2-resident, so DRAM traffic << algorithmic bytes",
           "us_per_launch": round(e["us_per_launch"], 2),
           "peak_note": "hbm: MEASURED_PEAKS.json hbm_gbs (burst); tensor: "
                        "dense tf32 = measured bf16 x 1.1/2.25; fp64: 37 "
                        "TFLOP/s nominal",
           "kernels": {k: {"bound": v["bound"],
                           "achieved": round(v["achieved"], 3),
                           "unit": v["unit"], "frac": round(v["frac"], 5),
                           "us_per_launch": round(v["us_per_launch"], 2),
                           "ms_per_episode": round(v["ms_per_episode"], 4)}
                       for k, v in sorted(table.items(),
                                          key=lambda kv: -kv[1]["ms_per_episode"])}}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--population", type=int, default=None)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
        dist.init_process_group("nccl")
    r = run_gpu(args, rank, world)
    total_ms, e2e_ms = r["total_ms"], r["e2e_ms"]
    if world > 1:
        import torch
        import torch.distributed as dist
        t = torch.tensor([total_ms, e2e_ms], dtype=torch.float64,
                         device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, e2e_ms = float(t[0]), float(t[1])
    if rank != 0:
        return
    visits_all = r["visits"] * world
    value = visits_all / (total_ms / 1e3)
    e2e = r["e2e_visits"] * world / (e2e_ms / 1e3)
    tb = build_workload(args.config, P)["tables"]
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "fp32 networks + fp64 features/GBT/PPO",
        "data": "synthetic (random-init reference architecture, synthetic "
                "50-tree depth-6 GBT)",
        "config": {"workload": cfgd["workload"], "population_per_gpu": P,
                   "episode": "cull_window 20, episode_len 40, "
                              "min_tracks P/2 (60 steps, P*40 visits)",
                   "hidden": [128, 128], "step": "one full _run_episode",
                   "l2": "flushed (256 MiB write) between timed episodes",
                   "parallelism": f"independent task replicas x{world}"
                   if world > 1 else "single GPU"},
        "e2e": {"value": round(e2e, 1), "unit": UNIT,
                "h2d_bytes_per_step": int(r["h2d"]),
                "d2h_bytes_per_step": int(r["d2h"]),
                "ms_per_step_parts": {k: round(v / max(1, min(args.steps, 3)), 3)
                                      for k, v in r["e2e_parts"].items()}},
        "gpu_launches": int(r["launches"]),
        "clocks": r["clocks"],
        "roofline": roofline_entry(r["native"], r["kstats"], tb, 128, P),
        "kernel_ms_per_episode": {k: round(v["ms"], 4)
                                  for k, v in r["kstats"].items()},
    }
    if not args.no_cpu_baseline and world == 1:   # rank 0 at N=1 only
        steps = 2
        visits, secs = cpu_episode_sample(args.config, P, steps)
        line["cpu_baseline"] = {
            "value": round(visits / secs, 1), "unit": UNIT, "cores": 1,
            "kind": "port",
            "sample": f"oracle episode, {P} tracks x {steps} steps "
                      f"({visits} visits) on 1 core, OPENBLAS_NUM_THREADS=1"}
    print(json.dumps(line))


def reference_arm(args, P, cfgd):
    procs = len(os.sched_getaffinity(0))
    steps = 2
    # each "step" of the reference arm: one bounded sample of the workload
    for _ in range(max(0, min(args.warmup, 1))):
        cpu_parallel(args.config, min(P, 2048), 1, min(procs, 2))
    tot_v, tot_s = 0, 0.0
    for _ in range(args.steps):
        v, slowest, wall = cpu_parallel(args.config, P, steps, procs)
        tot_v += v
        tot_s += slowest
    value = tot_v / tot_s
    line = {"metric": METRIC, "value": round(value, 1), "unit": UNIT,
            "impl": "reference", "n_gpus": 0, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1e3 * tot_s / args.steps, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "fp64 (numpy)", "data": "synthetic",
            "config": {"workload": cfgd["workload"], "population": P,
                       "sample": f"{procs} processes x {P // procs} tracks x "
                                 f"{steps} steps per timed step"},
            "cpu_baseline": {"value": round(value, 1), "unit": UNIT,
                             "cores": procs, "kind": "port",
                             "sample": f"{procs} independent oracle sessions "
                                       f"x {max(2, P // procs)} tracks x "
                                       f"{steps} steps"},
            "e2e": {"value": round(value, 1), "unit": UNIT,
                    "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# C4: the ResNet-50 task set through the reference session (drop-in)


def _ref_import():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(ref) and ref not in sys.path:
        sys.path.insert(0, ref)
    import schedtune  # noqa: F401  (raises ImportError when absent)


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
