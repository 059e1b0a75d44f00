"""The B200 episode engine: ``TuningSession._run_episode`` (tuner.py:350-440)
with the population on device.

Per step, for the m live rows (the first m alive tracks in index order,
tuner.py:373-375), the device runs

  1. ``policy_step``  select_actions + decode/apply  (K4 + K2)
  2. ``featurize``    X' of the new states            (K3)
  3. ``gbt_predict``  new scores + rewards            (K6)
  4. ``value_estimate`` V(X), V(X')                   (K5)
  5. ``finish_step``  advantage/TD, replay push, entry log, Track.advance

and the host keeps the decisions the reference keeps on the host: the
adaptive cull every ``cull_window`` steps (stopping.py:68-86, vectorised
``lexsort`` on the device-computed advantages) and the replay minibatch
indices (``Generator.choice``, rlcore.py:267-274) drawn from the SAME numpy
generator the device sampled from.  The RNG stream is consumed in exactly
the reference's order, so an episode is the reference's episode up to fp32
rounding in the networks (which can flip a sampled action whose uniform
lands within ~1e-7 of a CDF boundary).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import ctypes as C

import numpy as np
import torch

import os

from . import _native as N
from . import device as D
from . import profiling as PF
from . import rng as R
from .agent import AgentState, RlConfig
from .space import SketchTables


# HARL_FUSED_STEP=1: policy -> sample/apply -> featurize as one kernel per
# 128-row tile (k_policy_step_fused).  Correct, but with one 16-warp CTA per
# SM the sampler's rows run in two serial passes and it measured slower
# (49.7 us) than the three separate kernels (policy 19.3 + sampler 21.8 +
# featurize 11.4 us at ~28 warps/SM), so the split launches are the default.
_FUSED_STEP = os.environ.get("HARL_FUSED_STEP") == "1"

# HARL_SPLIT_FEATURIZE=1: featurize as its own launch (k_featurize2) instead
# of inside the sampler kernel (A/B and parity cross-check)
_SPLIT_FEATURIZE = os.environ.get("HARL_SPLIT_FEATURIZE") == "1"

# the graphed episode's cull decision: harl_cull_select (C++ radix select,
# branch-free marking) by default; HARL_NATIVE_CULL=0 uses numpy's
# partition (_cull_rows) instead, kept for A/B (the same decision)
_PY_CULL = os.environ.get("HARL_NATIVE_CULL") == "0"

# HARL_SPLIT_FINISH=1: separate GBT and finish launches (k_gbt_predict2 +
# k_finish_step) instead of the fused k_gbt_finish (A/B and fallback path)
_SPLIT_FINISH = os.environ.get("HARL_SPLIT_FINISH") == "1"

# HARL_SAMPLE_GBT=1: the cost model scored inside the sampler (k_sample_gbt:
# the featurized successor rows never leave shared memory before the forest
# walk) and the step's finish run in the value kernel's epilogue
# (harl_value_finish_tc: one launch fewer per step); =2: sampler-side only,
# the finish as its own launch.  Bit-identical to the default, measured no
# faster at C2 (5.44 / 5.40 vs 5.40 ms per episode: the forest walk adds
# ~7 us to the sampler and the finish ~8 us to the value pass, the launch
# they save costs ~18 us), so the separate k_gbt_finish stays the default.
_SAMPLE_GBT = os.environ.get("HARL_SAMPLE_GBT", "0") in ("1", "2")
_VALUE_FINISH = os.environ.get("HARL_SAMPLE_GBT", "0") == "1"

# graph mode: the next step's policy network on a forked stream beside the
# value and GBT passes of steps without a PPO update or cull
# (HARL_OVERLAP_POLICY=0: strictly sequential launches)
_OVERLAP_POLICY = os.environ.get("HARL_OVERLAP_POLICY", "1") != "0"

# HARL_PAR_VALUE=1: the value pass on a forked stream, concurrent with the
# GBT pass (both read only X'); the finish kernel joins them (split finish).
# Measured slower at 16 K tracks (5.95 vs 5.82 ms per C2 episode): both
# kernels hold most of an SM's shared memory, so they do not co-reside
_PAR_VALUE = os.environ.get("HARL_PAR_VALUE") == "1"

# HARL_EAGER_CAPTURE=1: capture a plan's graphs on its first episode
# instead of its second (C4 first visits, P = 4 K: 13.5 ms eager vs 18.5 ms
# capture + replay per episode, profiles/c4_rounds.py)
_LAZY_CAPTURE = os.environ.get("HARL_EAGER_CAPTURE") != "1"

# host-side timeline of the graphed episode (profiles/host_probe.py sets a
# list here; None = off)
_HOST_TRACE = None


@dataclass(frozen=True)
class EpisodeConfig:
    """The slice of TunerConfig/StopConfig an episode reads (tuner.py:51-150,
    stopping.py:16-28)."""

    tracks: int
    track_len: int
    cull_window: int | None = 20
    cull_fraction: float = 0.5
    min_tracks: int = 64
    rl: bool = True
    adaptive: bool = True

    @property
    def budget(self) -> int:
        return self.tracks * self.track_len

    @classmethod
    def from_tuner(cls, cfg, searcher: str) -> "EpisodeConfig":
        """From a reference ``TunerConfig`` (or a dict of its fields) and
        the searcher name (tuner.py:37-48,105-113,131-134)."""
        get = (lambda k, d=None: cfg.get(k, d)) if isinstance(cfg, dict) \
            else (lambda k, d=None: getattr(cfg, k, d))
        min_tracks = get("min_tracks", 64)
        cw = get("cull_window", 20)
        tracks = get("initial_tracks") or 2 * min_tracks
        track_len = get("episode_len") or 2 * cw
        s = getattr(searcher, "value", searcher)
        rl = s in ("rl", "rl-fixed-length", "rl-greedy-subgraph")
        adaptive = s in ("rl", "rl-greedy-subgraph")
        return cls(tracks=tracks, track_len=track_len,
                   cull_window=cw if adaptive else None,
                   cull_fraction=get("cull_fraction", 0.5),
                   min_tracks=min_tracks, rl=rl, adaptive=adaptive)


_PLANS: dict = {}


def schedule(cfg: EpisodeConfig, replay_count: int, rl_cfg: RlConfig):
    """The episode's step plan, known before it starts: the live-row count
    per step, where culls happen and how many rows they keep, and the
    replay size at each PPO step.  None of it depends on the data
    (tuner.py:371-432, stopping.py:68-95).  Memoised (the configs are
    frozen): the returned plan is shared and must not be modified."""
    key = (cfg, replay_count, rl_cfg)
    plan = _PLANS.get(key)
    if plan is None:
        if len(_PLANS) > 256:
            _PLANS.clear()
        plan = _PLANS[key] = _schedule(cfg, replay_count, rl_cfg)
    return plan


def _schedule(cfg: EpisodeConfig, replay_count: int, rl_cfg: RlConfig):
    alive, used, t = cfg.tracks, 0, 0
    count = replay_count
    plan = []
    while not (alive < cfg.min_tracks or used >= cfg.budget):
        t += 1
        m = min(alive, cfg.budget - used)
        used += m
        step = {"t": t, "m": m, "cull": None, "ppo": None}
        if cfg.rl:
            count = min(rl_cfg.buffer_capacity, count + m)
        if cfg.adaptive and cfg.cull_window is not None and \
                t % cfg.cull_window == 0 and used < cfg.budget:
            n_elim = min(int(math.floor(cfg.cull_fraction * alive)),
                         alive - cfg.min_tracks)
            if n_elim > 0:
                step["cull"] = n_elim
                alive -= n_elim
        if cfg.rl and t % rl_cfg.train_interval == 0 and count >= 2:
            step["ppo"] = min(rl_cfg.minibatch, count)
        plan.append(step)
    return plan


@dataclass
class EpisodeResult:
    """Device-resident outcome of one episode (the reference's return value
    plus its side effects, materialised lazily)."""

    tables: SketchTables
    visits: int
    order_start: int
    log_tiles: torch.Tensor       # [slots][V] int16
    log_knobs: torch.Tensor       # [3][V] uint8
    log_score: torch.Tensor       # [V] f64
    log_reward: torch.Tensor      # [V] f64
    log_track: torch.Tensor       # [V] int32
    step_rows: list               # m per step
    culls: list                   # (step, eliminated track ids, alive after)
    train: list                   # (step, losses tensor view)
    track_steps: torch.Tensor
    track_best_step: torch.Tensor
    alive: np.ndarray
    extra: dict = field(default_factory=dict)

    def states(self):
        """(tiles [V, slots] u16, knobs [V, 3] u8) on the host."""
        return D.states_to_host(self.tables, self.log_tiles, self.log_knobs,
                                self.visits)

    def scores(self) -> np.ndarray:
        return self.log_score[:self.visits].cpu().numpy()

    def top_entries(self, k: int, exclude=None, scratch=None,
                    pending=None):
        """``rank_scores(model, entries, k, exclude)`` on the device entry
        log (costmodel.py:266-286): (visit indices ascending, host tiles
        [n, slots] u16, knobs [n, 3] u8, features [n, F] f64, scores [n],
        stats).  See ``device.rank_topk`` for the superset contract.
        ``pending``: from ``top_entries_launch`` with the same arguments."""
        if pending is None:
            pending = self.top_entries_launch(k, exclude, scratch)
        didx, n, stats = D.rank_topk_finish(pending)
        t, kn, sc, _, f = D.gather_entries(self.tables, self.log_tiles,
                                           self.log_knobs, self.log_score,
                                           self.log_track, didx[:n],
                                           self.extra.get("dsk"))
        # one synchronisation for the five results (pinned, async copies)
        pins = scratch.host_pins(n, self.tables) if scratch is not None \
            else None
        if pins is None:
            idx = didx[:n].cpu().numpy().astype(np.int64)
            tiles, knobs = D.states_to_host(self.tables, t, kn, n)
            f, sc = f.cpu().numpy(), sc.cpu().numpy()
            PF.xfer("d2h", idx.nbytes + tiles.nbytes + knobs.nbytes +
                    f.nbytes + sc.nbytes)
        else:
            S = self.tables.local_slots
            pi, pt, pk, pf, ps = pins
            pi[:n].copy_(didx[:n], non_blocking=True)
            pt[:S, :n].copy_(t[:S, :n], non_blocking=True)
            pk[:, :n].copy_(kn[:, :n], non_blocking=True)
            pf[:n].copy_(f[:n], non_blocking=True)
            ps[:n].copy_(sc[:n], non_blocking=True)
            PF.xfer("d2h", pi[:n], pt[:S, :n], pk[:, :n], pf[:n], ps[:n])
            torch.cuda.current_stream().synchronize()
            idx = pi[:n].numpy().astype(np.int64)
            tiles = np.ascontiguousarray(
                pt[:S, :n].numpy().astype(np.uint16).T)
            knobs = np.ascontiguousarray(pk[:, :n].numpy().T)
            f, sc = pf[:n].numpy().copy(), ps[:n].numpy().copy()
        o = np.argsort(idx, kind="stable")
        return (idx[o], tiles[o], knobs[o], f[o], sc[o], stats)

    def top_entries_launch(self, k: int, exclude=None, scratch=None):
        """Queue the selection's kernels (``top_entries`` finishes)."""
        return D.rank_topk(self.tables, self.log_tiles, self.log_knobs,
                           self.log_score, self.visits, k, exclude, scratch,
                           sort=False, launch_only=True)

    def rewards_per_step(self):
        r = self.log_reward[:self.visits].cpu().numpy()
        out, p = [], 0
        for m in self.step_rows:
            out.append(r[p:p + m])
            p += m
        return out


# sharded PPO: "rows" (default; the minibatch rows all-reduced, the
# single-device update on every rank) or "grads" (per-shard gradients
# all-reduced)
_SHARD_PPO = os.environ.get("HARL_SHARD_PPO", "rows")


class _StagingRing:
    """B replay rows in the ring layout the PPO kernels read (X, actions,
    scalars, move/shift bits), all views of one byte buffer so a single
    collective moves them."""

    def __init__(self, cap: int, F: int, dev):
        import torch
        self.cap = cap
        sizes = [("X", (cap, F), torch.float64),
                 ("scalars", (cap, 4), torch.float64),
                 ("move_bits", (cap,), torch.int64),
                 ("actions", (cap, 4), torch.int32),
                 ("shift_bits", (cap,), torch.int32)]
        nbytes = [int(np.prod(sh)) * torch.empty(0, dtype=dt).element_size()
                  for _, sh, dt in sizes]
        self.buf = torch.zeros(sum((n + 15) // 16 * 16 for n in nbytes),
                               dtype=torch.uint8, device=dev)
        off = 0
        for (name, sh, dt), n in zip(sizes, nbytes):
            setattr(self, name, self.buf[off:off + n].view(dt).view(sh))
            off += (n + 15) // 16 * 16
        d = N.ReplayRing()
        d.X = d.Xn = self.X.data_ptr()
        d.actions, d.scalars = self.actions.data_ptr(), self.scalars.data_ptr()
        d.move_bits = self.move_bits.data_ptr()
        d.shift_bits = self.shift_bits.data_ptr()
        d.cap = cap
        self.desc = d


class _Buffers:
    """Device buffers of one episode geometry (population, entry log, step
    scratch, per-step parameter tables).  Kept alive across episodes so the
    captured CUDA graphs' baked pointers stay valid."""

    def __init__(self, eng, tables, P, V, plan, forest):
        dev = eng.dev
        self.tables, self.P, self.V, self.plan = tables, P, V, plan
        self.forest = forest
        self.dsk = D.DeviceSketch(tables, dev)
        self.pop = [eng._pop(tables, P), eng._pop(tables, P)]
        self.rt = [torch.empty(P, dtype=torch.int32, device=dev),
                   torch.empty(P, dtype=torch.int32, device=dev)]
        self.steps = torch.zeros(P, dtype=torch.int32, device=dev)
        self.best = torch.full((P,), -math.inf, dtype=torch.float64,
                               device=dev)
        self.best_step = torch.zeros(P, dtype=torch.int32, device=dev)
        self.ts = N.TrackStats(self.steps.data_ptr(), self.best.data_ptr(),
                               self.best_step.data_ptr())
        slots = max(tables.local_slots, 1)
        Vm = max(V, 1)
        self.log_tiles = torch.empty((slots, Vm), dtype=torch.int16, device=dev)
        self.log_knobs = torch.empty((3, Vm), dtype=torch.uint8, device=dev)
        self.log_score = torch.empty(Vm, dtype=torch.float64, device=dev)
        self.log_reward = torch.empty(Vm, dtype=torch.float64, device=dev)
        self.log_track = torch.empty(Vm, dtype=torch.int32, device=dev)
        self.elog = N.EntryLog(self.log_tiles.data_ptr(),
                               self.log_knobs.data_ptr(),
                               self.log_score.data_ptr(),
                               self.log_reward.data_ptr(),
                               self.log_track.data_ptr(), Vm)
        n_steps = len(plan)
        self.n_ppo = sum(1 for s in plan if s["ppo"])
        self.status = torch.full((max(n_steps, 1),), -1, dtype=torch.int64,
                                 device=dev)
        self.losses = torch.zeros((max(self.n_ppo, 1), 16),
                                  dtype=torch.float64, device=dev)
        self.pol_out = {
            "actions": torch.empty((4, P), dtype=torch.int32, device=dev),
            "logp": torch.empty(P, dtype=torch.float64, device=dev),
            "move_bits": torch.empty(P, dtype=torch.int64, device=dev),
            "shift_bits": torch.empty(P, dtype=torch.int32, device=dev),
            "head0_col": torch.empty(P, dtype=torch.int32, device=dev)}
        self.reward = torch.empty(P, dtype=torch.float64, device=dev)
        # V buffers alternate by step parity: step k writes V(X') into
        # vbuf[k % 2] and reads/writes V(X) in vbuf[(k + 1) % 2], which
        # already holds V(X'_{k-1}) = V(X_k) whenever no update or cull
        # came in between (then V(X) is not recomputed)
        self.vbuf = [torch.empty(P, dtype=torch.float32, device=dev),
                     torch.empty(P, dtype=torch.float32, device=dev)]
        self.adv = torch.empty(P, dtype=torch.float64, device=dev)
        self.keep = torch.empty(P, dtype=torch.int32, device=dev)
        # per-step tables for graph replay (host fills them each episode),
        # views of one device block mirrored by one pinned block: an upload
        # is one copy
        Bmax = max([s["ppo"] or 0 for s in plan] + [1])
        ns, npp = max(n_steps, 1), max(self.n_ppo, 1)
        a16 = lambda n: (n + 15) // 16 * 16  # noqa: E731
        o_wpos = a16(ns * 16)
        o_slot = o_wpos + a16(ns * 8)
        o_adam = o_slot + a16(npp * Bmax * 4)
        nbytes = o_adam + npp * 4 * 8
        self.tab = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
        self.tab_pin = torch.zeros(nbytes, dtype=torch.uint8,
                                   pin_memory=dev.type == "cuda")

        def views(t):
            return (t[:ns * 16].view(torch.int64).view(ns, 2),
                    t[o_wpos:o_wpos + ns * 8].view(torch.int64),
                    t[o_slot:o_slot + npp * Bmax * 4].view(torch.int32)
                    .view(npp, Bmax),
                    t[o_adam:o_adam + npp * 32].view(torch.float64)
                    .view(npp, 4))
        self.rng_tab, self.wpos_tab, self.slot_tab, self.adam_tab = \
            views(self.tab)
        self.pins = dict(zip(("rng", "wpos", "slot", "adam"),
                             views(self.tab_pin)))
        self.graphs = None      # list of (first_step, last_step, CUDAGraph)


class EpisodeEngine:
    """Device state of one subgraph agent: parameters + Adam (DeviceAgent)
    and the replay ring, persistent across that subgraph's episodes like the
    reference's ``self.agents[sg]``/``self.buffers[sg]``.

    ``run_episode`` replays each inter-cull segment of the episode as one
    captured CUDA graph (the whole plan -- live-row counts, cull points,
    PPO steps, minibatch sizes -- is fixed before the episode starts; the
    per-step values that do change between episodes, i.e. the RNG base
    state, replay write position, minibatch slots and Adam bias
    corrections, are read by the kernels from device tables the host fills
    before launching).  Parity hooks (``inject``/``record``/
    ``cull_override``) run the same launch sequence eagerly."""

    def __init__(self, agent: AgentState, rl_cfg: RlConfig, levels: int,
                 device=None, use_graphs: bool = True, shard=None):
        N.load()
        self.dev = D._dev(device)
        self.agent = agent
        self.rl_cfg = rl_cfg
        self.levels = levels
        self.dagent = D.DeviceAgent(agent, levels, self.dev)
        N.check(N.load().harl_prepare(), "harl_prepare")
        self.replay = D.DeviceReplay(rl_cfg.buffer_capacity, agent.feature_len,
                                     self.dev)
        self._ppo_scratch = None
        self.use_graphs = use_graphs
        self._cache = {}
        # population sharding: (world, rank, process group or None)
        self.shard = shard
        if shard is not None:
            from .shard import GlobalReplayIndex
            self._gidx = GlobalReplayIndex(rl_cfg.buffer_capacity, shard[0])

    # -----------------------------------------------------------------------

    def _buffers(self, tables, cfg, forest, plan):
        key = (id(tables), cfg, id(forest), id(plan))   # plans are memoised
        b = self._cache.get(key)
        if b is None:
            if len(self._cache) > 8:
                self._cache.clear()
            b = _Buffers(self, tables, cfg.tracks, cfg.budget, plan, forest)
            b.keepalive = (tables, forest, plan)
            self._cache[key] = b
        return b

    @staticmethod
    def _v_reusable(plan, k):
        """V(X_k) == V(X'_{k-1}) bit for bit when step k-1 was followed by
        neither a PPO update nor a cull (same weights, same rows)."""
        return k > 0 and not plan[k - 1]["ppo"] and not plan[k - 1]["cull"]

    def _launch_step(self, b, k, step, cur, nxt, rt, used, graph_mode,
                     gen=None, inj=None, want_logits=False, m=None,
                     grow=None, m_total=0, keep_from=None):
        """Issue every launch of search step k (policy+walker, featurize,
        GBT+reward, V(X)/V(X'), finish).  In graph mode the RNG base state
        and the replay write position come from the device tables.

        Graph mode, a step without PPO update or cull before an equal-size
        step (_OVERLAP_POLICY): step k+1's policy network depends only on
        X' (the sampler's output) and unchanged weights, so it runs on a
        forked stream beside this step's value and GBT passes (disjoint
        SMs once the population is culled), joined before step k+1's
        sampler."""
        m = step["m"] if m is None else m
        pre = graph_mode and getattr(b, "pre_pol", None) == k
        b.pre_pol = None
        side = None
        if (graph_mode and _OVERLAP_POLICY and
                grow is None and inj is None and not want_logits and
                not _SPLIT_FEATURIZE and not _PAR_VALUE and not _FUSED_STEP
                and not step["ppo"] and not step["cull"] and
                k + 1 < len(b.plan) and b.plan[k + 1]["m"] == m):
            side = self._side_stream()
        try:
            return self._launch_step_body(b, k, step, cur, nxt, rt, used,
                                          graph_mode, gen, inj, want_logits,
                                          m, grow, m_total, keep_from, pre,
                                          side)
        finally:
            if side is not None:
                torch.cuda.current_stream().wait_stream(side)

    def _launch_step_body(self, b, k, step, cur, nxt, rt, used, graph_mode,
                          gen, inj, want_logits, m, grow, m_total, keep_from,
                          pre, side):
        tables, P = b.tables, b.P
        lib = N.load()
        out = dict(b.pol_out)
        out["tiles"], out["knobs"] = nxt["tiles"], nxt["knobs"]
        out["status"] = b.status[k:k + 1]
        res = D.policy_step(b.dsk, self.dagent, cur["feat"], cur["tiles"],
                            cur["knobs"], m, gen=gen, inject=inj, out=out,
                            want_logits=want_logits,
                            rng_dev=b.rng_tab[k] if graph_mode else None,
                            advance=not graph_mode, grow=grow,
                            m_total=m_total,
                            feat_out=None if _SPLIT_FEATURIZE else nxt["feat"],
                            fuse_tc=_FUSED_STEP, reset_status=False,
                            settled=k > 0 and not b.plan[k - 1]["ppo"] and
                            not b.plan[k - 1]["cull"],
                            gbt=(b.forest, cur["score"], nxt["score"], b.reward)
                            if _SAMPLE_GBT and not _SPLIT_FINISH and
                            not _PAR_VALUE and not _SPLIT_FEATURIZE else None,
                            split=D.STEP_SAMPLE_ONLY if pre else 0)
        gbt_done = res.get("gbt_fused", False)
        if side is not None:   # step k+1's policy network beside value + GBT
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                if D.policy_mlp(b.dsk, self.dagent, nxt["feat"], m):
                    b.pre_pol = k + 1
        if _SPLIT_FEATURIZE:
            D.featurize(b.dsk, nxt["tiles"], nxt["knobs"], m, nxt["feat"])
        # value pass first: the fused GBT kernel's finish epilogue needs
        # V(X) and V(X') (the GBT and value passes both read only X')
        v_cur, v_next = b.vbuf[(k + 1) % 2], b.vbuf[k % 2]
        reuse = self._v_reusable(b.plan, k)
        par = _PAR_VALUE
        po = b.pol_out
        io = N.StepBuffers(
            rt.data_ptr(), nxt["tiles"].data_ptr(), nxt["knobs"].data_ptr(),
            cur["feat"].data_ptr(), nxt["feat"].data_ptr(),
            nxt["score"].data_ptr(), b.reward.data_ptr(), v_cur.data_ptr(),
            v_next.data_ptr(), po["actions"].data_ptr(),
            po["head0_col"].data_ptr(), po["logp"].data_ptr(),
            po["move_bits"].data_ptr(), po["shift_bits"].data_ptr(),
            b.adv.data_ptr())
        cap = self.replay.cap
        keep_from = max(0, m - cap) if keep_from is None else keep_from
        wdev = D._ptr(b.wpos_tab[k:k + 1]) if graph_mode else None
        if gbt_done and _VALUE_FINISH and self.dagent.tc and not par:
            # the scores are in (sampler); the finish rides on the value pass
            with PF.span("value_tc", (0 if reuse else m) + m):
                rc = lib.harl_value_finish_tc(
                    C.byref(self.dagent.val_desc), cur["feat"].data_ptr(),
                    0 if reuse else m, nxt["feat"].data_ptr(), m,
                    tables.feature_len, v_cur.data_ptr(), v_next.data_ptr(),
                    self.dagent.packed["vt"].data_ptr(), D.WEIGHTS_SETTLED, io,
                    P, used, tables.local_slots, self.rl_cfg.discount, 1,
                    self.replay.desc, self.replay.wpos, keep_from, b.elog,
                    b.ts, wdev, D._stream())
            if rc == 0:
                return res
            if rc != N.E_LIMIT:
                N.check(rc, "harl_value_finish_tc")
        if par:
            main = torch.cuda.current_stream()
            side = self._side_stream()
            side.wait_stream(main)
            with torch.cuda.stream(side):
                D.value_pair(self.dagent, cur["feat"], 0 if reuse else m,
                             nxt["feat"], m, v_cur, v_next)
        else:
            # (the sampler or featurize launch precedes it: the weight
            # images were last written by an earlier Adam step)
            # (paired X/X' tiles per CTA when the next policy network runs
            # beside it: half the CTAs, the rest of the SMs for that one)
            D.value_pair(self.dagent, cur["feat"], 0 if reuse else m,
                         nxt["feat"], m, v_cur, v_next, settled=True,
                         paired=side is not None)
        if not _SPLIT_FINISH and not par and not gbt_done:
            with PF.span("gbt", m, launches=1):
                rc = lib.harl_gbt_finish_step(
                    C.byref(b.forest.desc), tables.feature_len,
                    cur["score"].data_ptr(), io, m, P, used,
                    tables.local_slots, self.rl_cfg.discount, 1,
                    self.replay.desc, self.replay.wpos, keep_from, b.elog,
                    b.ts, wdev, D._stream())
            if rc == 0:
                return res
            if rc != N.E_LIMIT:
                N.check(rc, "harl_gbt_finish_step")
        if not gbt_done:
            D.gbt_predict(b.forest, nxt["feat"], m, old_score=cur["score"],
                          out=nxt["score"], reward=b.reward)
        if par:
            main.wait_stream(side)
        with PF.span("finish", m, launches=1):
            N.check(lib.harl_finish_step(
                io, m, P, used, tables.local_slots, tables.feature_len,
                self.rl_cfg.discount, 1, self.replay.desc, self.replay.wpos,
                keep_from, b.elog, b.ts, wdev, D._stream()), "harl_finish_step")
        return res

    def _side_stream(self):
        s = getattr(self, "_side", None)
        if s is None:
            s = self._side = torch.cuda.Stream(device=self.dev)
        return s

    def _launch_step_uniform(self, b, k, step, cur, nxt, rt, used, gen,
                             inj=None):
        """Non-RL searchers (tuner.py:382-383): uniform valid actions, then
        the same walker/featurizer/cost model; no value/replay/PPO."""
        tables, m, P = b.tables, step["m"], b.P
        lib = N.load()
        acts = b.pol_out["actions"]
        if inj is None:
            D.uniform_actions(b.dsk, cur["tiles"], cur["knobs"], m, gen,
                              out=acts)
        else:
            acts.view(-1)[:4 * m].copy_(torch.from_numpy(
                np.ascontiguousarray(np.asarray(inj, np.int32).T).reshape(-1)))
        with PF.span("apply", m):
            N.check(lib.harl_apply_actions(
                C.byref(b.dsk.desc), D._ptr(cur["tiles"]), D._ptr(cur["knobs"]),
                m, P, D._ptr(acts), D._ptr(nxt["tiles"]), D._ptr(nxt["knobs"]),
                D._ptr(b.status[k:k + 1]), D._stream()), "harl_apply_actions")
        D.featurize(b.dsk, nxt["tiles"], nxt["knobs"], m, nxt["feat"])
        D.gbt_predict(b.forest, nxt["feat"], m, old_score=cur["score"],
                      out=nxt["score"], reward=b.reward)
        io = N.StepBuffers(
            rt.data_ptr(), nxt["tiles"].data_ptr(), nxt["knobs"].data_ptr(),
            cur["feat"].data_ptr(), nxt["feat"].data_ptr(),
            nxt["score"].data_ptr(), b.reward.data_ptr(), None, None, None,
            None, None, None, None, None)
        with PF.span("finish", m):
            N.check(lib.harl_finish_step(
                io, m, P, used, tables.local_slots, tables.feature_len, 0.0,
                0, None, 0, m, b.elog, b.ts, None, D._stream()),
                "harl_finish_step")

    def _launch_ppo(self, b, j, B, slots_t, t_pi, t_v, graph_mode):
        self._ensure_ppo_scratch(B)
        self.dagent.ppo_update(self.replay, slots_t, self.rl_cfg, t_pi, t_v,
                               scratch=self._ppo_scratch, losses=b.losses[j],
                               adam_dev=b.adam_tab[j] if graph_mode else None)

    def run_episode(self, tables: SketchTables, forest: D.DeviceForest, gen,
                    cfg: EpisodeConfig, order_counter: int = 0,
                    inject=None, record: list | None = None,
                    cull_override=None, defer_checks: bool = False
                    ) -> EpisodeResult:
        """Run one episode.  ``gen`` is the session's numpy Generator
        (PCG64), advanced exactly as the reference advances it.  ``inject``
        (optional callable ``step -> (m,4) actions``) replays externally
        chosen actions; ``record`` collects per-step device tensors for
        parity checks; ``cull_override(step, own_choice)`` may replace the
        eliminated track set (parity replays only).  ``defer_checks``: the
        per-step status words and the divergence flag are copied out
        asynchronously and checked by ``result.check()`` (the caller may
        issue more device work first); otherwise checked before returning."""
        # (graph replays update the parameters without passing through
        # DeviceAgent.ppo_update: the host copy is stale from here on)
        self.dagent._device_is_pin = False
        if self.shard is not None:
            return self._run_sharded(tables, forest, gen, cfg, order_counter)
        trace = _HOST_TRACE
        if trace is not None:
            trace.append(("episode", 0, 0, time.perf_counter()))
        plan = schedule(cfg, len(self.replay), self.rl_cfg)
        b = self._buffers(tables, cfg, forest, plan)
        if trace is not None:
            trace.append(("buffers", 0, 0, time.perf_counter()))
        # graphs for the production (tcgen05) path; the FFMA kernels used
        # by small test networks take their RNG state by value
        # a plan's first episode runs eagerly: capturing costs more than the
        # launches it saves once, and plans that change every episode (a
        # filling replay buffer, task sets visited once) never repay it
        b.uses = getattr(b, "uses", 0) + 1
        eager = (inject is not None or record is not None or
                 cull_override is not None or not self.use_graphs or
                 not self.dagent.tc or not cfg.rl or
                 (b.graphs is None and b.uses < 2 and _LAZY_CAPTURE))
        P = cfg.tracks
        # ---- population (outside any graph: the sampler may sync) -------
        cur, nxt = b.pop[0], b.pop[1]
        rt, rt_spare = b.rt[0], b.rt[1]
        cursor = None if eager else R.StreamCursor(gen)
        D.init_population(b.dsk, P, gen, cur["tiles"], cur["knobs"],
                          cursor=cursor)
        if trace is not None:
            trace.append(("init", 0, 0, time.perf_counter()))
        if getattr(b, "iota", None) is None:
            b.iota = torch.arange(P, dtype=torch.int32, device=self.dev)
        if eager:
            # (the graphed path records these launches in its first graph)
            self._episode_prologue(b, forest)
        if eager:
            res = self._run_eager(b, gen, cfg, order_counter, inject, record,
                                  cull_override)
        else:
            res = self._run_graphed(b, gen, cfg, order_counter, cursor)
        # the status words and the divergence flag in one pinned copy-out
        n = len(plan)
        pin = getattr(b, "check_pin", None)
        if pin is None:
            pin = b.check_pin = torch.empty(max(n, 1) + 1, dtype=torch.int64,
                                            pin_memory=True)
        pin[:n].copy_(b.status[:n], non_blocking=True)
        pin[n:n + 1].copy_(self.dagent.bad.to(torch.int64), non_blocking=True)
        PF.xfer("d2h", pin)
        ev = torch.cuda.Event()
        ev.record()
        words = pin[:n + 1]

        def check():
            ev.synchronize()
            w = words.numpy()
            for code in w[:n].view(np.uint64):
                D.raise_status(int(code))
            if int(w[n]):
                self.dagent.restore_diverged()
            D.raise_diverged(int(w[n]))
        res.check = check
        if not defer_checks:
            check()
        return res

    def _episode_prologue(self, b, forest):
        """The initial population's features and scores, and the per-episode
        resets (track stats, status words, divergence flag)."""
        P = b.P
        cur = b.pop[0]
        D.featurize(b.dsk, cur["tiles"], cur["knobs"], P, cur["feat"])
        D.gbt_predict(forest, cur["feat"], P, out=cur["score"])
        b.rt[0].copy_(b.iota)
        b.steps.zero_()
        b.best.fill_(-math.inf)
        b.best_step.zero_()
        b.status.fill_(-1)
        self.dagent.bad.zero_()

    def _result(self, b, cfg, order_counter, used, culls, train, alive):
        return EpisodeResult(tables=b.tables, visits=used,
                             order_start=order_counter,
                             log_tiles=b.log_tiles, log_knobs=b.log_knobs,
                             log_score=b.log_score, log_reward=b.log_reward,
                             log_track=b.log_track,
                             step_rows=[s["m"] for s in b.plan], culls=culls,
                             train=train, track_steps=b.steps,
                             track_best_step=b.best_step, alive=alive,
                             extra={"dsk": b.dsk})

    # ---- eager path (parity hooks) ------------------------------------------

    def _run_eager(self, b, gen, cfg, order_counter, inject, record,
                   cull_override):
        from . import rng as R
        P = cfg.tracks
        cur, nxt = b.pop[0], b.pop[1]
        rt, rt_spare = b.rt[0], b.rt[1]
        alive = np.ones(P, dtype=bool)
        culls, train = [], []
        used, ppo_k = 0, 0
        for k, step in enumerate(b.plan):
            m = step["m"]
            inj = inject(step["t"]) if inject is not None else None
            if not cfg.rl:
                self._launch_step_uniform(b, k, step, cur, nxt, rt, used, gen,
                                          inj)
                if record is not None:
                    po = b.pol_out
                    record.append({"t": step["t"], "m": m,
                                   "sel": rt[:m].clone(),
                                   "actions": po["actions"].view(-1)[:4 * m]
                                   .view(4, m).clone(),
                                   "new_feats": nxt["feat"][:m].clone(),
                                   "new_score": nxt["score"][:m].clone(),
                                   "rewards": b.reward[:m].clone()})
                cur, nxt = nxt, cur
                used += m
                continue
            # a record may name the steps it wants (``record.steps``): the
            # full-size parity tests keep a few steps of a 1 M-row episode
            want = record is not None and \
                (getattr(record, "steps", None) is None or
                 step["t"] in record.steps)
            if want:
                rng_before = gen.bit_generator.state
                params_before = self.dagent.params.clone()
            res = self._launch_step(b, k, step, cur, nxt, rt, used, False,
                                    gen=gen, inj=inj, want_logits=want)
            if inj is not None:
                R.skip_u64(gen, 4 * m)
            self.replay.note_push(m)
            if want:
                po = b.pol_out
                record.append({"t": step["t"], "m": m,
                               "rng_before": rng_before,
                               "params": params_before,
                               "tiles": cur["tiles"][:, :m].clone(),
                               "knobs": cur["knobs"][:, :m].clone(),
                               "sel": rt[:m].clone(),
                               "X": cur["feat"][:m].clone(),
                               "actions": po["actions"].view(-1)[:4 * m]
                               .view(4, m).clone(),
                               "logp": po["logp"][:m].clone(),
                               "logits": res["logits"].clone(),
                               "new_tiles": nxt["tiles"][:, :m].clone(),
                               "new_knobs": nxt["knobs"][:, :m].clone(),
                               "new_feats": nxt["feat"][:m].clone(),
                               "new_score": nxt["score"][:m].clone(),
                               "rewards": b.reward[:m].clone(),
                               "v_cur": b.vbuf[(k + 1) % 2][:m].clone(),
                               "v_next": b.vbuf[k % 2][:m].clone(),
                               "adv": b.adv[:m].clone()})
            cur, nxt = nxt, cur
            used += m
            if step["cull"]:
                tracks = rt[:m].cpu().numpy().astype(np.int64)
                before = alive.copy()
                gone = self._cull(tracks, b.adv, m, alive, cfg)
                if cull_override is not None:
                    forced = cull_override(step["t"], gone)
                    if forced is not None:
                        gone = np.sort(np.asarray(forced, dtype=np.int64))
                        alive[:] = before
                        alive[gone] = False
                culls.append((step["t"], gone, int(alive.sum())))
                keep = np.flatnonzero(alive[tracks])
                b.keep[:len(keep)].copy_(torch.from_numpy(keep.astype(np.int32)))
                self._compact(b, cur, rt, nxt, rt_spare, len(keep))
                cur, nxt = nxt, cur
                rt, rt_spare = rt_spare, rt
                if want:
                    record[-1]["cull"] = gone
            if step["ppo"]:
                B = step["ppo"]
                idx = gen.choice(len(self.replay), size=B, replace=False)
                # through this update's row of the pinned table block: a
                # pageable copy would synchronise the stream every update
                sl = self.replay.slots_of(idx)
                pin = b.pins["slot"]
                if pin.is_pinned() and B <= pin.shape[1] and ppo_k < pin.shape[0]:
                    pin[ppo_k, :B].numpy()[:] = sl
                    b.slot_tab[ppo_k, :B].copy_(pin[ppo_k, :B], non_blocking=True)
                    slots_t = b.slot_tab[ppo_k, :B]
                else:
                    slots_t = torch.from_numpy(sl).to(self.dev)
                a = self.agent
                a.opt_pi.t += 1
                a.opt_v.t += 1
                self._launch_ppo(b, ppo_k, B, slots_t, a.opt_pi.t, a.opt_v.t,
                                 False)
                train.append((step["t"], b.losses[ppo_k], B))
                if want:
                    record[-1]["ppo_idx"] = idx
                ppo_k += 1
        return self._result(b, cfg, order_counter, used, culls, train, alive)

    # ---- population-sharded path (one rank of G) ---------------------------

    def _allreduce_(self, t):
        import torch.distributed as dist
        group = self.shard[2]
        if dist.get_backend(group) == "nccl":
            dist.all_reduce(t, group=group)
        else:                                   # gloo: reduce a host copy
            h = t.cpu()
            dist.all_reduce(h, group=group)
            t.copy_(h)

    def _sharded_ppo_rows(self, slots_t, where_t, B, losses):
        """One PPO update of a sharded episode, identical bit for bit to the
        single-device update (so an episode does not depend on the world
        size): every rank writes the minibatch rows it owns (its ring slots
        ``slots_t``) into their minibatch positions ``where_t`` of a zeroed
        staging ring of B rows -- exactly one rank owns each row -- one
        NCCL all-reduce (uint8 sum: x + 0 = x for every byte) gives every
        rank the whole minibatch in minibatch order, and every rank runs
        the single-device ppo_update on it.  The all-reduce carries the
        B transitions' PPO inputs (B x (8F + 60) bytes, 115 KB at B = 256,
        F = 49) instead of the fp64 gradients (1.2 MB); the update itself,
        ~1.5 % of the step's flops at C2, is replicated."""
        import torch
        st = self._staging_ring(B)
        st.buf.zero_()
        ring = self.replay
        sl = slots_t.long()
        wh = where_t.long()
        st.X[wh] = ring.X[sl]
        st.actions[wh] = ring.actions[sl]
        st.scalars[wh] = ring.scalars[sl]
        st.move_bits[wh] = ring.move_bits[sl]
        st.shift_bits[wh] = ring.shift_bits[sl]
        self._allreduce_(st.buf)
        if getattr(self, "_iota_B", None) is None or self._iota_B.numel() < B:
            self._iota_B = torch.arange(B, dtype=torch.int32, device=self.dev)
        self._ensure_ppo_scratch(B)
        a = self.agent
        self.dagent.ppo_update(st, self._iota_B[:B], self.rl_cfg, a.opt_pi.t,
                               a.opt_v.t, scratch=self._ppo_scratch,
                               losses=losses)

    def _staging_ring(self, B):
        st = getattr(self, "_stage", None)
        if st is None or st.cap < B:
            st = self._stage = _StagingRing(B, self.agent.feature_len,
                                            self.dev)
        return st

    def _sharded_ppo_grads(self, slots_t, B, losses):
        """The gradient variant (HARL_SHARD_PPO=grads): per-shard gradient
        and loss partial sums over the owned rows (global 1/B), one
        all-reduce of {gradients, loss sums}, the identical Adam on every
        rank.  Rounded differently from the single-device sum."""
        import torch
        a = self.agent
        self._ensure_ppo_scratch(max(int(slots_t.numel()), 1))
        self.dagent.ppo_update(self.replay, slots_t, self.rl_cfg,
                               a.opt_pi.t, a.opt_v.t,
                               scratch=self._ppo_scratch,
                               losses=losses, B_norm=B, phase=1)
        n_g = self.dagent.grads.numel()
        buf = getattr(self, "_ar_buf", None)
        if buf is None or buf.numel() != n_g + 4:
            buf = self._ar_buf = torch.empty(n_g + 4, dtype=torch.float64,
                                             device=self.dev)
        buf[:n_g].copy_(self.dagent.grads.view(-1))
        buf[n_g:].copy_(losses[5:9])
        self._allreduce_(buf)
        self.dagent.grads.view(-1).copy_(buf[:n_g])
        losses[5:9].copy_(buf[n_g:])
        self.dagent.ppo_update(self.replay, slots_t, self.rl_cfg,
                               a.opt_pi.t, a.opt_v.t,
                               scratch=self._ppo_scratch,
                               losses=losses, B_norm=B, phase=2)

    def _gather_advantages(self, b, local_ids, m_l, P):
        """Every rank's (track id, advantage) of the cull step: one
        all-gather of fixed-size tensors (ceil(P / G) rows per rank, track
        id -1 for padding) on the device for NCCL, on the host for gloo."""
        import torch.distributed as dist
        world, _, group = self.shard
        cap = (P + world - 1) // world
        dev = self.dev
        mine = torch.full((2, cap), -1.0, dtype=torch.float64, device=dev)
        mine[0, :m_l] = torch.from_numpy(local_ids[:m_l].astype(np.float64)
                                         ).to(dev)
        mine[1, :m_l] = b.adv[:m_l]
        nccl = dist.get_backend(group) == "nccl"
        src = mine if nccl else mine.cpu()
        out = torch.empty((world * 2, cap), dtype=src.dtype,
                          device=src.device)
        dist.all_gather_into_tensor(out, src, group=group)
        o = out.cpu().numpy().reshape(world, 2, cap)
        ids = o[:, 0, :].reshape(-1)
        av = o[:, 1, :].reshape(-1)
        keep = ids >= 0
        return ids[keep].astype(np.int64), av[keep]

    def _run_sharded(self, tables, forest, gen, cfg, order_counter):
        """This rank's share of the episode: tracks i with i % G == rank
        (shard.py).  Every rank advances the same generator; uniforms are
        taken at the tracks' global rows; culls are decided on the
        all-gathered advantages; PPO gradients are per-shard sums, one
        all-reduce, then the identical Adam on every rank."""
        import torch.distributed as dist
        from . import rng as R
        from .shard import ShardLayout, cull_decision
        world, rank, group = self.shard
        if not cfg.rl:
            raise NotImplementedError("sharded episodes are RL-only")
        P = cfg.tracks
        lay = ShardLayout(P, world, rank)
        plan = schedule(cfg, len(self._gidx), self.rl_cfg)
        Pl = len(lay.local_ids)
        b = self._buffers(tables, cfg, forest, plan)
        dev = self.dev
        if not hasattr(b, "full"):
            b.full = self._pop(tables, P)
            b.full_rt = torch.arange(P, dtype=torch.int32, device=dev)
            b.grow = torch.zeros(P, dtype=torch.int32, device=dev)
        # every rank samples the whole population (identical draws), keeps
        # its own tracks
        D.init_population(b.dsk, P, gen, b.full["tiles"], b.full["knobs"])
        cur, nxt = b.pop[0], b.pop[1]
        rt, rt_spare = b.rt[0], b.rt[1]
        b.keep[:Pl].copy_(torch.from_numpy(lay.local_ids.astype(np.int32)))
        self._compact(b, b.full, b.full_rt, cur, rt, Pl)
        D.featurize(b.dsk, cur["tiles"], cur["knobs"], Pl, cur["feat"])
        D.gbt_predict(forest, cur["feat"], Pl, out=cur["score"])
        b.steps.zero_()
        b.best.fill_(-math.inf)
        b.best_step.zero_()
        b.status.fill_(-1)
        self.dagent.bad.zero_()
        alive = np.ones(P, dtype=bool)
        local_ids = lay.local_ids.copy()        # ids of the local rows
        culls, train = [], []
        used_local, used, ppo_k = 0, 0, 0
        local_rows = []
        cap = self.replay.cap
        grow_all = None                          # changes only at culls
        live = None
        for k, step in enumerate(plan):
            m = step["m"]
            if grow_all is None:
                # the local rows' global rows: fixed between culls, so one
                # (pinned, asynchronous) upload per segment -- a pageable
                # copy per step would synchronise the stream every step
                grow_all = lay.global_rows(alive, local_ids)
                live = np.flatnonzero(alive)
                if getattr(b, "grow_pin", None) is None:
                    b.grow_pin = torch.empty(Pl, dtype=torch.int32,
                                             pin_memory=True)
                n_g = len(grow_all)
                b.grow_pin[:n_g].numpy()[:] = grow_all
                b.grow[:n_g].copy_(b.grow_pin[:n_g], non_blocking=True)
            m_l = int(np.searchsorted(grow_all, m))   # local rows in sel
            keep_from = int(np.searchsorted(grow_all[:m_l], max(0, m - cap)))
            self._launch_step(b, k, step, cur, nxt, rt, used_local, False,
                              gen=gen, m=m_l, grow=b.grow, m_total=m,
                              keep_from=keep_from)
            self.replay.note_push(m_l)
            local_rows.append(m_l)
            self._gidx.push_step(live[:m] % world)
            cur, nxt = nxt, cur
            used_local += m_l
            used += m
            if step["cull"]:
                ids, av = self._gather_advantages(b, local_ids, m_l, P)
                gone = cull_decision(alive, ids, av, cfg.cull_fraction,
                                     cfg.min_tracks)
                alive[gone] = False
                grow_all = None
                culls.append((step["t"], gone, int(alive.sum())))
                keep = np.flatnonzero(alive[local_ids]).astype(np.int32)
                b.keep[:len(keep)].copy_(torch.from_numpy(keep))
                self._compact(b, cur, rt, nxt, rt_spare, len(keep))
                cur, nxt = nxt, cur
                rt, rt_spare = rt_spare, rt
                local_ids = local_ids[keep]
            if step["ppo"]:
                B = step["ppo"]
                pos = gen.choice(len(self._gidx), size=B, replace=False)
                owners, lpush = self._gidx.locate(pos)
                mine = owners == rank
                slots = (lpush[mine] % cap).astype(np.int32)
                where = np.flatnonzero(mine).astype(np.int32)
                # pinned ring of (slot, minibatch position) lists, one per
                # update of the episode: the copies stay asynchronous
                n_up = max(1, sum(1 for s_ in plan if s_["ppo"]))
                sp = getattr(b, "slot_pin", None)
                if sp is None or sp.shape[2] < B or sp.shape[1] < n_up:
                    sp = b.slot_pin = torch.empty((2, n_up, B),
                                                  dtype=torch.int32,
                                                  pin_memory=True)
                    b.slot_dev = torch.empty_like(sp, device=dev)
                k_ = len(slots)
                sp[0, ppo_k, :k_].numpy()[:] = slots
                sp[1, ppo_k, :k_].numpy()[:] = where
                b.slot_dev[:, ppo_k, :k_].copy_(sp[:, ppo_k, :k_],
                                                non_blocking=True)
                slots_t = b.slot_dev[0, ppo_k, :k_]
                a = self.agent
                a.opt_pi.t += 1
                a.opt_v.t += 1
                losses = b.losses[ppo_k]
                if _SHARD_PPO == "grads":
                    self._sharded_ppo_grads(slots_t, B, losses)
                else:
                    self._sharded_ppo_rows(slots_t,
                                           b.slot_dev[1, ppo_k, :k_], B,
                                           losses)
                train.append((step["t"], losses, B))
                ppo_k += 1
        st = b.status.cpu().numpy().view(np.uint64)
        PF.xfer("d2h", b.status)
        for code in st[:len(plan)]:
            D.raise_status(int(code))
        self.dagent.raise_if_diverged()
        res = self._result(b, cfg, order_counter, used_local, culls, train,
                           alive)
        res.extra["global_visits"] = used
        res.extra["local_ids_final"] = local_ids
        res.step_rows = local_rows
        return res

    # ---- graph path --------------------------------------------------------

    # graph boundaries at the start of an episode: the rows of the first
    # graph are prepared before any GPU work can start, each later graph's
    # while the previous one runs (host precompute ~10-30 us per step)
    # (a split after step 0: the first graph needs only step 0's RNG base,
    # so the first PPO minibatch draw is computed while it runs -- 0.20 ->
    # 0.15 ms before the first graph at C2; HARL_HEAD_SPLITS overrides)
    HEAD_SPLITS = tuple(int(x) for x in os.environ.get(
        "HARL_HEAD_SPLITS", "1,2,8").split(",") if x)

    def _segments(self, plan):
        """Step index ranges of the captured graphs: a host cull decision
        ends a segment (the next one starts with the survivor gather), and
        the first steps are split at HEAD_SPLITS so the host precompute of
        each graph overlaps the previous one.  Returns (first, last,
        starts_after_cull)."""
        segs, start, after_cull = [], 0, False
        for k, step in enumerate(plan):
            head_end = (k + 1) in self.HEAD_SPLITS and start <= k and \
                k < len(plan) - 1 and not step["cull"] and \
                all(not s["cull"] for s in plan[:k])
            if step["cull"] or k == len(plan) - 1 or head_end:
                segs.append((start, k, after_cull))
                after_cull = bool(step["cull"])
                start = k + 1
        return segs

    def _capture(self, b, gen):
        """Record each segment's launches once (pointer sequence fixed by
        the plan).  ``gen`` only supplies the stream increment (jump
        tables); states come from the device tables at replay."""
        from . import rng as R
        lib = N.load()
        N.check(lib.harl_prepare(), "harl_prepare")
        # the sampler's byte-sliced jump table must exist before capture
        N.check(lib.harl_rng_prepare(C.byref(R.to_struct(gen))),
                "harl_rng_prepare")
        b.graph_inc = int(gen.bit_generator.state["state"]["inc"])
        if self.dagent.tc:
            self.dagent.hid_scratch(b.P)
        self._ensure_ppo_scratch(max([s["ppo"] or 0 for s in b.plan] + [1]))
        segs = self._segments(b.plan)
        graphs = []
        b.pre_pol = None
        cur_i, rt_i, used, ppo_k = 0, 0, 0, 0
        wpos0 = self.replay.wpos
        count0 = self.replay.count
        stream = torch.cuda.Stream(device=self.dev)
        stream.wait_stream(torch.cuda.current_stream())
        for si, (k0, k1, after_cull) in enumerate(segs):
            g = torch.cuda.CUDAGraph()
            n0 = PF.launch_count()
            with torch.cuda.graph(g, stream=stream,
                                  capture_error_mode="relaxed"):
                if si == 0:
                    self._episode_prologue(b, b.forest)
                if after_cull:
                    n_keep = b.plan[k0 - 1]["m"] - b.plan[k0 - 1]["cull"]
                    self._compact(b, b.pop[cur_i], b.rt[rt_i],
                                  b.pop[1 - cur_i], b.rt[1 - rt_i], n_keep)
                    cur_i, rt_i = 1 - cur_i, 1 - rt_i
                for k in range(k0, k1 + 1):
                    step = b.plan[k]
                    self._launch_step(b, k, step, b.pop[cur_i],
                                      b.pop[1 - cur_i], b.rt[rt_i], used, True,
                                      gen=gen)
                    cur_i = 1 - cur_i
                    used += step["m"]
                    if step["ppo"]:
                        B = step["ppo"]
                        self._launch_ppo(b, ppo_k, B, b.slot_tab[ppo_k, :B],
                                         1, 1, True)
                        ppo_k += 1
            graphs.append((k0, k1, g, PF.launch_count() - n0, after_cull))
        torch.cuda.current_stream().wait_stream(stream)
        self.replay.wpos, self.replay.count = wpos0, count0
        b.graphs = graphs

    def _run_graphed(self, b, gen, cfg, order_counter, cursor=None):
        from . import rng as R
        P = cfg.tracks
        inc = int(gen.bit_generator.state["state"]["inc"])
        if b.graphs is not None and getattr(b, "graph_inc", None) != inc:
            b.graphs = None     # jump tables of another stream are baked in
        if b.graphs is None:
            self._capture(b, gen)
            PF.add_launches(-sum(g[3] for g in b.graphs))  # not executed
        # ---- host precompute of every per-step value (data-independent),
        # pipelined: the first segment's rows go up and its graph starts,
        # then the host prepares the remaining rows while the GPU runs
        n_steps = len(b.plan)
        pins = b.pins
        rng_np = pins["rng"].numpy().view(np.uint64)
        wpos_np = pins["wpos"].numpy()
        slot_np = pins["slot"].numpy()
        adam_np = pins["adam"].numpy()
        a = self.agent
        if cursor is None:
            cursor = R.StreamCursor(gen)
        pk = [0]

        def precompute(k0, k1):
            p0 = pk[0]
            for k in range(k0, k1 + 1):
                step = b.plan[k]
                st = cursor.s
                rng_np[k, 0] = st >> 64           # u128 {hi, lo} (common.cuh)
                rng_np[k, 1] = st & ((1 << 64) - 1)
                cursor.skip_u64(4 * step["m"])
                wpos_np[k] = self.replay.wpos
                self.replay.note_push(step["m"])
                if step["ppo"]:
                    B = step["ppo"]
                    cursor.sync_to()
                    idx = gen.choice(len(self.replay), size=B, replace=False)
                    cursor.sync_from()
                    slot_np[pk[0], :B] = self.replay.slots_of(idx)
                    a.opt_pi.t += 1
                    a.opt_v.t += 1
                    adam_np[pk[0]] = (1.0 - 0.9 ** a.opt_pi.t,
                                      1.0 - 0.999 ** a.opt_pi.t,
                                      1.0 - 0.9 ** a.opt_v.t,
                                      1.0 - 0.999 ** a.opt_v.t)
                    pk[0] += 1
            return p0, pk[0]

        def upload(k0, k1, p0, p1):
            # the whole table block in one stream-ordered copy (rows of
            # earlier segments are rewritten with the values they hold)
            b.tab.copy_(b.tab_pin, non_blocking=True)
            PF.xfer("h2d", b.tab)

        segs = b.graphs
        # rows of segment 0 first; then, before blocking anywhere, the rows
        # of the next segment(s) while the GPU runs the launched ones
        done = [-1]          # last step whose rows are uploaded

        trace = _HOST_TRACE

        def prepare(upto):
            if upto > done[0]:
                k0 = done[0] + 1
                if trace is not None:
                    trace.append(("pre", k0, upto, time.perf_counter()))
                rows = precompute(k0, upto)
                if trace is not None:
                    trace.append(("up", k0, upto, time.perf_counter()))
                upload(k0, upto, *rows)
                done[0] = upto
                if trace is not None:
                    trace.append(("done", k0, upto, time.perf_counter()))

        prepare(segs[0][1])
        # ---- replay the segments; host culls in between --------------------
        alive = np.ones(P, dtype=bool)
        culls, train = [], []
        used, ppo_k = 0, 0
        rt_i = 0
        for si, (k0, k1, g, nl, after_cull) in enumerate(segs):
            if after_cull:
                prev = b.plan[k0 - 1]
                m = prev["m"]
                if _PY_CULL:
                    tracks, adv_h = self._cull_inputs(b, rt_i, m)
                    gone, keep = self._cull_rows(tracks, adv_h, alive, cfg)
                    kp = b.keep_pin if getattr(b, "keep_pin", None) is not \
                        None else None
                    if kp is None:
                        kp = b.keep_pin = torch.empty(b.P, dtype=torch.int32,
                                                      pin_memory=True)
                    kp[:len(keep)].numpy()[:] = keep
                    b.keep[:len(keep)].copy_(kp[:len(keep)], non_blocking=True)
                    PF.xfer("h2d", b.keep[:len(keep)])
                else:
                    gone = self._cull_native(b, rt_i, m, alive, cfg)
                culls.append((prev["t"], gone, int(alive.sum())))
                rt_i = 1 - rt_i
            prepare(k1)
            if trace is not None:
                trace.append(("launch", k0, k1, time.perf_counter()))
            g.replay()
            if trace is not None:
                trace.append(("launched", k0, k1, time.perf_counter()))
            PF.add_launches(nl)
            # look ahead while this segment runs: the next segment's rows, or
            # all remaining rows when a cull (which blocks the host) comes
            # first
            if si + 1 < len(segs):
                nk0, nk1, _, _, n_after_cull = segs[si + 1]
                prepare(n_steps - 1 if n_after_cull else nk1)
            for k in range(k0, k1 + 1):
                step = b.plan[k]
                used += step["m"]
                if step["ppo"]:
                    train.append((step["t"], b.losses[ppo_k], step["ppo"]))
                    ppo_k += 1
        cursor.sync_to()
        return self._result(b, cfg, order_counter, used, culls, train, alive)

    # -----------------------------------------------------------------------

    def _pop(self, tables, P):
        dev = self.dev
        tiles, knobs = D.alloc_state(P, tables, dev)
        return {"tiles": tiles, "knobs": knobs,
                "feat": torch.empty((P, tables.feature_len),
                                    dtype=torch.float64, device=dev),
                "score": torch.empty(P, dtype=torch.float64, device=dev)}

    def _cull(self, tracks, adv, m, alive, cfg):
        """stopping.py:68-86 on the host: the n_elim lowest by
        (advantage, -index) go.  ``adv``: host array of the step's rows (or
        a device tensor).  A partition finds the cut value; only ties at the
        cut are ordered (higher index first), as the full sort would."""
        live = np.flatnonzero(alive)
        n = len(live)
        n_elim = min(int(math.floor(cfg.cull_fraction * n)),
                     n - cfg.min_tracks)
        if n_elim <= 0:
            return np.zeros(0, dtype=np.int64)
        a = adv[:m].cpu().numpy() if isinstance(adv, torch.Tensor) \
            else np.asarray(adv[:m])
        adv_full = np.zeros(len(alive))
        adv_full[tracks] = a
        v = adv_full[live]
        if np.isnan(v).any():      # the reference's own sort (shard.py)
            from .shard import eliminated
            gone = eliminated(live, v, n_elim)
        else:
            cut = np.partition(v, n_elim - 1)[n_elim - 1]
            below = live[v < cut]
            tied = live[v == cut]
            need = n_elim - len(below)
            gone = np.sort(np.concatenate([below, tied[::-1][:need]]))
        alive[gone] = False
        return gone

    def _cull_rows(self, tracks, adv, alive, cfg):
        """``_cull`` on the cull step's rows directly (row r = live track
        tracks[r], every live track has one row): (eliminated track ids
        ascending, surviving rows ascending)."""
        m = len(tracks)
        n_elim = min(int(math.floor(cfg.cull_fraction * m)),
                     m - cfg.min_tracks)
        if n_elim <= 0:
            return np.zeros(0, dtype=np.int64), np.arange(m, dtype=np.int32)
        if np.isnan(adv).any():          # the reference's sort (_cull)
            gone = self._cull(tracks, adv, m, alive, cfg)
            return gone, np.flatnonzero(alive[tracks]).astype(np.int32)
        cut = np.partition(adv, n_elim - 1)[n_elim - 1]
        out = adv < cut
        tie = np.flatnonzero(adv == cut)
        need = n_elim - int(np.count_nonzero(out))
        # ties go by higher track index first (stopping.py:81)
        out[tie[np.argsort(-tracks[tie], kind="stable")[:need]]] = True
        alive[tracks[out]] = False
        # ascending ids without a sort: the tracks that were live and are not
        dead = np.zeros(len(alive), dtype=bool)
        dead[tracks[out]] = True
        return np.flatnonzero(dead), np.flatnonzero(~out).astype(np.int32)

    def _cull_native(self, b, rt_i, m, alive, cfg):
        """The graphed episode's cull: one pinned D2H of the step's rows and
        advantages, harl_cull_select on the host (the same decision as
        ``_cull``), the survivor rows H2D from a pinned buffer."""
        live_n = int(alive.sum())
        n_elim = min(int(math.floor(cfg.cull_fraction * live_n)),
                     live_n - cfg.min_tracks)
        n_elim = max(n_elim, 0)
        if getattr(b, "cull_pin", None) is None:
            b.cull_pin = (torch.empty(b.P, dtype=torch.int32, pin_memory=True),
                          torch.empty(b.P, dtype=torch.float64,
                                      pin_memory=True))
            b.keep_pin = torch.empty(b.P, dtype=torch.int32, pin_memory=True)
            b.alive8 = np.zeros(b.P, dtype=np.uint8)
        pt, pa = b.cull_pin
        pt[:m].copy_(b.rt[rt_i][:m], non_blocking=True)
        pa[:m].copy_(b.adv[:m], non_blocking=True)
        PF.xfer("d2h", pt[:m], pa[:m])
        trace = _HOST_TRACE
        if trace is not None:
            trace.append(("cull_wait", 0, 0, time.perf_counter()))
        torch.cuda.current_stream().synchronize()
        if trace is not None:
            trace.append(("cull_synced", 0, 0, time.perf_counter()))
        if np.isnan(pa[:m].numpy()).any():   # the reference's sort (_cull)
            tracks = pt[:m].numpy().astype(np.int64)
            gone, keep = self._cull_rows(tracks, pa[:m].numpy().copy(),
                                         alive, cfg)
            b.keep_pin[:len(keep)].numpy()[:] = keep
            b.keep[:len(keep)].copy_(b.keep_pin[:len(keep)],
                                     non_blocking=True)
            PF.xfer("h2d", b.keep[:len(keep)])
            return gone
        # (bool and uint8 share a layout: the library marks alive in place)
        a8 = alive.view(np.uint8) if alive.dtype == np.bool_ and \
            alive.flags.c_contiguous else b.alive8
        if a8 is b.alive8:
            a8[:len(alive)] = alive
        gone = np.zeros(n_elim, dtype=np.int64)
        nk = C.c_int64(0)
        N.check(N.load().harl_cull_select(
            pa.data_ptr(), pt.data_ptr(), m, a8.ctypes.data, len(alive),
            n_elim, gone.ctypes.data, b.keep_pin.data_ptr(), C.byref(nk)),
            "harl_cull_select")
        if trace is not None:
            trace.append(("cull_selected", 0, 0, time.perf_counter()))
        if a8 is b.alive8:
            alive[:] = a8[:len(alive)].astype(bool)
        b.keep[:nk.value].copy_(b.keep_pin[:nk.value], non_blocking=True)
        PF.xfer("h2d", b.keep[:nk.value])
        if trace is not None:
            trace.append(("cull_done", 0, 0, time.perf_counter()))
        return gone

    def _cull_inputs(self, b, rt_i, m):
        """Row->track ids and advantages of the cull step in one pinned
        D2H round trip."""
        if getattr(b, "cull_pin", None) is None:
            b.cull_pin = (torch.empty(b.P, dtype=torch.int32, pin_memory=True),
                          torch.empty(b.P, dtype=torch.float64,
                                      pin_memory=True))
        pt, pa = b.cull_pin
        pt[:m].copy_(b.rt[rt_i][:m], non_blocking=True)
        pa[:m].copy_(b.adv[:m], non_blocking=True)
        PF.xfer("d2h", pt[:m], pa[:m])
        torch.cuda.current_stream().synchronize()
        return pt[:m].numpy().astype(np.int64), pa[:m].numpy().copy()

    def _compact(self, b, src, rt_src, dst, rt_dst, n_keep):
        """Survivor gather with row indices from ``b.keep`` (device)."""
        lib = N.load()
        tables = b.tables
        P = src["tiles"].shape[1]
        with PF.span("gather", n_keep):
            N.check(lib.harl_gather_rows(
                b.keep.data_ptr(), n_keep, tables.local_slots,
                tables.feature_len, src["tiles"].data_ptr(),
                src["knobs"].data_ptr(), src["feat"].data_ptr(),
                src["score"].data_ptr(), rt_src.data_ptr(), P,
                dst["tiles"].data_ptr(), dst["knobs"].data_ptr(),
                dst["feat"].data_ptr(), dst["score"].data_ptr(),
                rt_dst.data_ptr(), dst["tiles"].shape[1], D._stream()),
                "harl_gather_rows")

    def _ensure_ppo_scratch(self, B):
        lib = N.load()
        need = lib.harl_ppo_scratch_bytes(B, self.dagent.row_stride, 0)
        if self._ppo_scratch is None or self._ppo_scratch.numel() < need:
            # the old buffer is retired, not freed: graphs captured for
            # other cached geometries keep its address baked in
            if self._ppo_scratch is not None:
                self.dagent._retired.append(self._ppo_scratch)
            self._ppo_scratch = torch.empty(need, dtype=torch.uint8,
                                            device=self.dev)

    def sync_to_host(self):
        """Mirror device parameters/moments into the numpy agent lists."""
        self.dagent.download()
