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
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from . import device as D
from . import profiling as PF
from .agent import AgentState, RlConfig
from .space import SketchTables


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


def schedule(cfg: EpisodeConfig, replay_count: int, rl_cfg: RlConfig):
    """The episode's step plan, known before it starts: the live-row count
    per step, where culls happen and how many rows they keep, and the
    replay size at each PPO step.  None of it depends on the data
    (tuner.py:371-432, stopping.py:68-95)."""
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

    def rewards_per_step(self):
        r = self.log_reward[:self.visits].cpu().numpy()
        out, p = [], 0
        for m in self.step_rows:
            out.append(r[p:p + m])
            p += m
        return out


class EpisodeEngine:
    """Device state of one subgraph agent: parameters + Adam (DeviceAgent)
    and the replay ring, persistent across that subgraph's episodes like the
    reference's ``self.agents[sg]``/``self.buffers[sg]``."""

    def __init__(self, agent: AgentState, rl_cfg: RlConfig, levels: int,
                 device=None):
        N.load()
        self.dev = D._dev(device)
        self.agent = agent
        self.rl_cfg = rl_cfg
        self.levels = levels
        self.dagent = D.DeviceAgent(agent, levels, self.dev)
        self.replay = D.DeviceReplay(rl_cfg.buffer_capacity, agent.feature_len,
                                     self.dev)
        self._ppo_scratch = None

    # -----------------------------------------------------------------------

    def run_episode(self, tables: SketchTables, forest: D.DeviceForest, gen,
                    cfg: EpisodeConfig, order_counter: int = 0,
                    inject=None, record: list | None = None,
                    cull_override=None) -> EpisodeResult:
        """Run one episode.  ``gen`` is the session's numpy Generator
        (PCG64), advanced exactly as the reference advances it.  ``inject``
        (optional callable ``step -> (m,4) actions``) replays externally
        chosen actions; ``record`` collects per-step device tensors for
        parity checks; ``cull_override(step, own_choice)`` may replace the
        eliminated track set (parity replays only)."""
        dev = self.dev
        dsk = D.DeviceSketch(tables, dev)
        F = tables.feature_len
        P = cfg.tracks
        V = cfg.budget
        rl = cfg.rl
        plan = schedule(cfg, len(self.replay), self.rl_cfg)
        if not rl:
            raise NotImplementedError("non-RL searchers: uniform device "
                                      "actions are not implemented yet")
        # ---- population -------------------------------------------------
        cur = self._pop(tables, P)
        nxt = self._pop(tables, P)
        D.init_population(dsk, P, gen, cur["tiles"], cur["knobs"])
        D.featurize(dsk, cur["tiles"], cur["knobs"], P, cur["feat"])
        D.gbt_predict(forest, cur["feat"], P, out=cur["score"])
        rt = torch.arange(P, dtype=torch.int32, device=dev)
        rt_spare = torch.empty_like(rt)
        steps_t = torch.zeros(P, dtype=torch.int32, device=dev)
        best = torch.full((P,), -math.inf, dtype=torch.float64, device=dev)
        best_step = torch.zeros(P, dtype=torch.int32, device=dev)
        ts = N.TrackStats(steps_t.data_ptr(), best.data_ptr(),
                          best_step.data_ptr())
        # ---- entry log ----------------------------------------------------
        slots = max(tables.local_slots, 1)
        log_tiles = torch.empty((slots, max(V, 1)), dtype=torch.int16, device=dev)
        log_knobs = torch.empty((3, max(V, 1)), dtype=torch.uint8, device=dev)
        log_score = torch.empty(max(V, 1), dtype=torch.float64, device=dev)
        log_reward = torch.empty(max(V, 1), dtype=torch.float64, device=dev)
        log_track = torch.empty(max(V, 1), dtype=torch.int32, device=dev)
        elog = N.EntryLog(log_tiles.data_ptr(), log_knobs.data_ptr(),
                          log_score.data_ptr(), log_reward.data_ptr(),
                          log_track.data_ptr(), max(V, 1))
        # ---- per-step scratch ---------------------------------------------
        n_steps = len(plan)
        status = torch.full((max(n_steps, 1),), -1, dtype=torch.int64,
                            device=dev)
        n_ppo = sum(1 for s in plan if s["ppo"])
        losses = torch.zeros((max(n_ppo, 1), 8), dtype=torch.float64,
                             device=dev)
        pol_out = {
            "actions": torch.empty((4, P), dtype=torch.int32, device=dev),
            "logp": torch.empty(P, dtype=torch.float64, device=dev),
            "move_bits": torch.empty(P, dtype=torch.int64, device=dev),
            "shift_bits": torch.empty(P, dtype=torch.int32, device=dev),
            "head0_col": torch.empty(P, dtype=torch.int32, device=dev)}
        reward = torch.empty(P, dtype=torch.float64, device=dev)
        v_cur = torch.empty(P, dtype=torch.float32, device=dev)
        v_next = torch.empty(P, dtype=torch.float32, device=dev)
        adv = torch.empty(P, dtype=torch.float64, device=dev)
        alive = np.ones(P, dtype=bool)
        culls, train = [], []
        used = 0
        ppo_k = 0
        lib = N.load()
        for k, step in enumerate(plan):
            m = step["m"]
            out = dict(pol_out)
            out["tiles"], out["knobs"] = nxt["tiles"], nxt["knobs"]
            out["status"] = status[k:k + 1]
            inj = inject(step["t"]) if inject is not None else None
            res = D.policy_step(dsk, self.dagent, cur["feat"], cur["tiles"],
                                cur["knobs"], m, gen=gen, inject=inj, out=out,
                                want_logits=record is not None)
            if inj is not None:
                from . import rng as R
                R.skip_u64(gen, 4 * m)
            D.featurize(dsk, nxt["tiles"], nxt["knobs"], m, nxt["feat"])
            D.gbt_predict(forest, nxt["feat"], m, old_score=cur["score"],
                          out=nxt["score"], reward=reward)
            D.value_pair(self.dagent, cur["feat"], m, nxt["feat"], m, v_cur,
                         v_next)
            cap = self.replay.cap
            io = N.StepBuffers(
                rt.data_ptr(), nxt["tiles"].data_ptr(),
                nxt["knobs"].data_ptr(), cur["feat"].data_ptr(),
                nxt["feat"].data_ptr(), nxt["score"].data_ptr(),
                reward.data_ptr(), v_cur.data_ptr(), v_next.data_ptr(),
                pol_out["actions"].data_ptr(), pol_out["head0_col"].data_ptr(),
                pol_out["logp"].data_ptr(), pol_out["move_bits"].data_ptr(),
                pol_out["shift_bits"].data_ptr(), adv.data_ptr())
            with PF.span("finish", m):
              N.check(lib.harl_finish_step(
                io, m, P, used, tables.local_slots, F, self.rl_cfg.discount,
                1 if rl else 0, self.replay.desc, self.replay.wpos,
                max(0, m - cap), elog, ts, D._stream()), "harl_finish_step")
            self.replay.note_push(m)
            if record is not None:
                record.append({"t": step["t"], "m": m,
                               "sel": rt[:m].clone(),
                               "X": cur["feat"][:m].clone(),
                               "actions": pol_out["actions"].view(-1)[:4 * m]
                               .view(4, m).clone(),
                               "logp": pol_out["logp"][:m].clone(),
                               "logits": res["logits"].clone(),
                               "new_tiles": nxt["tiles"][:, :m].clone(),
                               "new_knobs": nxt["knobs"][:, :m].clone(),
                               "new_feats": nxt["feat"][:m].clone(),
                               "new_score": nxt["score"][:m].clone(),
                               "rewards": reward[:m].clone(),
                               "v_cur": v_cur[:m].clone(),
                               "v_next": v_next[:m].clone(),
                               "adv": adv[:m].clone()})
            # rows >= m (budget tail) keep their state: only happens on the
            # final step, so the swap below is safe
            cur, nxt = nxt, cur
            used += m
            if step["cull"]:
                tracks = rt[:m].cpu().numpy().astype(np.int64)
                before = alive.copy()
                gone = self._cull(tracks, adv, m, alive, cfg)
                if cull_override is not None:
                    forced = cull_override(step["t"], gone)
                    if forced is not None:
                        gone = np.sort(np.asarray(forced, dtype=np.int64))
                        alive[:] = before
                        alive[gone] = False
                culls.append((step["t"], gone, int(alive.sum())))
                keep = np.flatnonzero(alive[tracks])
                self._compact(tables, cur, rt, nxt, rt_spare, keep)
                cur, nxt = nxt, cur
                rt, rt_spare = rt_spare, rt
                if record is not None:
                    record[-1]["cull"] = gone
            if step["ppo"]:
                B = step["ppo"]
                idx = gen.choice(len(self.replay), size=B, replace=False)
                slots_np = self.replay.slots_of(idx)
                slots_t = torch.from_numpy(slots_np).to(dev)
                a = self.agent
                a.opt_pi.t += 1
                a.opt_v.t += 1
                self._ensure_ppo_scratch(B)
                self.dagent.ppo_update(self.replay, slots_t, self.rl_cfg,
                                       a.opt_pi.t, a.opt_v.t,
                                       scratch=self._ppo_scratch,
                                       losses=losses[ppo_k])
                train.append((step["t"], losses[ppo_k], B))
                if record is not None:
                    record[-1]["ppo_idx"] = idx
                ppo_k += 1
        # ---- errors in step order (the reference raises at the first) -----
        st = status.cpu().numpy().view(np.uint64)
        bad_ppo = int(self.dagent.bad.item())
        for code in st[:n_steps]:
            D.raise_status(int(code))
        if bad_ppo:
            from .errors import RlDivergedError
            raise RlDivergedError("non-finite loss or gradient in update")
        return EpisodeResult(tables=tables, visits=used,
                             order_start=order_counter, log_tiles=log_tiles,
                             log_knobs=log_knobs, log_score=log_score,
                             log_reward=log_reward, log_track=log_track,
                             step_rows=[s["m"] for s in plan], culls=culls,
                             train=train, track_steps=steps_t,
                             track_best_step=best_step, alive=alive)

    # -----------------------------------------------------------------------

    def _pop(self, tables, P):
        dev = self.dev
        tiles, knobs = D.alloc_state(P, tables, dev)
        return {"tiles": tiles, "knobs": knobs,
                "feat": torch.empty((P, tables.feature_len),
                                    dtype=torch.float64, device=dev),
                "score": torch.empty(P, dtype=torch.float64, device=dev)}

    def _cull(self, tracks, adv, m, alive, cfg):
        """stopping.py:68-86 on the host: lowest (advantage, -index) go."""
        live = np.flatnonzero(alive)
        n = len(live)
        n_elim = min(int(math.floor(cfg.cull_fraction * n)),
                     n - cfg.min_tracks)
        if n_elim <= 0:
            return np.zeros(0, dtype=np.int64)
        a = adv[:m].cpu().numpy()
        adv_full = np.zeros(len(alive))
        adv_full[tracks] = a
        order = np.lexsort((-live, adv_full[live]))
        gone = np.sort(live[order[:n_elim]])
        alive[gone] = False
        return gone

    def _compact(self, tables, src, rt_src, dst, rt_dst, keep_rows):
        lib = N.load()
        idx = torch.from_numpy(keep_rows.astype(np.int32)).to(self.dev)
        P = src["tiles"].shape[1]
        with PF.span("gather", len(keep_rows)):
          N.check(lib.harl_gather_rows(
            idx.data_ptr(), len(keep_rows), tables.local_slots,
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
            self._ppo_scratch = torch.empty(need, dtype=torch.uint8,
                                            device=self.dev)

    def sync_to_host(self):
        """Mirror device parameters/moments into the numpy agent lists."""
        self.dagent.download()
