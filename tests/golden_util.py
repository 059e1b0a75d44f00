"""Loading the committed reference fixtures (tests/golden/*.json|npz)."""

from __future__ import annotations

import glob
import hashlib
import json
import os

import numpy as np

from paper_2211_11172_b200 import workloads as W
from paper_2211_11172_b200.agent import RlConfig, init_session_agents
from paper_2211_11172_b200.space import SketchTables

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

RL_SEARCHERS = ("rl", "rl-fixed-length", "rl-greedy-subgraph")
ADAPTIVE = ("rl", "rl-greedy-subgraph")

TUNER_DEFAULTS = dict(seed=0, min_tracks=64, initial_tracks=None,
                      cull_window=20, cull_fraction=0.5, episode_len=None,
                      train_interval=2, discount=0.9, lr_actor=3e-4,
                      lr_critic=1e-3, clip_ratio=0.2, value_loss_weight=0.5,
                      entropy_weight=0.01, minibatch=256,
                      buffer_capacity=4096, hidden=(128, 128))


def digest(a) -> str:
    a = np.ascontiguousarray(np.asarray(a))
    h = hashlib.sha256()
    h.update(str(a.dtype.str).encode() + str(a.shape).encode())
    h.update(a.tobytes())
    return h.hexdigest()


def digest_list(arrs) -> str:
    h = hashlib.sha256()
    for a in arrs:
        h.update(digest(a).encode())
    return h.hexdigest()


def case_names():
    """Recorded sessions: a .json header with its .npz arrays (other
    fixtures -- sim_golden.json, gbt_fit_large.npz -- stand alone)."""
    return sorted(os.path.basename(p)[:-5]
                  for p in glob.glob(os.path.join(GOLDEN, "*.json"))
                  if os.path.exists(p[:-5] + ".npz"))


class GoldenCase:
    """A recorded reference session, rebuilt with this package's host
    mirror (workload parsing, sketch tables, agent init)."""

    def __init__(self, name: str):
        with open(os.path.join(GOLDEN, name + ".json")) as fh:
            self.rec = json.load(fh)
        self.arr = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
        self.name = name
        cfg = dict(TUNER_DEFAULTS)
        cfg.update(self.rec["cfg"])
        cfg["hidden"] = tuple(cfg["hidden"])
        self.cfg = cfg
        net = W.loads_network(self.rec["yaml"])
        tg = self.rec["target"]
        self.target = W.gpu_target() if tg.get("name") == "gpu" else \
            W.TargetConfig(**tg)
        self.net = net
        sketches = {sg.id: W.generate_sketches(sg, self.target)
                    for sg in net.subgraphs}
        slots = [(sg.id, max(k.space.num_tile_slots for k in sketches[sg.id]))
                 for sg in net.subgraphs]
        self.sg = net.subgraphs[self.rec["sg"]]
        self.sketches = sketches[self.sg.id]
        self.slots = dict(slots)[self.sg.id]
        assert self.slots == self.rec["slots"]
        flen = SketchTables(self.sg, self.sketches[0], self.target,
                            self.slots).feature_len
        self.rl = RlConfig(lr_actor=cfg["lr_actor"], lr_critic=cfg["lr_critic"],
                           discount=cfg["discount"],
                           clip_ratio=cfg["clip_ratio"],
                           value_loss_weight=cfg["value_loss_weight"],
                           entropy_weight=cfg["entropy_weight"],
                           hidden=cfg["hidden"], minibatch=cfg["minibatch"],
                           buffer_capacity=cfg["buffer_capacity"],
                           train_interval=cfg["train_interval"])
        rng = np.random.default_rng(cfg["seed"])
        self.agents = init_session_agents(slots, flen, self.rl, rng)
        self.agent = self.agents[self.sg.id]
        self.feature_len = flen

    def tables(self, sketch_idx: int) -> SketchTables:
        return SketchTables(self.sg, self.sketches[sketch_idx], self.target,
                            self.slots)

    @property
    def tracks(self):
        c = self.cfg
        return c["initial_tracks"] if c["initial_tracks"] is not None \
            else 2 * c["min_tracks"]

    @property
    def track_len(self):
        c = self.cfg
        return c["episode_len"] if c["episode_len"] is not None \
            else 2 * c["cull_window"]

    @property
    def is_rl(self):
        return self.rec["searcher"] in RL_SEARCHERS

    @property
    def adaptive(self):
        return self.rec["searcher"] in ADAPTIVE

    def trees(self):
        out = []
        for i in range(self.rec["n_trees"]):
            p = f"tree{i:03d}_"
            out.append((self.arr[p + "feature"].astype(np.int64),
                        self.arr[p + "threshold"],
                        self.arr[p + "left"].astype(np.int64),
                        self.arr[p + "right"].astype(np.int64),
                        self.arr[p + "value"]))
        return out

    @property
    def model_base(self):
        return float(self.arr["model_base"][0])

    @staticmethod
    def rng_from(state: dict) -> np.random.Generator:
        g = np.random.Generator(np.random.PCG64())
        st = dict(state)
        st["state"] = {"state": int(state["state"]["state"]),
                       "inc": int(state["state"]["inc"])}
        g.bit_generator.state = st
        return g
