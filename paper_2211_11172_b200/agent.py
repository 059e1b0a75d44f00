"""Actor-critic parameters and optimizer state (host side, fp64 master).

The numpy float64 parameter lists are canonical, exactly as in the reference
(``rlcore.py:74-178``): the policy is a tanh trunk ``F -> hidden...`` whose
last layer also goes through tanh (rlcore.py:139), followed by four
single-layer heads of widths ``(S*S+1, 3, 3, 3)``; the value net is
``F -> hidden... -> 1``.  Parameter order is ``[W0, b0, W1, b1, ...]`` for the
trunk, then ``[W, b]`` per head (rlcore.py:88-93,130-134).

``init_session_agents`` reproduces the reference session's draw order
(tuner.py:268-280: per subgraph, PolicyNet then ValueNet, Glorot-normal
``sqrt(2/(fin+fout))`` with head output scale 0.01, zero biases,
rlcore.py:77-86) so a standalone engine starts from the same weights as a
reference session with the same seed.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class RlConfig:
    """rlcore.py:24-45 (validated the same way)."""

    lr_actor: float = 3e-4
    lr_critic: float = 1e-3
    discount: float = 0.9
    clip_ratio: float = 0.2
    value_loss_weight: float = 0.5
    entropy_weight: float = 0.01
    hidden: tuple = (128, 128)
    minibatch: int = 256
    buffer_capacity: int = 4096
    train_interval: int = 2

    def __post_init__(self):
        if not 0.0 <= self.discount <= 1.0:
            raise ValueError("discount must be in [0, 1]")
        if not 0.0 < self.clip_ratio < 1.0:
            raise ValueError("clip_ratio must be in (0, 1)")
        if self.lr_actor <= 0 or self.lr_critic <= 0:
            raise ValueError("learning rates must be positive")
        if self.train_interval < 1 or self.minibatch < 1:
            raise ValueError("train_interval and minibatch must be >= 1")


def _dense_params(sizes, rng, out_scale=1.0):
    params = []
    last = len(sizes) - 2
    for i in range(len(sizes) - 1):
        fin, fout = sizes[i], sizes[i + 1]
        scale = math.sqrt(2.0 / (fin + fout)) * (out_scale if i == last else 1.0)
        params.append(rng.normal(0.0, scale, size=(fin, fout)))
        params.append(np.zeros(fout))
    return params


def init_policy_params(feature_len, num_slots, hidden, rng):
    params = _dense_params([feature_len, *hidden], rng)
    for k in (num_slots * num_slots + 1, 3, 3, 3):
        params += _dense_params([hidden[-1], k], rng, out_scale=0.01)
    return params


def init_value_params(feature_len, hidden, rng):
    return _dense_params([feature_len, *hidden, 1], rng)


@dataclass
class AdamState:
    """rlcore.py:48-71: moments aligned with the parameter list."""

    lr: float
    m: list
    v: list
    t: int = 0
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8

    @classmethod
    def for_params(cls, params, lr):
        return cls(lr=lr, m=[np.zeros_like(p) for p in params],
                   v=[np.zeros_like(p) for p in params])


@dataclass
class AgentState:
    """One subgraph's agent: fp64 params (updated in place) + Adam."""

    policy: list
    value: list
    opt_pi: AdamState
    opt_v: AdamState
    hidden: tuple
    num_slots: int
    feature_len: int
    extra: dict = field(default_factory=dict)

    @property
    def n_trunk(self) -> int:
        return len(self.hidden)


def init_session_agents(subgraph_slots, feature_len, cfg: RlConfig, rng):
    """Per subgraph (in network order) PolicyNet then ValueNet draws."""
    out = {}
    for sg_id, s in subgraph_slots:
        pol = init_policy_params(feature_len, s, cfg.hidden, rng)
        val = init_value_params(feature_len, cfg.hidden, rng)
        out[sg_id] = AgentState(policy=pol, value=val,
                                opt_pi=AdamState.for_params(pol, cfg.lr_actor),
                                opt_v=AdamState.for_params(val, cfg.lr_critic),
                                hidden=tuple(cfg.hidden), num_slots=s,
                                feature_len=feature_len)
    return out
