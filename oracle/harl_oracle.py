"""ORACLE — CPU restatement of the reference's HARL inner search step.

THIS IS TEST INFRASTRUCTURE.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline / ``--impl reference`` leg may import it, and
only as the checker or as the timed CPU reference.  The product path
(``paper_2211_11172_b200``) never imports, calls or falls back to it.

What it restates (reference files under ``/root/reference/pkg/src/schedtune``):

* ``TuningSession._run_episode`` ............... tuner.py:350-440
* ``sample_initial_schedules`` ................. schedspace.py:165-178
* ``action_mask`` / ``decode_action`` /
  ``apply_action`` ............................. schedspace.py:196-301
* ``SketchContext.stage_footprints/featurize`` . schedspace.py:372-438
* ``_Tree.predict`` / ``SurrogateModel.predict`` costmodel.py:67-78,219-230
* ``Mlp``/``PolicyNet``/``ValueNet`` fwd+bwd ... rlcore.py:74-178
* ``masked_log_softmax`` / ``sample_categorical``
  / ``select_actions`` / ``advantage`` ......... rlcore.py:185-234
* ``ReplayBuffer`` / ``batch_arrays`` .......... rlcore.py:253-286
* ``actor_grads`` / ``critic_grads`` /
  ``ppo_update`` / ``Adam.step`` ............... rlcore.py:48-71,293-378
* ``TrackSet.cull`` / ``episode_done`` ......... stopping.py:68-95
* ``rank_scores`` ............................... costmodel.py:266-286
* ``_fit_tree`` / ``fit_incremental`` (GBT refit) costmodel.py:81-141,190-212
* ``simulate_time`` / ``brute_force_best`` ........ measure.py:78-167

It is written population-at-once (structure-of-arrays numpy) instead of the
reference's per-track objects, but every floating-point operation is the
same numpy/libm call in the same order, so on the same inputs and the same
``numpy.random.Generator`` it reproduces the reference bit for bit.  That
claim is pinned by ``tests/test_oracle_golden.py`` against fixtures recorded
from the reference itself (``tests/golden/make_golden.py``) and by the
reference's own known-answer tests restated in ``tests/test_oracle_pins.py``.

Third-party arithmetic on the path: numpy (BLAS ``@``, ``exp``/``log``,
``cumsum``, ``Generator``) and glibc libm (``math.log2``/``math.log10``) —
called directly, exactly as the reference does.
"""

from __future__ import annotations

import math
from collections import deque
from dataclasses import dataclass, field

import numpy as np

PREDICTION_FLOOR = 1e-6


class OracleInvalidAction(ValueError):
    def __init__(self, subspace: str, detail: str):
        super().__init__(f"invalid {subspace} action: {detail}")
        self.subspace = subspace


class OracleDiverged(RuntimeError):
    pass


# ---------------------------------------------------------------------------
# schedule space (population SoA: tiles u16 [B, ndims*L], knobs u8 [B, 3])


def sample_initial(tb, count: int, rng: np.random.Generator):
    """schedspace.py:165-178 — per track: one ``integers`` per tiled dim
    (index into ``list_tilings``), then compute-at, parallel, unroll.

    ``Generator.integers`` with an array of upper bounds consumes the stream
    exactly like the reference's sequential scalar calls (checked in tests),
    so the draws are made track-major in one call."""
    nd = tb.ndims
    per = np.concatenate([tb.tiling_counts,
                          [tb.ncas, tb.max_fusible + 1, tb.n_unroll]])
    draws = rng.integers(0, np.tile(per, count)).reshape(count, nd + 3)
    tiles = np.zeros((count, tb.local_slots), dtype=np.uint16)
    for d in range(nd):
        rows = tb.tiling_table[tb.tiling_offsets[d] + draws[:, d]]
        tiles[:, d * tb.levels:(d + 1) * tb.levels] = rows
    knobs = draws[:, nd:].astype(np.uint8)
    return tiles, knobs


def action_masks(tb, tiles, knobs, num_slots: int):
    """schedspace.py:226-262 for a batch; returns 4 boolean arrays."""
    B = len(tiles)
    S, L = num_slots, tb.levels
    tiling = np.zeros((B, S * S + 1), dtype=bool)
    tiling[:, -1] = True
    for src in range(tb.local_slots):
        movable = tiles[:, src] > 1
        base = (src // L) * L
        for dst in range(base, base + L):
            if dst != src:
                tiling[:, src * S + dst] = movable

    def shift(pos, top):
        return np.stack([pos > 0, np.ones(B, dtype=bool), pos < top], axis=1)

    k = knobs.astype(np.int64)
    return (tiling, shift(k[:, 0], tb.ncas - 1),
            shift(k[:, 1], tb.max_fusible), shift(k[:, 2], tb.n_unroll - 1))


def decode(actions, num_slots: int):
    """schedspace.py:196-210 for a batch -> (src, dst, d_ca, d_par, d_ur)."""
    a = np.asarray(actions, dtype=np.int64)
    noop = a[:, 0] == num_slots * num_slots
    src = np.where(noop, -1, a[:, 0] // num_slots)
    dst = np.where(noop, -1, a[:, 0] % num_slots)
    return src, dst, a[:, 1] - 1, a[:, 2] - 1, a[:, 3] - 1


def spf(n: int) -> int:
    if n % 2 == 0:
        return 2
    p = 3
    while p * p <= n:
        if n % p == 0:
            return p
        p += 2
    return n


def apply_actions(tb, tiles, knobs, actions, num_slots: int):
    """schedspace.py:265-301 row by row semantics; the first offending row
    (in row order) raises, with the same subspace check order."""
    L = tb.levels
    src, dst, dca, dpar, dur = decode(actions, num_slots)
    new_t = tiles.copy()
    new_k = knobs.astype(np.int64).copy()
    for r in range(len(tiles)):
        s, d = int(src[r]), int(dst[r])
        if s >= 0:
            if s >= tb.local_slots or d >= tb.local_slots or d < 0:
                raise OracleInvalidAction("tiling", "slot outside this sketch")
            if s // L != d // L:
                raise OracleInvalidAction(
                    "tiling", "move crosses dimensions, product not conserved")
            if s == d:
                raise OracleInvalidAction("tiling", "source equals destination")
            f = int(new_t[r, s])
            if f <= 1:
                raise OracleInvalidAction("tiling", "source factor is 1")
            p = spf(f)
            new_t[r, s] = f // p
            new_t[r, d] = int(new_t[r, d]) * p
        ca = new_k[r, 0] + dca[r]
        if not 0 <= ca < tb.ncas:
            raise OracleInvalidAction("compute_at", f"index {ca} out of range")
        par = new_k[r, 1] + dpar[r]
        if not 0 <= par <= tb.max_fusible:
            raise OracleInvalidAction("parallel", f"count {par} out of range")
        ur = new_k[r, 2] + dur[r]
        if not 0 <= ur < tb.n_unroll:
            raise OracleInvalidAction("unroll", f"index {ur} out of range")
        new_k[r] = (ca, par, ur)
    return new_t, new_k.astype(np.uint8)


def footprints(tb, tiles, knobs):
    """schedspace.py:372-411: exact integer (l1, l2) per candidate (int64;
    the tables guarantee every value < 2^53, so ``float()`` is exact)."""
    L = tb.levels
    t = tiles.astype(np.int64)
    t1 = t[:, L - 1::L] if tb.ndims else np.zeros((len(t), 0), np.int64)
    t2 = (t[:, L - 2::L] * t[:, L - 1::L]) if L >= 2 else t1
    root = knobs[:, 0].astype(np.int64) == 0
    l1 = np.zeros(len(t), dtype=np.int64)
    l2 = np.zeros(len(t), dtype=np.int64)
    for tensors, inter, extra, _ in tb.stages:
        s1 = np.zeros(len(t), dtype=np.int64)
        s2 = np.zeros(len(t), dtype=np.int64)
        o1 = o2 = None
        for terms in tensors:
            e1 = np.ones(len(t), dtype=np.int64)
            e2 = np.ones(len(t), dtype=np.int64)
            for gi, sc, off in terms:
                e1 *= sc * t1[:, gi] + off
                e2 *= sc * t2[:, gi] + off
            s1 += e1
            s2 += e2
            o1, o2 = e1, e2
        s1 += (inter + extra) * o1
        s2 += extra * o2 + np.where(root, inter * o2, 0)
        l1 += s1
        l2 += s2
    return l1, l2


def featurize(tb, tiles, knobs):
    """schedspace.py:415-438; glibc ``math.log2``/``math.log10`` per value."""
    B = len(tiles)
    L = tb.levels
    x = np.zeros((B, tb.feature_len), dtype=np.float64)
    for s in range(tb.local_slots):
        x[:, s] = [math.log2(int(v)) / 10.0 for v in tiles[:, s]]
    pos = tb.max_feature_dims * L
    k = knobs.astype(np.int64)
    x[:, pos] = [c / (tb.ncas - 1) if tb.ncas > 1 else 0.0 for c in k[:, 0]]
    x[:, pos + 1] = [p / tb.max_fusible if tb.max_fusible else 0.0
                     for p in k[:, 1]]
    x[np.arange(B), pos + 2 + k[:, 2]] = 1.0
    pos += 2 + tb.n_unroll
    l1, l2 = footprints(tb, tiles, knobs)
    x[:, pos] = [math.log10(1.0 + float(v)) / 6.0 for v in l1]
    x[:, pos + 1] = [math.log10(1.0 + float(v)) / 6.0 for v in l2]
    x[:, pos + 2] = math.log10(max(tb.flops, 1.0)) / 12.0
    return x


# ---------------------------------------------------------------------------
# cost model inference


@dataclass
class GbtModel:
    """Trees as the reference stores them (costmodel.py:59-78)."""

    base: float = 1.0
    learning_rate: float = 0.3
    fitted: bool = False
    trees: list = field(default_factory=list)   # (feat, thr, left, right, val)

    def predict(self, X):
        """costmodel.py:219-230: ``pred = pred + lr*leaf`` per tree, floor."""
        X = np.atleast_2d(np.asarray(X, dtype=np.float64))
        if not self.fitted:
            return np.maximum(np.ones(len(X)), PREDICTION_FLOOR)
        pred = np.full(len(X), self.base)
        rows = np.arange(len(X))
        for feat, thr, left, right, val in self.trees:
            node = np.zeros(len(X), dtype=np.int64)
            for _ in range(64):
                f = feat[node]
                live = f >= 0
                if not live.any():
                    break
                go_left = X[rows, np.maximum(f, 0)] <= thr[node]
                node = np.where(live, np.where(go_left, left[node],
                                               right[node]), node)
            pred = pred + self.learning_rate * val[node]
        return np.maximum(pred, PREDICTION_FLOOR)


def fit_tree(X, y, max_depth: int, min_leaf: int):
    """costmodel.py:81-141: exact greedy variance-reduction split search.
    Nodes are numbered as the reference creates them (an explicit stack,
    left child processed first, children allocated at the parent's split).
    Returns (feature, threshold, left, right, value) arrays."""
    feature, threshold, left, right, value = [], [], [], [], []

    def add_node():
        feature.append(-1)
        threshold.append(0.0)
        left.append(-1)
        right.append(-1)
        value.append(0.0)
        return len(feature) - 1

    root = add_node()
    stack = [(root, np.arange(len(y)), 0)]
    while stack:
        nid, idx, depth = stack.pop()
        ys = y[idx]
        mean = float(ys.mean())
        value[nid] = mean
        if depth >= max_depth or len(idx) < 2 * min_leaf:
            continue
        if float(((ys - mean) ** 2).sum()) <= 1e-24:
            continue
        Xs = X[idx]
        order = np.argsort(Xs, axis=0, kind="stable")
        Xsort = np.take_along_axis(Xs, order, axis=0)
        csum = np.cumsum(ys[order], axis=0)
        total = float(ys.sum())
        m = len(idx)
        pos = np.arange(1, m, dtype=np.float64)
        sum_l = csum[:-1]
        gain = (sum_l ** 2) / pos[:, None] + \
            ((total - sum_l) ** 2) / (m - pos)[:, None]
        ok = Xsort[1:] != Xsort[:-1]
        if min_leaf > 1:
            ok &= ((pos >= min_leaf) & (m - pos >= min_leaf))[:, None]
        gain = np.where(ok, gain, -np.inf)
        flat = int(np.argmax(gain))
        if not np.isfinite(gain.flat[flat]):
            continue
        split_pos, feat = divmod(flat, X.shape[1])
        thr = 0.5 * (Xsort[split_pos, feat] + Xsort[split_pos + 1, feat])
        go_left = Xs[:, feat] <= thr
        li, ri = idx[go_left], idx[~go_left]
        if len(li) == 0 or len(ri) == 0:
            continue
        lid, rid = add_node(), add_node()
        feature[nid] = int(feat)
        threshold[nid] = float(thr)
        left[nid] = lid
        right[nid] = rid
        stack.append((rid, ri, depth + 1))
        stack.append((lid, li, depth + 1))
    return (np.asarray(feature, np.int64), np.asarray(threshold, np.float64),
            np.asarray(left, np.int64), np.asarray(right, np.int64),
            np.asarray(value, np.float64))


def tree_predict(tree, X):
    """_Tree.predict (costmodel.py:67-78)."""
    feat, thr, left, right, val = tree
    node = np.zeros(len(X), dtype=np.int64)
    rows = np.arange(len(X))
    for _ in range(64):
        f = feat[node]
        live = f >= 0
        if not live.any():
            break
        go_left = X[rows, np.maximum(f, 0)] <= thr[node]
        node = np.where(live, np.where(go_left, left[node], right[node]), node)
    return val[node]


def gbt_fit(X, y, n_trees: int = 50, max_depth: int = 6,
            learning_rate: float = 0.3, min_leaf: int = 1):
    """SurrogateModel.fit_incremental (costmodel.py:190-212) on a prepared
    (X, y): returns (base, trees, final training predictions)."""
    X = np.asarray(X, np.float64)
    y = np.asarray(y, np.float64)
    base = float(y.mean())
    trees = []
    pred = np.full(len(y), base)
    for _ in range(n_trees):
        resid = y - pred
        if float(np.abs(resid).max()) <= 1e-12:
            break
        tree = fit_tree(X, resid, max_depth, min_leaf)
        pred = pred + learning_rate * tree_predict(tree, X)
        trees.append(tree)
    return base, trees, pred


SIM_DEFAULTS = dict(cores=32, cap_l1=4096.0, cap_l2=131072.0,
                    miss_penalty_l1=0.3, miss_penalty_l2=0.6,
                    parallel_overhead=0.02,
                    unroll_factors=((0, 1.00), (16, 0.97), (64, 0.95),
                                    (512, 0.98), (1024, 1.00)),
                    peak_flops=1e11)


def _miss_factor(l1, l2, p):
    """measure.py:78-81."""
    m1 = 1.0 + p["miss_penalty_l1"] * max(0.0, l1 / p["cap_l1"] - 1.0)
    m2 = 1.0 + p["miss_penalty_l2"] * max(0.0, l2 / p["cap_l2"] - 1.0)
    return m1 * m2


def sim_time(tb, tiles_row, knobs_row, params=None):
    """measure.simulate_time (measure.py:99-112) for one state given as the
    flat tile row + (ca, par, ur), over the host mirror's stage tables."""
    p = dict(SIM_DEFAULTS)
    p.update(params or {})
    L = tb.levels
    t = [int(v) for v in tiles_row]
    ca, par, ur = (int(v) for v in knobs_row)
    depth = tb.unroll_depths[ur]
    u = dict(p["unroll_factors"]).get(depth, 1.0)
    t1 = [t[d * L + L - 1] for d in range(tb.ndims)]
    t2 = [t[d * L + L - 2] * t[d * L + L - 1] for d in range(tb.ndims)] \
        if L >= 2 else list(t1)
    total = 0.0
    for s_i, (tensors, inter, extra, flops) in enumerate(tb.stages):
        def el(terms, tl):
            n = 1
            for gi, sc, off in terms:
                n *= sc * tl[gi] + off
            return n
        l1 = sum(el(tt, t1) for tt in tensors)
        l2 = sum(el(tt, t2) for tt in tensors)
        l1 += (inter + extra) * el(tensors[-1], t1)
        l2 += extra * el(tensors[-1], t2)
        if ca == 0:
            l2 += inter * el(tensors[-1], t2)
        m = _miss_factor(float(l1), float(l2), p)
        spatial = tb.sim_spatial[s_i]
        if par == 0 or not spatial:
            spd = 1.0
        else:
            extent = 1
            for gi in spatial:
                for lv in range(par):
                    extent *= t[gi * L + lv]
            used = min(extent, p["cores"])
            balance = extent / (math.ceil(extent / p["cores"]) * p["cores"])
            spd = used * balance * (1.0 - p["parallel_overhead"] * (par - 1))
        total += (flops / p["peak_flops"]) * m * u / spd
    for flops, l1, l2 in tb.sim_skipped:
        total += (flops / p["peak_flops"]) * _miss_factor(l1, l2, p)
    return total


def brute_force_best(tb, params=None):
    """measure.brute_force_best (measure.py:135-167): (tiles, knobs, time)
    of the minimum, ties on the canonical text."""
    import itertools
    L = tb.levels
    per_dim = [tb.tiling_table[int(tb.tiling_offsets[d]):
                               int(tb.tiling_offsets[d]) +
                               int(tb.tiling_counts[d])]
               for d in range(tb.ndims)]
    best = (math.inf, "", None, None)
    for combo in itertools.product(*per_dim):
        row = np.concatenate(combo) if combo else np.zeros(0, np.uint16)
        for ca in range(tb.ncas):
            for par in range(tb.max_fusible + 1):
                for ur in range(tb.n_unroll):
                    tm = sim_time(tb, row, (ca, par, ur), params)
                    if tm < best[0] or (tm == best[0] and
                                        tb.canonical(row, (ca, par, ur))
                                        < best[1]):
                        best = (tm, tb.canonical(row, (ca, par, ur)),
                                row.copy(), (ca, par, ur))
    return best[2], best[3], best[0]


# ---------------------------------------------------------------------------
# actor-critic networks (parameters are the reference's numpy lists)


def dense_forward(Ws, bs, x, tanh_last: bool):
    """rlcore.py:95-103 (+ the trunk tanh of rlcore.py:139 when tanh_last)."""
    acts = [x]
    a = x
    for i, (W, b) in enumerate(zip(Ws, bs)):
        z = a @ W + b
        a = np.tanh(z) if (i < len(Ws) - 1) else z
        acts.append(a)
    if tanh_last:
        a = np.tanh(a)
    return a, acts


def dense_backward(Ws, acts, dout):
    """rlcore.py:105-116."""
    n = len(Ws)
    grads = [None] * (2 * n)
    d = dout
    for i in range(n - 1, -1, -1):
        if i != n - 1:
            d = d * (1.0 - acts[i + 1] ** 2)
        grads[2 * i] = acts[i].T @ d
        grads[2 * i + 1] = d.sum(axis=0)
        d = d @ Ws[i].T
    return grads, d


@dataclass
class Agent:
    """Policy (trunk + 4 single-layer heads) and value net, fp64 master."""

    trunk_W: list
    trunk_b: list
    head_W: list
    head_b: list
    val_W: list
    val_b: list

    def policy_params(self):
        out = []
        for W, b in zip(self.trunk_W, self.trunk_b):
            out += [W, b]
        for W, b in zip(self.head_W, self.head_b):
            out += [W, b]
        return out

    def value_params(self):
        out = []
        for W, b in zip(self.val_W, self.val_b):
            out += [W, b]
        return out

    @classmethod
    def from_param_lists(cls, pi: list, vf: list, n_trunk: int):
        return cls(trunk_W=pi[0:2 * n_trunk:2], trunk_b=pi[1:2 * n_trunk:2],
                   head_W=pi[2 * n_trunk::2], head_b=pi[2 * n_trunk + 1::2],
                   val_W=vf[0::2], val_b=vf[1::2])

    def policy_forward(self, X):
        hid, trunk_acts = dense_forward(self.trunk_W, self.trunk_b, X,
                                        tanh_last=True)
        logits = [hid @ W + b for W, b in zip(self.head_W, self.head_b)]
        return logits, (trunk_acts, hid)

    def value(self, X):
        out, acts = dense_forward(self.val_W, self.val_b, X, tanh_last=False)
        return out[:, 0], acts


def masked_log_softmax(logits, mask):
    """rlcore.py:185-199."""
    if not mask.any(axis=1).all():
        raise OracleDiverged("action mask with no valid entry")
    z = np.where(mask, logits, -np.inf)
    zmax = z.max(axis=1, keepdims=True)
    e = np.exp(z - zmax)
    s = e.sum(axis=1, keepdims=True)
    return z - zmax - np.log(s), e / s


def categorical_from_uniform(p, u):
    """rlcore.py:202-213 given the uniforms ``u`` (shape (B,))."""
    c = np.cumsum(p, axis=1)
    idx = np.minimum((c < u[:, None]).sum(axis=1), p.shape[1] - 1)
    bad = np.nonzero(p[np.arange(len(p)), idx] <= 0.0)[0]
    for r in bad:
        j = int(idx[r])
        while j > 0 and p[r, j] <= 0.0:
            j -= 1
        idx[r] = j
    return idx.astype(np.int64)


def select_actions(agent: Agent, X, masks, rng, forced=None, record=None):
    """rlcore.py:216-228: one ``rng.random((B,1))`` per head, head-major.
    ``forced`` (B,4) replays externally chosen actions but still consumes
    the uniforms so the generator stays in lock-step."""
    logits, _ = agent.policy_forward(X)
    B = len(X)
    actions = np.zeros((B, len(logits)), dtype=np.int64)
    logp = np.zeros(B)
    for h, (lg, mk) in enumerate(zip(logits, masks)):
        lp, p = masked_log_softmax(lg, mk)
        u = rng.random((B, 1))[:, 0]
        a = categorical_from_uniform(p, u)
        if record is not None:
            record.append({"logits": lg, "p": p, "u": u, "a": a})
        if forced is not None:
            a = np.asarray(forced[:, h], dtype=np.int64)
        actions[:, h] = a
        logp += lp[np.arange(B), a]
    return actions, logp


# ---------------------------------------------------------------------------
# PPO update


@dataclass
class Adam:
    """rlcore.py:48-71 state: moments per parameter, step count."""

    lr: float
    m: list
    v: list
    t: int = 0
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8

    @classmethod
    def zeros_like(cls, params, lr):
        return cls(lr=lr, m=[np.zeros_like(p) for p in params],
                   v=[np.zeros_like(p) for p in params])

    def step(self, params, grads):
        self.t += 1
        c1 = 1.0 - self.beta1 ** self.t
        c2 = 1.0 - self.beta2 ** self.t
        for p, g, m, v in zip(params, grads, self.m, self.v):
            m *= self.beta1
            m += (1.0 - self.beta1) * g
            v *= self.beta2
            v += (1.0 - self.beta2) * (g * g)
            p -= self.lr * (m / c1) / (np.sqrt(v / c2) + self.eps)


@dataclass(frozen=True)
class RlCfg:
    lr_actor: float = 3e-4
    lr_critic: float = 1e-3
    discount: float = 0.9
    clip_ratio: float = 0.2
    value_loss_weight: float = 0.5
    entropy_weight: float = 0.01
    minibatch: int = 256
    buffer_capacity: int = 4096
    train_interval: int = 2


def ppo_grads(agent: Agent, X, masks, actions, logp_old, adv, td, cfg: RlCfg,
              norm: int | None = None):
    """rlcore.py:293-358 -> (actor loss, actor grads, stats, value loss,
    value grads).  ``norm`` (sharding checks only) replaces the batch size
    in the gradient normalisation so per-shard gradients sum to the full
    one; ``None`` is the reference."""
    logits, (trunk_acts, hid) = agent.policy_forward(X)
    B = len(X)
    Bn = B if norm is None else norm
    rows = np.arange(B)
    logp_new = np.zeros(B)
    ent_total = np.zeros(B)
    heads = []
    for h, (lg, mk) in enumerate(zip(logits, masks)):
        lp, p = masked_log_softmax(lg, mk)
        lp_safe = np.where(mk, lp, 0.0)
        ent = -(p * lp_safe).sum(axis=1)
        ent_total += ent
        logp_new += lp[rows, actions[:, h]]
        heads.append((lp_safe, p, ent))
    ratio = np.exp(logp_new - logp_old)
    clipped = np.clip(ratio, 1.0 - cfg.clip_ratio, 1.0 + cfg.clip_ratio)
    s_un = ratio * adv
    s_cl = clipped * adv
    policy_loss = -np.minimum(s_un, s_cl).mean()
    entropy = ent_total.mean()
    a_loss = float(policy_loss - cfg.entropy_weight * entropy)
    coef = np.where(s_un <= s_cl, ratio * adv, 0.0)
    dlogp = -coef / Bn
    dhid = np.zeros_like(hid)
    head_grads = []
    for h, (lp_safe, p, ent) in enumerate(heads):
        onehot = np.zeros_like(p)
        onehot[rows, actions[:, h]] = 1.0
        dz = dlogp[:, None] * (onehot - p)
        dz += (cfg.entropy_weight / Bn) * p * (lp_safe + ent[:, None])
        head_grads += [hid.T @ dz, dz.sum(axis=0)]
        dhid += dz @ agent.head_W[h].T
    dtrunk = dhid * (1.0 - hid ** 2)
    trunk_grads, _ = dense_backward(agent.trunk_W, trunk_acts, dtrunk)
    stats = {"policy_loss": float(policy_loss), "entropy": float(entropy),
             "mean_ratio": float(ratio.mean())}
    v, vacts = agent.value(X)
    v_loss = float(cfg.value_loss_weight * np.mean((v - td) ** 2))
    dv = cfg.value_loss_weight * 2.0 * (v - td) / (len(X) if norm is None
                                                    else norm)
    v_grads, _ = dense_backward(agent.val_W, vacts, dv[:, None])
    return a_loss, trunk_grads + head_grads, stats, v_loss, v_grads


def ppo_update(agent: Agent, opt_pi: Adam, opt_v: Adam, batch, cfg: RlCfg):
    """rlcore.py:361-378.  ``batch`` = (X, actions, logp_old, adv, td,
    masks) stacked like ``batch_arrays`` (rlcore.py:277-286)."""
    X, actions, logp_old, adv, td, masks = batch
    a_loss, a_grads, stats, v_loss, v_grads = ppo_grads(
        agent, X, masks, actions, logp_old, adv, td, cfg)
    for name, val in (("actor loss", a_loss), ("critic loss", v_loss)):
        if not math.isfinite(val):
            raise OracleDiverged(f"{name} is not finite: {val}")
    for g in a_grads + v_grads:
        if not np.isfinite(g).all():
            raise OracleDiverged("non-finite gradient in update")
    opt_pi.step(agent.policy_params(), a_grads)
    opt_v.step(agent.value_params(), v_grads)
    return {"actor_loss": a_loss, "value_loss": v_loss, **stats,
            "batch": len(X)}


class Replay:
    """rlcore.py:253-274: FIFO of the last ``capacity`` transitions."""

    def __init__(self, capacity: int):
        self.items = deque(maxlen=capacity)

    def __len__(self):
        return len(self.items)

    def push_rows(self, X, Xn, acts, logp, rew, adv, td, masks):
        for i in range(len(X)):
            self.items.append((X[i], Xn[i], acts[i].copy(), float(logp[i]),
                               float(rew[i]), float(adv[i]), float(td[i]),
                               tuple(m[i].copy() for m in masks)))

    def sample(self, rng, size):
        n = len(self.items)
        if n == 0:
            return None, np.zeros(0, dtype=np.int64)
        idx = rng.choice(n, size=min(size, n), replace=False)
        items = list(self.items)
        chosen = [items[int(i)] for i in idx]
        X = np.stack([c[0] for c in chosen])
        acts = np.stack([c[2] for c in chosen])
        logp = np.asarray([c[3] for c in chosen])
        adv = np.asarray([c[5] for c in chosen])
        td = np.asarray([c[6] for c in chosen])
        masks = [np.stack([c[7][h] for c in chosen]) for h in range(4)]
        return (X, acts, logp, adv, td, masks), idx


# ---------------------------------------------------------------------------
# adaptive stopping (host logic in the product as well)


def cull(alive, adv_by_track, fraction, min_tracks):
    """stopping.py:68-86: eliminate the lowest ``(adv, -index)``."""
    live = np.flatnonzero(alive)
    n = len(live)
    n_elim = min(int(math.floor(fraction * n)), n - min_tracks)
    if n_elim <= 0:
        return np.zeros(0, dtype=np.int64)
    order = np.lexsort((-live, adv_by_track[live]))
    gone = np.sort(live[order[:n_elim]])
    alive[gone] = False
    return gone


# ---------------------------------------------------------------------------
# the episode


@dataclass
class EpisodeCfg:
    tracks: int
    track_len: int
    cull_window: int | None
    cull_fraction: float
    min_tracks: int
    rl: bool = True
    adaptive: bool = True
    rl_cfg: RlCfg = field(default_factory=RlCfg)


@dataclass
class Entry:
    tiles: np.ndarray
    knobs: np.ndarray
    features: np.ndarray
    score: float
    order: int


def rank_scores(canonicals, scores, orders, k: int, exclude=()):
    """costmodel.py:266-286 over parallel lists: drop excluded and repeated
    canonical strings (first occurrence wins), then the top ``k`` by
    ``(-score, order)``.  ``scores`` are the model's predictions of each
    entry (predict is pointwise, so scoring the pool after dedup equals
    indexing the per-entry scores).  Returns positions into the lists."""
    exclude = set(exclude or ())
    seen = set()
    pool = []
    for i, c in enumerate(canonicals):
        if c in exclude or c in seen:
            continue
        seen.add(c)
        pool.append(i)
    ranked = sorted(pool, key=lambda i: (-float(scores[i]), orders[i]))
    return ranked[:k]


def run_episode(tb, num_slots, cfg: EpisodeCfg, agent: Agent, opt_pi: Adam,
                opt_v: Adam, replay: Replay, model: GbtModel, rng,
                order_counter: int, trace: list | None = None,
                follow=None, log: list | None = None):
    """tuner.py:350-440.  Returns (entries, new order_counter, summary).

    ``follow(step, info)`` (optional) returns a dict that may override the
    sampled actions (``"actions"``), the culled tracks (``"cull"``) or the
    network outputs pushed into the replay FIFO (``"logp"``/``"adv"``/
    ``"td"``, phase "push") so a GPU trajectory can be replayed and checked
    step by step."""
    p = cfg.tracks
    budget = p * cfg.track_len
    tiles, knobs = sample_initial(tb, p, rng)
    feats = featurize(tb, tiles, knobs)
    score = model.predict(feats)
    alive = np.ones(p, dtype=bool)
    steps = np.zeros(p, dtype=np.int64)
    best = np.full(p, -np.inf)
    best_step = np.zeros(p, dtype=np.int64)
    if trace is not None:
        trace.append({"init_tiles": tiles.copy(), "init_knobs": knobs.copy(),
                      "init_feats": feats.copy(), "init_score": score.copy()})
    entries = []
    used = 0
    t = 0
    rl_cfg = cfg.rl_cfg
    while not (alive.sum() < cfg.min_tracks or used >= budget):
        t += 1
        live = np.flatnonzero(alive)
        m = min(len(live), budget - used)
        sel = live[:m]
        X = feats[sel]
        masks = action_masks(tb, tiles[sel], knobs[sel], num_slots)
        rec = {"step": t, "sel": sel.copy(), "X": X.copy()}
        forced = None
        if follow is not None:
            forced = follow(t, {"phase": "act", "sel": sel}).get("actions")
        heads = []
        if cfg.rl:
            acts, logp = select_actions(agent, X, masks, rng, forced=forced,
                                        record=heads)
        else:
            acts = np.zeros((m, 4), dtype=np.int64)
            for h, mk in enumerate(masks):
                for r in range(m):
                    valid = np.flatnonzero(mk[r])
                    acts[r, h] = valid[int(rng.integers(len(valid)))]
            if forced is not None:
                acts = np.asarray(forced, dtype=np.int64)
            logp = None
        nt, nk = apply_actions(tb, tiles[sel], knobs[sel], acts, num_slots)
        nf = featurize(tb, nt, nk)
        old = score[sel]
        new = model.predict(nf)
        rewards = (new - old) / old
        adv = td = v_cur = v_next = None
        if cfg.rl:
            v_cur, _ = agent.value(X)
            v_next, _ = agent.value(nf)
            adv = rewards + rl_cfg.discount * v_next - v_cur
            td = rewards + rl_cfg.discount * v_next
            push = (logp, adv, td)
            if follow is not None:
                # optional: the replayed trajectory's own network outputs
                # go into the FIFO, so later PPO updates see its inputs
                ov = follow(t, {"phase": "push"})
                push = tuple(ov.get(k) if ov.get(k) is not None else v
                             for k, v in zip(("logp", "adv", "td"), push))
            replay.push_rows(X, nf, acts, push[0], rewards, push[1], push[2],
                             masks)
        tiles[sel], knobs[sel], feats[sel], score[sel] = nt, nk, nf, new
        steps[sel] += 1
        better = new > best[sel]
        best[sel] = np.where(better, new, best[sel])
        best_step[sel] = np.where(better, steps[sel], best_step[sel])
        for i in range(m):
            entries.append(Entry(nt[i].copy(), nk[i].copy(), nf[i].copy(),
                                 float(new[i]), order_counter + i))
        order_counter += m
        used += m
        rec.update({"masks": masks, "actions": acts, "logp": logp,
                    "heads": heads, "new_tiles": nt, "new_knobs": nk,
                    "new_feats": nf, "new_score": new, "rewards": rewards,
                    "v_cur": v_cur, "v_next": v_next, "adv": adv, "td": td})
        if log is not None:
            log.append({"event": "episode_step", "step": t, "alive": m,
                        "mean_reward": float(np.mean(rewards)),
                        "rewards": [float(r) for r in rewards]})
        if cfg.adaptive and cfg.cull_window is not None and \
                t % cfg.cull_window == 0 and used < budget:
            adv_full = np.zeros(p)
            adv_full[sel] = adv
            probe = alive.copy()
            gone = cull(probe, adv_full, cfg.cull_fraction, cfg.min_tracks)
            if follow is not None:
                ov = follow(t, {"phase": "cull", "sel": sel, "gone": gone,
                                "adv": adv_full}).get("cull")
                if ov is not None:
                    gone = np.asarray(ov, dtype=np.int64)
                    probe = alive.copy()
                    probe[gone] = False
            alive = probe
            rec["cull"] = gone
        if cfg.rl and t % rl_cfg.train_interval == 0 and len(replay) >= 2:
            batch, idx = replay.sample(rng, rl_cfg.minibatch)
            rec["ppo_idx"] = idx
            rec["ppo"] = ppo_update(agent, opt_pi, opt_v, batch, rl_cfg)
            if trace is not None:
                rec["ppo_policy"] = [a.copy() for a in agent.policy_params()]
                rec["ppo_value"] = [a.copy() for a in agent.value_params()]
        if trace is not None:
            trace.append(rec)
    summary = {"visited": used, "steps": steps, "best_step": best_step,
               "alive": alive, "n_steps": t}
    return entries, order_counter, summary
