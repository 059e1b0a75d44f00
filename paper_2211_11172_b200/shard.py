"""Population sharding across ranks.

Track ``i`` of the episode's population lives on rank ``i % G``
(interleaved, so the replay tail, the culls and the budget tail stay
balanced; a contiguous split would put every replay row -- and hence every
PPO minibatch -- on the last rank at P >= 4096, rlcore.py:253-265).
Parameters and trees are replicated; the only data-path collective is one
all-reduce per PPO update: of the minibatch rows (default, every rank then
runs the single-device update -- bit-identical at any world size) or of the
per-shard gradient and loss partial sums (HARL_SHARD_PPO=grads).

Everything here is host arithmetic that keeps a sharded episode *the same
episode* as the single-device one:

* **global rows** -- the reference processes the live tracks in index
  order (tuner.py:373-375); a track's global row is its rank among the
  alive track ids, and its uniforms are draws ``h*m + row + 1`` of the
  step (rlcore.py:223-225), whichever device holds it;
* **replay ownership** -- the FIFO keeps the last ``cap`` pushes in global
  (step, row) order; each rank's ring holds its own rows, and a global
  buffer position maps to (rank, local slot);
* **cull** -- every rank sees all advantages (all-gather) and takes the
  identical decision (stopping.py:68-86).
"""

from __future__ import annotations

import math

import numpy as np


class ShardLayout:
    def __init__(self, tracks: int, world: int, rank: int):
        if not 0 <= rank < world:
            raise ValueError("bad rank")
        self.P, self.G, self.rank = tracks, world, rank
        self.local_ids = np.arange(rank, tracks, world, dtype=np.int64)

    @staticmethod
    def owner(track_ids, world):
        return np.asarray(track_ids) % world

    def global_rows(self, alive: np.ndarray, local_alive_ids: np.ndarray):
        """Global row (rank among all alive ids) of each locally alive id.
        (Callers cache it: it changes only when a cull changes ``alive``.)"""
        csum = np.cumsum(alive) - 1
        return csum[local_alive_ids].astype(np.int64)


class GlobalReplayIndex:
    """Which rank/local slot holds each position of the global replay FIFO.

    Pushes arrive per step in global-row order; every rank appends its own
    rows to its local ring (capacity ``cap`` each, more than enough since a
    rank only ever needs the rows that survive globally).  Kept as a numpy
    ring of (owner rank, local push number) -- one vectorised append per
    step, no per-row Python."""

    def __init__(self, cap: int, world: int):
        self.cap, self.G = cap, world
        self._rank = np.zeros(cap, dtype=np.int64)
        self._push = np.zeros(cap, dtype=np.int64)
        self._n = 0                         # total global pushes so far
        self.local_pushes = np.zeros(world, dtype=np.int64)

    def __len__(self):
        return min(self._n, self.cap)

    def push_step(self, owners_in_row_order):
        o = np.asarray(owners_in_row_order, dtype=np.int64)
        m = len(o)
        if m == 0:
            return
        # local push number of each row: the owner's running count
        onehot = o[:, None] == np.arange(self.G)[None, :]
        before = np.cumsum(onehot, axis=0) - onehot
        num = self.local_pushes[o] + before[np.arange(m), o]
        self.local_pushes += onehot.sum(axis=0)
        keep = min(m, self.cap)             # only the last cap rows survive
        pos = (self._n + np.arange(m - keep, m)) % self.cap
        self._rank[pos] = o[m - keep:]
        self._push[pos] = num[m - keep:]
        self._n += m

    def locate(self, positions):
        """Global FIFO positions (0 = oldest kept) -> (rank, local push
        number) arrays."""
        p = np.asarray(positions, dtype=np.int64)
        first = self._n - len(self)
        slot = (first + p) % self.cap
        return self._rank[slot].copy(), self._push[slot].copy()


def eliminated(live, adv_live, n_elim):
    """The ``n_elim`` tracks TrackSet.cull eliminates (stopping.py:80-86):
    ``sorted(live, key=(advantage, -index))[:n_elim]``, ascending ids.
    ``live`` ascending track ids, ``adv_live`` their advantages.

    Finite keys: a lexsort, the same total order.  With a NaN key Python's
    tuple comparisons are no longer a total order (every comparison with
    NaN is False), so the outcome depends on timsort's comparison sequence
    over the input order; that case runs the reference's own ``sorted``
    over the same keys in the same (index) order -- the identical
    decision, not "NaN last"."""
    live = np.asarray(live, dtype=np.int64)
    adv_live = np.asarray(adv_live, dtype=np.float64)
    if n_elim <= 0:
        return np.zeros(0, dtype=np.int64)
    if np.isnan(adv_live).any():
        keys = [(float(a), -int(i)) for i, a in zip(live.tolist(),
                                                     adv_live.tolist())]
        order = sorted(range(len(keys)), key=keys.__getitem__)
        return np.sort(live[np.asarray(order[:n_elim], dtype=np.int64)])
    order = np.lexsort((-live, adv_live))
    return np.sort(live[order[:n_elim]])


def cull_decision(alive, track_ids, adv, fraction, min_tracks):
    """stopping.py:68-86 on the merged advantages of every rank."""
    live = np.flatnonzero(alive)
    n = len(live)
    n_elim = min(int(math.floor(fraction * n)), n - min_tracks)
    if n_elim <= 0:
        return np.zeros(0, dtype=np.int64)
    full = np.zeros(len(alive))
    full[np.asarray(track_ids, dtype=np.int64)] = adv
    return eliminated(live, full[live], n_elim)


def shard_tasks(n_tasks: int, world: int, rank: int) -> list:
    """Independent subgraph tasks of a task set (config C4): task i on rank
    i mod world.  Each rank tunes its tasks in its own session (no
    collective on the data path; SURVEY.md §8(e) task sharding)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return [i for i in range(n_tasks) if i % world == rank]
