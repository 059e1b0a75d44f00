"""Chunked oracle checks of one search step at north-star sizes (>= 64 K
rows), where the oracle cannot hold a whole step's fp64 intermediates at
once but can restate it chunk by chunk:

* policy logits of every head (rlcore.py:136-146) and the joint logp of the
  device's own actions (rlcore.py:185-199, 216-228) within the north-star
  tolerance ``1e-4 * max(|ref|, rms(ref))`` (rms over the chunk);
* every sampled index against the oracle's fp64 CDF on the same uniforms
  (head-major ``rng.random((B,1))`` draws): equal, or a flip whose uniform
  sits within float distance of a CDF boundary; flips bounded;
* V(X), V(X') (rlcore.py:173-174) and the advantage r + 0.9 V(X') - V(X)
  (rlcore.py:231-234, tuner.py:395-398) from the device's bit-exact rewards;
* the walker's successor states bit for bit (schedspace.py:265-301).
"""

import numpy as np

from gpu_util import REL_TOL
from oracle import harl_oracle as O


def scaled_err(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert np.array_equal(np.isfinite(got), np.isfinite(ref))
    fin = np.isfinite(ref)
    if not fin.any():
        return 0.0
    rms = float(np.sqrt(np.mean(ref[fin] ** 2)))
    scale = np.maximum(np.abs(ref[fin]), rms)
    return float((np.abs(got[fin] - ref[fin]) /
                  np.where(scale > 0, scale, 1.0)).max())


class StepCheck:
    """Accumulates the per-chunk comparisons of one step."""

    def __init__(self):
        self.err = {}
        self.draws = 0
        self.flips = 0
        self.rows = 0

    def note(self, what, e):
        self.err[what] = max(self.err.get(what, 0.0), e)

    def assert_ok(self, tol=REL_TOL):
        bad = {k: v for k, v in self.err.items() if v > tol}
        assert not bad, f"scaled errors above {tol}: {bad}"
        assert self.flips <= max(2, self.draws // 1000), \
            f"{self.flips} flips in {self.draws} draws"


def uniforms(rng_state, m):
    """The step's uniforms (4, m): rng.random((m,1)) per head, head-major."""
    g = np.random.default_rng()
    g.bit_generator.state = rng_state
    return g.random(4 * m).reshape(4, m)


def check_policy_rows(chk, tb, oa, X, tiles, knobs, u, acts, logp, logits,
                      cols, chunk=131072, new_tiles=None, new_knobs=None):
    """One step's policy outputs (device arrays on the host: actions (n,4),
    logp (n,), compact logits (n, C0+9), successor states) vs the oracle.
    ``tiles``/``knobs``: the current states [n, slots] / [n, 3]."""
    n = len(X)
    C0 = len(cols)
    for c0 in range(0, n, chunk):
        sl = slice(c0, min(n, c0 + chunk))
        rows = sl.stop - sl.start
        ref_lg, _ = oa.policy_forward(X[sl])
        chk.note("logits_head0", scaled_err(logits[sl, :C0],
                                            ref_lg[0][:, cols]))
        for h in range(3):
            chk.note(f"logits_head{h + 1}",
                     scaled_err(logits[sl, C0 + 3 * h:C0 + 3 * h + 3],
                                ref_lg[h + 1]))
        masks = O.action_masks(tb, tiles[sl], knobs[sl], tb.num_slots)
        lp_ref = np.zeros(rows)
        for h in range(4):
            lp, p = O.masked_log_softmax(ref_lg[h], masks[h])
            a_ref = O.categorical_from_uniform(p, u[h, sl])
            a_dev = np.asarray(acts[sl, h], np.int64)   # full head index
            chk.draws += rows
            diff = np.flatnonzero(a_dev != a_ref)
            chk.flips += len(diff)
            if len(diff):
                c = np.cumsum(p[diff], axis=1)
                a = a_dev[diff]
                hi = c[np.arange(len(diff)), a]
                lo = np.where(a > 0, c[np.arange(len(diff)),
                                       np.maximum(a - 1, 0)], 0.0)
                uu = u[h, sl][diff]
                assert (p[diff, a] > 0).all(), "flip onto a masked action"
                assert ((lo - 1e-5 <= uu) & (uu <= hi + 1e-5)).all(), \
                    "flip away from a CDF boundary"
            lp_ref += lp[np.arange(rows), a_dev]
        chk.note("logp", scaled_err(logp[sl], lp_ref))
        if new_tiles is not None:
            rt, rk = O.apply_actions(tb, tiles[sl], knobs[sl],
                                     np.asarray(acts[sl], np.int64),
                                     tb.num_slots)
            assert np.array_equal(new_tiles[sl], rt), "walker tiles"
            assert np.array_equal(new_knobs[sl], rk), "walker knobs"
        chk.rows += rows


def check_values(chk, oa, X, got, what, chunk=262144):
    for c0 in range(0, len(X), chunk):
        sl = slice(c0, min(len(X), c0 + chunk))
        ref, _ = oa.value(X[sl])
        chk.note(what, scaled_err(got[sl], ref))


def check_advantage(chk, oa, X, Xn, rewards, adv, discount=0.9,
                    chunk=262144):
    for c0 in range(0, len(X), chunk):
        sl = slice(c0, min(len(X), c0 + chunk))
        vc, _ = oa.value(X[sl])
        vn, _ = oa.value(Xn[sl])
        ref = rewards[sl] + discount * vn - vc
        chk.note("adv", scaled_err(adv[sl], ref))
