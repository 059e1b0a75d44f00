"""harl_agent_copy (host C++, no GPU): the copy plan that moves the agent's
numpy arrays (rlcore.py PolicyNet/ValueNet weights, Adam m/v) into the flat
parameter layout and back -- contiguous arrays and the tiling head's
column gather/scatter -- against the numpy restatement."""

import numpy as np

from paper_2211_11172_b200 import _native as N


def test_agent_copy_round_trip_matches_numpy():
    lib = N.load(require_device=False)
    rng = np.random.default_rng(0)
    H, Cfull, NH = 8, 40, 0
    cols = np.sort(rng.choice(Cfull, 11, replace=False)).astype(np.int64)
    C0 = len(cols)
    NH = C0 + 3
    W0 = rng.normal(size=(5, H))
    b0 = rng.normal(size=H)
    hW = rng.normal(size=(H, Cfull))
    hb = rng.normal(size=Cfull)
    sW = rng.normal(size=(H, 3))
    sb = rng.normal(size=3)
    off_W0, off_b0 = 0, 40
    off_hW = 48
    off_hb = off_hW + H * NH
    n = off_hb + NH
    ops = [(off_W0, 0, W0.ctypes.data, 0, 1, W0.size, None),
           (off_b0, 0, b0.ctypes.data, 0, 1, H, None),
           (off_hW, NH, hW.ctypes.data, Cfull, H, C0, cols.ctypes.data),
           (off_hb, 0, hb.ctypes.data, 0, 1, C0, cols.ctypes.data),
           (off_hW + C0, NH, sW.ctypes.data, 3, H, 3, None),
           (off_hb + C0, 0, sb.ctypes.data, 0, 1, 3, None)]
    arr = (N.CopyOp * len(ops))(*[N.CopyOp(*o) for o in ops])
    flat = np.full(n, np.nan)
    assert lib.harl_agent_copy(arr, len(ops), flat.ctypes.data, 0) == 0
    ref = np.full(n, np.nan)
    ref[:40] = W0.ravel()
    ref[40:48] = b0
    blk = ref[off_hW:off_hW + H * NH].reshape(H, NH)
    blk[:, :C0] = hW[:, cols]
    blk[:, C0:] = sW
    ref[off_hb:off_hb + C0] = hb[cols]
    ref[off_hb + C0:] = sb
    assert flat.tobytes() == ref.tobytes()
    # back: every covered element rewritten, the head's illegal columns kept
    flat2 = rng.normal(size=n)
    keep = hW.copy()
    assert lib.harl_agent_copy(arr, len(ops), flat2.ctypes.data, 1) == 0
    assert W0.ravel().tobytes() == flat2[:40].tobytes()
    blk2 = flat2[off_hW:off_hW + H * NH].reshape(H, NH)
    exp = keep.copy()
    exp[:, cols] = blk2[:, :C0]
    assert hW.tobytes() == exp.tobytes()
    assert sW.tobytes() == np.ascontiguousarray(blk2[:, C0:]).tobytes()
    assert hb[cols].tobytes() == flat2[off_hb:off_hb + C0].tobytes()
    assert lib.harl_agent_copy(arr, -1, flat.ctypes.data, 0) != 0
