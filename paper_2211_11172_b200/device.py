"""Device-resident tables and batch operators (the reference's per-call API,
one call per population batch).

Every function here launches hand-written sm_100a kernels through the C ABI
(``_native``); torch is used only for device allocation and the current
stream.  Reference functions mirrored (``pkg/src/schedtune``):

=============================  ==========================================
this module                    reference
=============================  ==========================================
``init_population``            schedspace.sample_initial_schedules 165-178
``featurize``                  SketchContext.featurize 415-438
``action_masks``               schedspace.action_mask 226-262
``apply_actions``              decode_action + apply_action 196-301
``gbt_predict``                SurrogateModel.predict 219-230 (+ reward)
``policy_step``                select_actions 216-228 (+ walker)
``value_estimate``             ValueNet.estimate 173-174
``DeviceAgent.ppo_update``     ppo_update 361-378
``rank_topk``                  costmodel.rank_scores 266-286
``simulate_time``              measure.simulate_time 99-112
``brute_force_best``           measure.brute_force_best 135-167
``gbt_fit``                    SurrogateModel.fit_incremental 190-212
                               (+ _fit_tree 81-141)
=============================  ==========================================
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from . import _native as N
from . import profiling as PF
from . import rng as R
from .errors import DeviceError, InvalidActionError, RlDivergedError
from .space import SketchTables, head_columns


# rows per launch up to which the sampler featurizes in-kernel
# (HARL_SAMPLE_FEAT_MAX_ROWS in harl_b200.cu)
SAMPLE_FEAT_MAX_ROWS = 16384


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _stream() -> int:
    """The current CUDA stream of the current device as a raw handle (the
    torch internals behind ``torch.cuda.current_stream().cuda_stream``,
    without building a Stream object per launch)."""
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


def _dev(device=None):
    return torch.device("cuda", torch.cuda.current_device()) \
        if device is None else torch.device(device)


_SUBSPACE = {N.ST_TILING: "tiling", N.ST_COMPUTE_AT: "compute_at",
             N.ST_PARALLEL: "parallel", N.ST_UNROLL: "unroll"}


def raise_status(code_word: int, where: str = "") -> None:
    """Translate a device status word (row*16 + HARL_ST_*) into the
    reference's exception."""
    if code_word == (1 << 64) - 1 or code_word < 0:
        return
    row, code = divmod(int(code_word), 16)
    if code in _SUBSPACE:
        raise InvalidActionError(_SUBSPACE[code],
                                 f"row {row}{' ' + where if where else ''}")
    if code == N.ST_NO_VALID:
        raise RlDivergedError("action mask with no valid entry")
    if code == N.ST_NONFINITE:
        raise RlDivergedError("non-finite loss or gradient in update")
    raise DeviceError(f"unknown device status {code} at row {row}")


# ---------------------------------------------------------------------------
# per-sketch tables


class DeviceSketch:
    """``SketchTables`` uploaded to the device plus its C descriptor."""

    def __init__(self, tables: SketchTables, device=None):
        N.load()
        dev = _dev(device)
        self.tables = tb = tables
        self.device = dev
        self.log2_lut = torch.from_numpy(tb.log2_lut).to(dev)
        self.spf_lut = torch.from_numpy(tb.spf_lut.astype(np.int16)).to(dev)
        table = tb.tiling_table if tb.tiling_table.size else \
            np.zeros((1, tb.levels), np.uint16)
        self.tiling_table = torch.from_numpy(
            np.ascontiguousarray(table).astype(np.int16)).to(dev)
        cols = tb.head_cols
        if len(cols) > N.MAX_HEAD0:
            raise DeviceError("tiling head too wide for the device tables")
        d = N.SketchDesc()
        d.levels, d.ndims, d.local_slots = tb.levels, tb.ndims, tb.local_slots
        d.num_slots, d.ncas, d.max_fusible = tb.num_slots, tb.ncas, \
            tb.max_fusible
        d.n_unroll, d.max_feature_dims = tb.n_unroll, tb.max_feature_dims
        d.feature_len = tb.feature_len
        d.n_stages, d.n_tensors = len(tb.stage_first), len(tb.tensor_first)
        d.n_terms, d.max_extent = len(tb.term_gi), tb.max_extent
        d.n_head0 = len(cols)
        for i in range(tb.ndims):
            d.extents[i] = int(tb.extents[i])
            d.tiling_counts[i] = int(tb.tiling_counts[i])
            d.tiling_offsets[i] = int(tb.tiling_offsets[i])
        for name in ("term_gi", "term_sc", "term_off", "tensor_first",
                     "tensor_nterms", "stage_first", "stage_ntensors",
                     "stage_inter", "stage_extra"):
            arr = getattr(tb, name)
            dst = getattr(d, name)
            for i, v in enumerate(arr):
                dst[i] = int(v)
        S = tb.num_slots
        for j, c in enumerate(cols):
            if j == len(cols) - 1:
                d.head0_src[j], d.head0_dst[j] = -1, -1
            else:
                d.head0_src[j], d.head0_dst[j] = int(c) // S, int(c) % S
        d.flops_feature = tb.flops_feature
        d.log2_lut = self.log2_lut.data_ptr()
        d.spf_lut = self.spf_lut.data_ptr()
        d.tiling_table = self.tiling_table.data_ptr()
        # a device copy of the descriptor (dev_self NULL inside it): kernels
        # staging the column/term tables read them with coalesced loads
        raw = np.frombuffer(C.string_at(C.addressof(d), C.sizeof(d)), np.uint8)
        self.desc_dev = torch.from_numpy(raw.copy()).to(dev)
        d.dev_self = self.desc_dev.data_ptr()
        self.desc = d
        self.head_cols = cols

    @property
    def n_head0(self) -> int:
        return len(self.head_cols)


def alloc_state(n: int, tables: SketchTables, device=None, ld: int | None = None):
    dev = _dev(device)
    ld = n if ld is None else ld
    tiles = torch.zeros((max(tables.local_slots, 1), max(ld, 1)),
                        dtype=torch.int16, device=dev)
    knobs = torch.zeros((3, max(ld, 1)), dtype=torch.uint8, device=dev)
    return tiles, knobs


def states_to_device(tables: SketchTables, tiles_np, knobs_np, device=None):
    """Host [B, slots] u16 / [B, 3] u8 -> device SoA (slot-major)."""
    dev = _dev(device)
    t = np.ascontiguousarray(np.asarray(tiles_np, np.uint16).T)
    if t.size == 0:
        t = np.zeros((1, max(len(knobs_np), 1)), np.uint16)
    k = np.ascontiguousarray(np.asarray(knobs_np, np.uint8).T)
    return (torch.from_numpy(t.astype(np.int16)).to(dev),
            torch.from_numpy(k).to(dev))


def states_to_host(tables: SketchTables, tiles, knobs, n: int):
    t = tiles[:tables.local_slots, :n].cpu().numpy().astype(np.uint16).T
    k = knobs[:, :n].cpu().numpy().T
    return np.ascontiguousarray(t), np.ascontiguousarray(k)


# ---------------------------------------------------------------------------
# batch operators


def init_population(dsk: DeviceSketch, count: int, gen: np.random.Generator,
                    tiles=None, knobs=None, cursor=None):
    """sample_initial_schedules on device, advancing ``gen`` exactly (or,
    given a ``rng.StreamCursor`` over it, the cursor instead)."""
    lib = N.load()
    tb = dsk.tables
    if tiles is None:
        tiles, knobs = alloc_state(count, tb, dsk.device)
    scratch = getattr(dsk, "_init_scratch", None)
    if scratch is None:
        scratch = dsk._init_scratch = torch.zeros(4, dtype=torch.int64,
                                                  device=dsk.device)
    st = cursor.struct() if cursor is not None else R.to_struct(gen)
    used = C.c_int64(0)
    with PF.span("init", count):
        N.check(lib.harl_init_population(
            C.byref(dsk.desc), C.byref(st), count, _ptr(tiles), _ptr(knobs),
            tiles.shape[1], C.byref(used), _ptr(scratch), _stream()),
            "harl_init_population")
    if cursor is not None:
        cursor.skip_u32(used.value)
    else:
        R.skip_u32(gen, used.value)
    return tiles, knobs


def uniform_actions(dsk: DeviceSketch, tiles, knobs, n: int, gen, out=None):
    """TuningSession._uniform_actions (tuner.py:341-348) on device; advances
    ``gen`` exactly.  Returns int32 [4][n] (head-major) full indices."""
    lib = N.load()
    if out is None:
        out = torch.empty((4, max(n, 1)), dtype=torch.int32, device=dsk.device)
    scratch = torch.empty(lib.harl_uniform_scratch_bytes(max(n, 1)),
                          dtype=torch.uint8, device=dsk.device)
    st = R.to_struct(gen)
    used = C.c_int64(0)
    with PF.span("uniform", n, launches=3):
        N.check(lib.harl_uniform_actions(
            C.byref(dsk.desc), _ptr(tiles), _ptr(knobs), n, tiles.shape[1],
            C.byref(st), _ptr(out), _ptr(scratch), C.byref(used), _stream()),
            "harl_uniform_actions")
    R.skip_u32(gen, used.value)
    return out


def featurize(dsk: DeviceSketch, tiles, knobs, n: int, out=None):
    lib = N.load()
    F = dsk.tables.feature_len
    if out is None:
        out = torch.empty((max(n, 1), F), dtype=torch.float64,
                          device=dsk.device)
    with PF.span("featurize", n):
        N.check(lib.harl_featurize(C.byref(dsk.desc), _ptr(tiles), _ptr(knobs),
                                   n, tiles.shape[1], _ptr(out), _stream()),
                "harl_featurize")
    return out[:n]


def format_floats(values, threads: int = 0) -> str:
    """", ".join of json's float rendering (float.__repr__, NaN/Infinity)
    of a host float64 array, in the native library's threaded formatter
    (harl_format_floats) -- the trajectory log's reward lists."""
    lib = N.load(require_device=False)
    v = np.ascontiguousarray(values, dtype=np.float64)
    if v.size == 0:
        return ""
    cap = 40 * v.size + 16
    out = C.create_string_buffer(cap)
    n = lib.harl_format_floats(v.ctypes.data, v.size, out, cap, threads)
    if n < 0:
        raise DeviceError("harl_format_floats: buffer too small")
    return out.raw[:n].decode("ascii")


class RankScratch:
    """Reusable device scratch of ``rank_topk`` (grown on demand)."""

    def __init__(self, device=None):
        self.device = _dev(device)
        self.buf = None
        self.out = None
        self.stats = torch.zeros(4, dtype=torch.int64, device=self.device)

    def host_pins(self, n: int, tables: SketchTables):
        """Pinned host buffers for a selection of n entries (grown on
        demand): (indices, tiles [slots][cap], knobs [3][cap], features,
        scores)."""
        S, F = max(tables.local_slots, 1), tables.feature_len
        cur = getattr(self, "_pins", None)
        if cur is None or cur[0].numel() < n or cur[1].shape[0] < S or \
                cur[3].shape[1] != F:
            cap = max(n, 256)
            pin = dict(pin_memory=True)
            self._pins = (torch.empty(cap, dtype=torch.int32, **pin),
                          torch.empty((S, cap), dtype=torch.int16, **pin),
                          torch.empty((3, cap), dtype=torch.uint8, **pin),
                          torch.empty((cap, F), dtype=torch.float64, **pin),
                          torch.empty(cap, dtype=torch.float64, **pin))
        return self._pins

    def ensure(self, n_visits: int, n_excluded: int, k: int):
        need = N.load().harl_rank_scratch_bytes(n_visits, n_excluded)
        if self.buf is None or self.buf.numel() < need:
            self.buf = torch.empty(need, dtype=torch.uint8, device=self.device)
        cap = k + n_visits
        if self.out is None or self.out.numel() < cap:
            self.out = torch.empty(max(cap, 1), dtype=torch.int32,
                                   device=self.device)


def rank_topk(tables: SketchTables, log_tiles, log_knobs, log_score,
              n_visits: int, k: int, exclude=None, scratch=None,
              sort: bool = True, launch_only: bool = False):
    """``rank_scores(model, entries, k, exclude)`` (costmodel.py:266-286)
    over a device entry log whose ``log_score`` holds each visit's model
    score (the episode's per-visit GBT predictions, which equal
    ``model.predict(features)`` since predict is pointwise and the model is
    fixed within an episode).

    ``exclude``: optional host ``(tiles [E, slots] u16, knobs [E, 3] u8)``
    of already-measured states of this sketch.  Returns the selected visit
    indices (ascending, so first occurrences come first) and the device
    stats ``{selected, kept, collisions, k_target}``; ``sort=False``
    returns (device int32 indices, unordered; count; stats) instead.  The selection is a
    superset of the reference's answer on which ``rank_scores`` returns
    exactly that answer (it equals the answer when ``collisions == 0``)."""
    lib = N.load()
    dev = log_score.device
    sc = scratch if scratch is not None else RankScratch(dev)
    E = 0
    ex_t = ex_k = None
    if exclude is not None and len(exclude[1]):
        E = len(exclude[1])
        ex_t, ex_k = states_to_device(tables, exclude[0], exclude[1], dev)
        PF.xfer("h2d", ex_t, ex_k)
    sc.ensure(n_visits, E, k)
    elog = N.EntryLog(log_tiles.data_ptr(), log_knobs.data_ptr(),
                      log_score.data_ptr(), 0, 0, log_tiles.shape[1])
    with PF.span("rank", n_visits):
        N.check(lib.harl_rank_topk(
            C.byref(elog), tables.local_slots, n_visits, _ptr(ex_t),
            _ptr(ex_k), 0 if ex_t is None else ex_t.shape[1], E, k,
            sc.buf.data_ptr(), sc.buf.numel(), sc.out.data_ptr(),
            sc.out.numel(), sc.stats.data_ptr(), _stream()),
            "harl_rank_topk")
    # the stats through a pinned buffer and an event: ``launch_only``
    # returns here (the caller may queue more work), ``rank_topk_finish``
    # completes the call
    if getattr(sc, "stats_pin", None) is None:
        sc.stats_pin = torch.empty(4, dtype=torch.int64, pin_memory=True)
    sc.stats_pin.copy_(sc.stats, non_blocking=True)
    PF.xfer("d2h", sc.stats)
    ev = torch.cuda.Event()
    ev.record()
    pend = (sc, ev, sort)
    if launch_only:
        return pend
    return rank_topk_finish(pend)


def rank_topk_finish(pend):
    """The second half of ``rank_topk(..., launch_only=True)``."""
    sc, ev, sort = pend
    ev.synchronize()
    st = sc.stats_pin.numpy()
    n = int(st[0])
    stats = {"selected": n, "kept": int(st[1]), "collisions": int(st[2]),
             "k_target": int(st[3])}
    if not sort:
        return sc.out, n, stats
    return np.sort(sc.out[:n].cpu().numpy().astype(np.int64)), stats


def gather_entries(tables: SketchTables, log_tiles, log_knobs, log_score,
                   log_track, idx, dsk=None):
    """Device gather of visits ``idx`` of an entry log -> device SoA
    (tiles, knobs), scores and tracks, plus their features (featurize on
    device: the features the reference stored in the CandidateEntry)."""
    lib = N.load()
    dev = log_score.device
    n = len(idx)
    didx = idx if isinstance(idx, torch.Tensor) else \
        torch.from_numpy(np.asarray(idx, np.int32)).to(dev)
    tiles, knobs = alloc_state(n, tables, dev)
    score = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    track = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    if n:
        N.check(lib.harl_gather_rows(
            didx.data_ptr(), n, tables.local_slots, 0,
            log_tiles.data_ptr(), log_knobs.data_ptr(), None,
            log_score.data_ptr(), log_track.data_ptr(), log_tiles.shape[1],
            tiles.data_ptr(), knobs.data_ptr(), None, score.data_ptr(),
            track.data_ptr(), tiles.shape[1], _stream()),
            "harl_gather_rows")
    feats = featurize(dsk if dsk is not None else DeviceSketch(tables, dev),
                      tiles, knobs, n)
    return tiles, knobs, score[:n], track[:n], feats


class GbtFit:
    """A device refit: ``base``, ``trees`` as the reference stores them
    ((feature, threshold, left, right, value) arrays, nodes numbered in
    _fit_tree's creation order) and ``pred``, the final training
    predictions (fit_incremental's ``pred``)."""

    def __init__(self, base, trees, pred):
        self.base, self.trees, self.pred = base, trees, pred


def heap_tree_to_reference(feat_h, thr_h, val_h):
    """Heap-layout tree (children of k at 2k+1, 2k+2) -> the reference's
    node numbering: _fit_tree pops a stack (left child first) and allocates
    both children when it splits a node (costmodel.py:86-141)."""
    feature, threshold, left, right, value = [-1], [0.0], [-1], [-1], [0.0]
    ref = {0: 0}
    stack = [0]
    while stack:
        h = stack.pop()
        nid = ref[h]
        value[nid] = float(val_h[h])
        f = int(feat_h[h])
        if f < 0:
            continue
        lid, rid = len(feature), len(feature) + 1
        for _ in range(2):
            feature.append(-1)
            threshold.append(0.0)
            left.append(-1)
            right.append(-1)
            value.append(0.0)
        ref[2 * h + 1], ref[2 * h + 2] = lid, rid
        feature[nid] = f
        threshold[nid] = float(thr_h[h])
        left[nid], right[nid] = lid, rid
        stack.append(2 * h + 2)
        stack.append(2 * h + 1)
    return (np.asarray(feature, np.int64), np.asarray(threshold, np.float64),
            np.asarray(left, np.int64), np.asarray(right, np.int64),
            np.asarray(value, np.float64))


class _FitGraph:
    """A captured GBT refit for training sets of up to ``ncap`` rows: the
    ~2,000 launches of one fit recorded once (the kernels read the row count
    from device memory), replayed per round with the new data copied into
    the workspace -- the launch latency, not the work, dominates small
    fits."""

    def __init__(self, ncap, F, n_trees, max_depth, lr, min_leaf, dev):
        lib = N.load()
        self.ncap, self.F, self.T = ncap, F, max(n_trees, 1)
        self.K = (1 << (max_depth + 1)) - 1
        f64 = dict(dtype=torch.float64, device=dev)
        self.X = torch.zeros((ncap, F), **f64)
        self.y = torch.zeros(ncap, **f64)
        self.pred = torch.zeros(ncap, **f64)
        self.base = torch.zeros(1, **f64)
        self.nt = torch.zeros(1, dtype=torch.int32, device=dev)
        self.n_dev = torch.zeros(1, dtype=torch.int32, device=dev)
        self.feat = torch.empty((self.T, self.K), dtype=torch.int32,
                                device=dev)
        self.thr = torch.empty((self.T, self.K), **f64)
        self.val = torch.empty((self.T, self.K), **f64)
        need = lib.harl_gbt_fit_scratch_bytes(ncap, F, max_depth)
        self.scratch = torch.empty(need, dtype=torch.uint8, device=dev)
        self.args = (n_trees, max_depth, lr, min_leaf)
        self.n_dev.fill_(1)
        self._call()                       # eager once: attributes, checks
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, capture_error_mode="relaxed"):
            self._call()

    def _call(self):
        lib = N.load()
        n_trees, max_depth, lr, min_leaf = self.args
        N.check(lib.harl_gbt_fit(
            _ptr(self.X), _ptr(self.y), self.ncap, self.F, n_trees, max_depth,
            lr, min_leaf, _ptr(self.scratch), self.scratch.numel(),
            _ptr(self.feat), _ptr(self.thr), _ptr(self.val), _ptr(self.pred),
            _ptr(self.base), _ptr(self.nt), _ptr(self.n_dev), _stream()),
            "harl_gbt_fit")

    def run(self, Xd, yd, n):
        self.X[:n].copy_(Xd)
        self.y[:n].copy_(yd)
        self.n_dev.fill_(n)
        self.graph.replay()


_FIT_GRAPHS: dict = {}


def gbt_fit(X, y, n_trees: int = 50, max_depth: int = 6,
            learning_rate: float = 0.3, min_leaf: int = 1, device=None):
    """SurrogateModel.fit_incremental (costmodel.py:190-212) on the device:
    (X [n][F], y [n]) host or device arrays -> ``GbtFit``, bit-exact with
    the reference's trees.  Runs as a captured graph per (power-of-two row
    capacity, F, config) -- HARL_FIT_EAGER=1 launches directly."""
    lib = N.load()
    dev = _dev(device)
    Xd = torch.as_tensor(np.ascontiguousarray(X, np.float64)
                         if not isinstance(X, torch.Tensor) else X,
                         dtype=torch.float64).to(dev).contiguous()
    yd = torch.as_tensor(np.ascontiguousarray(y, np.float64)
                         if not isinstance(y, torch.Tensor) else y,
                         dtype=torch.float64).to(dev).contiguous()
    n, F = Xd.shape
    if lib.harl_gbt_fit_scratch_bytes(n, F, max_depth) < 0 or n > 16384:
        raise DeviceError(f"gbt_fit: unsupported shape n={n} F={F} "
                          f"depth={max_depth}")
    if os.environ.get("HARL_FIT_EAGER") == "1":
        fg = None
    else:
        ncap = 1024
        while ncap < n:
            ncap <<= 1
        key = (ncap, F, n_trees, max_depth, float(learning_rate), min_leaf,
               dev)
        fg = _FIT_GRAPHS.get(key)
        if fg is None:
            fg = _FIT_GRAPHS[key] = _FitGraph(ncap, F, n_trees, max_depth,
                                              float(learning_rate), min_leaf,
                                              dev)
    with PF.span("gbt_fit", n, launches=None):
        if fg is not None:
            fg.run(Xd, yd, n)
            feat, thr, val, pred = fg.feat, fg.thr, fg.val, fg.pred
            base, nt = fg.base, fg.nt
        else:
            need = lib.harl_gbt_fit_scratch_bytes(n, F, max_depth)
            scratch = torch.empty(need, dtype=torch.uint8, device=dev)
            K = (1 << (max_depth + 1)) - 1
            T = max(n_trees, 1)
            feat = torch.empty((T, K), dtype=torch.int32, device=dev)
            thr = torch.empty((T, K), dtype=torch.float64, device=dev)
            val = torch.empty((T, K), dtype=torch.float64, device=dev)
            pred = torch.empty(n, dtype=torch.float64, device=dev)
            base = torch.empty(1, dtype=torch.float64, device=dev)
            nt = torch.zeros(1, dtype=torch.int32, device=dev)
            N.check(lib.harl_gbt_fit(
                _ptr(Xd), _ptr(yd), n, F, n_trees, max_depth, learning_rate,
                min_leaf, _ptr(scratch), need, _ptr(feat), _ptr(thr),
                _ptr(val), _ptr(pred), _ptr(base), _ptr(nt), None,
                _stream()), "harl_gbt_fit")
    k = int(nt.item())
    fh = np.ascontiguousarray(feat[:k].cpu().numpy())
    th = np.ascontiguousarray(thr[:k].cpu().numpy())
    vh = np.ascontiguousarray(val[:k].cpu().numpy())
    return GbtFit(float(base.item()), heap_trees_to_reference(fh, th, vh),
                  pred[:n].cpu().numpy())


def heap_trees_to_reference(fh, th, vh):
    """All trees of a fit through the native renumbering
    (harl_heap_to_creation_order; ``heap_tree_to_reference`` is the same
    rule in Python)."""
    T, K = fh.shape if fh.ndim == 2 else (0, 1)
    if T == 0:
        return []
    lib = N.load(require_device=False)
    fo = np.empty((T, K), np.int64)
    to = np.empty((T, K), np.float64)
    lo = np.empty((T, K), np.int64)
    ro = np.empty((T, K), np.int64)
    vo = np.empty((T, K), np.float64)
    sz = np.empty(T, np.int32)
    # (arrays bound to names: a temporary's buffer may be freed before the
    # call reads it)
    fh = np.ascontiguousarray(fh, dtype=np.int32)
    th = np.ascontiguousarray(th, dtype=np.float64)
    vh = np.ascontiguousarray(vh, dtype=np.float64)
    rc = lib.harl_heap_to_creation_order(
        fh.ctypes.data, th.ctypes.data, vh.ctypes.data, K, T,
        fo.ctypes.data, to.ctypes.data, lo.ctypes.data, ro.ctypes.data,
        vo.ctypes.data, sz.ctypes.data)
    if rc != 0:
        raise DeviceError(f"harl_heap_to_creation_order failed ({rc})")
    return [(fo[t, :sz[t]].copy(), to[t, :sz[t]].copy(), lo[t, :sz[t]].copy(),
             ro[t, :sz[t]].copy(), vo[t, :sz[t]].copy()) for t in range(T)]


# ---------------------------------------------------------------------------
# the analytic measurement model (measure.py)


SIM_DEFAULTS = dict(cores=32, cap_l1=4096.0, cap_l2=131072.0,
                    miss_penalty_l1=0.3, miss_penalty_l2=0.6,
                    parallel_overhead=0.02,
                    unroll_factors=((0, 1.00), (16, 0.97), (64, 0.95),
                                    (512, 0.98), (1024, 1.00)),
                    peak_flops=1e11)


def _sim_param(params, name):
    if params is None:
        return SIM_DEFAULTS[name]
    if isinstance(params, dict):
        return params.get(name, SIM_DEFAULTS[name])
    return getattr(params, name)


def sim_desc(tables: SketchTables, params=None) -> "N.SimDesc":
    """The simulator's descriptor for one sketch: SimHwParams (the
    reference's dataclass or a dict; defaults measure.py:41-60) and the
    sketch's stage data.  Noise is ignored (brute_force_best and the pure
    model)."""
    d = N.SimDesc()
    d.cores = int(_sim_param(params, "cores"))
    d.cap_l1 = float(_sim_param(params, "cap_l1"))
    d.cap_l2 = float(_sim_param(params, "cap_l2"))
    d.miss_l1 = float(_sim_param(params, "miss_penalty_l1"))
    d.miss_l2 = float(_sim_param(params, "miss_penalty_l2"))
    d.par_overhead = float(_sim_param(params, "parallel_overhead"))
    d.peak_flops = float(_sim_param(params, "peak_flops"))
    table = dict(_sim_param(params, "unroll_factors"))
    for i, depth in enumerate(tables.unroll_depths):
        d.unroll_factor[i] = float(table.get(depth, 1.0))
    if len(tables.stage_flops) > N.MAX_STAGES or \
            len(tables.sim_skipped) > N.MAX_STAGES:
        raise DeviceError("too many stages for the simulator tables")
    for s_i, (fl, sp) in enumerate(zip(tables.stage_flops,
                                       tables.sim_spatial)):
        d.stage_flops[s_i] = float(fl)
        d.stage_spatial_n[s_i] = len(sp)
        for j, gi in enumerate(sp):
            d.stage_spatial[s_i][j] = gi
    d.n_skipped = len(tables.sim_skipped)
    for k, (fl, l1, l2) in enumerate(tables.sim_skipped):
        d.skipped_flops[k], d.skipped_l1[k], d.skipped_l2[k] = fl, l1, l2
    return d


def simulate_time(dsk: DeviceSketch, tiles, knobs, n: int, params=None,
                  out=None):
    """measure.simulate_time (measure.py:99-112) for n device states:
    seconds under the analytic model, bit-exact."""
    lib = N.load()
    if out is None:
        out = torch.empty(max(n, 1), dtype=torch.float64, device=dsk.device)
    d = sim_desc(dsk.tables, params)
    with PF.span("sim", n):
        N.check(lib.harl_sim_time(C.byref(dsk.desc), C.byref(d), _ptr(tiles),
                                  _ptr(knobs), n, tiles.shape[1], _ptr(out),
                                  _stream()), "harl_sim_time")
    return out[:n]


def space_states(tables: SketchTables) -> int:
    """space_size (schedspace.py:88-95) from the tables."""
    n = 1
    for c in tables.tiling_counts:
        n *= int(c)
    return n * tables.ncas * (tables.max_fusible + 1) * tables.n_unroll


def decode_state_number(tables: SketchTables, x: int):
    """State number -> (tiles [local_slots] u16, knobs (ca, par, ur)) in
    brute_force_best's enumeration order (dim 0's tilings slowest)."""
    L = tables.levels
    ur = x % tables.n_unroll
    x //= tables.n_unroll
    par = x % (tables.max_fusible + 1)
    x //= tables.max_fusible + 1
    ca = x % tables.ncas
    x //= tables.ncas
    tiles = np.zeros(tables.local_slots, dtype=np.uint16)
    for d in range(tables.ndims - 1, -1, -1):
        c = int(tables.tiling_counts[d])
        idx = x % c
        x //= c
        tiles[d * L:(d + 1) * L] = tables.tiling_table[
            int(tables.tiling_offsets[d]) + idx]
    return tiles, (int(ca), int(par), int(ur))


def brute_force_best(tables: SketchTables, params=None,
                     cap: int = 1_000_000, device=None):
    """measure.brute_force_best (measure.py:135-167): the noise-free optimum
    of one sketch's space, ties broken on the canonical text.  The device
    sweeps every state (the minimum time, then the canonically smallest
    state attaining it, compared on rendered text).  Returns (tiles, (ca,
    par, ur), time)."""
    from .errors import SpaceTooLarge
    size = space_states(tables)
    if size > cap:
        raise SpaceTooLarge(size, cap)
    lib = N.load()
    dev = _dev(device)
    dsk = DeviceSketch(tables, dev)
    d = sim_desc(tables, params)
    best = torch.empty(1, dtype=torch.int64, device=dev)
    win = torch.empty(1, dtype=torch.int64, device=dev)
    scratch = torch.empty(4096, dtype=torch.int64, device=dev)
    with PF.span("brute", size):
        N.check(lib.harl_brute_force(C.byref(dsk.desc), C.byref(d), 0, size,
                                     _ptr(best), _ptr(win), _ptr(scratch),
                                     scratch.numel(), _stream()),
                "harl_brute_force")
    bits = int(best.item()) & ((1 << 64) - 1)
    raw = bits & ((1 << 63) - 1) if bits >> 63 else (~bits) & ((1 << 64) - 1)
    t = float(np.asarray([raw], dtype=np.uint64).view(np.float64)[0])
    tl, kn = decode_state_number(tables, int(win.item()))
    return tl, kn, t


def action_masks(dsk: DeviceSketch, tiles, knobs, n: int):
    lib = N.load()
    S = dsk.tables.num_slots
    tiling = torch.empty((max(n, 1), S * S + 1), dtype=torch.uint8,
                         device=dsk.device)
    shift = torch.empty((max(n, 1), 9), dtype=torch.uint8, device=dsk.device)
    N.check(lib.harl_action_masks(C.byref(dsk.desc), _ptr(tiles), _ptr(knobs),
                                  n, tiles.shape[1], _ptr(tiling), _ptr(shift),
                                  _stream()), "harl_action_masks")
    sh = shift[:n].bool()
    return (tiling[:n].bool(), sh[:, 0:3], sh[:, 3:6], sh[:, 6:9])


def apply_actions(dsk: DeviceSketch, tiles, knobs, n: int, actions):
    """actions: host array [n][4] (the reference's (B, 4) layout); raises
    InvalidActionError like the reference."""
    lib = N.load()
    a = torch.from_numpy(np.ascontiguousarray(
        np.asarray(actions, dtype=np.int32).reshape(n, 4).T)).to(dsk.device)
    t_out, k_out = alloc_state(n, dsk.tables, dsk.device, tiles.shape[1])
    status = torch.full((1,), -1, dtype=torch.int64, device=dsk.device)
    N.check(lib.harl_apply_actions(C.byref(dsk.desc), _ptr(tiles), _ptr(knobs),
                                   n, tiles.shape[1], _ptr(a), _ptr(t_out),
                                   _ptr(k_out), _ptr(status), _stream()),
            "harl_apply_actions")
    raise_status(int(status.item()) & ((1 << 64) - 1))
    return t_out, k_out


# ---------------------------------------------------------------------------
# cost model


class DeviceForest:
    """A GBT ensemble in the device layout (costmodel.py:59-78).

    ``trees`` are ``(feature, threshold, left, right, value)`` arrays per
    tree; ``learning_rate * value`` is formed here with numpy, the same
    fp64 product the reference computes per prediction.

    The buffers have a capacity: ``load`` writes a refitted ensemble into
    the same device memory and its scalars into a device header the kernels
    read at run time, so CUDA graphs recorded against this forest stay valid
    across refits (one capture per session, not per round)."""

    NODE = np.dtype([("v", "<f8"), ("feat", "<i2"), ("left", "<i2"),
                     ("right", "<i2"), ("pad", "<i2")])
    HDR = np.dtype([("n_trees", "<i4"), ("fitted", "<i4"), ("base", "<f8"),
                    ("floor_value", "<f8"), ("n_nodes", "<i8"),
                    ("max_depth", "<i4"), ("perfect_depth", "<i4"),
                    ("perfect", "<u8"), ("perfect_bytes", "<i8")])
    PERFECT_MAX = 7       # gbt_kernels.cuh GBT_PERFECT_MAX

    def __init__(self, trees, base: float, learning_rate: float,
                 fitted: bool = True, floor_value: float = 1e-6,
                 device=None, node_capacity: int = 0, tree_capacity: int = 0):
        N.load()
        dev = _dev(device)
        cols = self._columns(trees)
        self.cap_nodes = max(int(cols[0].sum()), int(node_capacity), 1)
        self.cap_trees = max(len(trees), int(tree_capacity), 1)
        self.nodes = torch.zeros(self.cap_nodes * 16, dtype=torch.uint8,
                                 device=dev)
        self.tree_first = torch.zeros(self.cap_trees, dtype=torch.int32,
                                      device=dev)
        self.hdr = torch.zeros(self.HDR.itemsize, dtype=torch.uint8,
                               device=dev)
        # perfect-tree image (forests of depth <= PERFECT_MAX), capacity-
        # sized like the node records
        self.perfect = torch.zeros(
            self.perfect_bytes(self.cap_trees, self.PERFECT_MAX),
            dtype=torch.uint8, device=dev)
        d = N.ForestDesc()
        d.n_trees = self.cap_trees
        d.n_nodes = self.cap_nodes
        d.tree_first = self.tree_first.data_ptr()
        d.nodes = self.nodes.data_ptr()
        d.dev_hdr = self.hdr.data_ptr()
        self.desc = d
        self.device = dev
        # pinned staging of everything _write uploads (node records, perfect
        # image, tree firsts, header), written by harl_forest_pack in place
        pb = self.perfect_bytes(self.cap_trees, self.PERFECT_MAX)
        a16 = lambda n: (n + 15) // 16 * 16  # noqa: E731
        self._o_img = a16(self.cap_nodes * 16)
        self._o_first = self._o_img + a16(pb)
        self._o_hdr = self._o_first + a16(self.cap_trees * 4)
        self._stage = torch.empty(self._o_hdr + a16(self.HDR.itemsize),
                                  dtype=torch.uint8, pin_memory=True)
        self._stage_np = self._stage.numpy()
        self._stage_done = None
        self._write(cols, learning_rate, base, fitted, floor_value)

    @staticmethod
    def _columns(trees):
        """(sizes i64, feature i64, threshold f64, left i64, right i64,
        value f64): the trees' arrays concatenated (harl_forest_pack's
        input)."""
        if len(trees) > 1024:
            raise DeviceError("more than 1024 trees")
        if not trees:
            z = np.zeros(0, np.int64)
            return (z, z, z.astype(np.float64), z, z, z.astype(np.float64))
        sizes = np.fromiter((len(t[0]) for t in trees), np.int64, len(trees))
        cat = [np.concatenate([t[j] for t in trees]).astype(dt, copy=False)
               for j, dt in ((0, np.int64), (1, np.float64), (2, np.int64),
                             (3, np.int64), (4, np.float64))]
        return (sizes, *(np.ascontiguousarray(c) for c in cat))

    @classmethod
    def _native_pack(cls, cols, learning_rate, nodes_out, firsts_out,
                     img_out):
        """harl_forest_pack of ``cols`` into the given host arrays ->
        (depth, perfect-image bytes written)."""
        lib = N.load(require_device=False)
        pbytes = C.c_longlong(0)
        ptr = lambda a: a.ctypes.data  # noqa: E731
        depth = int(lib.harl_forest_pack(
            len(cols[0]), ptr(cols[0]), ptr(cols[1]), ptr(cols[2]),
            ptr(cols[3]), ptr(cols[4]), ptr(cols[5]), float(learning_rate),
            ptr(nodes_out), ptr(firsts_out), cls.PERFECT_MAX, ptr(img_out),
            img_out.nbytes, C.byref(pbytes)))
        if depth < 0:
            raise DeviceError({
                -1: "tree deeper than the reference's 64-step walk",
                -2: "empty tree or child index outside its tree",
                -3: "tree too large for int16 node indices",
                -4: "perfect-tree image beyond its capacity"}.get(
                    depth, f"harl_forest_pack failed ({depth})"))
        return depth, int(pbytes.value)

    @classmethod
    def pack_host(cls, trees, learning_rate):
        """The native packing on its own (host arrays, no device): (node
        records, firsts, depth, perfect image or None) -- what ``_records``
        and ``perfect_image`` restate in numpy."""
        cols = cls._columns(trees)
        nodes = np.zeros(int(cols[0].sum()), cls.NODE)
        firsts = np.zeros(len(cols[0]), np.int32)
        img = np.zeros(cls.perfect_bytes(len(cols[0]), cls.PERFECT_MAX),
                       np.uint8)
        depth, pb = cls._native_pack(cols, learning_rate, nodes.view(np.uint8)
                                     if len(nodes) else np.zeros(16, np.uint8),
                                     firsts if len(firsts)
                                     else np.zeros(1, np.int32), img)
        return nodes, firsts, depth, (img[:pb] if pb else None)

    @classmethod
    def _records(cls, trees, learning_rate):
        """All trees' node records in one vectorised pass (the per-round
        host cost of a refit reload), and the forest's depth (internal
        levels of its deepest tree), with which the kernels walk several
        trees side by side for a fixed number of levels."""
        if len(trees) > 1024:
            raise DeviceError("more than 1024 trees")
        if not trees:
            return np.zeros(0, cls.NODE), np.zeros(0, np.int32), 0
        sizes = np.fromiter((len(t[0]) for t in trees), np.int64, len(trees))
        if sizes.max() > 32767:
            raise DeviceError("tree too large for int16 node indices")
        firsts = np.zeros(len(trees), np.int64)
        np.cumsum(sizes[:-1], out=firsts[1:])
        feat = np.concatenate([np.asarray(t[0]) for t in trees])
        thr = np.concatenate([np.asarray(t[1], np.float64) for t in trees])
        left = np.concatenate([np.asarray(t[2]) for t in trees])
        right = np.concatenate([np.asarray(t[3]) for t in trees])
        val = np.concatenate([np.asarray(t[4], np.float64) for t in trees])
        leaf = feat < 0
        off = np.repeat(firsts, sizes)
        depth = _check_depth_all(feat, np.where(leaf, 0, left) + off,
                                 np.where(leaf, 0, right) + off, firsts)
        rec = np.zeros(len(feat), dtype=cls.NODE)
        # leaves carry learning_rate * value: the reference's fp64
        # product (costmodel.py:224), formed here once
        rec["v"] = np.where(leaf, learning_rate * val, thr)
        rec["feat"] = feat.astype(np.int16)
        rec["left"] = np.where(leaf, 0, left).astype(np.int16)
        rec["right"] = np.where(leaf, 0, right).astype(np.int16)
        return rec, firsts.astype(np.int32), depth

    @staticmethod
    def perfect_bytes(T: int, D: int) -> int:
        """gbt_kernels.cuh gbt_perfect_bytes."""
        leaf = (T * ((1 << D) - 1) * 8 + 15) & ~15
        feat = leaf + T * (1 << D) * 8
        return (feat + T * ((1 << D) - 1) * 2 + 15) & ~15

    @classmethod
    def perfect_image(cls, nodes, firsts, D: int) -> np.ndarray:
        """The perfect-tree image of a forest of depth <= D (gbt_kernels.cuh):
        breadth-first complete trees of D levels; a leaf above the last
        level becomes pass-through slots (feature 0, threshold +inf) whose
        subtree repeats its value.  Built level by level for all trees at
        once."""
        T = len(firsts)
        NI, NL = (1 << D) - 1, 1 << D
        feat = nodes["feat"].astype(np.int64)
        v = nodes["v"]
        sizes = np.diff(np.append(firsts, len(nodes))).astype(np.int64)
        off = np.repeat(firsts.astype(np.int64), sizes)
        left = nodes["left"].astype(np.int64) + off
        right = nodes["right"].astype(np.int64) + off
        thr_p = np.empty((T, NI), np.float64)
        feat_p = np.empty((T, NI), np.int16)
        cur = firsts.astype(np.int64)[:, None]
        for d in range(D):
            leaf = feat[cur] < 0
            lo = (1 << d) - 1
            thr_p[:, lo:lo + (1 << d)] = np.where(leaf, np.inf, v[cur])
            feat_p[:, lo:lo + (1 << d)] = np.where(leaf, 0, feat[cur])
            cur = np.stack([np.where(leaf, cur, left[cur]),
                            np.where(leaf, cur, right[cur])],
                           axis=-1).reshape(T, -1)
        if not (feat[cur] < 0).all():
            raise DeviceError("forest deeper than its perfect image")
        leaf_p = v[cur]
        out = np.zeros(cls.perfect_bytes(T, D), np.uint8)
        b_leaf = (T * NI * 8 + 15) & ~15
        out[:T * NI * 8] = thr_p.reshape(-1).view(np.uint8)
        out[b_leaf:b_leaf + T * NL * 8] = leaf_p.reshape(-1).view(np.uint8)
        b_feat = b_leaf + T * NL * 8
        out[b_feat:b_feat + T * NI * 2] = feat_p.reshape(-1).view(np.uint8)
        return out

    def _write(self, cols, learning_rate, base, fitted, floor_value):
        """Pack ``cols`` (``_columns``) with harl_forest_pack straight into
        the pinned staging buffer and upload it (async copies on the
        current stream; the next write waits for them)."""
        lib = N.load()
        sizes = cols[0]
        T, n_nodes = len(sizes), int(sizes.sum())
        if self._stage_done is not None:
            self._stage_done.synchronize()
        st = self._stage_np
        depth, pb = self._native_pack(
            cols, learning_rate, st,
            st[self._o_first:self._o_first + 4 * T].view(np.int32),
            st[self._o_img:self._o_first])
        self._depth = depth
        self.n_nodes, self.n_trees = n_nodes, T
        h = st[self._o_hdr:self._o_hdr + self.HDR.itemsize].view(self.HDR)
        h["n_trees"], h["fitted"] = T, 1 if fitted else 0
        h["base"], h["floor_value"] = float(base), float(floor_value)
        h["n_nodes"] = n_nodes
        h["max_depth"] = depth
        h["perfect_depth"] = depth if pb else 0
        h["perfect"] = self.perfect.data_ptr()
        h["perfect_bytes"] = pb
        stg = self._stage
        if n_nodes:
            self.nodes[:n_nodes * 16].copy_(stg[:n_nodes * 16],
                                            non_blocking=True)
        if pb:
            self.perfect[:pb].copy_(stg[self._o_img:self._o_img + pb],
                                    non_blocking=True)
        if T:
            self.tree_first[:T].copy_(
                stg[self._o_first:self._o_first + 4 * T].view(torch.int32),
                non_blocking=True)
        self.hdr.copy_(stg[self._o_hdr:self._o_hdr + self.HDR.itemsize],
                       non_blocking=True)
        self._stage_done = torch.cuda.Event()
        self._stage_done.record()
        PF.xfer("h2d", n_nodes * 16 + 4 * T + self.HDR.itemsize + pb)
        # host mirrors (informational; the kernels read the header)
        self.desc.fitted = 1 if fitted else 0
        self.desc.base = float(base)
        self.desc.floor_value = float(floor_value)

    def load(self, trees, base: float, learning_rate: float,
             fitted: bool = True, floor_value: float = 1e-6) -> bool:
        """Load another ensemble in place; False if it exceeds the
        capacity (build a new forest then)."""
        self._loaded = None
        cols = self._columns(trees)
        if int(cols[0].sum()) > self.cap_nodes or len(trees) > self.cap_trees:
            return False
        self._write(cols, learning_rate, base, fitted, floor_value)
        return True

    @staticmethod
    def _model_trees(model):
        return [(t.feature, t.threshold, t.left, t.right, t.value)
                for t in model.trees]

    @classmethod
    def from_model(cls, model, device=None, node_capacity: int = 0,
                   tree_capacity: int = 0):
        """From a reference ``SurrogateModel`` (duck-typed)."""
        trees = cls._model_trees(model)
        f = cls(trees, model.base, model.cfg.learning_rate,
                fitted=model.fitted, device=device,
                node_capacity=node_capacity, tree_capacity=tree_capacity)
        f._loaded = ((model.base, model.cfg.learning_rate, bool(model.fitted),
                      len(trees)), trees)
        return f

    def load_model(self, model) -> bool:
        """Load a reference ``SurrogateModel``; a no-op when it still holds
        the very tree arrays (and scalars) loaded last time -- the
        reference refits by building new trees (costmodel.py:190-212),
        so an unchanged model is skipped without re-packing it."""
        trees = self._model_trees(model)
        sig = (model.base, model.cfg.learning_rate, bool(model.fitted),
               len(trees))
        last = getattr(self, "_loaded", None)
        if last is not None and last[0] == sig and all(
                a is b for ta, tb in zip(trees, last[1])
                for a, b in zip(ta, tb)):
            return True
        ok = self.load(trees, model.base, model.cfg.learning_rate,
                       fitted=model.fitted)
        # the arrays are held, so their identities stay unique
        self._loaded = (sig, trees) if ok else None
        return ok


def _check_depth_all(feat, left_g, right_g, roots):
    """The reference walks at most 64 levels (costmodel.py:67-78); reject
    deeper trees.  All trees at once: global child indices, one
    level-synchronous walk from every root."""
    frontier = np.asarray(roots, dtype=np.int64)
    for depth in range(64):
        inner = frontier[feat[frontier] >= 0]
        if inner.size == 0:
            return depth
        frontier = np.concatenate([left_g[inner], right_g[inner]])
    raise DeviceError("tree deeper than the reference's 64-step walk")


def gbt_predict(forest: DeviceForest, feat, n: int, old_score=None,
                out=None, reward=None):
    lib = N.load()
    F = feat.shape[1]
    if out is None:
        out = torch.empty(max(n, 1), dtype=torch.float64, device=feat.device)
    if old_score is not None and reward is None:
        reward = torch.empty(max(n, 1), dtype=torch.float64, device=feat.device)
    with PF.span("gbt", n):
        N.check(lib.harl_gbt_predict(C.byref(forest.desc), _ptr(feat), n, F,
                                     _ptr(out), _ptr(old_score), _ptr(reward),
                                     _stream()),
                "harl_gbt_predict")
    return (out[:n], reward[:n]) if old_score is not None else out[:n]


# ---------------------------------------------------------------------------
# agent parameters on device


class DeviceAgent:
    """fp64 master parameters + Adam moments + fp32 rollout copy in one flat
    layout per subgraph agent.  The tiling head is stored compact over
    ``head_columns(S, L)``: every other column of the reference's
    ``S*S+1``-wide head has probability zero for every state, hence zero
    gradient and zero Adam moments forever, so it never changes and is left
    untouched in the host arrays."""

    def __init__(self, agent, levels: int, device=None):
        N.load()
        dev = _dev(device)
        self.agent = agent
        self.device = dev
        hidden = tuple(agent.hidden)
        S = agent.num_slots
        F = agent.feature_len
        if len(hidden) > N.MAX_LAYERS or max(hidden) > N.MAX_HIDDEN or \
                F > N.MAX_FEATURES:
            raise DeviceError("network shape beyond the device kernels' limits")
        self.cols = head_columns(S, levels)
        self.C0 = len(self.cols)
        self._hw0 = np.zeros((hidden[-1], self.C0))
        self.NH = self.C0 + 9
        self.hidden, self.F, self.S = hidden, F, S
        nt = len(hidden)
        # ---- flat layout ----
        off = 0
        pl = N.NetLayout()
        pl.n_layers = nt
        dims = [F, *hidden]
        for i, d in enumerate(dims):
            pl.dims[i] = d
        for l in range(nt):
            pl.off_W[l] = off
            off += dims[l] * dims[l + 1]
            pl.off_b[l] = off
            off += dims[l + 1]
        H = hidden[-1]
        pl.off_hW = off
        off += H * self.NH
        pl.off_hb = off
        off += self.NH
        pl.n_head_cols = self.NH
        self.n_pi = off
        vl = N.NetLayout()
        vdims = [F, *hidden, 1]
        vl.n_layers = len(vdims) - 1
        for i, d in enumerate(vdims):
            vl.dims[i] = d
        for l in range(vl.n_layers):
            vl.off_W[l] = off
            off += vdims[l] * vdims[l + 1]
            vl.off_b[l] = off
            off += vdims[l + 1]
        self.n_params = off
        # ---- per-row PPO scratch offsets ----
        r = 0
        pl.row_act[0] = vl.row_act[0] = r
        r += F
        for l in range(1, nt + 1):
            pl.row_act[l] = r
            r += dims[l]
        pl.row_head = r
        r += self.NH
        for l in range(nt):
            pl.row_delta[l] = r
            r += dims[l + 1]
        for l in range(1, vl.n_layers + 1):
            vl.row_act[l] = r
            r += vdims[l]
        for l in range(vl.n_layers):
            vl.row_delta[l] = r
            r += vdims[l + 1]
        self.row_stride = r
        self.pol_layout, self.val_layout = pl, vl
        # parameters and both Adam moments in one [3][n] block (one copy
        # each way per episode), staged through one pinned host block
        # (rows 3-5: the speculative update's pre-update backup)
        self._pmv6 = torch.zeros((6, self.n_params), dtype=torch.float64,
                                 device=dev)
        self.pmv = self._pmv6[:3]
        self.params, self.m, self.v = self.pmv[0], self.pmv[1], self.pmv[2]
        self._pin = torch.empty((3, self.n_params), dtype=torch.float64,
                                pin_memory=True)
        self._pin_np = self._pin.numpy()
        self._pin_done = None
        self._pin_views = [self._views(self._pin_np[i]) for i in range(3)]
        self.grads = torch.zeros_like(self.params)
        self.params32 = torch.zeros(self.n_params, dtype=torch.float32,
                                    device=dev)
        self.losses = torch.zeros(16, dtype=torch.float64, device=dev)
        # bad[0]: ppo_update's finiteness flags; bad[1]: the speculative
        # update's per-update snapshot of bad[0]
        self._badw = torch.zeros(2, dtype=torch.int32, device=dev)
        self.bad = self._badw[:1]
        # transposed fp64 copies for the PPO backward (kept current by Adam)
        self.wt = torch.zeros(max(1, int(N.load().harl_ppo_wt_doubles(
            C.byref(pl), C.byref(vl)))), dtype=torch.float64, device=dev)
        self.tc = (hidden == (128, 128) and F <= 64 and self.NH <= 128
                   and os.environ.get("HARL_KERNELS", "tc") != "ffma")
        self._hid = None
        self._retired = []      # scratch buffers graphs may still address
        self.packed = None
        if self.tc:
            lib = N.load()
            self.packed = {
                "pt": torch.empty(lib.harl_tc_packed_bytes(0, self.NH),
                                  dtype=torch.uint8, device=dev),
                "ph": torch.empty(lib.harl_tc_packed_bytes(1, self.NH),
                                  dtype=torch.uint8, device=dev),
                "vt": torch.empty(lib.harl_tc_packed_bytes(0, self.NH),
                                  dtype=torch.uint8, device=dev)}
        self.head0_src = np.asarray(
            [int(c) // S if j < self.C0 - 1 else 0
             for j, c in enumerate(self.cols)], dtype=np.int16)
        self._build_descs()
        self.upload()

    def repack(self):
        """Rebuild the tcgen05 weight images from the fp32 rollout copy
        (after upload and after every PPO update)."""
        if not self.tc:
            return
        lib = N.load()
        with PF.span("pack", 0, launches=None):
            N.check(lib.harl_pack_tc_weights(
                C.byref(self.pol_desc), C.byref(self.val_desc), self.F,
                _ptr(self.packed["pt"]), _ptr(self.packed["ph"]),
                _ptr(self.packed["vt"]), _stream()), "harl_pack_tc_weights")

    # -- host <-> device --------------------------------------------------

    def _views(self, flat: np.ndarray):
        """1-D views of a flat parameter vector in the numpy lists' order:
        (policy trunk W/b..., the compact head's [H][NH] and [NH] blocks,
        value W/b...)."""
        pl, vl = self.pol_layout, self.val_layout
        nt = len(self.hidden)
        dims = [self.F, *self.hidden]
        trunk = []
        for l in range(nt):
            n = dims[l] * dims[l + 1]
            trunk.append(flat[pl.off_W[l]:pl.off_W[l] + n])
            trunk.append(flat[pl.off_b[l]:pl.off_b[l] + dims[l + 1]])
        H = self.hidden[-1]
        hW = flat[pl.off_hW:pl.off_hW + H * self.NH].reshape(H, self.NH)
        hb = flat[pl.off_hb:pl.off_hb + self.NH]
        vdims = [self.F, *self.hidden, 1]
        val = []
        for l in range(vl.n_layers):
            n = vdims[l] * vdims[l + 1]
            val.append(flat[vl.off_W[l]:vl.off_W[l] + n])
            val.append(flat[vl.off_b[l]:vl.off_b[l] + vdims[l + 1]])
        return trunk, hW, hb, val

    def _copy_plan(self, pol_list, val_list):
        """harl_agent_copy's op list moving these arrays to / from the flat
        layout (the _views / _pack order), cached while the arrays are the
        same objects; None if one is not a C-contiguous float64 array of
        its layout shape (the numpy copies handle it then)."""
        key = tuple(id(a) for a in pol_list) + tuple(id(a) for a in val_list)
        cache = getattr(self, "_plans", None)
        if cache is None:
            cache = self._plans = {}
        hit = cache.get(key)
        if hit is not None:
            return hit[0]
        arrs = list(pol_list) + list(val_list)
        if any(not isinstance(a, np.ndarray) or a.dtype != np.float64 or
               not a.flags.c_contiguous for a in arrs):
            return None
        pl, vl = self.pol_layout, self.val_layout
        nt = len(self.hidden)
        dims = [self.F, *self.hidden]
        H, NH, C0 = self.hidden[-1], self.NH, self.C0
        cols = np.ascontiguousarray(self.cols, dtype=np.int64)
        ops = []

        def flat_op(off, a, n):
            if a.size != n:
                raise ValueError
            ops.append((off, 0, a.ctypes.data, 0, 1, n, None))
        try:
            for l in range(nt):
                flat_op(pl.off_W[l], pol_list[2 * l], dims[l] * dims[l + 1])
                flat_op(pl.off_b[l], pol_list[2 * l + 1], dims[l + 1])
            heads = pol_list[2 * nt:]
            if heads[0].shape[0] != H or heads[1].size != heads[0].shape[1]:
                raise ValueError
            ops.append((pl.off_hW, NH, heads[0].ctypes.data, heads[0].shape[1],
                        H, C0, cols.ctypes.data))
            ops.append((pl.off_hb, 0, heads[1].ctypes.data, 0, 1, C0,
                        cols.ctypes.data))
            for h in range(3):
                w, b = heads[2 + 2 * h], heads[3 + 2 * h]
                if w.shape != (H, 3) or b.size != 3:
                    raise ValueError
                ops.append((pl.off_hW + C0 + 3 * h, NH, w.ctypes.data, 3, H, 3,
                            None))
                ops.append((pl.off_hb + C0 + 3 * h, 0, b.ctypes.data, 0, 1, 3,
                            None))
            vdims = [self.F, *self.hidden, 1]
            for l in range(vl.n_layers):
                flat_op(vl.off_W[l], val_list[2 * l], vdims[l] * vdims[l + 1])
                flat_op(vl.off_b[l], val_list[2 * l + 1], vdims[l + 1])
        except (ValueError, IndexError):
            return None
        arr = (N.CopyOp * len(ops))(*[N.CopyOp(*o) for o in ops])
        if len(cache) > 16:
            cache.clear()
        cache[key] = ((arr, len(ops)), arrs, cols)   # keeps the ids valid
        return cache[key][0]

    def _native_copy(self, flat: np.ndarray, pol_list, val_list,
                     to_host: bool) -> bool:
        plan = self._copy_plan(pol_list, val_list)
        if plan is None:
            return False
        N.check(N.load().harl_agent_copy(plan[0], plan[1], flat.ctypes.data,
                                         1 if to_host else 0),
                "harl_agent_copy")
        return True

    def _lists(self):
        a = self.agent
        return ((a.policy, a.value), (a.opt_pi.m, a.opt_v.m),
                (a.opt_pi.v, a.opt_v.v))

    def _host_matches_pin(self) -> bool:
        """The numpy parameters and moments equal, bit for bit, the pinned
        block (False when a list cannot be compared natively).  In line: a
        pool dispatch costs more than the three ~30 us compares."""
        lib = N.load()
        plans = [self._copy_plan(pol, val) for pol, val in self._lists()]
        if any(p is None for p in plans):
            return False

        def cmp(i):
            return lib.harl_agent_copy(plans[i][0], plans[i][1],
                                       self._pin_np[i].ctypes.data, 2) == 0
        return all(cmp(i) for i in range(3))

    def _unpack_all(self):
        """The pinned block -> the numpy lists (native plans, the three
        lists on the host pool's threads; numpy copies where no plan)."""
        pin, vw = self._pin_np, self._pin_views
        lists = self._lists()

        def one(i):
            pol, val = lists[i]
            return self._native_copy(pin[i], pol, val, True)
        done = list(_host_pool().map(one, range(3))) if _POOL_ON else \
            [one(i) for i in range(3)]
        for i, ok in enumerate(done):
            if not ok:
                self._unpack_into(pin[i], *lists[i], vw[i])

    def _pack(self, pol_list, val_list, out=None, views=None) -> np.ndarray:
        """The numpy lists -> the flat layout (every element written)."""
        if out is None:
            out = np.zeros(self.n_params, dtype=np.float64)
        trunk, hW, hb, val = views if views is not None else self._views(out)
        nt2 = len(trunk)
        for dst, src in zip(trunk, pol_list):
            np.copyto(dst, src.reshape(-1))
        heads = pol_list[nt2:]
        C0 = self.C0
        np.take(heads[0], self.cols, axis=1, out=self._hw0)
        hW[:, :C0] = self._hw0
        hb[:C0] = heads[1][self.cols]
        for h in range(3):
            hW[:, C0 + 3 * h:C0 + 3 * h + 3] = heads[2 + 2 * h]
            hb[C0 + 3 * h:C0 + 3 * h + 3] = heads[3 + 2 * h]
        for dst, src in zip(val, val_list):
            np.copyto(dst, src.reshape(-1))
        return out

    def _unpack_into(self, flat: np.ndarray, pol_list, val_list, views=None):
        trunk, hW, hb, val = views if views is not None else self._views(flat)
        nt2 = len(trunk)
        for src, dst in zip(trunk, pol_list):
            np.copyto(dst, src.reshape(dst.shape))
        heads = pol_list[nt2:]
        C0 = self.C0
        heads[0][:, self.cols] = hW[:, :C0]
        heads[1][self.cols] = hb[:C0]
        for h in range(3):
            np.copyto(heads[2 + 2 * h], hW[:, C0 + 3 * h:C0 + 3 * h + 3])
            np.copyto(heads[3 + 2 * h], hb[C0 + 3 * h:C0 + 3 * h + 3])
        for src, dst in zip(val, val_list):
            np.copyto(dst, src.reshape(dst.shape))

    def upload(self):
        """The numpy parameters and moments -> the device: packed into the
        pinned block, one async copy, then the derived copies (fp32
        rollout parameters, transposes, weight images) on the device."""
        a = self.agent
        if self._pin_done is not None:      # the last copy out of _pin
            self._pin_done.synchronize()
        if _UPLOAD_SKIP and getattr(self, "_device_is_pin", False) and \
                self._host_matches_pin():
            # the device state is what the last download wrote into the
            # lists, and nobody changed them since: nothing to upload
            return
        pin, vw = self._pin_np, self._pin_views
        for i, (pol, val) in enumerate(((a.policy, a.value),
                                        (a.opt_pi.m, a.opt_v.m),
                                        (a.opt_pi.v, a.opt_v.v))):
            if not self._native_copy(pin[i], pol, val, False):
                self._pack(pol, val, pin[i], vw[i])
        self.pmv.copy_(self._pin, non_blocking=True)
        self._pin_done = torch.cuda.Event()
        self._pin_done.record()
        self.params32.copy_(self.params)
        PF.xfer("h2d", self.pmv)
        self.refresh_derived()
        self._device_is_pin = True

    def refresh_derived(self):
        """Rebuild every device copy derived from the master parameters:
        the fp64 transposes the PPO backward reads and the tcgen05 weight
        images (the Adam kernel keeps both current afterwards)."""
        lib = N.load()
        with PF.span("wt_fill", 0):
            N.check(lib.harl_ppo_wt_fill(C.byref(self.pol_layout),
                                         C.byref(self.val_layout),
                                         _ptr(self.params), _ptr(self.wt),
                                         _stream()), "harl_ppo_wt_fill")
        if getattr(self, "packed", None) is not None:
            self.repack()

    def download_async(self):
        """Start the device -> pinned copy of params and moments on a side
        stream (ordered after everything issued so far on the current
        stream) so the caller can issue other device work meanwhile;
        ``download`` finishes it."""
        if self._pin_done is not None:
            self._pin_done.synchronize()
        main = torch.cuda.current_stream()
        side = getattr(self, "_side", None)
        if side is None:
            side = self._side = torch.cuda.Stream(device=self.device)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            self._pin.copy_(self.pmv, non_blocking=True)
            self._dl_done = torch.cuda.Event()
            self._dl_done.record()
        self.pmv.record_stream(side)

    def download_start_unpack(self):
        """After ``download_async``: wait for the copy and write the numpy
        lists on the host pool (the caller keeps working; ``download``
        joins).  Call only when nothing else touches the lists meanwhile."""
        dl = getattr(self, "_dl_done", None)
        if dl is None:
            return
        self._dl_done = None

        if not _POOL_ON:
            self._dl_done = dl       # download() finishes it in line
            return

        def job():
            dl.synchronize()
            self._unpack_all()
        self._unpack_job = _host_pool().submit(job)

    def download(self):
        """Write device params and moments back into the numpy lists."""
        job = getattr(self, "_unpack_job", None)
        if job is not None:       # started by download_start_unpack
            self._unpack_job = None
            job.result()
        else:
            dl = getattr(self, "_dl_done", None)
            if dl is not None:    # started by download_async
                self._dl_done = None
                dl.synchronize()
            else:
                if self._pin_done is not None:
                    self._pin_done.synchronize()
                self._pin.copy_(self.pmv, non_blocking=True)
                torch.cuda.current_stream().synchronize()
            self._unpack_all()
        self._pin_done = None
        self._device_is_pin = True
        PF.xfer("d2h", self.pmv)

    def _build_descs(self):
        base = self.params32.data_ptr()
        f4 = 4
        pl, vl = self.pol_layout, self.val_layout
        pd = N.MlpDesc()
        pd.n_layers = pl.n_layers
        for i in range(pl.n_layers + 1):
            pd.dims[i] = pl.dims[i]
        for l in range(pl.n_layers):
            pd.W[l] = base + f4 * pl.off_W[l]
            pd.b[l] = base + f4 * pl.off_b[l]
        pd.head_W = base + f4 * pl.off_hW
        pd.head_b = base + f4 * pl.off_hb
        pd.n_head_cols = self.NH
        vd = N.MlpDesc()
        vd.n_layers = vl.n_layers
        for i in range(vl.n_layers + 1):
            vd.dims[i] = vl.dims[i]
        for l in range(vl.n_layers):
            vd.W[l] = base + f4 * vl.off_W[l]
            vd.b[l] = base + f4 * vl.off_b[l]
        self.pol_desc, self.val_desc = pd, vd

    def hid_scratch(self, n: int):
        """The logits scratch of the tcgen05 policy path, grown on demand.
        A replaced buffer is retired, not freed: CUDA graphs captured
        against it (other episode geometries cached by the engine) keep
        its address baked in."""
        if self._hid is None or self._hid.shape[0] < n:
            if self._hid is not None:
                self._retired.append(self._hid)
            self._hid = torch.empty((max(n, 1), 128), dtype=torch.float32,
                                    device=self.device)
        return self._hid

    def raise_if_diverged(self):
        """ppo_update's finiteness checks (rlcore.py:368-373): the kernels
        set ``bad`` (1: a loss, 2: a gradient) and skip the Adam step; the
        host raises the reference's RlDivergedError."""
        code = int(self.bad.item())
        if code:
            self.restore_diverged()
        raise_diverged(code)

    def restore_diverged(self):
        """After a flagged speculative update (harl_ppo_update with
        HARL_PPO_SPECULATIVE): parameters and moments back to their values
        before it (the backup rows), derived copies rebuilt -- the state
        the reference leaves when ppo_update raises before stepping."""
        if not getattr(self, "_spec_used", False):
            return
        self.pmv.copy_(self._pmv6[3:])
        self.params32.copy_(self.params)
        self.refresh_derived()
        self._device_is_pin = False

    # -- PPO ----------------------------------------------------------------

    def ppo_update(self, ring, slots, cfg, t_pi: int, t_v: int,
                   scratch=None, losses=None, adam_dev=None, B_norm=None,
                   phase: int = 3):
        """One ppo_update on replay ``slots`` (device int32 ring slots).
        ``t_pi``/``t_v`` are the Adam step counts AFTER this update."""
        self._device_is_pin = False
        lib = N.load()
        B = int(slots.shape[0])
        hp = N.PpoHyper()
        hp.clip_ratio = cfg.clip_ratio
        hp.entropy_weight = cfg.entropy_weight
        hp.value_loss_weight = cfg.value_loss_weight
        hp.lr_actor, hp.lr_critic = cfg.lr_actor, cfg.lr_critic
        b1, b2 = 0.9, 0.999
        hp.beta1, hp.beta2 = b1, b2
        hp.one_m_beta1, hp.one_m_beta2 = 1.0 - b1, 1.0 - b2
        hp.eps = 1e-8
        hp.b1t_pi, hp.b2t_pi = 1.0 - b1 ** t_pi, 1.0 - b2 ** t_pi
        hp.b1t_v, hp.b2t_v = 1.0 - b1 ** t_v, 1.0 - b2 ** t_v
        if scratch is None:
            nbytes = lib.harl_ppo_scratch_bytes(max(B, 1), self.row_stride, 0)
            scratch = torch.empty(nbytes, dtype=torch.uint8,
                                  device=self.device)
        if losses is None:
            losses = self.losses
        src = self.head0_src.ctypes.data_as(C.c_void_p)
        # speculative gradients + Adam (single device, not the cooperative
        # variant); the backup restores a flagged update (restore_diverged)
        spec = _PPO_SPEC and phase == 3 and not _PPO_COOP
        # (launch count from the library: 2 when wgrad and Adam run as one
        # kernel, 3 otherwise)
        with PF.span("ppo", B, launches=None):
          N.check(lib.harl_ppo_update(
            C.byref(self.pol_layout), C.byref(self.val_layout), C.byref(hp),
            C.byref(ring.desc), _ptr(slots), B, self.F, self.C0, src,
            self.row_stride, _ptr(self.params), _ptr(self.grads), _ptr(self.m),
            _ptr(self.v), _ptr(self.params32), self.n_pi, self.n_params,
            _ptr(losses), _ptr(self.bad), _ptr(scratch), _ptr(adam_dev),
            *(([_ptr(self.packed["pt"]), _ptr(self.packed["ph"]),
                _ptr(self.packed["vt"])]) if self.tc else [None, None, None]),
            _ptr(self.wt), int(B_norm or B),
            phase | (PPO_SPECULATIVE if spec else 0), _stream()),
            "harl_ppo_update")
        if spec:
            self._spec_used = True
        return losses


def policy_step(dsk: DeviceSketch, agent: DeviceAgent, feat, tiles, knobs,
                n: int, gen=None, inject=None, out=None, want_logits=False,
                rng_dev=None, advance=True, grow=None, m_total: int = 0,
                feat_out=None, fuse_tc: bool = False, reset_status=True,
                settled: bool = False, gbt=None, split: int = 0):
    """select_actions + decode/apply for n rows.  Consumes 4*n doubles of
    ``gen`` (head-major, like rlcore.py:223-225) unless ``inject`` is given.
    ``feat_out`` (optional f64 [n][F]): also featurize the new states (in
    the sampler kernel on the tcgen05 path; ``fuse_tc``: in the one fused
    policy->sample->featurize kernel instead).  ``reset_status=False``: the
    caller already set ``out["status"]`` to -1 (the engine fills its
    per-step status table once per episode, not once per step).
    ``settled``: the weight images were not written by the previous launch
    (see ``value_pair``).  ``gbt`` (optional ``(forest, old_score, score,
    reward)``): score the featurized successor rows with the forest inside
    the sampler (harl_policy_step_tc_gbt); ``out["gbt_fused"]`` says
    whether the library took it (else the caller scores them).
    ``split=STEP_SAMPLE_ONLY``: the policy network already ran for these
    rows (``policy_mlp``), only the sampler launches.  Returns a dict of
    device tensors; ``status`` must be checked by the caller
    (``raise_status``)."""
    lib = N.load()
    dev = dsk.device
    if out is None:
        ld = tiles.shape[1]
        t_o, k_o = alloc_state(n, dsk.tables, dev, ld)
        out = {"actions": torch.empty((4, max(n, 1)), dtype=torch.int32,
                                      device=dev),
               "logp": torch.empty(max(n, 1), dtype=torch.float64, device=dev),
               "tiles": t_o, "knobs": k_o,
               "move_bits": torch.empty(max(n, 1), dtype=torch.int64,
                                        device=dev),
               "shift_bits": torch.empty(max(n, 1), dtype=torch.int32,
                                         device=dev),
               "head0_col": torch.empty(max(n, 1), dtype=torch.int32,
                                        device=dev),
               "status": torch.full((1,), -1, dtype=torch.int64, device=dev)}
    elif reset_status:
        out["status"].fill_(-1)
    logits = None
    if want_logits:
        logits = torch.empty((max(n, 1), agent.NH), dtype=torch.float32,
                             device=dev)
    st = R.to_struct(gen) if gen is not None else None
    inj = None
    if inject is not None:
        inj = torch.as_tensor(np.ascontiguousarray(np.asarray(inject).T),
                              dtype=torch.int32).to(dev).contiguous()
    args = [C.byref(dsk.desc), C.byref(agent.pol_desc), _ptr(feat),
            _ptr(tiles), _ptr(knobs), n, tiles.shape[1],
            C.byref(st) if st is not None else None, _ptr(inj),
            _ptr(out["actions"]), _ptr(out["logp"]), _ptr(out["tiles"]),
            _ptr(out["knobs"]), _ptr(out["move_bits"]),
            _ptr(out["shift_bits"]), _ptr(out["head0_col"]), _ptr(logits),
            _ptr(out["status"])]
    out["gbt_fused"] = False
    if agent.tc:
        flags = (STEP_FUSED if fuse_tc else 0) | \
            (WEIGHTS_SETTLED if settled else 0) | split
        tc_args = [*args, _ptr(agent.hid_scratch(n)), _ptr(rng_dev),
                   _ptr(agent.packed["pt"]), _ptr(agent.packed["ph"]),
                   _ptr(grow), m_total, _ptr(feat_out), flags]
        with PF.span("policy_tc", n, launches=None):
            rc = N.E_LIMIT
            if gbt is not None and feat_out is not None and not fuse_tc:
                forest, old_score, score, reward = gbt
                rc = lib.harl_policy_step_tc_gbt(
                    *tc_args, C.byref(forest.desc), _ptr(old_score),
                    _ptr(score), _ptr(reward), _stream())
                if rc != N.E_LIMIT:
                    N.check(rc, "harl_policy_step_tc_gbt")
                    out["gbt_fused"] = True
            if rc == N.E_LIMIT:
                N.check(lib.harl_policy_step_tc(*tc_args, _stream()),
                        "harl_policy_step_tc")
        if feat_out is not None and not fuse_tc and n > SAMPLE_FEAT_MAX_ROWS:
            # the library featurized with k_featurize2 inside the call: its
            # rows belong to the featurize span (per-kernel roofline rows)
            with PF.span("featurize", n, launches=0):
                pass
    else:
        with PF.span("policy", n):
            N.check(lib.harl_policy_step(*args, _ptr(grow), m_total, _stream()),
                    "harl_policy_step")
        if feat_out is not None:
            featurize(dsk, out["tiles"], out["knobs"], n, feat_out)
    if gen is not None and inject is None and advance:
        R.skip_u64(gen, 4 * (m_total or n))
    if want_logits:
        out["logits"] = logits[:n]
    return out


def value_estimate(agent: DeviceAgent, feat, n: int, out=None):
    lib = N.load()
    if out is None:
        out = torch.empty(max(n, 1), dtype=torch.float32, device=feat.device)
    with PF.span("value", n):
        N.check(lib.harl_value_forward(C.byref(agent.val_desc), _ptr(feat), n,
                                       feat.shape[1], _ptr(out), _stream()),
                "harl_value_forward")
    return out[:n]


# harl_policy_step_tc / harl_value_pair_tc flags (include/harl_b200.h)
# DeviceAgent.upload skips the copy while the numpy lists still hold what
# the last download wrote (HARL_UPLOAD_SKIP=0: always upload; A/B)
_UPLOAD_SKIP = os.environ.get("HARL_UPLOAD_SKIP", "1") != "0"

STEP_FUSED, WEIGHTS_SETTLED = 1, 2
STEP_MLP_ONLY, STEP_SAMPLE_ONLY, VALUE_PAIRED = 4, 8, 16
PPO_SPECULATIVE = 8
# gradients + Adam in one launch, restored on divergence
# (HARL_PPO_SPEC=0: the separate k_ppo_wgrad + k_ppo_adam launches)
_PPO_SPEC = os.environ.get("HARL_PPO_SPEC", "1") != "0"
_PPO_COOP = os.environ.get("HARL_PPO_FUSED_ADAM") == "1"


_POOL = None
# HARL_HOST_POOL=1: the agent lists are unpacked on a host thread while the
# entry list is built -- measured slower at C2 (e2e 6.29-6.43 vs 5.95-6.00
# ms per call: the worker contends for the GIL with the entry building),
# so the copies run in line by default
_POOL_ON = os.environ.get("HARL_HOST_POOL", "0") == "1"


def _host_pool():
    """A small persistent host thread pool for the native agent copies
    (ctypes releases the GIL, so the three lists copy in parallel)."""
    global _POOL
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(max_workers=3,
                                   thread_name_prefix="harl-agent")
    return _POOL


def raise_diverged(code: int) -> None:
    """DeviceAgent.bad as ppo_update's exception (rlcore.py:368-373)."""
    if code & 1:
        raise RlDivergedError("actor or critic loss is not finite")
    if code:
        raise RlDivergedError("non-finite gradient in update")


def policy_mlp(dsk: DeviceSketch, agent: DeviceAgent, feat, n: int,
               settled: bool = True) -> bool:
    """The policy network alone (PolicyNet.forward, rlcore.py:136-146) for
    n rows into the agent's logits scratch, for a later
    ``policy_step(..., split=STEP_SAMPLE_ONLY)`` on the same rows.  False
    (nothing launched) off the 3xFP16 path."""
    if not agent.tc:
        return False
    lib = N.load()
    z = [None] * 10
    with PF.span("policy_tc", n, launches=None):
        rc = lib.harl_policy_step_tc(
            C.byref(dsk.desc), C.byref(agent.pol_desc), _ptr(feat), None, None,
            n, 0, None, *z, _ptr(agent.hid_scratch(n)), None,
            _ptr(agent.packed["pt"]), _ptr(agent.packed["ph"]), None, 0, None,
            STEP_MLP_ONLY | (WEIGHTS_SETTLED if settled else 0), _stream())
    if rc == N.E_LIMIT:
        return False
    N.check(rc, "harl_policy_step_tc")
    return True


def value_pair(agent: DeviceAgent, feat0, n0: int, feat1, n1: int,
               out0, out1, settled: bool = False, paired: bool = False):
    """V(X) and V(X') (tuner.py:395-396); one tcgen05 launch for the
    production shape, otherwise two FFMA launches.  ``settled``: the
    weight images were not written by the previous launch (the kernel may
    prefetch them ahead of its PDL wait)."""
    lib = N.load()
    if agent.tc:
        with PF.span("value_tc", n0 + n1):
            N.check(lib.harl_value_pair_tc(C.byref(agent.val_desc),
                                           _ptr(feat0), n0, _ptr(feat1), n1,
                                           feat0.shape[1], _ptr(out0),
                                           _ptr(out1), _ptr(agent.packed["vt"]),
                                           (WEIGHTS_SETTLED if settled else 0) |
                                           (VALUE_PAIRED if paired else 0),
                                           _stream()),
                    "harl_value_pair_tc")
        return out0[:n0], out1[:n1]
    return (value_estimate(agent, feat0, n0, out0),
            value_estimate(agent, feat1, n1, out1))


class DeviceReplay:
    """The replay FIFO as a device ring (rlcore.py:253-274)."""

    def __init__(self, capacity: int, feature_len: int, device=None):
        dev = _dev(device)
        self.cap = int(capacity)
        self.F = feature_len
        self.X = torch.zeros((self.cap, feature_len), dtype=torch.float64,
                             device=dev)
        self.Xn = torch.zeros_like(self.X)
        self.actions = torch.zeros((self.cap, 4), dtype=torch.int32, device=dev)
        self.scalars = torch.zeros((self.cap, 4), dtype=torch.float64,
                                   device=dev)
        self.move_bits = torch.zeros(self.cap, dtype=torch.int64, device=dev)
        self.shift_bits = torch.zeros(self.cap, dtype=torch.int32, device=dev)
        self.count = 0
        self.wpos = 0
        d = N.ReplayRing()
        d.X, d.Xn = self.X.data_ptr(), self.Xn.data_ptr()
        d.actions, d.scalars = self.actions.data_ptr(), self.scalars.data_ptr()
        d.move_bits = self.move_bits.data_ptr()
        d.shift_bits = self.shift_bits.data_ptr()
        d.cap = self.cap
        self.desc = d
        self.device = dev

    def __len__(self):
        return self.count

    def slots_of(self, idx: np.ndarray) -> np.ndarray:
        """Buffer positions (0 = oldest) -> ring slots."""
        start = (self.wpos - self.count) % self.cap
        return ((start + np.asarray(idx, dtype=np.int64)) % self.cap) \
            .astype(np.int32)

    def note_push(self, n: int):
        self.wpos = (self.wpos + n) % self.cap
        self.count = min(self.cap, self.count + n)


def masks_to_bits(masks, num_slots: int, levels: int):
    """ActionMask arrays (tiling [B, S*S+1], 3x [B, 3]) -> (move bits,
    shift bits).  A slot is movable iff any same-dim move out of it is
    legal (schedspace.py:241-248)."""
    tiling = np.asarray(masks[0], dtype=bool)
    B = len(tiling)
    S, L = num_slots, levels
    move = np.zeros(B, dtype=np.uint64)
    if L >= 2:
        for src in range(S):
            dst = (src // L) * L + (src % L + 1) % L
            move |= tiling[:, src * S + dst].astype(np.uint64) << np.uint64(src)
    shift = np.zeros(B, dtype=np.uint32)
    for h in range(3):
        m = np.asarray(masks[1 + h], dtype=bool)
        for j in range(3):
            shift |= m[:, j].astype(np.uint32) << np.uint32(3 * h + j)
    return move, shift


def bits_to_masks(move, shift, num_slots: int, levels: int):
    """Inverse of masks_to_bits (materialises the reference's boolean
    masks, e.g. for checkpoints, tuner.py:683-684)."""
    move = np.asarray(move).astype(np.uint64)
    shift = np.asarray(shift).astype(np.uint32)
    B = len(move)
    S, L = num_slots, levels
    tiling = np.zeros((B, S * S + 1), dtype=bool)
    tiling[:, -1] = True
    for src in range(S):
        bit = ((move >> np.uint64(src)) & np.uint64(1)).astype(bool)
        base = (src // L) * L
        for dst in range(base, base + L):
            if dst != src:
                tiling[:, src * S + dst] = bit
    out = [tiling]
    for h in range(3):
        out.append(np.stack([((shift >> np.uint32(3 * h + j)) & 1).astype(bool)
                             for j in range(3)], axis=1))
    return tuple(out)


def _replay_load(self, X, Xn, actions, logp, reward, adv, td, masks,
                 num_slots: int, levels: int):
    """Replace the ring contents with host transitions (oldest first),
    like rebuilding the reference's deque (tuner.py:752-768)."""
    n = len(X)
    if n > self.cap:
        raise ValueError("more transitions than ring capacity")
    cols = head_columns(num_slots, levels)
    col_of = {int(c): j for j, c in enumerate(cols)}
    acts = np.asarray(actions, dtype=np.int64).reshape(n, 4).copy()
    acts[:, 0] = [col_of[int(a)] for a in acts[:, 0]]
    move, shift = masks_to_bits(masks, num_slots, levels)
    dev = self.device
    if n:
        self.X[:n].copy_(torch.from_numpy(np.asarray(X, np.float64)))
        self.Xn[:n].copy_(torch.from_numpy(np.asarray(Xn, np.float64)))
        self.actions[:n].copy_(torch.from_numpy(acts.astype(np.int32)))
        sc = np.stack([logp, reward, adv, td], axis=1).astype(np.float64)
        self.scalars[:n].copy_(torch.from_numpy(sc))
        self.move_bits[:n].copy_(torch.from_numpy(move.view(np.int64)))
        self.shift_bits[:n].copy_(torch.from_numpy(shift.view(np.int32)))
    self.count = n
    self.wpos = n % self.cap
    del dev


def _replay_export(self, num_slots: int, levels: int):
    """Ring contents oldest-first as host arrays with full head indices and
    materialised boolean masks."""
    n = self.count
    start = (self.wpos - n) % self.cap
    order = (start + np.arange(n)) % self.cap
    idx = torch.from_numpy(order).to(self.device)
    cols = head_columns(num_slots, levels)
    acts = self.actions[idx].cpu().numpy().astype(np.int64)
    if n:
        acts[:, 0] = cols[acts[:, 0]]
    sc = self.scalars[idx].cpu().numpy()
    move = self.move_bits[idx].cpu().numpy().view(np.uint64)
    shift = self.shift_bits[idx].cpu().numpy().view(np.uint32)
    return {"X": self.X[idx].cpu().numpy(), "Xn": self.Xn[idx].cpu().numpy(),
            "actions": acts, "logp": sc[:, 0], "reward": sc[:, 1],
            "adv": sc[:, 2], "td": sc[:, 3],
            "masks": bits_to_masks(move, shift, num_slots, levels)}


DeviceReplay.load = _replay_load
DeviceReplay.export = _replay_export
