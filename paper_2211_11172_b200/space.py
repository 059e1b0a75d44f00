"""Schedule-space host utilities and the per-sketch device tables.

Host mirror of the parts of the reference's ``schedspace.py`` that the B200
engine needs off the hot path:

* tiling combinatorics (``list_tilings`` etc., reference schedspace.py:39-100)
* the ``ScheduleState`` value type and its canonical text
  (schedspace.py:107-120)
* ``SketchTables``: everything ``SketchContext.__init__`` precomputes
  (schedspace.py:324-368), flattened into the integer/float arrays that the
  CUDA kernels read from constant memory: tiled-dim extents, the footprint
  term table per anchor stage, the log2/10 lookup over tile factors, the
  smallest-prime-factor lookup, the enumerated tilings used by the
  initial-state sampler, and the feature-vector layout.

The tables are built from duck-typed sketch objects, so both the reference's
``Sketch``/``SubgraphSpec`` and this package's mirrors work.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from .errors import ScheduleError

# Limits shared with the CUDA side (csrc/harl_common.cuh).
MAX_DIMS = 16          # tiled dims per sketch (feature budget is usually 10)
MAX_LEVELS = 8
MAX_SLOTS = 64         # agent-wide slots S (ndims * levels)
MAX_STAGES = 16
MAX_TENSORS = 48       # over all stages
MAX_TERMS = 160        # over all tensors
MAX_FACTOR = 65535     # tile factors are stored as u16


@lru_cache(maxsize=None)
def divisors(n: int) -> tuple:
    """Ascending divisors of ``n``."""
    lo, hi = [], []
    d = 1
    while d * d <= n:
        if n % d == 0:
            lo.append(d)
            if d * d != n:
                hi.append(n // d)
        d += 1
    return tuple(lo + hi[::-1])


@lru_cache(maxsize=None)
def enumerate_tilings(extent: int, levels: int) -> int:
    """Number of ordered factorizations (reference schedspace.py:51-59)."""
    if extent < 1 or levels < 1:
        raise ScheduleError("extent and levels must be >= 1")
    if levels == 1:
        return 1
    return sum(enumerate_tilings(extent // d, levels - 1)
               for d in divisors(extent))


@lru_cache(maxsize=None)
def list_tilings(extent: int, levels: int) -> tuple:
    """Ordered factorizations in lexicographic order (schedspace.py:62-71)."""
    if levels == 1:
        return ((extent,),)
    return tuple((d,) + rest for d in divisors(extent)
                 for rest in list_tilings(extent // d, levels - 1))


def smallest_prime_factor(n: int) -> int:
    if n < 2:
        raise ScheduleError(f"no prime factor of {n}")
    if n % 2 == 0:
        return 2
    p = 3
    while p * p <= n:
        if n % p == 0:
            return p
        p += 2
    return n


def space_size(sketch) -> int:
    sp = sketch.space
    total = len(sp.unroll_depths) * (sp.max_fusible + 1) * \
        len(sp.compute_at_candidates)
    for td in sp.tiled_dims:
        total *= enumerate_tilings(td.extent, sp.levels)
    return total


@dataclass(frozen=True)
class ScheduleState:
    """Complete parameter assignment below one sketch (schedspace.py:107)."""

    sketch_id: str
    tiles: tuple
    compute_at_index: int = 0
    parallel_fuse_count: int = 0
    unroll_index: int = 0

    def canonical(self) -> str:
        return canonical_text(self.sketch_id, self.tiles,
                              self.compute_at_index, self.parallel_fuse_count,
                              self.unroll_index)


def canonical_text(sketch_id, tiles, ca, par, ur) -> str:
    """``sk|t=a.b;c.d|ca=..|par=..|ur=..`` (reference schedspace.py:117-120)."""
    t = ";".join(".".join(map(str, dim)) for dim in tiles)
    return f"{sketch_id}|t={t}|ca={ca}|par={par}|ur={ur}"


def fast_dataclass_maker(cls, names):
    """``(*values) -> cls(**dict(zip(names, values)))`` for a frozen
    dataclass whose fields are exactly ``names`` (in order) with plain
    ``__init__`` semantics (no ``__post_init__``, no slots, no converters):
    the instance dict is filled directly, skipping the per-field
    ``object.__setattr__`` of the frozen ``__init__`` (~5x cheaper; equal
    and hash-equal objects).  Any other class gets its constructor."""
    import dataclasses
    ok = (dataclasses.is_dataclass(cls) and
          not hasattr(cls, "__post_init__") and
          "__slots__" not in cls.__dict__ and
          tuple(f.name for f in dataclasses.fields(cls)) == tuple(names) and
          all(f.init for f in dataclasses.fields(cls)))
    if not ok:
        return lambda *v: cls(**dict(zip(names, v)))
    new = object.__new__

    def make(*v):
        o = new(cls)
        o.__dict__.update(zip(names, v))
        return o
    return make


def canonical_texts(sketch_id, tiles, knobs, levels: int) -> list:
    """``canonical_text`` of every row of (tiles [n, slots] u16, knobs
    [n, 3] u8), formatted natively (harl_format_canonical)."""
    import ctypes as C
    from . import _native as N
    t = np.ascontiguousarray(tiles, dtype=np.uint16)
    k = np.ascontiguousarray(knobs, dtype=np.uint8)
    n = len(k)
    if n == 0:
        return []
    t = t.reshape(n, -1)
    pre = sketch_id.encode()
    cap = n * (len(pre) + 6 * t.shape[1] + 64)
    buf = C.create_string_buffer(cap)
    nb = N.load(require_device=False).harl_format_canonical(
        t.ctypes.data, k.ctypes.data, n, t.shape[1], levels, pre, len(pre),
        buf, cap)
    if nb < 0:
        raise ValueError("canonical text buffer too small")
    return buf.raw[:nb].decode().split("\0")[:-1]


@dataclass(frozen=True)
class ModificationAction:
    tile_src: int = -1
    tile_dst: int = -1
    ca_delta: int = 0
    par_delta: int = 0
    unr_delta: int = 0


def decode_action(indices, num_slots: int) -> ModificationAction:
    """Head indices -> modification (reference schedspace.py:196-210)."""
    t, ca, par, ur = (int(i) for i in indices)
    src, dst = (-1, -1) if t == num_slots * num_slots else divmod(t, num_slots)
    return ModificationAction(src, dst, ca - 1, par - 1, ur - 1)


def head_columns(num_slots: int, levels: int) -> np.ndarray:
    """Tiling-head columns that can ever be legal, ascending, no-op last.

    A move ``src*S+dst`` is only ever legal when both slots belong to the
    same tiled dimension (slots ``d*L .. d*L+L-1``) and ``src != dst``
    (reference schedspace.py:241-248); every other column is masked to
    probability zero for every state of every sketch of the subgraph, so the
    policy head can be evaluated on this compact set exactly.
    """
    S, L = num_slots, levels
    cols = [src * S + dst for src in range(S) for dst in range(S)
            if src // L == dst // L and src != dst]
    cols.append(S * S)
    return np.asarray(cols, dtype=np.int32)


def _val(x):
    return getattr(x, "value", x)


class SketchTables:
    """Flattened per-sketch tables for the device kernels.

    Mirrors what ``SketchContext.__init__`` derives (reference
    schedspace.py:324-368): anchor stages with their tensor footprint terms
    ``(global dim, scale, offset)``, ``inter_mult`` / ``extra_out_mult``,
    and ``feature_len = max_feature_dims*L + 2 + len(unroll) + 3``.
    """

    def __init__(self, sg, sketch, target, num_slots: int | None = None):
        from .workloads import tensor_specs as _specs, effective_flops

        sp = sketch.space
        self.sketch_id = sketch.id
        self.levels = L = int(sp.levels)
        self.ndims = len(sp.tiled_dims)
        self.local_slots = self.ndims * L
        self.num_slots = int(num_slots if num_slots is not None
                             else self.local_slots)
        if self.num_slots < self.local_slots:
            raise ScheduleError("agent slot count below sketch slot count")
        self.extents = np.asarray([td.extent for td in sp.tiled_dims],
                                  dtype=np.int64)
        self.ncas = len(sp.compute_at_candidates)
        self.max_fusible = int(sp.max_fusible)
        self.n_unroll = len(sp.unroll_depths)
        self.max_feature_dims = int(target.max_feature_dims)
        self.feature_len = self.max_feature_dims * L + 2 + self.n_unroll + 3
        if self.ndims > MAX_DIMS or L > MAX_LEVELS or \
                self.num_slots > MAX_SLOTS:
            raise ScheduleError("sketch exceeds device table limits")
        if self.ndims > self.max_feature_dims:
            raise ScheduleError("more tiled dims than feature slots")
        if self.extents.size and int(self.extents.max()) > MAX_FACTOR:
            raise ScheduleError(
                f"extent above {MAX_FACTOR} is not supported on device")

        # -- anchor stages and footprint terms -----------------------------
        slot_of = {(td.node, td.dim): i for i, td in enumerate(sp.tiled_dims)}
        b_eff = effective_flops(sg, sketch)
        stages = []
        # simulator data (SketchContext.stages / .skipped, schedspace.py:
        # 337-364): per anchor stage its flops and spatial slots; per
        # non-anchor node (flops, full footprint, full footprint)
        self.sim_spatial = []
        self.sim_skipped = []
        self.unroll_depths = tuple(int(d) for d in sp.unroll_depths)
        for node in sg.nodes:
            st = _val(sketch.structure_of(node.name))
            if st == "inlined":
                continue
            mnode = _mirror_node(node)
            if st == "skipped":
                full = {d: e for d, e in mnode.shape}
                l_full = float(sum(t.elements(full) for t in _specs(mnode)))
                self.sim_skipped.append((float(b_eff[node.name]), l_full,
                                         l_full))
                continue
            self.sim_spatial.append(tuple(slot_of[(node.name, d)]
                                          for d, _ in mnode.shape
                                          if mnode.is_spatial(d)))
            specs = _specs(mnode)
            tensors = [[(slot_of[(node.name, d)], int(sc), int(off))
                        for d, sc, off in t.terms] for t in specs]
            inter = {"tiled": 0, "tiled_fused": 1, "cache_write_tiled": 1,
                     "rfactor_tiled": 2}[st]
            extra = 1 if st == "tiled_fused" else 0
            stages.append((tensors, inter, extra, b_eff[node.name]))
        self.stages = stages
        self.stage_flops = [s[3] for s in stages]

        term_gi, term_sc, term_off = [], [], []
        tens_first, tens_n = [], []
        stage_first, stage_n, stage_inter, stage_extra = [], [], [], []
        for tensors, inter, extra, _ in stages:
            stage_first.append(len(tens_first))
            stage_n.append(len(tensors))
            stage_inter.append(inter)
            stage_extra.append(extra)
            for terms in tensors:
                tens_first.append(len(term_gi))
                tens_n.append(len(terms))
                for gi, sc, off in terms:
                    term_gi.append(gi)
                    term_sc.append(sc)
                    term_off.append(off)
        if len(stages) > MAX_STAGES or len(tens_first) > MAX_TENSORS or \
                len(term_gi) > MAX_TERMS:
            raise ScheduleError("footprint table exceeds device limits")
        i32 = lambda v: np.asarray(v, dtype=np.int32)  # noqa: E731
        self.term_gi, self.term_sc, self.term_off = \
            i32(term_gi), i32(term_sc), i32(term_off)
        self.tensor_first, self.tensor_nterms = i32(tens_first), i32(tens_n)
        self.stage_first, self.stage_ntensors = i32(stage_first), i32(stage_n)
        self.stage_inter, self.stage_extra = i32(stage_inter), i32(stage_extra)
        self._check_footprint_bound()

        # -- scalar features -------------------------------------------------
        # log10(max(flops, 1)) / 12 (reference schedspace.py:437), host libm.
        self.flops = float(sg.flops)
        self.flops_feature = math.log10(max(self.flops, 1.0)) / 12.0

        # -- lookup tables over factor values ------------------------------
        vmax = int(self.extents.max()) if self.ndims else 1
        self.max_extent = vmax
        # log2(f)/10 for every factor value (schedspace.py:425); only
        # divisors of an extent ever occur, the rest are unused filler.
        self.log2_lut = np.zeros(vmax + 1, dtype=np.float64)
        for v in range(1, vmax + 1):
            self.log2_lut[v] = math.log2(v) / 10.0
        spf = np.zeros(vmax + 1, dtype=np.uint16)
        for v in range(2, vmax + 1):
            if spf[v] == 0:
                spf[v::v][spf[v::v] == 0] = v
        self.spf_lut = spf

        # -- enumerated tilings for the initial sampler -------------------
        # schedspace.py:165-178 draws one list_tilings index per dim.
        per_dim = [list_tilings(int(e), L) for e in self.extents]
        self.tiling_counts = np.asarray([len(t) for t in per_dim],
                                        dtype=np.int64)
        self.tiling_offsets = np.zeros(self.ndims, dtype=np.int64)
        if self.ndims:
            self.tiling_offsets[1:] = np.cumsum(self.tiling_counts)[:-1]
        flat = [f for tl in per_dim for t in tl for f in t]
        self.tiling_table = np.asarray(flat, dtype=np.uint16).reshape(-1, L) \
            if flat else np.zeros((0, L), dtype=np.uint16)

        self.head_cols = head_columns(self.num_slots, L)

    def _check_footprint_bound(self):
        """Footprints are exact int64 and exactly representable as fp64."""
        ext = self.extents
        worst = 0
        for tensors, inter, extra, _ in self.stages:
            out = 1
            tot = 0
            for terms in tensors:
                n = 1
                for gi, sc, off in terms:
                    n *= max(1, sc * int(ext[gi]) + off)
                tot += n
                out = n
            worst += tot + (inter + extra) * out
        if worst >= 2 ** 53:
            raise ScheduleError("footprint could exceed 2^53; unsupported")

    # -- host-side helpers used by tests and the engine ---------------------

    def state_arrays(self, states) -> tuple:
        """List of states -> (tiles u16 [B, ndims*L], knobs u8 [B, 3])."""
        B = len(states)
        tiles = np.zeros((B, self.local_slots), dtype=np.uint16)
        knobs = np.zeros((B, 3), dtype=np.uint8)
        for i, s in enumerate(states):
            if self.local_slots:
                tiles[i] = np.asarray(s.tiles, dtype=np.uint16).reshape(-1)
            knobs[i] = (s.compute_at_index, s.parallel_fuse_count,
                        s.unroll_index)
        return tiles, knobs

    def states_from_arrays(self, tiles, knobs, state_cls=ScheduleState,
                           canonical: bool = False):
        """(tiles [B, slots], knobs [B, 3]) -> ``state_cls`` objects (and,
        with ``canonical``, their canonical texts as a second list)."""
        L, sk = self.levels, self.sketch_id
        out = []
        make = fast_dataclass_maker(state_cls, ("sketch_id", "tiles",
                                                "compute_at_index",
                                                "parallel_fuse_count",
                                                "unroll_index"))
        for t, k in zip(np.asarray(tiles).tolist(), np.asarray(knobs).tolist()):
            it = iter(t)
            tl = tuple(zip(*([it] * L))) if L else ()
            out.append(make(sk, tl, k[0], k[1], k[2]))
        if canonical:
            texts = canonical_texts(sk, tiles, knobs, L)
        return (out, texts) if canonical else out

    def arrays_from_canonical(self, texts) -> tuple:
        """Canonical strings of this sketch (``sk|t=a.b;..|ca=|par=|ur=``,
        schedspace.py:117-120) -> (tiles u16 [E, local_slots], knobs u8
        [E, 3]); strings of other sketches are skipped."""
        tiles, knobs = [], []
        for c in texts:
            sk, t, ca, par, ur = c.rsplit("|", 4)
            if sk != self.sketch_id:
                continue
            flat = [int(v) for d in t[2:].split(";") if d
                    for v in d.split(".")]
            if len(flat) != self.local_slots:
                raise ValueError(f"canonical state {c!r} does not match "
                                 f"sketch {self.sketch_id}")
            tiles.append(flat)
            knobs.append((int(ca[3:]), int(par[4:]), int(ur[3:])))
        return (np.asarray(tiles, np.uint16).reshape(len(tiles),
                                                     self.local_slots),
                np.asarray(knobs, np.uint8).reshape(len(knobs), 3))

    def canonical(self, tiles_row, knobs_row) -> str:
        L = self.levels
        tl = [tiles_row[d * L:(d + 1) * L] for d in range(self.ndims)]
        return canonical_text(self.sketch_id, [[int(v) for v in t] for t in tl],
                              int(knobs_row[0]), int(knobs_row[1]),
                              int(knobs_row[2]))


def _mirror_node(node):
    """Adapt a reference ``TensorOpDef`` to this package's ``tensor_specs``."""
    from .workloads import OpKind, TensorOpDef
    if isinstance(node, TensorOpDef):
        return node
    return TensorOpDef(name=node.name, kind=OpKind(_val(node.kind)),
                       shape=tuple(node.shape),
                       has_data_reuse=node.has_data_reuse,
                       is_inlinable=node.is_inlinable,
                       has_reduction=node.has_reduction,
                       consumers=tuple(node.consumers),
                       stride=node.stride, padding=node.padding)
