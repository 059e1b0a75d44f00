"""Workload descriptions and loop-structure sketches (host side).

This module is the host-side mirror of the reference's workload layer
(``pkg/src/schedtune/workload.py``).  It exists so that the B200 episode
engine can run standalone (on the GPU box the reference package is not
installed): it parses the same YAML schema, derives the same iteration
spaces, flop counts, footprint terms and sketch list, and exposes objects
whose attribute names match the reference's (``sg.nodes``, ``sketch.space
.tiled_dims`` ...), so the engine accepts either the reference's objects or
these ones.

Semantics followed (reference file:line, relative to ``pkg/src/schedtune``):

* operator defaults / reduction axes ............ workload.py:35-66
* flop counts ................................... workload.py:152-165
* footprint terms per tensor .................... workload.py:168-212
* YAML loading + validation ..................... workload.py:263-419
* sketch enumeration ............................ workload.py:484-575
* inline absorption / effective flops ........... workload.py:578-621

None of this is on the per-step hot path; it runs once per session.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass
from typing import Iterable

import yaml

from .errors import WorkloadError


class OpKind(str, enum.Enum):
    MATMUL = "matmul"
    BATCH_MATMUL = "batch_matmul"
    CONV1D = "conv1d"
    CONV2D = "conv2d"
    CONV3D = "conv3d"
    TRANSPOSED_CONV2D = "transposed_conv2d"
    ELEMENTWISE = "elementwise"
    SOFTMAX = "softmax"
    REDUCTION = "reduction"


class Structure(str, enum.Enum):
    TILED = "tiled"
    TILED_FUSED = "tiled_fused"
    CACHE_WRITE_TILED = "cache_write_tiled"
    RFACTOR_TILED = "rfactor_tiled"
    INLINED = "inlined"
    SKIPPED = "skipped"


ANCHOR_STRUCTURES = (Structure.TILED, Structure.TILED_FUSED,
                     Structure.CACHE_WRITE_TILED, Structure.RFACTOR_TILED)

# Removable intermediate buffer size (in output tiles) and the extra
# non-removable output-shaped buffer, per anchor structure
# (reference schedspace.py:357-360).
INTERMEDIATE_MULT = {Structure.TILED: 0, Structure.TILED_FUSED: 1,
                     Structure.CACHE_WRITE_TILED: 1,
                     Structure.RFACTOR_TILED: 2}
EXTRA_OUT_MULT = {Structure.TILED: 0, Structure.TILED_FUSED: 1,
                  Structure.CACHE_WRITE_TILED: 0,
                  Structure.RFACTOR_TILED: 0}

_MAC = frozenset({OpKind.MATMUL, OpKind.BATCH_MATMUL, OpKind.CONV1D,
                  OpKind.CONV2D, OpKind.CONV3D, OpKind.TRANSPOSED_CONV2D})

# kind -> (has_data_reuse, is_inlinable, has_reduction) defaults
_DEFAULT_FLAGS = {k: (True, False, True) for k in _MAC}
_DEFAULT_FLAGS.update({OpKind.ELEMENTWISE: (False, True, False),
                       OpKind.SOFTMAX: (False, False, True),
                       OpKind.REDUCTION: (False, False, True)})

_REDUCTION_AXES = {
    OpKind.MATMUL: ("k",), OpKind.BATCH_MATMUL: ("k",),
    OpKind.CONV1D: ("ci", "kw"), OpKind.CONV2D: ("ci", "kh", "kw"),
    OpKind.CONV3D: ("ci", "kd", "kh", "kw"),
    OpKind.TRANSPOSED_CONV2D: ("ci", "kh", "kw"),
}


@dataclass(frozen=True)
class TargetConfig:
    """Target knobs shaping the schedule space (reference workload.py:69-91)."""

    name: str = "cpu"
    tiling_levels: int = 4
    unroll_depths: tuple = (0, 16, 64, 512)
    parallel_fuse_cap: int = 3
    max_feature_dims: int = 10

    def __post_init__(self):
        if self.tiling_levels < 1:
            raise WorkloadError("tiling_levels must be >= 1")
        if not self.unroll_depths:
            raise WorkloadError("unroll_depths must be non-empty")


def gpu_target(tiling_levels: int = 4) -> TargetConfig:
    return TargetConfig(name="gpu", tiling_levels=tiling_levels,
                        unroll_depths=(0, 16, 64, 512, 1024))


@dataclass(frozen=True)
class TensorSpec:
    """Tensor footprint as affine terms ``(dim, scale, offset)`` per axis."""

    name: str
    terms: tuple

    def elements(self, tile: dict) -> int:
        n = 1
        for dim, scale, off in self.terms:
            n *= scale * tile[dim] + off
        return n


@dataclass(frozen=True)
class TensorOpDef:
    name: str
    kind: OpKind
    shape: tuple            # ((dim, extent), ...) in loop order
    has_data_reuse: bool
    is_inlinable: bool
    has_reduction: bool
    consumers: tuple = ()
    stride: int = 1
    padding: int = 0

    @property
    def extents(self):
        return tuple(e for _, e in self.shape)

    @property
    def dim_names(self):
        return tuple(d for d, _ in self.shape)

    def reduce_dims(self):
        if self.kind in _REDUCTION_AXES:
            return _REDUCTION_AXES[self.kind]
        if self.kind in (OpKind.SOFTMAX, OpKind.REDUCTION):
            return self.dim_names[-1:]
        return ()

    def is_spatial(self, dim: str) -> bool:
        return dim not in self.reduce_dims()


@dataclass(frozen=True)
class SubgraphSpec:
    id: str
    weight: int
    nodes: tuple
    flops: float = 0.0
    similarity_key: str = ""

    def node(self, name: str) -> TensorOpDef:
        for n in self.nodes:
            if n.name == name:
                return n
        raise KeyError(name)


@dataclass(frozen=True)
class NetworkSpec:
    name: str
    subgraphs: tuple

    def subgraph(self, sg_id: str) -> SubgraphSpec:
        for sg in self.subgraphs:
            if sg.id == sg_id:
                return sg
        raise KeyError(sg_id)

    @property
    def total_flops(self) -> float:
        return sum(sg.weight * sg.flops for sg in self.subgraphs)


@dataclass(frozen=True)
class TiledDim:
    node: str
    dim: str
    extent: int
    is_spatial: bool


@dataclass(frozen=True)
class SpaceDescriptor:
    tiled_dims: tuple
    levels: int
    compute_at_candidates: tuple
    max_fusible: int
    unroll_depths: tuple

    @property
    def num_tile_slots(self) -> int:
        return self.levels * len(self.tiled_dims)


@dataclass(frozen=True)
class Sketch:
    id: str
    subgraph_id: str
    structures: tuple
    space: SpaceDescriptor
    absorbed_by: tuple = ()

    def structure_of(self, node: str) -> Structure:
        for name, st in self.structures:
            if name == node:
                return st
        raise KeyError(node)


# ---------------------------------------------------------------------------
# flops and footprint terms


def _product(values: Iterable[int]) -> int:
    out = 1
    for v in values:
        out *= v
    return out


def _kind(node) -> OpKind:
    return OpKind(getattr(node.kind, "value", node.kind))


def flop_count(node) -> float:
    """Flops of one operator execution (reference workload.py:152-165)."""
    points = _product(e for _, e in node.shape)
    kind = _kind(node)
    if kind in _MAC:
        f = 2.0 * points
        if kind is OpKind.TRANSPOSED_CONV2D:
            f /= float(node.stride * node.stride)
        return f
    if kind is OpKind.SOFTMAX:
        return 4.0 * points
    return float(points)


def _plain(name: str, dims) -> TensorSpec:
    return TensorSpec(name, tuple((d, 1, 0) for d in dims))


def _window(dim: str, stride: int, kernel: int):
    return (dim, stride, kernel - stride)


def tensor_specs(node: TensorOpDef) -> tuple:
    """Inputs then output, in footprint-term form (workload.py:168-212)."""
    k, s = node.kind, node.stride
    ext = dict(node.shape)
    if k is OpKind.MATMUL:
        return (_plain("a", "mk"), _plain("b", "kn"), _plain("out", "mn"))
    if k is OpKind.BATCH_MATMUL:
        return (_plain("a", "bmk"), _plain("b", "bkn"), _plain("out", "bmn"))
    if k is OpKind.CONV1D:
        inp = TensorSpec("in", (("n", 1, 0), _window("lo", s, ext["kw"]),
                                ("ci", 1, 0)))
        return (inp, _plain("w", ("kw", "ci", "co")),
                _plain("out", ("n", "lo", "co")))
    if k is OpKind.CONV2D:
        inp = TensorSpec("in", (("n", 1, 0), _window("ho", s, ext["kh"]),
                                _window("wo", s, ext["kw"]), ("ci", 1, 0)))
        return (inp, _plain("w", ("kh", "kw", "ci", "co")),
                _plain("out", ("n", "ho", "wo", "co")))
    if k is OpKind.CONV3D:
        inp = TensorSpec("in", (("n", 1, 0), _window("do", s, ext["kd"]),
                                _window("ho", s, ext["kh"]),
                                _window("wo", s, ext["kw"]), ("ci", 1, 0)))
        return (inp, _plain("w", ("kd", "kh", "kw", "ci", "co")),
                _plain("out", ("n", "do", "ho", "wo", "co")))
    if k is OpKind.TRANSPOSED_CONV2D:
        inp = TensorSpec("in", (("n", 1, 0), ("ho", 1, ext["kh"]),
                                ("wo", 1, ext["kw"]), ("ci", 1, 0)))
        return (inp, _plain("w", ("kh", "kw", "ci", "co")),
                _plain("out", ("n", "ho", "wo", "co")))
    dims = node.dim_names
    if k is OpKind.REDUCTION:
        return (_plain("in", dims), _plain("out", dims[:-1]))
    return (_plain("in", dims), _plain("out", dims))


# ---------------------------------------------------------------------------
# YAML loading


def _conv_extent(n: int, kernel: int, stride: int, pad: int) -> int:
    return (n + 2 * pad - kernel) // stride + 1


def _iteration_space(kind: OpKind, raw: dict, where: str):
    stride = int(raw.get("stride", 1))
    pad = int(raw.get("padding", 0))
    kern = int(raw.get("kernel", 1))
    if stride < 1:
        raise WorkloadError(f"{where}: stride must be >= 1")
    if pad < 0:
        raise WorkloadError(f"{where}: padding must be >= 0")

    def fields(*names):
        missing = [n for n in names if n not in raw]
        if missing:
            raise WorkloadError(f"{where}: missing shape field '{missing[0]}'")
        return [int(raw[n]) for n in names]

    if kind is OpKind.MATMUL:
        m, k, n = fields("m", "k", "n")
        dims = [("m", m), ("k", k), ("n", n)]
    elif kind is OpKind.BATCH_MATMUL:
        b, m, k, n = fields("b", "m", "k", "n")
        dims = [("b", b), ("m", m), ("k", k), ("n", n)]
    elif kind is OpKind.CONV1D:
        n, length, ci, co = fields("n", "l", "ci", "co")
        dims = [("n", n), ("lo", _conv_extent(length, kern, stride, pad)),
                ("co", co), ("ci", ci), ("kw", kern)]
    elif kind in (OpKind.CONV2D, OpKind.TRANSPOSED_CONV2D):
        n, h, w, ci, co = fields("n", "h", "w", "ci", "co")
        if kind is OpKind.CONV2D:
            ho = _conv_extent(h, kern, stride, pad)
            wo = _conv_extent(w, kern, stride, pad)
        else:
            ho = (h - 1) * stride - 2 * pad + kern
            wo = (w - 1) * stride - 2 * pad + kern
        dims = [("n", n), ("ho", ho), ("wo", wo), ("co", co), ("ci", ci),
                ("kh", kern), ("kw", kern)]
    elif kind is OpKind.CONV3D:
        n, d, h, w, ci, co = fields("n", "d", "h", "w", "ci", "co")
        dims = [("n", n), ("do", _conv_extent(d, kern, stride, pad)),
                ("ho", _conv_extent(h, kern, stride, pad)),
                ("wo", _conv_extent(w, kern, stride, pad)), ("co", co),
                ("ci", ci), ("kd", kern), ("kh", kern), ("kw", kern)]
    else:
        dims = [(str(key), int(val)) for key, val in raw.items()
                if key not in ("stride", "padding", "kernel")]
        if not dims:
            raise WorkloadError(f"{where}: shape has no dimensions")
    for dname, ext in dims:
        if ext < 1:
            raise WorkloadError(
                f"{where}: extent '{dname}' must be >= 1, got {ext}")
    return tuple(dims), stride, pad


def _parse_node(raw, where: str) -> TensorOpDef:
    if not isinstance(raw, dict):
        raise WorkloadError(f"{where}: node entry must be a mapping")
    name = raw.get("name")
    if not name:
        raise WorkloadError(f"{where}: node missing 'name'")
    where = f"{where} node '{name}'"
    try:
        kind = OpKind(raw.get("kind", ""))
    except ValueError:
        raise WorkloadError(
            f"{where}: unknown kind {raw.get('kind')!r}") from None
    shape_raw = raw.get("shape")
    if not isinstance(shape_raw, dict):
        raise WorkloadError(f"{where}: 'shape' must be a mapping")
    shape, stride, pad = _iteration_space(kind, shape_raw, where)
    d_reuse, d_inl, d_red = _DEFAULT_FLAGS[kind]
    reuse = bool(raw.get("has_data_reuse", d_reuse))
    inl = bool(raw.get("is_inlinable", d_inl))
    red = bool(raw.get("has_reduction", d_red))
    if kind is OpKind.ELEMENTWISE and not inl:
        raise WorkloadError(f"{where}: elementwise operators must be inlinable")
    if kind in _MAC and not (reuse and red):
        raise WorkloadError(
            f"{where}: multiply-accumulate kinds need data reuse and reduction")
    return TensorOpDef(name=str(name), kind=kind, shape=shape,
                       has_data_reuse=reuse, is_inlinable=inl,
                       has_reduction=red,
                       consumers=tuple(str(c) for c in raw.get("consumers", [])),
                       stride=stride, padding=pad)


def _parse_subgraph(raw, where: str) -> SubgraphSpec:
    if not isinstance(raw, dict):
        raise WorkloadError(f"{where}: subgraph entry must be a mapping")
    sg_id = raw.get("id")
    if not sg_id:
        raise WorkloadError(f"{where}: subgraph missing 'id'")
    where = f"subgraph '{sg_id}'"
    weight = int(raw.get("weight", 1))
    if weight < 1:
        raise WorkloadError(f"{where}: weight must be >= 1")
    raw_nodes = raw.get("nodes")
    if not raw_nodes:
        raise WorkloadError(f"{where}: needs at least one node")
    nodes = tuple(_parse_node(n, where) for n in raw_nodes)
    position = {}
    for i, n in enumerate(nodes):
        if n.name in position:
            raise WorkloadError(f"{where}: duplicate node names")
        position[n.name] = i
    for n in nodes:
        for c in n.consumers:
            if c not in position:
                raise WorkloadError(
                    f"{where}: node '{n.name}' lists unknown consumer '{c}'")
            if position[c] <= position[n.name]:
                raise WorkloadError(
                    f"{where}: consumer '{c}' must come after '{n.name}'")
    flops = sum(flop_count(n) for n in nodes)
    if flops <= 0:
        raise WorkloadError(f"{where}: total flop count must be positive")
    return SubgraphSpec(id=str(sg_id), weight=weight, nodes=nodes,
                        flops=flops,
                        similarity_key="|".join(sorted(n.kind.value
                                                       for n in nodes)))


def parse_network(raw) -> NetworkSpec:
    if not isinstance(raw, dict):
        raise WorkloadError("workload file must contain a mapping at top level")
    sgs = raw.get("subgraphs")
    if not sgs:
        raise WorkloadError("workload must define a non-empty 'subgraphs' list")
    subgraphs = tuple(_parse_subgraph(s, f"subgraphs[{i}]")
                      for i, s in enumerate(sgs))
    if len({sg.id for sg in subgraphs}) != len(subgraphs):
        raise WorkloadError("duplicate subgraph ids")
    return NetworkSpec(name=str(raw.get("name", "network")),
                       subgraphs=subgraphs)


def load_network(path: str) -> NetworkSpec:
    """Parse and validate a workload YAML file (reference workload.py:399)."""
    try:
        with open(path, "r", encoding="utf-8") as fh:
            raw = yaml.safe_load(fh)
    except OSError as exc:
        raise WorkloadError(f"cannot read workload file: {exc}") from exc
    except yaml.YAMLError as exc:
        raise WorkloadError(f"workload parse error: {exc}") from exc
    return parse_network(raw)


def loads_network(text: str) -> NetworkSpec:
    try:
        raw = yaml.safe_load(text)
    except yaml.YAMLError as exc:
        raise WorkloadError(f"workload parse error: {exc}") from exc
    return parse_network(raw)


# ---------------------------------------------------------------------------
# sketches


def _structure_choices(node: TensorOpDef, consumer, decided: dict):
    """Applicable structures in rule order (reference workload.py:484-509)."""
    if node.is_inlinable and consumer is not None:
        return [Structure.INLINED]
    if not node.has_data_reuse:
        return [Structure.SKIPPED] + ([Structure.RFACTOR_TILED]
                                      if node.has_reduction else [])
    out = [Structure.TILED]
    if consumer is not None and decided.get(consumer) in (Structure.SKIPPED,
                                                          Structure.INLINED):
        out.append(Structure.TILED_FUSED)
    if consumer is None:
        out.append(Structure.CACHE_WRITE_TILED)
    if node.has_reduction:
        out.append(Structure.RFACTOR_TILED)
    return out


def _absorption(sg: SubgraphSpec, decided: dict):
    fused_into = {n.consumers[0]: n.name for n in sg.nodes
                  if decided[n.name] is Structure.TILED_FUSED and n.consumers}
    out = []
    for node in sg.nodes:
        if decided[node.name] is not Structure.INLINED:
            continue
        cur, hops = node.name, 0
        while hops <= len(sg.nodes) and decided.get(cur) is Structure.INLINED:
            if cur in fused_into:
                cur = fused_into[cur]
                break
            nxt = sg.node(cur).consumers
            if not nxt:
                break
            cur, hops = nxt[0], hops + 1
        out.append((node.name, cur))
    return out


def generate_sketches(sg: SubgraphSpec, target: TargetConfig) -> list:
    """Deterministic duplicate-free sketch list (workload.py:512-575)."""
    partial = [{}]
    for node in reversed(sg.nodes):
        consumer = node.consumers[0] if node.consumers else None
        grown = []
        for decided in partial:
            for st in _structure_choices(node, consumer, decided):
                d = dict(decided)
                d[node.name] = st
                if st is Structure.TILED_FUSED:
                    d[consumer] = Structure.INLINED
                grown.append(d)
        partial = grown

    levels = target.tiling_levels
    sketches, seen = [], set()
    for decided in partial:
        key = tuple((n.name, decided[n.name]) for n in sg.nodes)
        if key in seen:
            continue
        seen.add(key)
        anchors = [n for n in sg.nodes if decided[n.name] in ANCHOR_STRUCTURES]
        tiled = tuple(TiledDim(node=n.name, dim=d, extent=e,
                               is_spatial=n.is_spatial(d))
                      for n in anchors for d, e in n.shape)
        if len(tiled) > target.max_feature_dims:
            raise WorkloadError(
                f"subgraph '{sg.id}' tiles {len(tiled)} dimensions, above the "
                f"feature budget of {target.max_feature_dims}")
        with_inter = any(decided[n.name] in (Structure.TILED_FUSED,
                                             Structure.CACHE_WRITE_TILED,
                                             Structure.RFACTOR_TILED)
                         for n in anchors)
        ca = (("root", 0),)
        if with_inter and anchors:
            ca = ca + ((anchors[0].name, levels - 1),)
        spatial = any(t.is_spatial for t in tiled)
        space = SpaceDescriptor(
            tiled_dims=tiled, levels=levels, compute_at_candidates=ca,
            max_fusible=min(levels, target.parallel_fuse_cap) if spatial else 0,
            unroll_depths=tuple(target.unroll_depths))
        sketches.append(Sketch(id=f"{sg.id}::k{len(sketches)}",
                               subgraph_id=sg.id, structures=key, space=space,
                               absorbed_by=tuple(_absorption(sg, decided))))
    return sketches


def effective_flops(sg: SubgraphSpec, sketch) -> dict:
    """Per-stage flops with inlined nodes folded in (workload.py:604-621)."""
    out = {}
    for n in sg.nodes:
        st = sketch.structure_of(n.name)
        if getattr(st, "value", st) != Structure.INLINED.value:
            out[n.name] = flop_count(n)
    for name, host in dict(sketch.absorbed_by).items():
        extra = flop_count(sg.node(name))
        target_stage = host if host in out else next(iter(out))
        out[target_stage] += extra
    return out
