"""Shared helpers for the GPU parity tests."""

import numpy as np
import pytest

from paper_2211_11172_b200 import workloads as W
from paper_2211_11172_b200.space import SketchTables

torch = pytest.importorskip("torch")

needs_gpu = pytest.mark.skipif(not torch.cuda.is_available(),
                               reason="needs a CUDA device")

# north_star: "policy outputs, cost-model scores and advantages must agree
# within 1e-4 relative in fp32".  Pure relative error is unbounded near 0,
# so the scale is max(|ref|, rms(ref)).
REL_TOL = 1e-4


def assert_close_rel(got, ref, tol=REL_TOL, what=""):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    fin = np.isfinite(ref)
    assert np.array_equal(np.isfinite(got), fin), what
    if not fin.any():
        return
    rms = float(np.sqrt(np.mean(ref[fin] ** 2)))
    scale = np.maximum(np.abs(ref[fin]), rms)
    err = np.abs(got[fin] - ref[fin]) / np.where(scale > 0, scale, 1.0)
    assert err.max() <= tol, f"{what}: max scaled err {err.max():.3e}"


BMM_SOFTMAX = """
name: bert-attention
subgraphs:
  - id: bgemm_softmax
    weight: 12
    nodes:
      - name: bmm
        kind: batch_matmul
        shape: {b: 12, m: 128, k: 64, n: 128}
        consumers: [sm]
      - name: sm
        kind: softmax
        shape: {heads: 12, q: 128, k: 128}
"""

CONV = """
subgraphs:
  - id: c2d_14x256x256_k3
    nodes:
      - name: conv
        kind: conv2d
        shape: {n: 1, h: 14, w: 14, ci: 256, co: 256, kernel: 3, stride: 1, padding: 1}
"""

GEMM = """
subgraphs:
  - id: gemm_%d
    nodes: [{name: mm, kind: matmul, shape: {m: %d, k: %d, n: %d}}]
"""

TCONV = """
subgraphs:
  - id: tc
    nodes:
      - name: tconv
        kind: transposed_conv2d
        shape: {n: 1, h: 8, w: 8, ci: 32, co: 16, kernel: 4, stride: 2, padding: 1}
      - name: relu
        kind: elementwise
        shape: {n: 1, ho: 16, wo: 16, co: 16}
"""

ELEMENTWISE = """
subgraphs:
  - id: ew
    nodes: [{name: ew, kind: elementwise, shape: {t: 128, h: 768}}]
"""


def all_sketch_tables(yaml_text, target=None):
    """[(sg, sketch, tables)] for every sketch of every subgraph, with the
    agent-wide slot count of its subgraph."""
    target = target or W.TargetConfig()
    net = W.loads_network(yaml_text)
    out = []
    for sg in net.subgraphs:
        ks = W.generate_sketches(sg, target)
        S = max(k.space.num_tile_slots for k in ks)
        for k in ks:
            out.append((sg, k, SketchTables(sg, k, target, S)))
    return out


def config_tables():
    """Sketch tables for every benchmark config shape plus edge shapes."""
    cases = []
    cases += all_sketch_tables(GEMM % (1024, 1024, 1024, 1024))
    cases += all_sketch_tables(GEMM % (4096, 4096, 4096, 4096))
    cases += all_sketch_tables(CONV)
    cases += all_sketch_tables(BMM_SOFTMAX)
    cases += all_sketch_tables(GEMM % (64, 64, 64, 64),
                               W.TargetConfig(tiling_levels=2))
    cases += all_sketch_tables(GEMM % (1024, 1024, 1024, 1024), W.gpu_target())
    cases += all_sketch_tables(TCONV, W.TargetConfig(tiling_levels=3))
    cases += all_sketch_tables(ELEMENTWISE)
    return cases


def conv_tables():
    """Sketch k0 of the conv2d config (C2)."""
    return all_sketch_tables(CONV)[0][2]
