// K6: GBT cost-model inference + reward (costmodel.py:67-78,219-237,
// tuner.py:389-391).  fp64 and bit-exact: the walk is a chain of exact
// comparisons, each tree's leaf contribution is the host-computed product
// learning_rate*leaf_value, and the contributions are added to the base in
// tree order with explicit round-to-nearest adds -- exactly the
// reference's ``pred = pred + lr * tree.predict(X)`` loop.
//
// Parallelism is (row x tree-group): G threads share a row, each walks
// every G-th tree and parks its leaf contributions in shared memory; one
// thread per row then sums them in tree order.  Nodes are 16-byte records
// read through the read-only/L1 path (the whole forest, ~100-150 KB, stays
// L1/L2-resident), so many CTAs fit per SM to hide the dependent-load
// latency of the walk.
#pragma once

#include "common.cuh"
#include "tc_common.cuh"

namespace harl {

// device-side forest scalars (harl_forest_desc.dev_hdr)
struct GbtHdr {
  int32_t n_trees, fitted;
  double base, floor_value;
  int64_t n_nodes;
  int32_t max_depth;        // internal levels of the deepest tree
  int32_t perfect_depth;    // > 0: the perfect-tree image below is valid
  const uint8_t* perfect;   // perfect-tree image (device)
  int64_t perfect_bytes;    // its size (multiple of 16)
};

// Perfect-tree image of a forest of depth D <= GBT_PERFECT_MAX: every tree
// padded to a complete binary tree of D levels, breadth-first (children of
// slot i at 2i+1, 2i+2), so a walk needs no child links: thresholds
// f64 [T][2^D-1] | leaf lr*values f64 [T][2^D] | features i16 [T][2^D-1].
// A leaf above level D becomes pass-through slots (feature 0, threshold
// +inf) whose whole subtree repeats its value, so every route through
// them -- a NaN feature goes right, as in the reference's walk -- ends on
// the same leaf value.
constexpr int GBT_PERFECT_MAX = 7;
__host__ __device__ inline size_t gbt_perfect_off_leaf(int T, int D) {
  return ((size_t)T * ((1 << D) - 1) * 8 + 15) & ~(size_t)15;
}
__host__ __device__ inline size_t gbt_perfect_off_feat(int T, int D) {
  return gbt_perfect_off_leaf(T, D) + (size_t)T * (1 << D) * 8;
}
__host__ __device__ inline size_t gbt_perfect_bytes(int T, int D) {
  return (gbt_perfect_off_feat(T, D) + (size_t)T * ((1 << D) - 1) * 2 + 15) &
         ~(size_t)15;
}

struct __align__(16) GbtNode {
  double v;        // split threshold (internal) / lr*value (leaf)
  int16_t feat;    // -1 for a leaf
  int16_t left, right, pad;
};

constexpr int GBT_GROUPS = 8;      // threads per row
constexpr int GBT_THREADS = 256;   // 32 rows per CTA

__global__ void __launch_bounds__(GBT_THREADS)
k_gbt_predict(const GbtNode* __restrict__ nodes,
              const int32_t* __restrict__ tree_first, int32_t n_trees,
              int32_t fitted, double base, double floor_value,
              const double* __restrict__ feat, int64_t n, int32_t F,
              double* score, const double* old_score, double* reward,
              int32_t rows_per_cta, const GbtHdr* hdr) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  extern __shared__ double contrib[];  // [rows_per_cta][n_trees]
  if (hdr) {
    n_trees = hdr->n_trees;
    fitted = hdr->fitted;
    base = hdr->base;
    floor_value = hdr->floor_value;
  }
  const int g = threadIdx.x % GBT_GROUPS;
  const int rl = threadIdx.x / GBT_GROUPS;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r = r0 + rl;
  if (fitted && rl < rows_per_cta && r < n) {
    const double* x = feat + r * F;
    for (int t = g; t < n_trees; t += GBT_GROUPS) {
      const GbtNode* tree = nodes + tree_first[t];
      GbtNode nd = tree[0];
      // same 64-step cap as the reference's walk (trees are checked to be
      // shallower on the host)
      while (nd.feat >= 0) nd = tree[(__ldg(x + nd.feat) <= nd.v) ? nd.left : nd.right];
      contrib[rl * n_trees + t] = nd.v;
    }
  }
  __syncthreads();
  if (g != 0 || rl >= rows_per_cta || r >= n) return;
  double pred = 1.0;
  if (fitted) {
    pred = base;
    const double* c = contrib + rl * n_trees;
    for (int t = 0; t < n_trees; ++t) pred = __dadd_rn(pred, c[t]);
  }
  // np.maximum(pred, floor): NaN propagates
  const double s = (pred != pred) ? pred : (pred < floor_value ? floor_value : pred);
  score[r] = s;
  if (old_score) {
    const double o = old_score[r];
    reward[r] = __ddiv_rn(__dsub_rn(s, o), o);
  }
}

// Persistent variant: each CTA bulk-copies the forest (nodes and tree
// offsets) into shared memory once, then loops over 64-row tiles whose
// feature rows arrive by bulk copy too, double-buffered so the next tile's
// rows land while the current one is walked; every level of every walk is
// then two shared-memory loads.  SMEM_NODES=false keeps the nodes in global
// memory for forests too large to stage.
#ifndef HARL_GBT_GROUPS
#define HARL_GBT_GROUPS 8
#endif
// tree groups per tile (a warp pair walks every GROUPS-th tree for the
// tile's 64 rows); 16 groups (1024 threads) measured slower: the 64-register
// cap spills the fused finish epilogue (C2 20.5 -> 24.2 us)
constexpr int GBT2_GROUPS = HARL_GBT_GROUPS;

// one node record as a single 16-byte shared-memory load (the compiler
// otherwise splits it into four loads), and a shared-memory fp64 load
// through an explicit state space (the feature tile pointer is chosen at
// run time between two buffers, which demoted its loads to generic ones)
__device__ __forceinline__ void lds_node(uint32_t addr, double& v, int& feat,
                                         int& left, int& right) {
  uint32_t a, b, c, d;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(addr));
  v = __hiloint2double((int)b, (int)a);
  feat = (int)(int16_t)(c & 0xffffu);
  left = (int)(int16_t)(c >> 16);
  right = (int)(int16_t)(d & 0xffffu);
}
__device__ __forceinline__ int lds_s16(uint32_t addr) {
  short v;
  asm volatile("ld.shared.s16 %0, [%1];" : "=h"(v) : "r"(addr));
  return (int)v;
}
__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
#ifndef HARL_GBT_ILP
#define HARL_GBT_ILP 4
#endif
constexpr int GBT_ILP = HARL_GBT_ILP;    // trees walked side by side
constexpr int GBT_WALK_MAX_DEPTH = 24;   // fixed-depth walk up to this depth
constexpr int GBT2_ROWS = 64;
constexpr int GBT2_THREADS = GBT2_ROWS * GBT2_GROUPS;

__host__ __device__ inline size_t gbt2_align(size_t x) { return (x + 15) & ~(size_t)15; }

__host__ __device__ inline size_t gbt2_node_region(int64_t n_nodes, int T) {
  const size_t rec = gbt2_align((size_t)n_nodes * 16);
  const size_t per = gbt_perfect_bytes(T, GBT_PERFECT_MAX);
  return rec > per ? rec : per;
}
__host__ __device__ inline size_t gbt2_smem_bytes(bool smem_nodes, int64_t n_nodes,
                                                  int T, int F) {
  return (smem_nodes ? gbt2_node_region(n_nodes, T) : 0) +
         gbt2_align((size_t)T * 4) + 2 * gbt2_align((size_t)GBT2_ROWS * F * 8) +
         (size_t)GBT2_ROWS * T * 8;
}

struct GbtNoEpilogue {
  __device__ void operator()(int64_t, int, int, int) const {}
};

// epi(r0, rows, group, local row) runs after each tile's scores and rewards
// are in global memory (visible to the whole CTA)
template <bool SMEM_NODES, typename Epi>
__device__ __forceinline__ void gbt2_body(
    const GbtNode* __restrict__ gnodes, const int32_t* __restrict__ tree_first,
    int32_t n_trees, int64_t n_nodes, int32_t fitted, double base,
    double floor_value, const double* __restrict__ feat, int64_t n, int32_t F,
    double* score, const double* old_score, double* reward, const GbtHdr* hdr,
    int32_t t_cap, const Epi& epi) {
  dbg_ts(24);
  extern __shared__ __align__(16) unsigned char gsm[];
  __shared__ uint64_t fbar, xbar[2];
  int max_depth = 1 << 30;   // unknown: the while-loop walk
  int pdepth = 0;
  const uint8_t* perfect = nullptr;
  int64_t perfect_bytes = 0;
  if (hdr) {   // reloadable forest: the scalars live on the device
    n_trees = hdr->n_trees;
    fitted = hdr->fitted;
    base = hdr->base;
    floor_value = hdr->floor_value;
    n_nodes = hdr->n_nodes;
    max_depth = hdr->max_depth;
    pdepth = hdr->perfect_depth;
    perfect = hdr->perfect;
    perfect_bytes = hdr->perfect_bytes;
  }
  if (!SMEM_NODES || pdepth > GBT_PERFECT_MAX) pdepth = 0;
  size_t off = 0;
  const GbtNode* nodes = gnodes;
  GbtNode* sn = (GbtNode*)gsm;
  if (SMEM_NODES) {
    nodes = sn;
    // the node region is sized for either layout (t_cap: capacity in trees)
    off = gbt2_node_region(n_nodes, t_cap > n_trees ? t_cap : n_trees);
  }
  int32_t* s_first = (int32_t*)(gsm + off);
  off += gbt2_align((size_t)(n_trees > t_cap ? n_trees : t_cap) * 4);
  double* const xsb0 = (double*)(gsm + off);
  off += gbt2_align((size_t)GBT2_ROWS * F * 8);
  double* const xsb1 = (double*)(gsm + off);
  off += gbt2_align((size_t)GBT2_ROWS * F * 8);
  double* contrib = (double*)(gsm + off);
  const int64_t n_tiles = (n + GBT2_ROWS - 1) / GBT2_ROWS;
  // the forest (written by host copies only) streams in before the PDL wait
  if (threadIdx.x == 0) {
    tc::mbar_init(&fbar, 1);
    tc::mbar_init(&xbar[0], 1);
    tc::mbar_init(&xbar[1], 1);
    if (SMEM_NODES && pdepth > 0 && perfect_bytes > 0)
      tc::bulk_load(sn, perfect, (uint32_t)perfect_bytes, &fbar);
    else if (SMEM_NODES && n_nodes > 0) tc::bulk_load(sn, gnodes, (uint32_t)n_nodes * 16, &fbar);
    else asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(&fbar)) : "memory");
  }
  griddep_wait();  // PDL: the feature rows come from the predecessor
  if (threadIdx.x == 0) {
    if (blockIdx.x < n_tiles) {
      const int64_t r0 = (int64_t)blockIdx.x * GBT2_ROWS;
      tc::bulk_f64(xsb0, feat + r0 * F,
                   (uint32_t)(min((int64_t)GBT2_ROWS, n - r0) * F), &xbar[0]);
    }
  }
  for (int t = threadIdx.x; t < n_trees; t += blockDim.x) s_first[t] = tree_first[t];
  // a warp = 32 rows on the same tree group: node reads of a level are
  // mostly broadcasts and the 32 feature reads hit distinct bank pairs
  const int warp = threadIdx.x >> 5;
  const int g = warp / (GBT2_ROWS / 32);
  const int rl = (warp % (GBT2_ROWS / 32)) * 32 + (threadIdx.x & 31);
  __syncthreads();
  tc::mbar_wait(&fbar, 0);
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
    const int64_t r0 = tile * GBT2_ROWS;
    const int rows = (int)(n - r0 < GBT2_ROWS ? n - r0 : GBT2_ROWS);
    const int64_t r = r0 + rl;
    double o = 0.0;
    if (old_score && g == 0 && rl < rows) o = old_score[r];
    const int b = it & 1;
    tc::mbar_wait(&xbar[b], (it >> 1) & 1);
    if (threadIdx.x == 0) {
      const int64_t nt = tile + gridDim.x;
      if (nt < n_tiles) {   // the other buffer was released at the end of it-1
        const int64_t n0 = nt * GBT2_ROWS;
        tc::bulk_f64(b ? xsb0 : xsb1, feat + n0 * F,
                     (uint32_t)(min((int64_t)GBT2_ROWS, n - n0) * F), &xbar[b ^ 1]);
      }
    }
    if (it < 2) dbg_ts(25 + 3 * it);
    const double* xs = b ? xsb1 : xsb0;
    if (fitted && rl < rows) {
      const double* x = xs + rl * F;
      if (pdepth > 0) {
        // perfect-tree walk: slot 2i+1+(x > thr), no child links to load;
        // GBT_ILP trees side by side
        const int D = pdepth, NI = (1 << D) - 1, NLF = 1 << D;
        const uint32_t s_thr = tc::smem_u32(sn);
        const uint32_t s_leaf = s_thr + (uint32_t)gbt_perfect_off_leaf(n_trees, D);
        const uint32_t s_feat = s_thr + (uint32_t)gbt_perfect_off_feat(n_trees, D);
        const uint32_t s_x = tc::smem_u32(x);
        for (int t0 = g; t0 < n_trees; t0 += GBT_ILP * GBT2_GROUPS) {
          uint32_t tbase[GBT_ILP], idx[GBT_ILP];
#pragma unroll
          for (int k = 0; k < GBT_ILP; ++k) {
            const int t = t0 + k * GBT2_GROUPS;
            tbase[k] = (uint32_t)((t < n_trees ? t : t0) * NI);
            idx[k] = 0;
          }
          for (int lv = 0; lv < D; ++lv) {
            int f[GBT_ILP];
            double th[GBT_ILP], xv[GBT_ILP];
#pragma unroll
            for (int k = 0; k < GBT_ILP; ++k) {
              f[k] = lds_s16(s_feat + 2u * (tbase[k] + idx[k]));
              th[k] = lds_f64(s_thr + 8u * (tbase[k] + idx[k]));
            }
#pragma unroll
            for (int k = 0; k < GBT_ILP; ++k) xv[k] = lds_f64(s_x + 8u * (uint32_t)f[k]);
#pragma unroll
            for (int k = 0; k < GBT_ILP; ++k)
              idx[k] = 2u * idx[k] + (xv[k] <= th[k] ? 1u : 2u);
          }
#pragma unroll
          for (int k = 0; k < GBT_ILP; ++k) {
            const int t = t0 + k * GBT2_GROUPS;
            const double lv = lds_f64(s_leaf + 8u * ((uint32_t)t * NLF + idx[k] - (uint32_t)NI));
            if (t < n_trees) contrib[rl * n_trees + t] = lv;
          }
        }
      } else if (SMEM_NODES && max_depth <= GBT_WALK_MAX_DEPTH) {
        // GBT_ILP trees walked side by side for a fixed max_depth levels
        // (a walk that reached its leaf stays there): independent chains
        // of dependent shared-memory loads instead of one at a time
        const uint32_t s_nodes = tc::smem_u32(nodes), s_x = tc::smem_u32(x);
        for (int t0 = g; t0 < n_trees; t0 += GBT_ILP * GBT2_GROUPS) {
          uint32_t cur[GBT_ILP];   // node byte address
#pragma unroll
          for (int k = 0; k < GBT_ILP; ++k) {
            const int t = t0 + k * GBT2_GROUPS;
            cur[k] = s_nodes + 16u * (uint32_t)s_first[t < n_trees ? t : t0];
          }
          uint32_t tb[GBT_ILP];
#pragma unroll
          for (int k = 0; k < GBT_ILP; ++k) tb[k] = cur[k];
          for (int lv = 0; lv < max_depth; ++lv) {
            double v[GBT_ILP];
            int f[GBT_ILP], l[GBT_ILP], r_[GBT_ILP];
#pragma unroll
            for (int k = 0; k < GBT_ILP; ++k) lds_node(cur[k], v[k], f[k], l[k], r_[k]);
            double xv[GBT_ILP];
#pragma unroll
            for (int k = 0; k < GBT_ILP; ++k)
              xv[k] = lds_f64(s_x + 8u * (uint32_t)(f[k] < 0 ? 0 : f[k]));
#pragma unroll
            for (int k = 0; k < GBT_ILP; ++k)
              if (f[k] >= 0) cur[k] = tb[k] + 16u * (uint32_t)(xv[k] <= v[k] ? l[k] : r_[k]);
          }
#pragma unroll
          for (int k = 0; k < GBT_ILP; ++k) {
            const int t = t0 + k * GBT2_GROUPS;
            double v;
            int f, l, r_;
            lds_node(cur[k], v, f, l, r_);
            if (t < n_trees) contrib[rl * n_trees + t] = v;
          }
        }
      } else {
        for (int t = g; t < n_trees; t += GBT2_GROUPS) {
          const GbtNode* tree = nodes + s_first[t];
          GbtNode nd = tree[0];
          while (nd.feat >= 0) nd = tree[(x[nd.feat] <= nd.v) ? nd.left : nd.right];
          contrib[rl * n_trees + t] = nd.v;
        }
      }
    }
    __syncthreads();
    if (it < 2) dbg_ts(26 + 3 * it);
    if (g == 0 && rl < rows) {
      double pred = 1.0;
      if (fitted) {
        pred = base;
        const double* c = contrib + rl * n_trees;
        // sequential in tree order (the reference's pred = pred + lr*leaf),
        // the shared-memory loads of 8 terms issued ahead of their adds
        int t = 0;
        for (; t + 8 <= n_trees; t += 8) {
          double cc[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) cc[u] = c[t + u];
#pragma unroll
          for (int u = 0; u < 8; ++u) pred = __dadd_rn(pred, cc[u]);
        }
        for (; t < n_trees; ++t) pred = __dadd_rn(pred, c[t]);
      }
      const double s = (pred != pred) ? pred : (pred < floor_value ? floor_value : pred);
      score[r] = s;
      if (old_score) reward[r] = __ddiv_rn(__dsub_rn(s, o), o);
    }
    __syncthreads();
    if (it < 2) dbg_ts(27 + 3 * it);
    epi(r0, rows, g, rl);
  }
  griddep_trigger();
}

template <bool SMEM_NODES>
__global__ void __launch_bounds__(GBT2_THREADS)
k_gbt_predict2(const GbtNode* __restrict__ gnodes,
               const int32_t* __restrict__ tree_first, int32_t n_trees,
               int64_t n_nodes, int32_t fitted, double base,
               double floor_value, const double* __restrict__ feat, int64_t n,
               int32_t F, double* score, const double* old_score,
               double* reward, const GbtHdr* hdr, int32_t t_cap) {
  // (gbt2_body waits for the predecessor after its forest prologue)
  gbt2_body<SMEM_NODES>(gnodes, tree_first, n_trees, n_nodes, fitted, base,
                        floor_value, feat, n, F, score, old_score, reward, hdr,
                        t_cap, GbtNoEpilogue());
}

}  // namespace harl
