// GBT refit on the device: SurrogateModel.fit_incremental / _fit_tree
// (costmodel.py:81-141, 190-212), bit-exact with the reference.
//
// The reference grows each tree depth-first with numpy; every node's split
// depends only on the node's own sample set, so the device grows the same
// tree level by level (heap numbering: children of k are 2k+1 / 2k+2) and
// the host renumbers the nodes in the reference's creation order.  What has
// to match numpy operation for operation:
//   * ys.mean(), ys.sum(), ((ys - mean)**2).sum(): numpy's pairwise
//     summation (blocks of <= 128 with 8 accumulators, halves split at a
//     multiple of 8) over the node's samples in index order -- leaf blocks
//     summed in parallel, combined in the recursion's order;
//   * argsort(kind="stable") per feature: a presort of every feature column
//     by (value, index) once per fit; a node's sorted order is the stable
//     subsequence, kept by stable partitions level to level;
//   * cumsum: one sequential fp64 chain per (node, feature);
//   * gain = sum_l**2/pos + (total - sum_l)**2/(m - pos), no contraction;
//     argmax over the (position, feature) grid, first maximum;
//   * thr = 0.5 * (x_j + x_j+1); x <= thr routes left;
//   * pred = pred + lr * leaf value.
#pragma once

#include "common.cuh"

namespace harl {

constexpr int FIT_MAX_N = 16384;      // presort in one CTA's shared memory
constexpr int FIT_MAX_DEPTH = 12;
constexpr int FIT_CHUNK = 256;        // cumsum chunk staged per warp

enum FitState : int32_t { FS_NONE = 0, FS_OPEN = 1, FS_LEAF = 2, FS_PEND = 3, FS_SPLIT = 4 };

struct FitCtl {
  int32_t stop;       // residuals all <= 1e-12: no more trees
  int32_t n_built;
  unsigned long long maxres_bits;
  double base;
};

struct FitArgs {
  const double* X;    // [n][F]
  const double* y;    // [n]
  int32_t n, F, K, max_depth, min_leaf;
  int32_t ncap;       // row capacity: stride of the [F][ncap] lists
  const int32_t* n_dev;  // optional: the row count read at run time
                         // (a captured fit graph replayed for any n <= ncap)
  double lr;
  double* pred;       // [n]
  double* resid;      // [n]
  const int32_t* sorted_all;   // [F][n] presorted by (x, index)
  int32_t* ord[2];    // [n] samples by node, index order (ping-pong)
  int32_t* srt[2];    // [F][n] samples by node, (x, index) order
  int32_t* node_of;   // [n] heap id of the sample's node
  int32_t* goleft;    // [n]
  int32_t* seg_start; // [K]
  int32_t* seg_count; // [K]
  int32_t* state;     // [K]
  int32_t* nleft;     // [K]
  int32_t* feat;      // [K]
  double* thr;        // [K]
  double* total;      // [K]
  double* bgain;      // [level nodes][F]
  int32_t* bpos;      // [level nodes][F]
  FitCtl* ctl;
  int32_t* out_feat;  // [n_trees][K]: >= 0 split feature, -1 leaf, -2 none
  double* out_thr;    // [n_trees][K]
  double* out_val;    // [n_trees][K]
};

__device__ __forceinline__ int fit_n(const FitArgs& a) {
  return a.n_dev ? *a.n_dev : a.n;
}

// ---- presort: one CTA per feature, bitonic sort of (x, index) ------------

__device__ __forceinline__ bool fit_less(double xa, int ia, double xb, int ib) {
  return xa < xb || (!(xb < xa) && ia < ib);
}

__global__ void k_fit_presort(const double* __restrict__ X, int n_host,
                              const int32_t* n_dev, int F, int P2, int ncap,
                              int32_t* sorted_all) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  extern __shared__ __align__(16) unsigned char fsm_[];
  double* key = (double*)fsm_;
  int32_t* idx = (int32_t*)(key + P2);
  const int f = blockIdx.x;
  const int n = n_dev ? *n_dev : n_host;
  for (int i = threadIdx.x; i < P2; i += blockDim.x) {
    key[i] = i < n ? X[(int64_t)i * F + f] : INFINITY;
    idx[i] = i < n ? i : 0x7fffffff;
  }
  __syncthreads();
  for (int k = 2; k <= P2; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < P2 / 2; t += blockDim.x) {
        const int i = 2 * t - (t & (j - 1));
        const int l = i + j;
        const bool up = (i & k) == 0;
        const double ka = key[i], kb = key[l];
        const int ia = idx[i], ib = idx[l];
        if (fit_less(kb, ib, ka, ia) == up) {
          key[i] = kb; key[l] = ka;
          idx[i] = ib; idx[l] = ia;
        }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    sorted_all[(int64_t)f * ncap + i] = idx[i];
}

// ---- numpy pairwise summation over an index list --------------------------

// element i of the summed sequence: v[list[i]] or (v[list[i]] - mean)^2
__device__ __forceinline__ double fit_elem(const double* v, const int32_t* list,
                                           int i, bool sq, double mean) {
  const double x = v[list[i]];
  if (!sq) return x;
  const double d = __dsub_rn(x, mean);
  return __dmul_rn(d, d);
}

// numpy's pairwise_sum for n <= 128 (loops_utils.h: 8 accumulators)
__device__ double fit_pw_block(const double* v, const int32_t* list, int lo,
                               int n, bool sq, double mean) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, fit_elem(v, list, lo + i, sq, mean));
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = fit_elem(v, list, lo + j, sq, mean);
  int i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], fit_elem(v, list, lo + i + j, sq, mean));
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, fit_elem(v, list, lo + i, sq, mean));
  return res;
}

// leaves of the pairwise recursion of n elements (left to right)
__device__ int fit_pw_leaves(int lo, int n, int* starts, int* lens, int cnt) {
  if (n <= 128) {
    starts[cnt] = lo;
    lens[cnt] = n;
    return cnt + 1;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  cnt = fit_pw_leaves(lo, n2, starts, lens, cnt);
  return fit_pw_leaves(lo + n2, n - n2, starts, lens, cnt);
}

// combine the leaf sums in the recursion's order
__device__ double fit_pw_combine(int n, const double* sums, int* k) {
  if (n <= 128) return sums[(*k)++];
  int n2 = n / 2;
  n2 -= n2 % 8;
  const double a = fit_pw_combine(n2, sums, k);
  const double b = fit_pw_combine(n - n2, sums, k);
  return __dadd_rn(a, b);
}

constexpr int FIT_MAX_LEAVES = 320;   // pairwise leaves are >= 57 elements

// CTA-wide pairwise sum of the n-element sequence (list[lo..lo+n))
__device__ double fit_pw_cta(const double* v, const int32_t* list, int lo, int n,
                             bool sq, double mean, int* s_starts, int* s_lens,
                             double* s_sums, int* s_cnt) {
  if (threadIdx.x == 0) *s_cnt = fit_pw_leaves(lo, n, s_starts, s_lens, 0);
  __syncthreads();
  const int cnt = *s_cnt;
  for (int b = threadIdx.x; b < cnt; b += blockDim.x)
    s_sums[b] = fit_pw_block(v, list, s_starts[b], s_lens[b], sq, mean);
  __syncthreads();
  __shared__ double res;
  if (threadIdx.x == 0) {
    int k = 0;
    res = fit_pw_combine(n, s_sums, &k);
  }
  __syncthreads();
  const double r = res;
  __syncthreads();
  return r;
}

// ---- per fit / per tree ----------------------------------------------------

// base = y.mean(); pred = base (one CTA)
__global__ void k_fit_base(FitArgs a) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  __shared__ int s_starts[FIT_MAX_LEAVES], s_lens[FIT_MAX_LEAVES], s_cnt;
  __shared__ double s_sums[FIT_MAX_LEAVES];
  // identity list: pairwise over y in index order (ord[0] holds 0..n-1)
  const int n = fit_n(a);
  const double tot = fit_pw_cta(a.y, a.ord[0], 0, n, false, 0.0, s_starts,
                                s_lens, s_sums, &s_cnt);
  const double base = __ddiv_rn(tot, (double)n);
  for (int i = threadIdx.x; i < n; i += blockDim.x) a.pred[i] = base;
  if (threadIdx.x == 0) {
    a.ctl->base = base;
    a.ctl->stop = 0;
    a.ctl->n_built = 0;
    a.ctl->maxres_bits = 0ull;
  }
}

__global__ void k_fit_iota(int32_t* ord, int n_host, const int32_t* n_dev) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  const int n = n_dev ? *n_dev : n_host;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    ord[i] = i;
}

// resid = y - pred, max |resid|, level-0 lists and node table reset
__global__ void k_fit_tree_init(FitArgs a) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  if (a.ctl->stop) return;
  unsigned long long mx = 0ull;
  const int n = fit_n(a);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += gridDim.x * blockDim.x) {
    const double r = __dsub_rn(a.y[i], a.pred[i]);
    a.resid[i] = r;
    const unsigned long long b = (unsigned long long)__double_as_longlong(fabs(r));
    mx = b > mx ? b : mx;
    a.ord[0][i] = i;
    a.node_of[i] = 0;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = t > mx ? t : mx;
  }
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(&a.ctl->maxres_bits, mx);
  for (int64_t e = blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)a.F * a.ncap;
       e += gridDim.x * blockDim.x)
    if ((int)(e % a.ncap) < n) a.srt[0][e] = a.sorted_all[e];
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < a.K;
       k += gridDim.x * blockDim.x) {
    a.state[k] = k == 0 ? FS_OPEN : FS_NONE;
    a.seg_start[k] = 0;
    a.seg_count[k] = k == 0 ? n : 0;
    a.nleft[k] = 0;
  }
}

// tree t is built only if max |resid| > 1e-12 (fit_incremental's break)
__global__ void k_fit_tree_check(FitArgs a, int t) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  if (a.ctl->stop) return;
  const double mx = __longlong_as_double((long long)a.ctl->maxres_bits);
  if (mx <= 1e-12) a.ctl->stop = 1;
  else a.ctl->n_built = t + 1;
  a.ctl->maxres_bits = 0ull;
  const int K = a.K;
  for (int k = 0; k < K; ++k) a.out_feat[(int64_t)t * K + k] = -2;
}

// (level d) node stats: value = mean, leaf tests; one CTA per level node
__global__ void k_fit_stats(FitArgs a, int d, int t, int lists) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  if (a.ctl->stop) return;
  const int k = (1 << d) - 1 + blockIdx.x;
  if (a.state[k] != FS_OPEN) return;
  __shared__ int s_starts[FIT_MAX_LEAVES], s_lens[FIT_MAX_LEAVES], s_cnt;
  __shared__ double s_sums[FIT_MAX_LEAVES];
  const int s = a.seg_start[k], m = a.seg_count[k];
  const int32_t* list = a.ord[lists];
  const double tot = fit_pw_cta(a.resid, list, s, m, false, 0.0, s_starts,
                                s_lens, s_sums, &s_cnt);
  const double mean = __ddiv_rn(tot, (double)m);
  bool leaf = d >= a.max_depth || m < 2 * a.min_leaf;
  if (!leaf) {
    const double var = fit_pw_cta(a.resid, list, s, m, true, mean, s_starts,
                                  s_lens, s_sums, &s_cnt);
    leaf = var <= 1e-24;
  }
  if (threadIdx.x == 0) {
    const int64_t o = (int64_t)t * a.K + k;
    a.out_val[o] = mean;
    a.out_feat[o] = -1;
    a.out_thr[o] = 0.0;
    a.total[k] = tot;
    a.state[k] = leaf ? FS_LEAF : FS_OPEN;
  }
}

// (level d) best split of one feature for one node: a warp per (node, f);
// lane 0 runs the sequential cumsum over FIT_CHUNK staged residuals, then
// every lane evaluates gains for its positions and the warp keeps the first
// maximum
__global__ void k_fit_best(FitArgs a, int d, int lists) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  if (a.ctl->stop) return;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nl = 1 << d;
  const int node = warp / a.F, f = warp % a.F;
  if (node >= nl) return;
  const int k = nl - 1 + node;
  if (a.state[k] != FS_OPEN) return;
  __shared__ double s_c[8][FIT_CHUNK];
  __shared__ double s_x[8][FIT_CHUNK + 1];
  double* cs = s_c[(threadIdx.x >> 5) & 7];
  double* xs = s_x[(threadIdx.x >> 5) & 7];
  const int s = a.seg_start[k], m = a.seg_count[k];
  const int32_t* list = a.srt[lists] + (int64_t)f * a.ncap + s;
  const double total = a.total[k];
  const double mf = (double)m;
  double best = -INFINITY;
  int bpos = -1;
  double carry = 0.0;
  // software pipeline: the next chunk's residuals and feature values are
  // loaded into registers while lane 0 runs the current chunk's chain
  constexpr int PL = FIT_CHUNK / 32;
  double nr[PL], nx[PL];
  auto fetch = [&](int c0) {
#pragma unroll
    for (int u = 0; u < PL; ++u) {
      const int q = lane + 32 * u;
      const int j = c0 + q;
      if (j < m) {
        const int i = list[j];
        nr[u] = a.resid[i];
        nx[u] = a.X[(int64_t)i * a.F + f];
      }
    }
  };
  if (m > 1) fetch(0);
  for (int c0 = 0; c0 < m - 1; c0 += FIT_CHUNK) {
    const int cn = min(FIT_CHUNK, m - c0);           // elements staged
    // positions j = c0 .. c0+cn-1 need x_j and x_{j+1}
#pragma unroll
    for (int u = 0; u < PL; ++u) {
      const int q = lane + 32 * u;
      if (q < cn) {
        cs[q] = nr[u];
        xs[q] = nx[u];
      }
    }
    if (lane == 0)
      xs[cn] = (c0 + cn < m) ? a.X[(int64_t)list[c0 + cn] * a.F + f] : 0.0;
    __syncwarp();
    if (c0 + FIT_CHUNK < m - 1) fetch(c0 + FIT_CHUNK);
    if (lane == 0) {   // numpy cumsum: out[0] = a[0], out[j] = out[j-1] + a[j]
      double c = carry;
      int q = 0;
      if (c0 == 0) {
        c = cs[0];
        q = 1;
      }
      for (; q + 8 <= cn; q += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = cs[q + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          c = __dadd_rn(c, v[u]);
          v[u] = c;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) cs[q + u] = v[u];
      }
      for (; q < cn; ++q) {
        c = __dadd_rn(c, cs[q]);
        cs[q] = c;
      }
      carry = c;
    }
    __syncwarp();
    carry = __shfl_sync(0xffffffffu, carry, 0);
    for (int q = lane; q < cn; q += 32) {
      const int j = c0 + q;
      if (j >= m - 1) continue;
      const bool ok = xs[q] != xs[q + 1] &&
                      (a.min_leaf <= 1 || (j + 1 >= a.min_leaf && m - (j + 1) >= a.min_leaf));
      if (!ok) continue;
      const double sl = cs[q];
      const double pos = (double)(j + 1);
      const double tr = __dsub_rn(total, sl);
      const double g = __dadd_rn(__ddiv_rn(__dmul_rn(sl, sl), pos),
                                 __ddiv_rn(__dmul_rn(tr, tr), __dsub_rn(mf, pos)));
      if (g > best || (g == best && j < bpos)) {
        best = g;
        bpos = j;
      }
    }
    __syncwarp();
  }
  // first maximum over the warp (smaller position on ties)
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double og = __shfl_xor_sync(0xffffffffu, best, o);
    const int op = __shfl_xor_sync(0xffffffffu, bpos, o);
    if (og > best || (og == best && op >= 0 && (bpos < 0 || op < bpos))) {
      best = og;
      bpos = op;
    }
  }
  if (lane == 0) {
    a.bgain[(int64_t)node * a.F + f] = best;
    a.bpos[(int64_t)node * a.F + f] = bpos;
  }
}

// (level d) pick the split over features: argmax over the flattened
// (position, feature) grid = max gain, then smallest position, then
// smallest feature; threshold = midpoint of the sorted neighbours
__global__ void k_fit_split(FitArgs a, int d, int lists) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  if (a.ctl->stop) return;
  const int nl = 1 << d;
  const int node = blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= nl) return;
  const int k = nl - 1 + node;
  if (a.state[k] != FS_OPEN) return;
  double best = -INFINITY;
  int bp = -1, bf = -1;
  for (int f = 0; f < a.F; ++f) {
    const double g = a.bgain[(int64_t)node * a.F + f];
    const int p = a.bpos[(int64_t)node * a.F + f];
    if (p < 0) continue;
    if (bp < 0 || g > best || (g == best && p < bp)) {
      best = g;
      bp = p;
      bf = f;
    }
  }
  if (bp < 0 || !isfinite(best)) {
    a.state[k] = FS_LEAF;
    return;
  }
  const int s = a.seg_start[k];
  const int32_t* list = a.srt[lists] + (int64_t)bf * a.ncap + s;
  const double x0 = a.X[(int64_t)list[bp] * a.F + bf];
  const double x1 = a.X[(int64_t)list[bp + 1] * a.F + bf];
  a.feat[k] = bf;
  a.thr[k] = __dmul_rn(0.5, __dadd_rn(x0, x1));
  a.nleft[k] = 0;
  a.state[k] = FS_PEND;
}

// (level d) route every sample of a pending node: x <= thr goes left
__global__ void k_fit_route(FitArgs a) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  if (a.ctl->stop) return;
  const int n = fit_n(a);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += gridDim.x * blockDim.x) {
    const int k = a.node_of[i];
    if (a.state[k] != FS_PEND) continue;
    const int gl = a.X[(int64_t)i * a.F + a.feat[k]] <= a.thr[k];
    a.goleft[i] = gl;
    if (gl) atomicAdd(&a.nleft[k], 1);
  }
}

// (level d) a split whose midpoint collapsed onto one side stays a leaf;
// otherwise record it and open the children
__global__ void k_fit_commit(FitArgs a, int d, int t) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  if (a.ctl->stop) return;
  const int nl = 1 << d;
  const int node = blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= nl) return;
  const int k = nl - 1 + node;
  if (a.state[k] != FS_PEND) return;
  const int m = a.seg_count[k], L = a.nleft[k];
  if (L == 0 || L == m) {
    a.state[k] = FS_LEAF;
    return;
  }
  a.state[k] = FS_SPLIT;
  const int64_t o = (int64_t)t * a.K + k;
  a.out_feat[o] = a.feat[k];
  a.out_thr[o] = a.thr[k];
  const int s = a.seg_start[k];
  const int cl = 2 * k + 1, cr = 2 * k + 2;
  a.seg_start[cl] = s;
  a.seg_count[cl] = L;
  a.seg_start[cr] = s + L;
  a.seg_count[cr] = m - L;
  a.state[cl] = FS_OPEN;
  a.state[cr] = FS_OPEN;
}

// (level d) stable partition of every split node's segment, for the
// index-order list (q == F, also moving node_of to the child) and each
// feature's sorted list (q < F): one warp per (node, list)
__global__ void k_fit_partition(FitArgs a, int d, int lists) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  if (a.ctl->stop) return;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nl = 1 << d;
  const int node = warp / (a.F + 1), q = warp % (a.F + 1);
  if (node >= nl) return;
  const int k = nl - 1 + node;
  if (a.state[k] != FS_SPLIT) return;
  const int s = a.seg_start[k], m = a.seg_count[k], L = a.nleft[k];
  const int32_t* src = q == a.F ? a.ord[lists] : a.srt[lists] + (int64_t)q * a.ncap;
  int32_t* dst = q == a.F ? a.ord[lists ^ 1] : a.srt[lists ^ 1] + (int64_t)q * a.ncap;
  int nlw = 0, nrw = 0;
  constexpr int PB = 8;   // chunks of 32 with their loads in flight together
  for (int c0 = 0; c0 < m; c0 += 32 * PB) {
    int iv[PB];
    bool gv[PB];
#pragma unroll
    for (int u = 0; u < PB; ++u) {
      const int j = c0 + 32 * u + lane;
      iv[u] = j < m ? src[s + j] : -1;
    }
#pragma unroll
    for (int u = 0; u < PB; ++u) gv[u] = iv[u] >= 0 && a.goleft[iv[u]];
#pragma unroll
    for (int u = 0; u < PB; ++u) {
      const bool in = iv[u] >= 0;
      const unsigned bl = __ballot_sync(0xffffffffu, gv[u]);
      const unsigned br = __ballot_sync(0xffffffffu, in && !gv[u]);
      const unsigned below = (1u << lane) - 1u;
      if (in) {
        const int p = gv[u] ? s + nlw + __popc(bl & below)
                            : s + L + nrw + __popc(br & below);
        dst[p] = iv[u];
        if (q == a.F) a.node_of[iv[u]] = gv[u] ? 2 * k + 1 : 2 * k + 2;
      }
      nlw += __popc(bl);
      nrw += __popc(br);
    }
  }
}

// after the last level: pred = pred + lr * value[leaf]
__global__ void k_fit_pred(FitArgs a, int t) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  if (a.ctl->stop) return;
  const int n = fit_n(a);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += gridDim.x * blockDim.x) {
    const double v = a.out_val[(int64_t)t * a.K + a.node_of[i]];
    a.pred[i] = __dadd_rn(a.pred[i], __dmul_rn(a.lr, v));
  }
}

}  // namespace harl
