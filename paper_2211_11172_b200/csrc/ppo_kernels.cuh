// K7: the PPO update (rlcore.py:293-378) in fp64 on device.
//   (a) k_ppo_rows   row-parallel: gather the sampled transitions from the
//       replay ring, policy + value forward, per-row clipped-surrogate /
//       entropy / MSE terms and the per-layer deltas (dL/dz) for both nets
//       (rlcore.py:293-358, Mlp.backward 105-116, PolicyNet.backward 148-158)
//   (b) k_ppo_losses one warp: fixed-order means -> losses, finiteness
//   (c) k_ppo_wgrad  weight/bias gradients = sum over rows of act^T delta,
//       tiled through shared memory, fixed summation order (deterministic)
//   (d) k_ppo_adam   Adam.step (rlcore.py:62-71) with the reference's
//       operation order, skipped entirely when anything is non-finite
//       (ppo_update raises before stepping, rlcore.py:368-375); refreshes
//       the fp32 rollout copy of every parameter.
// Parameters live in one flat fp64 buffer (policy segment then value
// segment); the tiling head is stored compact (see space.head_columns).
#pragma once

#include "common.cuh"
#include "tc_common.cuh"

namespace harl {

typedef harl_net_layout NetLayout;

struct PpoArgs {
  int32_t B, F, C0, row_stride;
  // offsets (doubles) of the transposed copies used by the backward pass:
  // policy heads, policy W[l] and value W[l] for l >= 1
  int64_t wt_head, wt_P[HARL_MAX_LAYERS], wt_V[HARL_MAX_LAYERS];
  int32_t B_norm;           // batch size in the 1/B normalisation (global)
  double clip_lo, clip_hi, w_ent, w_val;
  int32_t* bad;             // optional: bad[1] = bad[0] at the update's start
                            // (the speculative Adam's skip decision)
  int16_t head0_src[HARL_MAX_HEAD0];
};

typedef harl_replay_ring PpoRing;

#ifndef HARL_PPO_WIDE
#define HARL_PPO_WIDE 2
#endif
#ifndef HARL_PPO_TM
#define HARL_PPO_TM 2          // minibatch rows per CTA
#endif
constexpr int PPO_TM = HARL_PPO_TM;
// HARL_PPO_WIDE x 4 warps per row: the loss terms use 4 warps per row, the
// dense layers split each output's reduction over the extra threads
constexpr int PPO_THREADS = 128 * PPO_TM * HARL_PPO_WIDE;
static_assert(PPO_TM >= 1 && HARL_PPO_WIDE >= 1 && PPO_THREADS <= 1024,
              "HARL_PPO_TM x HARL_PPO_WIDE: at most 1024 threads per CTA");

// Latency-bound small-batch layers: every thread keeps PPO_UNR weight
// loads in flight (issued before the FMAs that consume them); the CTA's
// row activations live in shared memory.
#ifndef HARL_PPO_UNR
#define HARL_PPO_UNR 16
#endif
constexpr int PPO_UNR = HARL_PPO_UNR;

// Each output is split over up to PPO_SPLIT threads along the reduction
// (contiguous k ranges summed in part order: deterministic), so a thread's
// chain of dependent weight-load rounds is PPO_SPLIT times shorter.
#ifndef HARL_PPO_SPLIT
#define HARL_PPO_SPLIT 4
#endif
constexpr int PPO_SPLIT = HARL_PPO_SPLIT;

__device__ inline int ppo_parts(int outputs) {
  int p = (int)blockDim.x / (outputs > 0 ? outputs : 1);
  return p < 1 ? 1 : (p > PPO_SPLIT ? PPO_SPLIT : p);
}

// out[r][c] = act(sum_k in[r][k] W[k][c] + b[c]) for r < rows
__device__ inline void dense64(const double* in, int ldi, int K,
                               const double* __restrict__ W,
                               const double* __restrict__ b, int N, double* out,
                               int ldo, bool act, int rows, double* part) {
  const int P = ppo_parts(N);
  const int kc = (K + P - 1) / P;
  for (int t = threadIdx.x; t < N * P; t += blockDim.x) {
    const int c = t % N, p = t / N;
    const int k1 = min(K, (p + 1) * kc);
    double acc[PPO_TM];
#pragma unroll
    for (int r = 0; r < PPO_TM; ++r) acc[r] = 0.0;
    int k = p * kc;
    for (; k + PPO_UNR <= k1; k += PPO_UNR) {
      double w[PPO_UNR];
#pragma unroll
      for (int q = 0; q < PPO_UNR; ++q) w[q] = __ldg(W + (int64_t)(k + q) * N + c);
#pragma unroll
      for (int q = 0; q < PPO_UNR; ++q)
#pragma unroll
        for (int r = 0; r < PPO_TM; ++r)
          if (r < rows) acc[r] = fma(in[r * ldi + k + q], w[q], acc[r]);
    }
    for (; k < k1; ++k) {
      const double w = __ldg(W + (int64_t)k * N + c);
#pragma unroll
      for (int r = 0; r < PPO_TM; ++r)
        if (r < rows) acc[r] = fma(in[r * ldi + k], w, acc[r]);
    }
    if (P == 1) {
      for (int r = 0; r < rows; ++r) {
        const double z = acc[r] + b[c];
        out[r * ldo + c] = act ? tanh(z) : z;
      }
    } else {
#pragma unroll
      for (int r = 0; r < PPO_TM; ++r) part[(p * PPO_TM + r) * N + c] = acc[r];
    }
  }
  if (P > 1) {
    __syncthreads();
    for (int t = threadIdx.x; t < N * rows; t += blockDim.x) {
      const int c = t % N, r = t / N;
      double z = part[r * N + c];
      for (int p = 1; p < P; ++p) z += part[(p * PPO_TM + r) * N + c];
      z += b[c];
      out[r * ldo + c] = act ? tanh(z) : z;
    }
  }
  __syncthreads();
}

__device__ inline double wsum64_(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// out[r][k] = (sum_c d[r][c] W[k][c]) * (1 - a[r][k]^2), reading the
// transposed copy WT[c][k] (kept current by the Adam kernel) so that
// threads over k load coalesced rows, with the same split reduction as
// dense64.
__device__ inline void back64(const double* d, int ldd, int N,
                              const double* __restrict__ WT, int K,
                              const double* a, int lda, double* out, int ldo,
                              int rows, double* part) {
  const int P = ppo_parts(K);
  const int ncs = (N + P - 1) / P;
  for (int t = threadIdx.x; t < K * P; t += blockDim.x) {
    const int k = t % K, p = t / K;
    const int c1 = min(N, (p + 1) * ncs);
    double acc[PPO_TM];
#pragma unroll
    for (int r = 0; r < PPO_TM; ++r) acc[r] = 0.0;
    int c = p * ncs;
    for (; c + PPO_UNR <= c1; c += PPO_UNR) {
      double w[PPO_UNR];
#pragma unroll
      for (int q = 0; q < PPO_UNR; ++q) w[q] = __ldg(WT + (int64_t)(c + q) * K + k);
#pragma unroll
      for (int q = 0; q < PPO_UNR; ++q)
#pragma unroll
        for (int r = 0; r < PPO_TM; ++r)
          if (r < rows) acc[r] = fma(d[r * ldd + c + q], w[q], acc[r]);
    }
    for (; c < c1; ++c) {
      const double w = __ldg(WT + (int64_t)c * K + k);
#pragma unroll
      for (int r = 0; r < PPO_TM; ++r)
        if (r < rows) acc[r] = fma(d[r * ldd + c], w, acc[r]);
    }
    if (P == 1) {
      for (int r = 0; r < rows; ++r) {
        const double av = a[r * lda + k];
        out[r * ldo + k] = acc[r] * (1.0 - av * av);
      }
    } else {
#pragma unroll
      for (int r = 0; r < PPO_TM; ++r) part[(p * PPO_TM + r) * K + k] = acc[r];
    }
  }
  if (P > 1) {
    __syncthreads();
    for (int t = threadIdx.x; t < K * rows; t += blockDim.x) {
      const int k = t % K, r = t / K;
      double z = part[r * K + k];
      for (int p = 1; p < P; ++p) z += part[(p * PPO_TM + r) * K + k];
      const double av = a[r * lda + k];
      out[r * ldo + k] = z * (1.0 - av * av);
    }
  }
  __syncthreads();
}

__device__ inline double wmax64(double v) {
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ inline double wsum64(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// per-row terms written to rowout[r*4 + {0..3}]:
//   min(s_un, s_cl), entropy total, ratio, (v - td)^2
// (2 CTAs per SM: the 2 x B/PPO_TM CTAs of a minibatch in one wave)
__global__ void __launch_bounds__(PPO_THREADS, 2)
k_ppo_rows(const __grid_constant__ PpoArgs a, const __grid_constant__ NetLayout P,
           const __grid_constant__ NetLayout V, PpoRing ring, const int32_t* idx,
           const double* params, const double* wt, double* rows,
           double* rowout) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  dbg_ts(40);
  extern __shared__ double srows[];
  // blockIdx.y: 0 = policy (forward, heads, surrogate/entropy terms,
  // backward), 1 = value (forward, squared error, backward) -- the two nets
  // share only X, so their chains run side by side in separate CTAs
  const int role = blockIdx.y;
  const int r0 = blockIdx.x * PPO_TM;
  // (nothing sets bad before this update's wgrad launch: a stable snapshot)
  if (a.bad && blockIdx.x == 0 && role == 0 && threadIdx.x == 0) a.bad[1] = a.bad[0];
  const int nrows = min(PPO_TM, a.B - r0);
  const int RS = a.row_stride;
  double* base = srows;  // this CTA's rows, copied out at the end
  double* wbuf = srows + PPO_TM * RS + 8;  // split-reduction partials
  __shared__ int16_t s_src[HARL_MAX_HEAD0];
  // the rows' transition fields, loaded with the gather (one round trip
  // behind idx) instead of where the loss terms use them
  __shared__ uint64_t s_mv[PPO_TM];
  __shared__ uint32_t s_sb[PPO_TM];
  __shared__ int32_t s_act[PPO_TM][4];
  __shared__ double s_sc[PPO_TM][4];
  if (threadIdx.x < nrows) {
    const int q = threadIdx.x;
    const int sl = idx[r0 + q];
    const int4 ac = *(const int4*)&ring.actions[(int64_t)sl * 4];
    const uint64_t mvq = ring.move_bits[sl];
    const uint32_t sbq = ring.shift_bits[sl];
    double sc[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) sc[j] = ring.scalars[(int64_t)sl * 4 + j];
    s_act[q][0] = ac.x;
    s_act[q][1] = ac.y;
    s_act[q][2] = ac.z;
    s_act[q][3] = ac.w;
    s_mv[q] = mvq;
    s_sb[q] = sbq;
#pragma unroll
    for (int j = 0; j < 4; ++j) s_sc[q][j] = sc[j];
  }
  for (int i = threadIdx.x; i < a.C0; i += blockDim.x) s_src[i] = a.head0_src[i];
  // gather X (shared by both nets: P.row_act[0] == V.row_act[0])
  for (int i = threadIdx.x; i < nrows * a.F; i += blockDim.x) {
    const int rr = i / a.F, k = i % a.F;
    base[rr * RS + P.row_act[0] + k] = ring.X[(int64_t)idx[r0 + rr] * a.F + k];
  }
  __syncthreads();
  dbg_ts(41);
  const int H = P.dims[P.n_layers];
  const int NH = P.n_head_cols;
  if (role == 0) {
    // policy trunk (every layer tanh: rlcore.py:95-103 + 139) and heads
    for (int l = 0; l < P.n_layers; ++l)
      dense64(base + P.row_act[l], RS, P.dims[l], params + P.off_W[l],
              params + P.off_b[l], P.dims[l + 1], base + P.row_act[l + 1], RS,
              true, nrows, wbuf);
    dbg_ts(42);
    dense64(base + P.row_act[P.n_layers], RS, H, params + P.off_hW,
            params + P.off_hb, NH, base + P.row_head, RS, false, nrows, wbuf);
    dbg_ts(43);
  } else {
    // value net (its last layer linear, rlcore.py:161-178)
    for (int l = 0; l < V.n_layers; ++l)
      dense64(base + V.row_act[l], RS, V.dims[l], params + V.off_W[l],
              params + V.off_b[l], V.dims[l + 1], base + V.row_act[l + 1], RS,
              l < V.n_layers - 1, nrows, wbuf);
    dbg_ts(44);
  }
  // per-row PPO terms: warp w takes (row w/4, head w%4); the exps of a
  // lane's columns are computed once and reused for the sum, the entropy
  // and the gradient.  Per-(row, head) results meet in shared memory.
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double invB = 1.0 / (double)a.B_norm;
  __shared__ double s_lp[PPO_TM][4], s_ent[PPO_TM][4];
  const int rr = warp >> 2, h = warp & 3;
  const bool active = role == 0 && rr < nrows &&
                      (PPO_THREADS / 32) >= 4 * PPO_TM;
  constexpr int HI = 4;      // cached columns per lane (C0 <= 128)
  double ev[HI];
  double hm = 0.0, hs = 1.0, hls = 0.0, hent = 0.0;
  int col = 0, c0 = 0, C = 0;
  uint64_t mv = 0;
  uint32_t sb = 0;
  double* z = nullptr;
  if (active) {
    z = base + rr * RS + P.row_head;
    mv = s_mv[rr];
    sb = s_sb[rr];
    c0 = h == 0 ? 0 : a.C0 + 3 * (h - 1);
    C = h == 0 ? a.C0 : 3;
    col = s_act[rr][h];
  }
  auto legal = [&](int j) -> bool {
    if (h == 0) return j == a.C0 - 1 || ((mv >> s_src[j]) & 1ull);
    return (sb >> (3 * (h - 1) + j)) & 1u;
  };
  if (active) {
    // pass 1: max, sum, entropy (rlcore.py:300-306)
    double m = -INFINITY;
    for (int j = lane; j < C; j += 32)
      if (legal(j)) m = fmax(m, z[c0 + j]);
    m = wmax64(m);
    double sacc = 0.0;
#pragma unroll
    for (int i = 0; i < HI; ++i) {
      const int j = lane + 32 * i;
      ev[i] = 0.0;
      if (j < C && legal(j)) ev[i] = exp(z[c0 + j] - m);
      sacc += ev[i];
    }
    for (int j = lane + 32 * HI; j < C; j += 32)   // wide heads (C0 > 128)
      if (legal(j)) sacc += exp(z[c0 + j] - m);
    const double sh = wsum64(sacc);
    const double ls = log(sh);
    double e = 0.0;
#pragma unroll
    for (int i = 0; i < HI; ++i) {
      const int j = lane + 32 * i;
      if (j < C && legal(j)) e -= (ev[i] / sh) * (z[c0 + j] - m - ls);
    }
    for (int j = lane + 32 * HI; j < C; j += 32)
      if (legal(j)) e -= (exp(z[c0 + j] - m) / sh) * (z[c0 + j] - m - ls);
    e = wsum64(e);
    hm = m;
    hs = sh;
    hls = ls;
    hent = e;
    if (lane == 0) {
      // log-prob of the taken action; ring actions hold the COMPACT column
      // for head 0 (policy kernel output head0_col)
      s_lp[rr][h] = z[c0 + col] - m - ls;
      s_ent[rr][h] = e;
    }
  }
  __syncthreads();
  if (active) {
    const double logp_new = ((s_lp[rr][0] + s_lp[rr][1]) + s_lp[rr][2]) + s_lp[rr][3];
    const double ent_total = ((s_ent[rr][0] + s_ent[rr][1]) + s_ent[rr][2]) + s_ent[rr][3];
    const double logp_old = s_sc[rr][0];
    const double adv = s_sc[rr][2];
    const double ratio = exp(logp_new - logp_old);
    const double clipped = fmin(fmax(ratio, a.clip_lo), a.clip_hi);
    const double s_un = ratio * adv, s_cl = clipped * adv;
    const double coef = (s_un <= s_cl) ? ratio * adv : 0.0;
    const double dlogp = -coef * invB;
    const double went = a.w_ent * invB;
    // pass 2: dz in place over the logits
    for (int j = lane, i = 0; j < C; j += 32, ++i) {
      {
        double dz;
        if (legal(j)) {
          const double lp = z[c0 + j] - hm - hls;
          double evj = 0.0;
#pragma unroll
          for (int q = 0; q < HI; ++q) evj = q == i ? ev[q] : evj;
          if (i >= HI) evj = exp(z[c0 + j] - hm);
          const double p = evj / hs;
          dz = dlogp * ((j == col ? 1.0 : 0.0) - p) + went * p * (lp + hent);
        } else {
          dz = dlogp * ((j == col ? 1.0 : 0.0) - 0.0);
        }
        z[c0 + j] = dz;
      }
    }
    if (h == 0 && lane == 0) {
      double* o = rowout + (int64_t)(r0 + rr) * 4;
      o[0] = fmin(s_un, s_cl);
      o[1] = ent_total;
      o[2] = ratio;
    }
  }
  if (role == 1 && threadIdx.x < nrows) {
    const int q = threadIdx.x;
    const double td = s_sc[q][3];
    const double v = base[q * RS + V.row_act[V.n_layers]];
    rowout[(int64_t)(r0 + q) * 4 + 3] = (v - td) * (v - td);
    // dv = w * 2 (v - td) / B is the value net's output delta
    base[q * RS + V.row_delta[V.n_layers - 1]] = a.w_val * 2.0 * (v - td) * invB;
  }
  __syncthreads();
  dbg_ts(45);
  if (role == 0) {
    // policy backward: dhid = dz . Wh^T, times (1 - hid^2)
    back64(base + P.row_head, RS, NH, wt + a.wt_head, H,
           base + P.row_act[P.n_layers], RS,
           base + P.row_delta[P.n_layers - 1], RS, nrows, wbuf);
    for (int l = P.n_layers - 1; l >= 1; --l)
      back64(base + P.row_delta[l], RS, P.dims[l + 1], wt + a.wt_P[l],
             P.dims[l], base + P.row_act[l], RS, base + P.row_delta[l - 1],
             RS, nrows, wbuf);
    dbg_ts(46);
  } else {
    for (int l = V.n_layers - 1; l >= 1; --l)
      back64(base + V.row_delta[l], RS, V.dims[l + 1], wt + a.wt_V[l],
             V.dims[l], base + V.row_act[l], RS, base + V.row_delta[l - 1],
             RS, nrows, wbuf);
    dbg_ts(47);
  }
  // each role writes its own segment of the rows: [X, policy acts, heads,
  // policy deltas] | [value acts, value deltas] (DeviceAgent row layout)
  const int seg0 = role == 0 ? 0 : V.row_act[1];
  const int seg1 = role == 0 ? V.row_act[1] : RS;
  const int sw = seg1 - seg0;
  double* out = rows + (int64_t)r0 * RS;
  for (int i = threadIdx.x; i < nrows * sw; i += blockDim.x) {
    const int q = i / sw, c = seg0 + i % sw;
    out[q * RS + c] = base[q * RS + c];
  }
  griddep_trigger();
  dbg_ts(48);
}

// ---------------------------------------------------------------------------
// (a') the same per-row work on fp64 tensor cores: 8 minibatch rows per CTA
// (mma.m8n8k4.f64: M = the 8 rows, N = 8 outputs per warp tile, K = 4 per
// instruction); each warp owns output tiles n0 = 8 * (warp + 16 i), loads
// all of its weight fragments before the dependent MMA chain, and writes
// act(z + b) / delta * (1 - a^2) for its tile.  Accumulation order differs
// from the SIMT kernel (fp64 rounding level; the parity tests' tolerance).
// Opt-in (HARL_PPO_TC=1): the full GPU suite passed with it as the default
// (PPO parity within tolerance), but at B = 256 it measured slower than
// k_ppo_rows (41 vs 29 us) -- 32 CTAs per chain, dependent MMA chains.

constexpr int PPO8_ROWS = 8;
constexpr int PPO8_THREADS = 512;
constexpr int PPO8_KMAX = 128;   // reduction length held in fragments

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a,
                                        double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 "
      "{%0, %1}, {%2}, {%3}, {%0, %1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// out[r][n] = epi(r, n, sum_k in[r][k] * Wm[k][n]) for r < 8, n < Nout;
// Wm row-major [Kred][Nout] in global memory, in (smem) row stride ldi.
template <typename Epi>
__device__ __forceinline__ void mma8_layer(const double* in, int ldi, int Kred,
                                           const double* __restrict__ Wm,
                                           int Nout, const Epi& epi) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int nwarps = blockDim.x >> 5;
  const int ksteps = (Kred + 3) / 4;
  for (int n0 = 8 * warp; n0 < Nout; n0 += 8 * nwarps) {
    const int col = n0 + gid;
    double d0 = 0.0, d1 = 0.0;
    for (int kb = 0; kb < ksteps; kb += 16) {
      double bf[16], af[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int k = 4 * (kb + u) + tig;
        bf[u] = (kb + u < ksteps && k < Kred && col < Nout)
                    ? __ldg(Wm + (int64_t)k * Nout + col) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int k = 4 * (kb + u) + tig;
        af[u] = (kb + u < ksteps && k < Kred) ? in[gid * ldi + k] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (kb + u < ksteps) dmma884(d0, d1, af[u], bf[u]);
    }
    const int c0 = n0 + 2 * tig;
    if (c0 < Nout) epi(gid, c0, d0);
    if (c0 + 1 < Nout) epi(gid, c0 + 1, d1);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(PPO8_THREADS, 1)
k_ppo_rows_tc(const __grid_constant__ PpoArgs a,
              const __grid_constant__ NetLayout P,
              const __grid_constant__ NetLayout V, PpoRing ring,
              const int32_t* idx, const double* params, const double* wt,
              double* rows, double* rowout) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  dbg_ts(40);
  extern __shared__ double srows[];
  const int role = blockIdx.y;   // 0 policy chain, 1 value chain
  const int r0 = blockIdx.x * PPO8_ROWS;
  if (a.bad && blockIdx.x == 0 && role == 0 && threadIdx.x == 0) a.bad[1] = a.bad[0];
  const int nrows = min(PPO8_ROWS, a.B - r0);
  const int RS = a.row_stride;
  double* base = srows;
  __shared__ int16_t s_src[HARL_MAX_HEAD0];
  __shared__ double s_st[PPO8_ROWS * 4][4];   // per (row, head): m, s, log s, ent
  __shared__ double s_lp[PPO8_ROWS][4], s_ent[PPO8_ROWS][4];
  for (int i = threadIdx.x; i < a.C0; i += blockDim.x) s_src[i] = a.head0_src[i];
  // rows past nrows are zeros (their fragments contribute nothing)
  for (int i = threadIdx.x; i < PPO8_ROWS * RS; i += blockDim.x) base[i] = 0.0;
  __syncthreads();
  for (int i = threadIdx.x; i < nrows * a.F; i += blockDim.x) {
    const int rr = i / a.F, k = i % a.F;
    base[rr * RS + P.row_act[0] + k] = ring.X[(int64_t)idx[r0 + rr] * a.F + k];
  }
  __syncthreads();
  dbg_ts(41);
  const int H = P.dims[P.n_layers];
  const int NH = P.n_head_cols;
  if (role == 0) {
    for (int l = 0; l < P.n_layers; ++l) {
      double* out = base + P.row_act[l + 1];
      const double* bb = params + P.off_b[l];
      mma8_layer(base + P.row_act[l], RS, P.dims[l], params + P.off_W[l],
                 P.dims[l + 1], [&](int r, int c, double z) {
                   out[r * RS + c] = tanh(z + bb[c]);
                 });
    }
    dbg_ts(42);
    {
      double* out = base + P.row_head;
      const double* bb = params + P.off_hb;
      mma8_layer(base + P.row_act[P.n_layers], RS, H, params + P.off_hW, NH,
                 [&](int r, int c, double z) { out[r * RS + c] = z + bb[c]; });
    }
    dbg_ts(43);
  } else {
    for (int l = 0; l < V.n_layers; ++l) {
      double* out = base + V.row_act[l + 1];
      const double* bb = params + V.off_b[l];
      const bool act = l < V.n_layers - 1;
      mma8_layer(base + V.row_act[l], RS, V.dims[l], params + V.off_W[l],
                 V.dims[l + 1], [&](int r, int c, double z) {
                   const double v = z + bb[c];
                   out[r * RS + c] = act ? tanh(v) : v;
                 });
    }
    dbg_ts(44);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const double invB = 1.0 / (double)a.B_norm;
  if (role == 0) {
    // per-(row, head) warps: max, sum, entropy (rlcore.py:300-306)
    for (int pr = warp; pr < nrows * 4; pr += nwarps) {
      const int rr = pr >> 2, h = pr & 3;
      const int slot = idx[r0 + rr];
      const double* z = base + rr * RS + P.row_head;
      const uint64_t mv = ring.move_bits[slot];
      const uint32_t sb = ring.shift_bits[slot];
      const int c0 = h == 0 ? 0 : a.C0 + 3 * (h - 1);
      const int C = h == 0 ? a.C0 : 3;
      auto legal = [&](int j) -> bool {
        if (h == 0) return j == a.C0 - 1 || ((mv >> s_src[j]) & 1ull);
        return (sb >> (3 * (h - 1) + j)) & 1u;
      };
      double m = -INFINITY;
      for (int j = lane; j < C; j += 32)
        if (legal(j)) m = fmax(m, z[c0 + j]);
      m = wmax64(m);
      double sacc = 0.0;
      for (int j = lane; j < C; j += 32)
        if (legal(j)) sacc += exp(z[c0 + j] - m);
      const double sh = wsum64(sacc);
      const double ls = log(sh);
      double e = 0.0;
      for (int j = lane; j < C; j += 32)
        if (legal(j)) e -= (exp(z[c0 + j] - m) / sh) * (z[c0 + j] - m - ls);
      e = wsum64(e);
      if (lane == 0) {
        const int col = ring.actions[slot * 4 + h];
        s_lp[rr][h] = z[c0 + col] - m - ls;
        s_ent[rr][h] = e;
        s_st[pr][0] = m;
        s_st[pr][1] = sh;
        s_st[pr][2] = ls;
        s_st[pr][3] = e;
      }
    }
    __syncthreads();
    // pass 2: dz in place over the logits
    for (int pr = warp; pr < nrows * 4; pr += nwarps) {
      const int rr = pr >> 2, h = pr & 3;
      const int slot = idx[r0 + rr];
      double* z = base + rr * RS + P.row_head;
      const uint64_t mv = ring.move_bits[slot];
      const uint32_t sb = ring.shift_bits[slot];
      const int c0 = h == 0 ? 0 : a.C0 + 3 * (h - 1);
      const int C = h == 0 ? a.C0 : 3;
      auto legal = [&](int j) -> bool {
        if (h == 0) return j == a.C0 - 1 || ((mv >> s_src[j]) & 1ull);
        return (sb >> (3 * (h - 1) + j)) & 1u;
      };
      const double hm = s_st[pr][0], hs = s_st[pr][1], hls = s_st[pr][2],
                   hent = s_st[pr][3];
      const double logp_new = ((s_lp[rr][0] + s_lp[rr][1]) + s_lp[rr][2]) + s_lp[rr][3];
      const double logp_old = ring.scalars[slot * 4 + 0];
      const double adv = ring.scalars[slot * 4 + 2];
      const double ratio = exp(logp_new - logp_old);
      const double clipped = fmin(fmax(ratio, a.clip_lo), a.clip_hi);
      const double s_un = ratio * adv, s_cl = clipped * adv;
      const double coef = (s_un <= s_cl) ? ratio * adv : 0.0;
      const double dlogp = -coef * invB;
      const double went = a.w_ent * invB;
      const int col = ring.actions[slot * 4 + h];
      for (int j = lane; j < C; j += 32) {
        double dz;
        if (legal(j)) {
          const double lp = z[c0 + j] - hm - hls;
          const double p = exp(z[c0 + j] - hm) / hs;
          dz = dlogp * ((j == col ? 1.0 : 0.0) - p) + went * p * (lp + hent);
        } else {
          dz = dlogp * ((j == col ? 1.0 : 0.0) - 0.0);
        }
        z[c0 + j] = dz;
      }
      if (h == 0 && lane == 0) {
        const double ent_total =
            ((s_ent[rr][0] + s_ent[rr][1]) + s_ent[rr][2]) + s_ent[rr][3];
        double* o = rowout + (int64_t)(r0 + rr) * 4;
        o[0] = fmin(s_un, s_cl);
        o[1] = ent_total;
        o[2] = ratio;
      }
    }
    __syncthreads();
    dbg_ts(45);
    // policy backward: dhid = dz . Wh^T, times (1 - hid^2)
    {
      const double* act = base + P.row_act[P.n_layers];
      double* out = base + P.row_delta[P.n_layers - 1];
      mma8_layer(base + P.row_head, RS, NH, wt + a.wt_head, H,
                 [&](int r, int c, double z) {
                   const double av = act[r * RS + c];
                   out[r * RS + c] = z * (1.0 - av * av);
                 });
    }
    for (int l = P.n_layers - 1; l >= 1; --l) {
      const double* act = base + P.row_act[l];
      double* out = base + P.row_delta[l - 1];
      mma8_layer(base + P.row_delta[l], RS, P.dims[l + 1], wt + a.wt_P[l],
                 P.dims[l], [&](int r, int c, double z) {
                   const double av = act[r * RS + c];
                   out[r * RS + c] = z * (1.0 - av * av);
                 });
    }
    dbg_ts(46);
  } else {
    if (threadIdx.x < nrows) {
      const int q = threadIdx.x;
      const int sl = idx[r0 + q];
      const double td = ring.scalars[sl * 4 + 3];
      const double v = base[q * RS + V.row_act[V.n_layers]];
      rowout[(int64_t)(r0 + q) * 4 + 3] = (v - td) * (v - td);
      base[q * RS + V.row_delta[V.n_layers - 1]] = a.w_val * 2.0 * (v - td) * invB;
    }
    __syncthreads();
    for (int l = V.n_layers - 1; l >= 1; --l) {
      const double* act = base + V.row_act[l];
      double* out = base + V.row_delta[l - 1];
      mma8_layer(base + V.row_delta[l], RS, V.dims[l + 1], wt + a.wt_V[l],
                 V.dims[l], [&](int r, int c, double z) {
                   const double av = act[r * RS + c];
                   out[r * RS + c] = z * (1.0 - av * av);
                 });
    }
    dbg_ts(47);
  }
  const int seg0 = role == 0 ? 0 : V.row_act[1];
  const int seg1 = role == 0 ? V.row_act[1] : RS;
  const int sw = seg1 - seg0;
  double* out = rows + (int64_t)r0 * RS;
  for (int i = threadIdx.x; i < nrows * sw; i += blockDim.x) {
    const int q = i / sw, c = seg0 + i % sw;
    out[q * RS + c] = base[q * RS + c];
  }
  griddep_trigger();
  dbg_ts(48);
}

// (b) loss terms: lane l sums rows l, l+32, ... in order, then a fixed xor
// tree (deterministic).  losses[5..8] = the per-row sums (min surrogate,
// entropy, ratio, squared value error) -- the quantities a sharded update
// all-reduces; k_ppo_finalize turns them into the reported means.
__device__ inline void ppo_loss_means(int B, double w_ent, double w_val,
                                      double* losses, int32_t* bad) {
  const double policy_loss = -(losses[5] / B);
  const double entropy = losses[6] / B;
  const double a_loss = policy_loss - w_ent * entropy;
  const double v_loss = w_val * (losses[8] / B);
  losses[0] = a_loss;
  losses[1] = v_loss;
  losses[2] = policy_loss;
  losses[3] = entropy;
  losses[4] = losses[7] / B;
  if (!isfinite(a_loss) || !isfinite(v_loss)) atomicOr(bad, 1);
}

// means_B > 0 (single device): also the reported means and the loss
// finiteness check, for a batch of means_B rows
__device__ inline void ppo_losses_warp(int B, const double* rowout,
                                       double* losses, int means_B,
                                       double w_ent, double w_val,
                                       int32_t* bad) {
  const int lane = threadIdx.x & 31;
  double q[4] = {0, 0, 0, 0};
  for (int r = lane; r < B; r += 32)
    for (int j = 0; j < 4; ++j) q[j] += rowout[r * 4 + j];
  for (int j = 0; j < 4; ++j) q[j] = wsum64(q[j]);
  if (lane == 0) {
    for (int j = 0; j < 4; ++j) losses[5 + j] = q[j];
    if (means_B > 0) ppo_loss_means(means_B, w_ent, w_val, losses, bad);
  }
}

__global__ void k_ppo_losses(int B, const double* rowout, double* losses,
                             int means_B, double w_ent, double w_val,
                             int32_t* bad) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  ppo_losses_warp(B, rowout, losses, means_B, w_ent, w_val, bad);
}

// means (rlcore.py:311-312,355; [0] actor loss, [1] value loss, [2] policy
// loss, [3] entropy, [4] mean ratio) + the finiteness checks of
// ppo_update (rlcore.py:368-373) over the (reduced) losses and gradients
__global__ void k_ppo_finalize(int B, double w_ent, double w_val,
                               double* losses, const double* grads,
                               int64_t n, int32_t* bad) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  if (blockIdx.x == 0 && threadIdx.x == 0) ppo_loss_means(B, w_ent, w_val, losses, bad);
  int nonfinite = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    nonfinite |= !isfinite(grads[i]);
  if (__any_sync(0xffffffffu, nonfinite) && (threadIdx.x & 31) == 0) atomicOr(bad, 2);
}

// (c) gradient jobs: grad[off + i*nj + j] = sum_r A[r][ai + i] * D[r][dj + j]
// (A column -1 means "ones": bias gradient)
struct GradJob {
  int32_t a_off, d_off, ni, nj;  // ni == 0 -> bias (A = 1)
  int64_t g_off;
  int32_t tile_first;            // first tile index of this job
};

constexpr int WG_T = 16;    // 16x16 output tile, one output per thread
constexpr int WG_RB = 128;  // rows staged per pass (static smem <= 48 KB)

struct GradJobs {
  GradJob j[4 * (HARL_MAX_LAYERS + 2)];
  int32_t n;
};

// Every gradient element is one thread's in-order sum over the batch rows
// (the same single-accumulator order as before, so results are unchanged);
// a CTA stages its 16 A columns and 16 D columns for 256 rows at a time
// with all loads in flight.  check_finite: flag non-finite gradients here
// (rlcore.py:368-373) so no separate scan is needed on a single device.
struct WgNoEpi {
  __device__ void operator()(int64_t, double, bool) const {}
};

template <typename Epi = WgNoEpi>
__device__ __forceinline__ void wgrad_body(
    const GradJobs& jt, int B, int RS, const double* __restrict__ rows,
    double* grads, int32_t* bad, int check_finite, const double* rowout,
    double* losses, int means_B, double w_ent, double w_val,
    const Epi& epi = Epi()) {
  dbg_ts(54);
  if (blockIdx.x == gridDim.x - 1) {   // the extra CTA: loss sums/means
    if (threadIdx.x < 32) ppo_losses_warp(B, rowout, losses, means_B, w_ent, w_val, bad);
    return;
  }
  const GradJob* jobs = jt.j;
  const int n_jobs = jt.n;
  __shared__ double sa[WG_RB][WG_T];
  __shared__ double sd[WG_RB][WG_T];
  __shared__ int s_job;
  if (threadIdx.x == 0) {
    int j = 0;
    while (j + 1 < n_jobs && jobs[j + 1].tile_first <= (int)blockIdx.x) ++j;
    s_job = j;
  }
  __syncthreads();
  const GradJob jb = jobs[s_job];
  const int tile = blockIdx.x - jb.tile_first;
  const int ni = jb.ni == 0 ? 1 : jb.ni;
  const int tiles_j = (jb.nj + WG_T - 1) / WG_T;
  const int i0 = (tile / tiles_j) * WG_T, j0 = (tile % tiles_j) * WG_T;
  const int tj = threadIdx.x % WG_T, ti = threadIdx.x / WG_T;
  const bool ones = jb.ni == 0;
  // fp64 tensor cores: warp w sums rows [16w, 16w + 16) of each 128-row
  // slab into a 16x16 partial with mma.m8n8k4.f64 (M = i, N = j, K = rows);
  // the 8 warps' partials are added in warp order at the end
  // (deterministic).  A fragment (m = i, k = r) = A[r][i], B fragment
  // (k = r, n = j) = D[r][j].
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  double pacc[2][2][2] = {{{0.0, 0.0}, {0.0, 0.0}}, {{0.0, 0.0}, {0.0, 0.0}}};
  for (int rb = 0; rb < B; rb += WG_RB) {
    const int nr = min(WG_RB, B - rb);
    // element e of the 128x16 slab: row e/16, column e%16
    constexpr int PER = WG_RB * WG_T / 256;   // 8 per thread per operand
    double va[PER], vd[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = threadIdx.x + 256 * u;
      const int rr = e / WG_T, cc = e % WG_T;
      const int64_t rowoff = (int64_t)(rb + rr) * RS;
      vd[u] = (rr < nr && j0 + cc < jb.nj) ? rows[rowoff + jb.d_off + j0 + cc] : 0.0;
      va[u] = ones ? (rr < nr ? 1.0 : 0.0)
                   : ((rr < nr && i0 + cc < ni) ? rows[rowoff + jb.a_off + i0 + cc] : 0.0);
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = threadIdx.x + 256 * u;
      sd[e / WG_T][e % WG_T] = vd[u];
      sa[e / WG_T][e % WG_T] = va[u];
    }
    __syncthreads();
    if (rb == 0) dbg_ts(55);
    // rows past nr were staged as zeros
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int r = warp * 16 + ks * 4 + tig;
      double af[2], bf[2];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        af[t] = sa[r][8 * t + gid];
        bf[t] = sd[r][8 * t + gid];
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
          asm volatile(
              "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 "
              "{%0, %1}, {%2}, {%3}, {%0, %1};"
              : "+d"(pacc[mt][nt][0]), "+d"(pacc[mt][nt][1])
              : "d"(af[mt]), "d"(bf[nt]));
    }
    __syncthreads();
  }
  dbg_ts(56);
  // partials -> shared (reusing sa: 8 warps x 256 doubles = 16 KB), then
  // one output per thread summed over warps in order
  double* part = &sa[0][0];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int q = 0; q < 2; ++q)
        part[warp * 256 + (8 * mt + gid) * 16 + 8 * nt + 2 * tig + q] =
            pacc[mt][nt][q];
  __syncthreads();
  double acc1 = 0.0;
  for (int w = 0; w < 8; ++w) acc1 += part[w * 256 + ti * 16 + tj];
  const double acc = acc1;
  const int i = i0 + ti, j = j0 + tj;
  if (i < ni && j < jb.nj) {
    const int64_t gi = jb.g_off + (int64_t)i * jb.nj + j;
    grads[gi] = acc;
    const bool fin = isfinite(acc);
    if (check_finite && !fin) atomicOr(bad, 2);
    epi(gi, acc, fin);
  }
}

__global__ void __launch_bounds__(256)
k_ppo_wgrad(const __grid_constant__ GradJobs jt, int B, int RS,
            const double* __restrict__ rows, double* grads, int32_t* bad,
            int check_finite, const double* rowout, double* losses,
            int means_B, double w_ent, double w_val) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  wgrad_body(jt, B, RS, rows, grads, bad, check_finite, rowout, losses,
             means_B, w_ent, w_val);
  griddep_trigger();
}

// (d) Adam over [0, n_pi) with the policy optimizer and [n_pi, n) with the
// value optimizer.  Scalars precomputed on the host exactly as numpy does.
// Where the updated fp32 weights also live in the tcgen05 weight images
// (tf32 hi/lo, K-major core layout; biases as plain floats), so the Adam
// pass refreshes the images directly instead of a separate re-pack.
struct PackMat {
  int64_t off;
  int32_t K, N, Kpad;
  float* hi;
  float* lo;
  // optional 3xFP16 image (mlp_f16.cuh): halves of p32 * (*sc16)
  uint16_t* h16;
  uint16_t* l16;
  const float* sc16;
};
struct PackVec {
  int64_t off;
  int32_t len;
  float* dst;
};
struct PackPlan {
  PackMat mat[6];
  PackVec vec[12];
  int32_t n_mat, n_vec;
};

// fp64 transposed copies of the matrices the PPO backward pass reads
// (WT[n][k] = W[k][n] at wt + dst)
struct TransMat {
  int64_t off, dst;
  int32_t K, N;
};
struct TransPlan {
  TransMat m[2 * HARL_MAX_LAYERS + 2];
  int32_t n;
  int64_t total;
};

struct AdamArgs {
  int64_t n_pi, n;
  harl_ppo_hyper h;
  PackPlan pk;
  TransPlan tp;
  double* wt;
};

__global__ void k_wt_fill(TransPlan tp, const double* params, double* wt) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  for (int q = 0; q < tp.n; ++q) {
    const TransMat& M = tp.m[q];
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
         e < (int64_t)M.K * M.N; e += (int64_t)gridDim.x * blockDim.x) {
      const int k = (int)(e / M.N), nn = (int)(e % M.N);
      wt[M.dst + (int64_t)nn * M.K + k] = params[M.off + e];
    }
  }
}

__device__ __forceinline__ void adam_one(const AdamArgs& a, double b1t_pi,
                                         double b2t_pi, double b1t_v,
                                         double b2t_v, int64_t i, double g,
                                         double* params, double* m, double* v,
                                         float* params32);

__device__ __forceinline__ void adam_body(const AdamArgs& a,
                                          const double* adam_dev,
                                          const double* grads, double* params,
                                          double* m, double* v,
                                          float* params32) {
  double b1t_pi = a.h.b1t_pi, b2t_pi = a.h.b2t_pi, b1t_v = a.h.b1t_v,
         b2t_v = a.h.b2t_v;
  if (adam_dev) {  // graph replay: this update's 1 - beta^t from device memory
    b1t_pi = adam_dev[0];
    b2t_pi = adam_dev[1];
    b1t_v = adam_dev[2];
    b2t_v = adam_dev[3];
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n;
       i += (int64_t)gridDim.x * blockDim.x)
    adam_one(a, b1t_pi, b2t_pi, b1t_v, b2t_v, i, grads[i], params, m, v, params32);
  dbg_ts(53);
}

// Adam.step (rlcore.py:62-71) for parameter i with gradient g, in the
// reference's operation order, and every derived copy of it (fp32 rollout
// value, tf32 / fp16 tcgen05 images, the backward pass's transposes)
__device__ __forceinline__ void adam_one(const AdamArgs& a, double b1t_pi,
                                         double b2t_pi, double b1t_v,
                                         double b2t_v, int64_t i, double g,
                                         double* params, double* m, double* v,
                                         float* params32) {
  {
    const bool pi = i < a.n_pi;
    const double lr = pi ? a.h.lr_actor : a.h.lr_critic;
    const double b1t = pi ? b1t_pi : b1t_v;
    const double b2t = pi ? b2t_pi : b2t_v;
    double mi = __dmul_rn(m[i], a.h.beta1);
    mi = __dadd_rn(mi, __dmul_rn(a.h.one_m_beta1, g));
    double vi = __dmul_rn(v[i], a.h.beta2);
    vi = __dadd_rn(vi, __dmul_rn(a.h.one_m_beta2, __dmul_rn(g, g)));
    m[i] = mi;
    v[i] = vi;
    const double num = __dmul_rn(lr, __ddiv_rn(mi, b1t));
    const double den = __dadd_rn(__dsqrt_rn(__ddiv_rn(vi, b2t)), a.h.eps);
    const double p = __dsub_rn(params[i], __ddiv_rn(num, den));
    params[i] = p;
    const float p32 = (float)p;
    params32[i] = p32;
    for (int q = 0; q < a.pk.n_mat; ++q) {
      const PackMat& M = a.pk.mat[q];
      const int64_t e = i - M.off;
      if (e >= 0 && e < (int64_t)M.K * M.N) {
        const uint32_t ue = (uint32_t)e, un = (uint32_t)M.N;
        const int k = (int)(ue / un), nn = (int)(ue % un);
        float hi, lo;
        tc::split_tf32(p32, hi, lo);
        const uint32_t o = tc::kmajor_off(nn, k, M.Kpad) / 4;
        M.hi[o] = hi;
        M.lo[o] = lo;
        if (M.h16)
          tc::store_split_f16(p32 * *M.sc16, M.h16, M.l16,
                              tc::kmajor16_off(nn, k, M.Kpad));
      }
    }
    for (int q = 0; q < a.pk.n_vec; ++q) {
      const PackVec& V = a.pk.vec[q];
      const int64_t e = i - V.off;
      if (e >= 0 && e < V.len) V.dst[e] = p32;
    }
    dbg_ts(52);
    if (a.wt)
      for (int q = 0; q < a.tp.n; ++q) {
        const TransMat& M = a.tp.m[q];
        const int64_t e = i - M.off;
        if (e >= 0 && e < (int64_t)M.K * M.N) {
          const uint32_t ue = (uint32_t)e, un = (uint32_t)M.N;
          const int k = (int)(ue / un), nn = (int)(ue % un);
          a.wt[M.dst + (int64_t)nn * M.K + k] = p;
        }
      }
  }
}

__global__ void k_ppo_adam(const __grid_constant__ AdamArgs a,
                           const double* adam_dev, const int32_t* bad,
                           const double* grads, double* params, double* m,
                           double* v, float* params32) {
  // __grid_constant__: the pack/transposition plans are indexed with
  // runtime loop counters; a by-value param would be copied to local memory
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  dbg_ts(50);
  if (*bad) return;
  dbg_ts(51);
  adam_body(a, adam_dev, grads, params, m, v, params32);
  griddep_trigger();
}

// Grid-wide barrier for a cooperative launch (all CTAs co-resident):
// arrival count + generation word, so it needs no reset between launches
// of different grid sizes.
__device__ inline void grid_barrier(unsigned int* count, unsigned int* gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int g0;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g0) : "l"(gen));
    __threadfence();
    if (atomicAdd(count, 1u) == gridDim.x - 1) {
      atomicExch(count, 0u);
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      unsigned int g;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(gen));
      } while (g == g0);
    }
  }
  __syncthreads();
}

// (c)+(d) in one cooperative launch: every CTA writes its gradient tile
// (the extra CTA the loss means and checks), one grid barrier publishes
// them and the global finiteness flag, then every CTA runs its grid-stride
// share of Adam -- one launch and one dependency gap less per update, same
// arithmetic as k_ppo_wgrad + k_ppo_adam.
__global__ void __launch_bounds__(256)
k_ppo_wgrad_adam(const __grid_constant__ GradJobs jt, int B, int RS,
                 const double* __restrict__ rows, double* grads, int32_t* bad,
                 const double* rowout, double* losses, int means_B,
                 double w_ent, double w_val, const __grid_constant__ AdamArgs a,
                 const double* adam_dev, double* params, double* m, double* v,
                 float* params32, unsigned int* bar) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  wgrad_body(jt, B, RS, rows, grads, bad, 1, rowout, losses, means_B, w_ent,
             w_val);
  grid_barrier(bar, bar + 1);
  if (*(volatile int32_t*)bad) return;
  adam_body(a, adam_dev, grads, params, m, v, params32);
}

// (c)+(d) speculatively, no grid barrier: each gradient tile's CTA applies
// Adam to its own parameters as soon as their gradients are summed (a
// parameter's gradient is one thread's complete in-order sum over the
// batch), after saving their pre-update values (params / m / v) into the
// backup block.  The reference steps nothing when any loss or gradient is
// non-finite (ppo_update raises first, rlcore.py:368-375): here the update
// flags `bad` as before, tiles with a finite gradient have already
// stepped, and the host restores the whole backup before raising
// (DeviceAgent.restore_diverged).  Updates after a flagged one skip
// entirely: the decision reads bad[1], the snapshot of bad[0] that this
// update's k_ppo_rows took before anything of this update could set it,
// so every CTA of the flagged update itself backs up and steps alike.
struct WgSpecEpi {
  const AdamArgs* a;
  double b1t_pi, b2t_pi, b1t_v, b2t_v;
  bool skip;
  double* params;
  double* m;
  double* v;
  float* params32;
  double* bk;   // [3][n]: params, m, v before this update
  __device__ void operator()(int64_t i, double g, bool fin) const {
    if (skip || i >= a->n) return;
    const int64_t n = a->n;
    bk[i] = params[i];
    bk[n + i] = m[i];
    bk[2 * n + i] = v[i];
    if (fin) adam_one(*a, b1t_pi, b2t_pi, b1t_v, b2t_v, i, g, params, m, v, params32);
  }
};

__global__ void __launch_bounds__(256)
k_ppo_wgrad_spec(const __grid_constant__ GradJobs jt, int B, int RS,
                 const double* __restrict__ rows, double* grads, int32_t* bad,
                 const double* rowout, double* losses, int means_B,
                 double w_ent, double w_val, const __grid_constant__ AdamArgs a,
                 const double* adam_dev, double* params, double* m, double* v,
                 float* params32, double* bk) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  WgSpecEpi e;
  e.a = &a;
  e.b1t_pi = adam_dev ? adam_dev[0] : a.h.b1t_pi;
  e.b2t_pi = adam_dev ? adam_dev[1] : a.h.b2t_pi;
  e.b1t_v = adam_dev ? adam_dev[2] : a.h.b1t_v;
  e.b2t_v = adam_dev ? adam_dev[3] : a.h.b2t_v;
  e.skip = bad[1] != 0;
  e.params = params;
  e.m = m;
  e.v = v;
  e.params32 = params32;
  e.bk = bk;
  wgrad_body(jt, B, RS, rows, grads, bad, 1, rowout, losses, means_B, w_ent,
             w_val, e);
  griddep_trigger();
}

}  // namespace harl
