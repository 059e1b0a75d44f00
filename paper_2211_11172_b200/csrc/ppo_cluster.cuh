// K7(a) on thread-block clusters: the per-row PPO work (rlcore.py:293-358;
// Mlp.backward 105-116, PolicyNet.backward 148-158) for the production
// network shape (hidden (128, 128), feature_len <= 64, policy head columns
// <= 128), in fp64 on the DMMA tensor cores.
//
// k_ppo_rows (ppo_kernels.cuh) gives every CTA 2 minibatch rows and all
// of a net's weights, streamed from L2: ~800 KB of weight reads per CTA and
// a dependent load chain per layer.  Here a cluster of 8 CTAs owns 32 rows
// and each CTA owns a 16-column slice of every layer, its weight slices
// resident in shared memory for the launch:
//   * a layer is [32 x K] . [K x 16] per CTA: 8 warps, one 8x8 output tile
//     each, mma.m8n8k4.f64 over K with two accumulator chains (fragment
//     loads are conflict-free: activation rows padded to 132 doubles,
//     weight slices to 20);
//   * its 16 output columns are pushed into the 7 peer CTAs' copies of the
//     activation block (distributed shared memory), then one cluster
//     barrier -- every CTA holds the full [32 x 128] input of the next layer;
//   * the loss terms (masked log-softmax per head, entropy, clipped ratio,
//     dz) run on CTA c's 4 rows, and the dz rows are pushed the same way;
//   * the backward layers use row slices of W (W[k][:] for the CTA's k).
// blockIdx.y = 0: policy chain, 1: value chain (they share only X).
// Output: the same per-row [X | acts | dz | deltas] rows and rowout terms
// as k_ppo_rows, which k_ppo_wgrad / k_ppo_adam then consume unchanged.
// Arithmetic: the same fp64 operations in another summation order (the
// parity tests' PPO tolerance).
#pragma once

#include <cooperative_groups.h>

#include "ppo_kernels.cuh"

namespace harl {

constexpr int PCL_CTAS = 8;          // CTAs per cluster
constexpr int PCL_R = 32;            // minibatch rows per cluster
constexpr int PCL_THREADS = 256;     // 8 warps: one 8x8 output tile each
constexpr int PCL_H = 128;           // hidden width
constexpr int PCL_NC = PCL_H / PCL_CTAS;   // columns per CTA
constexpr int PCL_LDA = PCL_H + 4;   // activation row stride (== 4 mod 16)
constexpr int PCL_LDW = PCL_NC + 4;  // column-slice stride   (== 4 mod 16)
constexpr int PCL_KX = 64;           // feature_len bound (X padded to 4)

struct PclLayout {   // offsets in doubles of the dynamic shared memory
  int x, a1, a2, z, w1c, w2c, whc, w2r, whr, b, total;
  int ldx;
};

__host__ __device__ inline PclLayout pcl_layout(int F) {
  PclLayout L;
  const int kx = (F + 3) / 4 * 4;
  L.ldx = kx + ((4 - kx % 16) + 16) % 16;   // >= kx, == 4 mod 16
  int o = 0;
  L.x = o;   o += PCL_R * L.ldx;
  L.a1 = o;  o += PCL_R * PCL_LDA;
  L.a2 = o;  o += PCL_R * PCL_LDA;   // also delta2 (in place)
  L.z = o;   o += PCL_R * PCL_LDA;   // logits -> dz (policy only)
  L.w1c = o; o += kx * PCL_LDW;
  L.w2c = o; o += PCL_H * PCL_LDW;
  L.whc = o; o += PCL_H * PCL_LDW;   // value: w3 (128)
  L.w2r = o; o += PCL_NC * PCL_LDA;
  L.whr = o; o += PCL_NC * PCL_LDA;
  L.b = o;   o += 3 * PCL_H + 2 * PCL_R;   // biases, v, dv
  L.total = o;
  return L;
}
__host__ __device__ inline size_t pcl_smem_bytes(int F) {
  return sizeof(double) * (size_t)pcl_layout(F).total;
}

// D(8x8) += A(8 x K) . B(K x 8): A rows at a (stride lda), element (k, n)
// of B at b[k * ldb + n] (BT: at b[n * ldb + k]); K a multiple of 4 with
// zero padding.  Two accumulator chains (even / odd k-steps).
template <bool BT>
__device__ __forceinline__ void pcl_tile(const double* a, int lda,
                                         const double* b, int ldb, int K,
                                         double& d0, double& d1) {
  const int lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
  const double* ap = a + gid * lda + tig;
  const double* bp = BT ? b + gid * ldb + tig : b + tig * ldb + gid;
  double e0 = 0.0, e1 = 0.0, f0 = 0.0, f1 = 0.0;
  int k = 0;
#pragma unroll 4
  for (; k + 8 <= K; k += 8) {
    const double a0 = ap[k], a1 = ap[k + 4];
    const double b0 = BT ? bp[k] : bp[k * ldb];
    const double b1 = BT ? bp[k + 4] : bp[(k + 4) * ldb];
    dmma884(e0, e1, a0, b0);
    dmma884(f0, f1, a1, b1);
  }
  if (k < K) dmma884(e0, e1, ap[k], BT ? bp[k] : bp[k * ldb]);
  d0 = e0 + f0;
  d1 = e1 + f1;
}

// push this CTA's 16 columns [c0, c0+16) of a [32][PCL_LDA] block to the
// other CTAs of the cluster, then a cluster barrier (release/acquire)
__device__ __forceinline__ void pcl_allgather(double* blk, int c0,
                                              bool stamp = false) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned me = cl.block_rank();
  __syncthreads();
  if (stamp) dbg_ts(57);
  // 32 rows x 8 double2 per peer: one double2 per thread per peer
  // (st.shared::cluster to the mapa-translated address)
  const int r = threadIdx.x >> 3, q = threadIdx.x & 7;
  double* src = blk + r * PCL_LDA + c0 + 2 * q;
  const double2 v = *reinterpret_cast<const double2*>(src);
  const uint32_t la = (uint32_t)__cvta_generic_to_shared(src);
#pragma unroll
  for (int p = 1; p < PCL_CTAS; ++p) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                 : "=r"(ra) : "r"(la), "r"((me + p) % PCL_CTAS));
    asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};"
                 ::"r"(ra), "d"(v.x), "d"(v.y) : "memory");
  }
  if (stamp) dbg_ts(58);
  cl.sync();
  if (stamp) dbg_ts(59);
}

__global__ void __cluster_dims__(PCL_CTAS, 1, 1) __launch_bounds__(PCL_THREADS, 1)
k_ppo_rows_cl(const __grid_constant__ PpoArgs a,
              const __grid_constant__ NetLayout P,
              const __grid_constant__ NetLayout V, PpoRing ring,
              const int32_t* idx, const double* params, double* rows,
              double* rowout) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) double pcs[];
  const int F = a.F, RS = a.row_stride, B = a.B;
  const PclLayout L = pcl_layout(F);
  const int kx = (F + 3) / 4 * 4;
  const int role = blockIdx.y;
  const NetLayout& N = role == 0 ? P : V;
  const int c = (int)cl.block_rank();
  const int c0 = c * PCL_NC;
  const int b0 = (int)(blockIdx.x / PCL_CTAS) * PCL_R;
  const int nrows = min(PCL_R, B - b0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NH = P.n_head_cols;
  double* X = pcs + L.x;
  double* A1 = pcs + L.a1;
  double* A2 = pcs + L.a2;
  double* Z = pcs + L.z;
  double* W1c = pcs + L.w1c;
  double* W2c = pcs + L.w2c;
  double* Whc = pcs + L.whc;
  double* W2r = pcs + L.w2r;
  double* Whr = pcs + L.whr;
  double* bs = pcs + L.b;             // b1 [128], b2 [128], bh / w3 [128]
  double* vv = bs + 3 * PCL_H;        // value: v [32], dv [32]
  __shared__ int16_t s_src[HARL_MAX_HEAD0];
  __shared__ double s_lp[4][4], s_ent[4][4];
  // ---- weight slices and the cluster's X rows (the ring rows come from
  // the preceding step kernels: everything follows the PDL wait) ---------
  griddep_wait();
  if (a.bad && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
    a.bad[1] = a.bad[0];   // the speculative Adam's per-update snapshot
  dbg_ts(40);
  // asynchronous 8-byte copies (no register staging, every load in flight
  // at once; rows of Wh / X need not be 16-byte aligned); padding is stored
  // as zeros directly
  auto cp8 = [](double* dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
  };
  const double* W1 = params + N.off_W[0];
  const double* W2 = params + N.off_W[1];
  for (int i = tid; i < kx * PCL_NC; i += PCL_THREADS) {
    const int k = i / PCL_NC, j = i % PCL_NC;
    if (k < F) cp8(&W1c[k * PCL_LDW + j], &W1[(int64_t)k * PCL_H + c0 + j]);
    else W1c[k * PCL_LDW + j] = 0.0;
  }
  for (int i = tid; i < PCL_H * PCL_NC; i += PCL_THREADS) {
    const int k = i / PCL_NC, j = i % PCL_NC;
    cp8(&W2c[k * PCL_LDW + j], &W2[(int64_t)k * PCL_H + c0 + j]);
  }
  // row slice of W2: W2r[kk][n] = W2[c0 + kk][n] (the backward's W^T)
  for (int i = tid; i < PCL_NC * PCL_H; i += PCL_THREADS) {
    const int kk = i / PCL_H, n = i % PCL_H;
    cp8(&W2r[kk * PCL_LDA + n], &W2[(int64_t)(c0 + kk) * PCL_H + n]);
  }
  for (int i = tid; i < PCL_H; i += PCL_THREADS) {
    cp8(&bs[i], &params[N.off_b[0] + i]);
    cp8(&bs[PCL_H + i], &params[N.off_b[1] + i]);
  }
  const int kh = (NH + 3) / 4 * 4;   // the heads' backward reduction length
  if (role == 0) {
    const double* Wh = params + P.off_hW;
    for (int i = tid; i < PCL_H * PCL_NC; i += PCL_THREADS) {
      const int k = i / PCL_NC, j = i % PCL_NC;
      if (c0 + j < NH) cp8(&Whc[k * PCL_LDW + j], &Wh[(int64_t)k * NH + c0 + j]);
      else Whc[k * PCL_LDW + j] = 0.0;
    }
    for (int i = tid; i < PCL_NC * PCL_H; i += PCL_THREADS) {
      const int kk = i / PCL_H, j = i % PCL_H;
      if (j < NH) cp8(&Whr[kk * PCL_LDA + j], &Wh[(int64_t)(c0 + kk) * NH + j]);
      else Whr[kk * PCL_LDA + j] = 0.0;
    }
    for (int i = tid; i < PCL_H; i += PCL_THREADS) {
      if (i < NH) cp8(&bs[2 * PCL_H + i], &params[P.off_hb + i]);
      else bs[2 * PCL_H + i] = 0.0;
    }
    for (int i = tid; i < a.C0; i += PCL_THREADS) s_src[i] = a.head0_src[i];
  } else {
    for (int i = tid; i < PCL_H; i += PCL_THREADS)
      cp8(&bs[2 * PCL_H + i], &params[V.off_W[2] + i]);   // w3 [128][1]
  }
  // X rows of the cluster (zero past B and past F)
  for (int i = tid; i < PCL_R * kx; i += PCL_THREADS) {
    const int r = i / kx, k = i % kx;
    if (r < nrows && k < F) cp8(&X[r * L.ldx + k], &ring.X[(int64_t)idx[b0 + r] * F + k]);
    else X[r * L.ldx + k] = 0.0;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  dbg_ts(41);
  // every CTA of the cluster is running before any shared memory of it is
  // written remotely (and the staging above is complete)
  cl.sync();
  const int rt = warp & 3, ct = warp >> 2;   // this warp's 8x8 output tile
  const int gid = lane >> 2, tig = lane & 3;
  const int orow = rt * 8 + gid;             // tile rows held by the lane
  const int ocol = c0 + ct * 8 + 2 * tig;    // global column (and +1)
  auto store_rows = [&](int seg, const double* blk, int ld) {
    // this CTA's 16 columns of rows b0.. (row-major [B][RS] rows)
    for (int i = tid; i < nrows * PCL_NC; i += PCL_THREADS) {
      const int r = i / PCL_NC, j = i % PCL_NC;
      rows[(int64_t)(b0 + r) * RS + seg + c0 + j] = blk[r * ld + c0 + j];
    }
  };
  // ---- forward trunk: A1 = tanh(X W1 + b1), A2 = tanh(A1 W2 + b2) -------
  {
    double d0, d1;
    pcl_tile<false>(X + rt * 8 * L.ldx, L.ldx, W1c + ct * 8, PCL_LDW, kx, d0, d1);
    A1[orow * PCL_LDA + ocol] = tanh(d0 + bs[ocol]);
    A1[orow * PCL_LDA + ocol + 1] = tanh(d1 + bs[ocol + 1]);
  }
  pcl_allgather(A1, c0);
  {
    double d0, d1;
    dbg_ts(47);
    pcl_tile<false>(A1 + rt * 8 * PCL_LDA, PCL_LDA, W2c + ct * 8, PCL_LDW,
                    PCL_H, d0, d1);
    A2[orow * PCL_LDA + ocol] = tanh(d0 + bs[PCL_H + ocol]);
    A2[orow * PCL_LDA + ocol + 1] = tanh(d1 + bs[PCL_H + ocol + 1]);
  }
  dbg_ts(44);
  pcl_allgather(A2, c0, true);
  dbg_ts(42);
  store_rows(N.row_act[1], A1, PCL_LDA);
  store_rows(N.row_act[2], A2, PCL_LDA);
  if (role == 0 && c == 0)
    for (int i = tid; i < nrows * F; i += PCL_THREADS) {
      const int r = i / F, k = i % F;
      rows[(int64_t)(b0 + r) * RS + P.row_act[0] + k] = X[r * L.ldx + k];
    }
  const double invB = 1.0 / (double)a.B_norm;
  if (role == 0) {
    // ---- heads: Z = A2 Wh + bh (columns >= NH stay zero) ----------------
    {
      double d0, d1;
      pcl_tile<false>(A2 + rt * 8 * PCL_LDA, PCL_LDA, Whc + ct * 8, PCL_LDW,
                      PCL_H, d0, d1);
      Z[orow * PCL_LDA + ocol] = d0 + bs[2 * PCL_H + ocol];
      Z[orow * PCL_LDA + ocol + 1] = d1 + bs[2 * PCL_H + ocol + 1];
    }
    pcl_allgather(Z, c0);
    dbg_ts(43);
    // ---- loss terms on rows 4c .. 4c+3: warp w -> row 4c + w/2, heads
    // 2(w&1), 2(w&1)+1 (rlcore.py:293-358) --------------------------------
    const int rr = 4 * c + (warp >> 1);
    const bool live = rr < nrows;
    const int slot = live ? idx[b0 + rr] : 0;
    const uint64_t mv = live ? ring.move_bits[slot] : 0;
    const uint32_t sb = live ? ring.shift_bits[slot] : 0;
    double* z = Z + rr * PCL_LDA;
    constexpr int HI = 4;                    // cached columns per lane
    double ev[2][HI], hm[2], hs[2], hls[2], hent[2];
    int cols[2];
    for (int q = 0; q < 2; ++q) {
      const int h = 2 * (warp & 1) + q;
      const int cb = h == 0 ? 0 : a.C0 + 3 * (h - 1);
      const int C = h == 0 ? a.C0 : 3;
      auto legal = [&](int j) -> bool {
        if (h == 0) return j == a.C0 - 1 || ((mv >> s_src[j]) & 1ull);
        return (sb >> (3 * (h - 1) + j)) & 1u;
      };
      double m = -INFINITY;
      for (int j = lane; j < C; j += 32)
        if (legal(j)) m = fmax(m, z[cb + j]);
      m = wmax64(m);
      double sacc = 0.0;
#pragma unroll
      for (int i = 0; i < HI; ++i) {
        const int j = lane + 32 * i;
        ev[q][i] = (j < C && legal(j)) ? exp(z[cb + j] - m) : 0.0;
        sacc += ev[q][i];
      }
      const double sh = wsum64(sacc);
      const double ls = log(sh);
      double e = 0.0;
#pragma unroll
      for (int i = 0; i < HI; ++i) {
        const int j = lane + 32 * i;
        if (j < C && legal(j)) e -= (ev[q][i] / sh) * (z[cb + j] - m - ls);
      }
      e = wsum64(e);
      hm[q] = m;
      hs[q] = sh;
      hls[q] = ls;
      hent[q] = e;
      cols[q] = live ? ring.actions[slot * 4 + h] : 0;
      if (lane == 0) {
        s_lp[warp >> 1][h] = z[cb + cols[q]] - m - ls;
        s_ent[warp >> 1][h] = e;
      }
    }
    __syncthreads();
    if (live) {
      const int rq = warp >> 1;
      const double logp_new = ((s_lp[rq][0] + s_lp[rq][1]) + s_lp[rq][2]) + s_lp[rq][3];
      const double ent_total = ((s_ent[rq][0] + s_ent[rq][1]) + s_ent[rq][2]) + s_ent[rq][3];
      const double logp_old = ring.scalars[slot * 4 + 0];
      const double adv = ring.scalars[slot * 4 + 2];
      const double ratio = exp(logp_new - logp_old);
      const double clipped = fmin(fmax(ratio, a.clip_lo), a.clip_hi);
      const double s_un = ratio * adv, s_cl = clipped * adv;
      const double coef = (s_un <= s_cl) ? ratio * adv : 0.0;
      const double dlogp = -coef * invB;
      const double went = a.w_ent * invB;
      for (int q = 0; q < 2; ++q) {
        const int h = 2 * (warp & 1) + q;
        const int cb = h == 0 ? 0 : a.C0 + 3 * (h - 1);
        const int C = h == 0 ? a.C0 : 3;
        auto legal = [&](int j) -> bool {
          if (h == 0) return j == a.C0 - 1 || ((mv >> s_src[j]) & 1ull);
          return (sb >> (3 * (h - 1) + j)) & 1u;
        };
#pragma unroll
        for (int i = 0; i < HI; ++i) {
          const int j = lane + 32 * i;
          if (j >= C) continue;
          const double onehot = j == cols[q] ? 1.0 : 0.0;
          double dz;
          if (legal(j)) {
            const double lp = z[cb + j] - hm[q] - hls[q];
            const double p = ev[q][i] / hs[q];
            dz = dlogp * (onehot - p) + went * p * (lp + hent[q]);
          } else {
            dz = dlogp * (onehot - 0.0);
          }
          z[cb + j] = dz;
        }
      }
      if ((warp & 1) == 0 && lane == 0) {
        double* o = rowout + (int64_t)(b0 + rr) * 4;
        o[0] = fmin(s_un, s_cl);
        o[1] = ent_total;
        o[2] = ratio;
      }
    }
    // dz rows 4c..4c+3 -> global rows and the peers' Z blocks
    __syncthreads();
    dbg_ts(45);
    for (int i = tid; i < 4 * NH; i += PCL_THREADS) {
      const int q = i / NH, j = i % NH;
      if (4 * c + q < nrows)
        rows[(int64_t)(b0 + 4 * c + q) * RS + P.row_head + j] =
            Z[(4 * c + q) * PCL_LDA + j];
    }
    {
      const unsigned me = cl.block_rank();
      for (int p = 1; p < PCL_CTAS; ++p) {
        double* dst = cl.map_shared_rank(Z, (me + p) % PCL_CTAS);
        for (int i = tid; i < 4 * NH; i += PCL_THREADS) {
          const int q = i / NH, j = i % NH;
          dst[(4 * c + q) * PCL_LDA + j] = Z[(4 * c + q) * PCL_LDA + j];
        }
      }
      cl.sync();
    }
    // ---- backward: delta2 = (dz Wh^T) * (1 - A2^2), in place over A2 ----
    {
      double d0, d1;
      pcl_tile<true>(Z + rt * 8 * PCL_LDA, PCL_LDA, Whr + ct * 8 * PCL_LDA,
                     PCL_LDA, kh, d0, d1);
      double* p2 = A2 + orow * PCL_LDA + ocol;
      p2[0] = d0 * (1.0 - p2[0] * p2[0]);
      p2[1] = d1 * (1.0 - p2[1] * p2[1]);
    }
  } else {
    // ---- value output: v = A2 w3 + b3 (every CTA, all 32 rows), the
    // squared error and dv = w 2 (v - td) / B (rlcore.py:161-178, 340-345)
    const double* w3 = bs + 2 * PCL_H;
    const double b3 = params[V.off_b[2]];
    for (int q = 0; q < 4; ++q) {
      const int r = 4 * warp + q;
      double acc = 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        acc = fma(A2[r * PCL_LDA + lane + 32 * i], w3[lane + 32 * i], acc);
      acc = wsum64(acc);
      if (lane == 0) {
        const double v = acc + b3;
        double dv = 0.0;
        if (r < nrows) {
          const double td = ring.scalars[(int64_t)idx[b0 + r] * 4 + 3];
          dv = a.w_val * 2.0 * (v - td) * invB;
          if (c == 0) {
            rowout[(int64_t)(b0 + r) * 4 + 3] = (v - td) * (v - td);
            rows[(int64_t)(b0 + r) * RS + V.row_act[3]] = v;
            rows[(int64_t)(b0 + r) * RS + V.row_delta[2]] = dv;
          }
        }
        vv[PCL_R + r] = dv;
      }
    }
    // every CTA of the cluster has read all of A2 before any overwrites
    // its columns with delta_v1 and pushes them
    cl.sync();
    // delta_v1 = dv w3^T * (1 - A2^2), in place over A2
    double* p2 = A2 + orow * PCL_LDA + ocol;
    const double dv = vv[PCL_R + orow];
    p2[0] = dv * w3[ocol] * (1.0 - p2[0] * p2[0]);
    p2[1] = dv * w3[ocol + 1] * (1.0 - p2[1] * p2[1]);
  }
  // ---- delta2 (policy) / delta_v1 (value): store, gather, back through
  // W2: delta1 = (delta2 W2^T) * (1 - A1^2) ---------------------------------
  const int seg_d2 = role == 0 ? P.row_delta[1] : V.row_delta[1];
  const int seg_d1 = role == 0 ? P.row_delta[0] : V.row_delta[0];
  pcl_allgather(A2, c0);
  dbg_ts(46);
  store_rows(seg_d2, A2, PCL_LDA);
  {
    double d0, d1;
    pcl_tile<true>(A2 + rt * 8 * PCL_LDA, PCL_LDA, W2r + ct * 8 * PCL_LDA,
                   PCL_LDA, PCL_H, d0, d1);
    const double* p1 = A1 + orow * PCL_LDA + ocol;
    if (orow < nrows) {
      double* o = rows + (int64_t)(b0 + orow) * RS + seg_d1 + ocol;
      o[0] = d0 * (1.0 - p1[0] * p1[0]);
      o[1] = d1 * (1.0 - p1[1] * p1[1]);
    }
  }
  // (the last remote stores precede the cluster barrier of the gather)
  griddep_trigger();
  dbg_ts(48);
}

}  // namespace harl
