// K4/K5 rollout networks on CUDA cores (fp32 FFMA, accurate tanhf/exp).
// Generic over the reference's hidden sizes (tests use (16,), (32,32),
// (128,128)); the tcgen05 path (mlp_tc.cuh) takes over for the (128,128)
// production shape.  A CTA owns TM population rows; activations stay in
// shared memory between layers, weights stream from L2.
//
// K4 = select_actions (rlcore.py:216-228) fused with decode/apply
// (schedspace.py:196-301):  trunk -> 4 heads (compact tiling head) ->
// masked log-softmax (rlcore.py:185-199) -> inverse-CDF sample on the
// numpy PCG64 stream (rlcore.py:202-213) -> walker.
#pragma once

#include "common.cuh"
#include "space_kernels.cuh"

namespace harl {

constexpr int MLP_TM = 32;        // rows per CTA
constexpr int MLP_THREADS = 256;  // 8 warps

// out[TM][N] = act(in[TM][K] . W[K][N] + b); in/out in smem with leading
// dims ldi/ldo.  Thread t owns column c = t%64 (+64 j) and rows t/64 + 4 i.
__device__ inline void dense_tile(const float* in, int ldi, int K,
                                  const float* __restrict__ W,
                                  const float* __restrict__ b, int N,
                                  float* out, int ldo, bool act) {
  const int c0 = threadIdx.x & 63;
  const int rg = threadIdx.x >> 6;  // 0..3
  for (int cb = 0; cb < N; cb += 256) {
    float acc[MLP_TM / 4][4];
#pragma unroll
    for (int i = 0; i < MLP_TM / 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    for (int k = 0; k < K; ++k) {
      float w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = cb + c0 + 64 * j;
        w[j] = (c < N) ? __ldg(W + (int64_t)k * N + c) : 0.f;
      }
#pragma unroll
      for (int i = 0; i < MLP_TM / 4; ++i) {
        const float a = in[(rg + 4 * i) * ldi + k];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a, w[j], acc[i][j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = cb + c0 + 64 * j;
      if (c >= N) continue;
      const float bj = b[c];
#pragma unroll
      for (int i = 0; i < MLP_TM / 4; ++i) {
        const float z = acc[i][j] + bj;
        out[(rg + 4 * i) * ldo + c] = act ? tanhf(z) : z;
      }
    }
  }
}

// load TM fp64 feature rows, convert to fp32, zero-fill beyond n
__device__ inline void load_rows(const double* feat, int64_t r0, int64_t n,
                                 int F, float* dst, int ld) {
  for (int i = threadIdx.x; i < MLP_TM * F; i += blockDim.x) {
    const int rr = i / F, k = i % F;
    const int64_t r = r0 + rr;
    dst[rr * ld + k] = (r < n) ? (float)feat[r * F + k] : 0.f;
  }
}

// run all layers of `net` over the tile; returns pointer to the final
// activation buffer (in one of bufA/bufB), its width in *width
__device__ inline float* run_layers(const harl_mlp_desc& net, float* bufA,
                                    float* bufB, int ld, int last_linear,
                                    int* width) {
  float* cur = bufA;
  float* nxt = bufB;
  for (int l = 0; l < net.n_layers; ++l) {
    const bool act = !(last_linear && l == net.n_layers - 1);
    dense_tile(cur, ld, net.dims[l], net.W[l], net.b[l], net.dims[l + 1], nxt,
               ld, act);
    __syncthreads();
    float* t = cur;
    cur = nxt;
    nxt = t;
  }
  *width = net.dims[net.n_layers];
  return cur;
}

struct StepRng {
  u128 s;  // PCG64 state at the start of this step's random((n,1)) draws
  const int32_t* grow;  // optional global row of each local row (shards)
  int64_t m_total;      // rows drawn this step over all shards (0 -> n)
};

__device__ inline uint64_t draw_index(const StepRng& g, int h, int64_t n,
                                      int64_t r) {
  const int64_t m = g.m_total > 0 ? g.m_total : n;
  const int64_t row = g.grow ? (int64_t)g.grow[r] : r;
  return (uint64_t)h * (uint64_t)m + (uint64_t)row + 1;
}

__device__ inline double warp_max(double v) {
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ inline double warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr int SAMPLE_MAXCH = 16;  // head-0 columns up to 512

// Masked log-softmax + inverse-CDF sample over `C` columns of one row,
// computed by one warp (rlcore.py:185-213).  Lane l owns columns
// l + 32 i; bit i of `lb` says whether that column is legal.  Returns the
// chosen column (with the reference's walk-back over zero-probability
// cells) and its log-probability; -1 when the walk ends on an illegal
// column 0 (the reference then picks full index 0).
__device__ inline int warp_sample_bits(const float* z, int C, uint32_t lb,
                                       double u, double* logp_out,
                                       bool* all_masked) {
  const int lane = threadIdx.x & 31;
  const int nch = (C + 31) >> 5;
  double zmax = -INFINITY;
#pragma unroll
  for (int i = 0; i < SAMPLE_MAXCH; ++i)
    if (i < nch && ((lb >> i) & 1u)) zmax = fmax(zmax, (double)z[lane + 32 * i]);
  zmax = warp_max(zmax);
  *all_masked = (zmax == -INFINITY);
  double e[SAMPLE_MAXCH];
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < SAMPLE_MAXCH; ++i) {
    e[i] = (i < nch && ((lb >> i) & 1u)) ? exp((double)z[lane + 32 * i] - zmax) : 0.0;
    s += e[i];
  }
  s = warp_sum(s);
  const double logs = log(s);
  // inclusive prefix sum of p = e/s in column order; count c < u
  int count = 0;
  double carry = 0.0;
#pragma unroll
  for (int i = 0; i < SAMPLE_MAXCH; ++i) {
    if (i >= nch) break;
    double c = e[i] / s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double t = __shfl_up_sync(0xffffffffu, c, o);
      if (lane >= o) c += t;
    }
    c += carry;
    if (lane + 32 * i < C && c < u) ++count;
    carry = __shfl_sync(0xffffffffu, c, 31);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) count += __shfl_xor_sync(0xffffffffu, count, o);
  int idx = min(count, C - 1);
  auto legal_at = [&](int j) -> bool {
    return (__shfl_sync(0xffffffffu, lb, j & 31) >> (j >> 5)) & 1u;
  };
  while (idx > 0 && !legal_at(idx)) --idx;
  const bool ok = legal_at(idx);
  *logp_out = ok ? ((double)z[idx] - zmax - logs) : -INFINITY;
  return ok ? idx : -1;
}

// The same for a 3-column shift head, computed redundantly by every lane
// with the reference's sequential cumsum.
__device__ inline int sample3(const float* z, uint32_t m3, double u,
                              double* logp_out, bool* all_masked) {
  double zmax = -INFINITY;
  for (int j = 0; j < 3; ++j)
    if ((m3 >> j) & 1u) zmax = fmax(zmax, (double)z[j]);
  *all_masked = (zmax == -INFINITY);
  double e[3], s = 0.0;
  for (int j = 0; j < 3; ++j) {
    e[j] = ((m3 >> j) & 1u) ? exp((double)z[j] - zmax) : 0.0;
    s += e[j];
  }
  int count = 0;
  double c = 0.0;
  for (int j = 0; j < 3; ++j) {
    c += e[j] / s;
    if (c < u) ++count;
  }
  int idx = min(count, 2);
  while (idx > 0 && !((m3 >> idx) & 1u)) --idx;
  const bool ok = (m3 >> idx) & 1u;
  *logp_out = ok ? ((double)z[idx] - zmax - log(s)) : -INFINITY;
  return ok ? idx : -1;
}

__device__ inline double logp3(const float* z, uint32_t m3, int a) {
  if (a < 0 || a > 2 || !((m3 >> a) & 1u)) return -INFINITY;
  double zmax = -INFINITY, s = 0.0;
  for (int j = 0; j < 3; ++j)
    if ((m3 >> j) & 1u) zmax = fmax(zmax, (double)z[j]);
  for (int j = 0; j < 3; ++j)
    if ((m3 >> j) & 1u) s += exp((double)z[j] - zmax);
  return (double)z[a] - zmax - log(s);
}

// decode + apply for one row by a whole warp (schedspace.py:196-210,
// 265-301): lane l writes slots l and l+32 of the new state; the checks
// follow the reference's order and are warp-uniform.
__device__ inline int apply_row_warp(const harl_sketch_desc& sk, int tv0,
                                     int tv1, int ca0, int par0, int ur0,
                                     const int* act, uint16_t* __restrict__ tiles_out,
                                     uint8_t* __restrict__ knobs_out, int64_t ld,
                                     int64_t r) {
  const int lane = threadIdx.x & 31;
  const int S = sk.num_slots, L = sk.levels;
  int src = -1, dst = -1;
  if (act[0] != S * S) {
    src = act[0] / S;
    dst = act[0] % S;
  }
  int code = HARL_ST_OK;
  int f_src = 0, f_dst = 0, p = 1;
  if (src >= 0) {
    if (src >= sk.local_slots || dst >= sk.local_slots || dst < 0 ||
        src / L != dst / L || src == dst) {
      code = HARL_ST_TILING;
    } else {
      f_src = __shfl_sync(0xffffffffu, src < 32 ? tv0 : tv1, src & 31);
      f_dst = __shfl_sync(0xffffffffu, dst < 32 ? tv0 : tv1, dst & 31);
      if (f_src <= 1) code = HARL_ST_TILING;
      else p = sk.spf_lut[f_src];
    }
  }
  if (code == HARL_ST_OK) {
    const int ca = ca0 + (act[1] - 1);
    const int par = par0 + (act[2] - 1);
    const int ur = ur0 + (act[3] - 1);
    if (ca < 0 || ca >= sk.ncas) code = HARL_ST_COMPUTE_AT;
    else if (par < 0 || par > sk.max_fusible) code = HARL_ST_PARALLEL;
    else if (ur < 0 || ur >= sk.n_unroll) code = HARL_ST_UNROLL;
    if (code == HARL_ST_OK && lane == 0) {
      knobs_out[r] = (uint8_t)ca;
      knobs_out[ld + r] = (uint8_t)par;
      knobs_out[2 * ld + r] = (uint8_t)ur;
    }
  }
  const bool moved = code == HARL_ST_OK && src >= 0;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int s = lane + 32 * half;
    if (s < sk.local_slots) {
      int v = half ? tv1 : tv0;
      if (moved && s == src) v = f_src / p;
      if (moved && s == dst) v = f_dst * p;
      tiles_out[(int64_t)s * ld + r] = (uint16_t)v;
    }
  }
  return code;
}

// Sampling epilogue for one row, executed by one warp: masked
// log-softmax per head, inverse-CDF draw on the PCG64 stream (or the
// injected action), then decode + apply.  Shared by the FFMA and tcgen05
// policy kernels.
__device__ inline void policy_row(
    const harl_sketch_desc& sk, const PcgJump& J, const StepRng& rng,
    const float* z, int NH, const uint16_t* tiles, const uint8_t* knobs,
    int64_t n, int64_t ld, int64_t r, const int32_t* inject, int32_t* actions,
    double* logp, uint16_t* tiles_out, uint8_t* knobs_out, uint64_t* move_bits,
    uint32_t* shift_bits, int32_t* head0_col, float* logits_out,
    unsigned long long* status, const int16_t* src_tab,
    const int16_t* dst_tab) {
  const int lane = threadIdx.x & 31;
  const int C0 = sk.n_head0;
  const int S = sk.num_slots;
  {
    if (logits_out)
      for (int j = lane; j < NH; j += 32) logits_out[r * NH + j] = z[j];
    // this lane's tile factors (slots lane, lane+32) and the movable mask
    const int tv0 = lane < sk.local_slots ? tiles[(int64_t)lane * ld + r] : 0;
    const int tv1 = lane + 32 < sk.local_slots ? tiles[(int64_t)(lane + 32) * ld + r] : 0;
    const uint64_t mv = (uint64_t)__ballot_sync(0xffffffffu, tv0 > 1) |
                        ((uint64_t)__ballot_sync(0xffffffffu, tv1 > 1) << 32);
    const int ca = knobs[r], par = knobs[ld + r], ur = knobs[2 * ld + r];
    const uint32_t sb = shift_bits_of(sk, ca, par, ur);
    int act[4];
    int col0 = 0;
    double lp_total = 0.0;
    bool dead = false;
    // head 0: compact tiling columns (no-op last); legal bits of my columns
    uint32_t lb = 0;
    for (int i = 0; (lane + 32 * i) < C0; ++i) {
      const int j = lane + 32 * i;
      const int src = src_tab[j];
      if (j == C0 - 1 || (src < sk.local_slots && ((mv >> src) & 1ull)))
        lb |= 1u << i;
    }
    {
      double lp;
      bool none;
      double u = 0.0;
      if (!inject) u = u64_to_unit(pcg_draw64(J, rng.s, draw_index(rng, 0, n, r)));
      const int j = warp_sample_bits(z, C0, lb, u, &lp, &none);
      dead |= none;
      if (inject) {
        const int a = inject[r];
        // full index -> compact column (if in the legal superset)
        int jj = -1;
        for (int c = lane; c < C0; c += 32) {
          const int full = (c == C0 - 1) ? S * S : src_tab[c] * S + dst_tab[c];
          if (full == a) jj = c;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) jj = max(jj, __shfl_xor_sync(0xffffffffu, jj, o));
        act[0] = a;
        col0 = jj < 0 ? 0 : jj;
        const bool ok = jj >= 0 &&
            ((__shfl_sync(0xffffffffu, lb, jj & 31) >> (jj >> 5)) & 1u);
        if (ok) {
          // log-prob of the injected column under the same softmax
          double zm = -INFINITY, ss = 0.0;
          for (int i = 0; (lane + 32 * i) < C0; ++i)
            if ((lb >> i) & 1u) zm = fmax(zm, (double)z[lane + 32 * i]);
          zm = warp_max(zm);
          for (int i = 0; (lane + 32 * i) < C0; ++i)
            if ((lb >> i) & 1u) ss += exp((double)z[lane + 32 * i] - zm);
          ss = warp_sum(ss);
          lp = (double)z[jj] - zm - log(ss);
        } else {
          lp = -INFINITY;
        }
      } else {
        act[0] = (j < 0) ? 0 : ((j == C0 - 1) ? S * S : src_tab[j] * S + dst_tab[j]);
        col0 = j < 0 ? 0 : j;
      }
      lp_total += lp;
    }
    // shift heads: 3 columns each at offsets C0, C0+3, C0+6
    for (int h = 1; h < 4; ++h) {
      const uint32_t m3 = (sb >> (3 * (h - 1))) & 7u;
      const float* zh = z + C0 + 3 * (h - 1);
      double lp;
      bool none;
      if (inject) {
        const int a = inject[h * n + r];
        act[h] = a;
        lp = logp3(zh, m3, a);
        none = m3 == 0;
      } else {
        const double u = u64_to_unit(pcg_draw64(J, rng.s, draw_index(rng, h, n, r)));
        const int j = sample3(zh, m3, u, &lp, &none);
        act[h] = (j < 0) ? 0 : j;
      }
      dead |= none;
      lp_total += lp;
    }
    const int code = dead ? HARL_ST_NO_VALID
                          : apply_row_warp(sk, tv0, tv1, ca, par, ur, act,
                                           tiles_out, knobs_out, ld, r);
    if (lane == 0) {
      for (int h = 0; h < 4; ++h) actions[h * n + r] = act[h];
      logp[r] = lp_total;
      move_bits[r] = mv;
      shift_bits[r] = sb;
      head0_col[r] = col0;
      report_status(status, r, code);
    }
    __syncwarp();
  }
}

__global__ void __launch_bounds__(MLP_THREADS)
k_policy_step(const __grid_constant__ harl_sketch_desc sk,
              const __grid_constant__ harl_mlp_desc net,
              const __grid_constant__ PcgJump J, StepRng rng,
              const double* feat, const uint16_t* tiles, const uint8_t* knobs,
              int64_t n, int64_t ld, const int32_t* inject, int32_t* actions,
              double* logp, uint16_t* tiles_out, uint8_t* knobs_out,
              uint64_t* move_bits, uint32_t* shift_bits, int32_t* head0_col,
              float* logits_out, unsigned long long* status, int ldbuf) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  extern __shared__ float smem[];
  float* bufA = smem;
  float* bufB = smem + MLP_TM * ldbuf;
  const int64_t r0 = (int64_t)blockIdx.x * MLP_TM;
  const int F = sk.feature_len;
  load_rows(feat, r0, n, F, bufA, ldbuf);
  __syncthreads();
  int width;
  float* hid = run_layers(net, bufA, bufB, ldbuf, 0, &width);
  float* logits = (hid == bufA) ? bufB : bufA;
  const int NH = net.n_head_cols;  // n_head0 + 9
  dense_tile(hid, ldbuf, width, net.head_W, net.head_b, NH, logits, ldbuf, false);
  __syncthreads();

  __shared__ int16_t s_src[HARL_MAX_HEAD0], s_dst[HARL_MAX_HEAD0];
  for (int i = threadIdx.x; i < sk.n_head0; i += blockDim.x) {
    s_src[i] = sk.head0_src[i];
    s_dst[i] = sk.head0_dst[i];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  for (int rr = warp; rr < MLP_TM; rr += MLP_THREADS / 32) {
    const int64_t r = r0 + rr;
    if (r >= n) break;
    policy_row(sk, J, rng, logits + rr * ldbuf, NH, tiles, knobs, n, ld, r,
               inject, actions, logp, tiles_out, knobs_out, move_bits,
               shift_bits, head0_col, logits_out, status, s_src, s_dst);
  }
}

// ValueNet.estimate (rlcore.py:161-178): hidden tanh layers, last layer
// linear (width 1).
__global__ void __launch_bounds__(MLP_THREADS)
k_value_forward(const __grid_constant__ harl_mlp_desc net, const double* feat,
                int64_t n, int32_t F, float* v_out, int ldbuf) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  extern __shared__ float smem[];
  float* bufA = smem;
  float* bufB = smem + MLP_TM * ldbuf;
  const int64_t r0 = (int64_t)blockIdx.x * MLP_TM;
  load_rows(feat, r0, n, F, bufA, ldbuf);
  __syncthreads();
  harl_mlp_desc hidden = net;
  hidden.n_layers = net.n_layers - 1;
  int width;
  float* hid = run_layers(hidden, bufA, bufB, ldbuf, 0, &width);
  const float* w = net.W[net.n_layers - 1];
  const float b = net.b[net.n_layers - 1][0];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int rr = warp; rr < MLP_TM; rr += MLP_THREADS / 32) {
    const int64_t r = r0 + rr;
    if (r >= n) break;
    float acc = 0.f;
    for (int k = lane; k < width; k += 32) acc = fmaf(hid[rr * ldbuf + k], __ldg(w + k), acc);
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) v_out[r] = acc + b;
  }
}

}  // namespace harl
