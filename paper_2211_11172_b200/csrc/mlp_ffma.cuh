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
};

__device__ inline double warp_max(double v) {
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ inline double warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Masked log-softmax + inverse-CDF sample over `C` columns of one row,
// computed by one warp.  legal(j) supplied as a predicate functor.
// Returns the chosen column (walk-back semantics of rlcore.py:206-212) and
// its log-probability; *all_masked set when no column is legal.
template <typename Legal>
__device__ inline int warp_sample(const float* z, int C, Legal legal, double u,
                                  double* logp_out, bool* all_masked) {
  const int lane = threadIdx.x & 31;
  double zmax = -INFINITY;
  for (int j = lane; j < C; j += 32)
    if (legal(j)) zmax = fmax(zmax, (double)z[j]);
  zmax = warp_max(zmax);
  *all_masked = (zmax == -INFINITY);
  double s = 0.0;
  for (int j = lane; j < C; j += 32)
    if (legal(j)) s += exp((double)z[j] - zmax);
  s = warp_sum(s);
  const double logs = log(s);
  // inclusive prefix sum in column order, chunk by chunk; count c < u
  int count = 0;
  double carry = 0.0;
  for (int base = 0; base < C; base += 32) {
    const int j = base + lane;
    double p = (j < C && legal(j)) ? exp((double)z[j] - zmax) / s : 0.0;
    double c = p;
    for (int o = 1; o < 32; o <<= 1) {
      const double t = __shfl_up_sync(0xffffffffu, c, o);
      if (lane >= o) c += t;
    }
    c += carry;
    if (j < C && c < u) ++count;
    carry = __shfl_sync(0xffffffffu, c, 31);
  }
  for (int o = 16; o; o >>= 1) count += __shfl_xor_sync(0xffffffffu, count, o);
  int idx = min(count, C - 1);
  // float-edge landing on a zero-probability cell: walk back
  while (idx > 0 && !legal(idx)) --idx;
  const bool ok = legal(idx);
  *logp_out = ok ? ((double)z[idx] - zmax - logs) : -INFINITY;
  return ok ? idx : -1;  // -1: reference would land on full index 0
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
    unsigned long long* status) {
  const int lane = threadIdx.x & 31;
  const int C0 = sk.n_head0;
  const int S = sk.num_slots;
  {
    if (logits_out)
      for (int j = lane; j < NH; j += 32) logits_out[r * NH + j] = z[j];
    // movable slots of the current state
    uint64_t mv = 0;
    for (int s0 = 0; s0 < sk.local_slots; s0 += 32) {
      const int s = s0 + lane;
      const bool m = (s < sk.local_slots) && tiles[(int64_t)s * ld + r] > 1;
      mv |= (uint64_t)__ballot_sync(0xffffffffu, m) << s0;
    }
    const int ca = knobs[r], par = knobs[ld + r], ur = knobs[2 * ld + r];
    const uint32_t sb = shift_bits_of(sk, ca, par, ur);
    int act[4];
    int col0 = 0;
    double lp_total = 0.0;
    bool dead = false;
    // head 0: compact tiling columns (no-op last)
    {
      auto legal = [&](int j) -> bool {
        if (j == C0 - 1) return true;
        const int src = sk.head0_src[j];
        return src < sk.local_slots && ((mv >> src) & 1ull);
      };
      double lp;
      bool none;
      double u = 0.0;
      if (!inject) u = u64_to_unit(pcg_draw64(J, rng.s, (uint64_t)r + 1));
      int j = warp_sample(z, C0, legal, u, &lp, &none);
      dead |= none;
      if (inject) {
        const int a = inject[r];
        // full index -> compact column (if legal-superset)
        int jj = -1;
        for (int c = lane; c < C0; c += 32) {
          const int full = (c == C0 - 1) ? S * S : sk.head0_src[c] * S + sk.head0_dst[c];
          if (full == a) jj = c;
        }
        for (int o = 16; o; o >>= 1) jj = max(jj, __shfl_xor_sync(0xffffffffu, jj, o));
        act[0] = a;
        col0 = jj < 0 ? 0 : jj;
        if (jj >= 0 && legal(jj)) {
          // recompute log-prob of the injected column
          double zm = -INFINITY, ss = 0.0;
          for (int c = lane; c < C0; c += 32)
            if (legal(c)) zm = fmax(zm, (double)z[c]);
          zm = warp_max(zm);
          for (int c = lane; c < C0; c += 32)
            if (legal(c)) ss += exp((double)z[c] - zm);
          ss = warp_sum(ss);
          lp = (double)z[jj] - zm - log(ss);
        } else {
          lp = -INFINITY;
        }
      } else {
        act[0] = (j < 0) ? 0 : ((j == C0 - 1) ? S * S : sk.head0_src[j] * S + sk.head0_dst[j]);
        col0 = j < 0 ? 0 : j;
      }
      lp_total += lp;
    }
    // shift heads: 3 columns each at offsets C0, C0+3, C0+6
    for (int h = 1; h < 4; ++h) {
      const uint32_t m3 = (sb >> (3 * (h - 1))) & 7u;
      auto legal = [&](int j) -> bool { return (m3 >> j) & 1u; };
      const float* zh = z + C0 + 3 * (h - 1);
      double lp;
      bool none;
      double u = 0.0;
      if (!inject) u = u64_to_unit(pcg_draw64(J, rng.s, (uint64_t)h * n + r + 1));
      int j = warp_sample(zh, 3, legal, u, &lp, &none);
      dead |= none;
      if (inject) {
        const int a = inject[h * n + r];
        act[h] = a;
        if (a >= 0 && a < 3 && legal(a)) {
          double zm = -INFINITY, ss = 0.0;
          for (int c = 0; c < 3; ++c)
            if (legal(c)) zm = fmax(zm, (double)zh[c]);
          for (int c = 0; c < 3; ++c)
            if (legal(c)) ss += exp((double)zh[c] - zm);
          lp = (double)zh[a] - zm - log(ss);
        } else {
          lp = -INFINITY;
        }
      } else {
        act[h] = (j < 0) ? 0 : j;
      }
      lp_total += lp;
    }
    if (lane == 0) {
      for (int h = 0; h < 4; ++h) actions[h * n + r] = act[h];
      logp[r] = lp_total;
      move_bits[r] = mv;
      shift_bits[r] = sb;
      head0_col[r] = col0;
      int code = dead ? HARL_ST_NO_VALID
                      : apply_row(sk, tiles, knobs, ld, r, act[0], act[1], act[2],
                                  act[3], tiles_out, knobs_out, ld, r);
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

  const int warp = threadIdx.x >> 5;
  for (int rr = warp; rr < MLP_TM; rr += MLP_THREADS / 32) {
    const int64_t r = r0 + rr;
    if (r >= n) break;
    policy_row(sk, J, rng, logits + rr * ldbuf, NH, tiles, knobs, n, ld, r,
               inject, actions, logp, tiles_out, knobs_out, move_bits,
               shift_bits, head0_col, logits_out, status);
  }
}

// ValueNet.estimate (rlcore.py:161-178): hidden tanh layers, last layer
// linear (width 1).
__global__ void __launch_bounds__(MLP_THREADS)
k_value_forward(const __grid_constant__ harl_mlp_desc net, const double* feat,
                int64_t n, int32_t F, float* v_out, int ldbuf) {
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
