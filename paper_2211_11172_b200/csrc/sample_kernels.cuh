// K4 epilogue as its own full-occupancy kernel: masked log-softmax per head
// (rlcore.py:185-199), inverse-CDF sampling on the numpy PCG64 stream
// (rlcore.py:202-213, select_actions 216-228) and decode + apply
// (schedspace.py:196-301), ONE THREAD PER ROW.  (A warp per row spends
// ~50x more issue slots on the same work: the heads are short and
// sequential.)
//
// Uniforms: draw #(h*n + r + 1) after the step's base state.  Each warp
// jumps once from the base state to its first row (warp-uniform), then
// every lane applies its precomputed lane offset (A^l, C_l) -- one 128-bit
// multiply-add per lane instead of a full jump per lane.
#pragma once

#include "common.cuh"
#include "space_kernels.cuh"

namespace harl {

constexpr int SAMPLE_THREADS = 128;

struct LaneJump {
  u128 A[32];
  u128 C[32];
};

struct SampleArgs {
  const float* logits;   // [n][ldz] (head0 compact columns, then 3x3)
  int32_t ldz;
  int64_t n, ld;
  const int32_t* inject; // [4][n] or null
  int32_t* actions;      // [4][n]
  double* logp;          // [n]
  uint16_t* tiles_out;
  uint8_t* knobs_out;
  uint64_t* move_bits;
  uint32_t* shift_bits;
  int32_t* head0_col;
  unsigned long long* status;
};

// masked log-softmax + inverse CDF over C columns of one row (one thread);
// exp in fp32 (the logits are fp32), sums/cumsum in fp64.  Walk-back over
// zero-probability cells as in the reference; returns -1 when the walk ends
// on an illegal column 0.
template <typename Legal>
__device__ inline int row_sample(const float* z, int C, Legal legal, double u,
                                 double* logp_out, bool* none) {
  float zmax = -INFINITY;
  for (int j = 0; j < C; ++j)
    if (legal(j)) zmax = fmaxf(zmax, z[j]);
  *none = (zmax == -INFINITY);
  double s = 0.0;
  for (int j = 0; j < C; ++j)
    if (legal(j)) s += (double)expf(z[j] - zmax);
  const double inv = 1.0 / s;
  int count = 0;
  double c = 0.0;
  for (int j = 0; j < C; ++j) {
    if (legal(j)) c += (double)expf(z[j] - zmax) * inv;
    count += (c < u);
  }
  int idx = min(count, C - 1);
  while (idx > 0 && !legal(idx)) --idx;
  const bool ok = legal(idx);
  *logp_out = ok ? ((double)z[idx] - (double)zmax - log(s)) : -INFINITY;
  return ok ? idx : -1;
}

template <typename Legal>
__device__ inline double row_logp(const float* z, int C, Legal legal, int a) {
  if (a < 0 || a >= C || !legal(a)) return -INFINITY;
  float zmax = -INFINITY;
  for (int j = 0; j < C; ++j)
    if (legal(j)) zmax = fmaxf(zmax, z[j]);
  double s = 0.0;
  for (int j = 0; j < C; ++j)
    if (legal(j)) s += (double)expf(z[j] - zmax);
  return (double)z[a] - (double)zmax - log(s);
}

__global__ void __launch_bounds__(SAMPLE_THREADS)
k_sample_rows(const __grid_constant__ harl_sketch_desc sk,
              const __grid_constant__ PcgJump J,
              const __grid_constant__ LaneJump LJ, u128 base_arg,
              const u128* base_dev, const uint16_t* __restrict__ tiles,
              const uint8_t* __restrict__ knobs, SampleArgs a) {
  __shared__ int16_t s_src[HARL_MAX_HEAD0], s_dst[HARL_MAX_HEAD0];
  __shared__ u128 s_la[32], s_lc[32];
  for (int i = threadIdx.x; i < sk.n_head0; i += blockDim.x) {
    s_src[i] = sk.head0_src[i];
    s_dst[i] = sk.head0_dst[i];
  }
  if (threadIdx.x < 32) {
    s_la[threadIdx.x] = LJ.A[threadIdx.x];
    s_lc[threadIdx.x] = LJ.C[threadIdx.x];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t r_lane0 = r - lane;
  if (r_lane0 >= a.n) return;  // whole warp out of range
  // uniforms for the 4 heads (computed by every lane of a live warp); the
  // step's base state comes from device memory in graph-replay mode
  const u128 base = base_dev ? *base_dev : base_arg;
  double u[4] = {0, 0, 0, 0};
  if (!a.inject) {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const u128 w = pcg_advance(J, base, (uint64_t)h * a.n + r_lane0 + 1);
      const u128 s = add128(mul128(s_la[lane], w), s_lc[lane]);
      u[h] = u64_to_unit(pcg_output(s));
    }
  }
  if (r >= a.n) return;
  const int S = sk.num_slots, L = sk.levels, C0 = sk.n_head0;
  // current state
  uint64_t mv = 0;
  for (int s = 0; s < sk.local_slots; ++s)
    if (tiles[(int64_t)s * a.ld + r] > 1) mv |= 1ull << s;
  const int ca0 = knobs[r], par0 = knobs[a.ld + r], ur0 = knobs[2 * a.ld + r];
  const uint32_t sb = shift_bits_of(sk, ca0, par0, ur0);
  const float* z = a.logits + r * a.ldz;
  int act[4];
  int col0 = 0;
  double lp_total = 0.0;
  bool dead = false;
  {
    auto legal = [&](int j) -> bool {
      return j == C0 - 1 || ((mv >> s_src[j]) & 1ull);
    };
    double lp;
    bool none = false;
    if (a.inject) {
      const int full = a.inject[r];
      int jj = -1;
      if (full == S * S) jj = C0 - 1;
      else if (full >= 0 && full < S * S) {
        const int src = full / S, dst = full % S;
        for (int c = 0; c < C0 - 1; ++c)
          if (s_src[c] == src && s_dst[c] == dst) jj = c;
      }
      act[0] = full;
      col0 = jj < 0 ? 0 : jj;
      lp = jj < 0 ? -INFINITY : row_logp(z, C0, legal, jj);
    } else {
      const int j = row_sample(z, C0, legal, u[0], &lp, &none);
      act[0] = (j < 0) ? 0 : ((j == C0 - 1) ? S * S : s_src[j] * S + s_dst[j]);
      col0 = j < 0 ? 0 : j;
    }
    dead |= none;
    lp_total += lp;
  }
  for (int h = 1; h < 4; ++h) {
    const uint32_t m3 = (sb >> (3 * (h - 1))) & 7u;
    auto legal = [&](int j) -> bool { return (m3 >> j) & 1u; };
    const float* zh = z + C0 + 3 * (h - 1);
    double lp;
    bool none = (m3 == 0);
    if (a.inject) {
      act[h] = a.inject[h * a.n + r];
      lp = row_logp(zh, 3, legal, act[h]);
    } else {
      const int j = row_sample(zh, 3, legal, u[h], &lp, &none);
      act[h] = (j < 0) ? 0 : j;
    }
    dead |= none;
    lp_total += lp;
  }
  for (int h = 0; h < 4; ++h) a.actions[h * a.n + r] = act[h];
  a.logp[r] = lp_total;
  a.move_bits[r] = mv;
  a.shift_bits[r] = sb;
  a.head0_col[r] = col0;
  const int code = dead ? HARL_ST_NO_VALID
                        : apply_row(sk, tiles, knobs, a.ld, r, act[0], act[1],
                                    act[2], act[3], a.tiles_out, a.knobs_out,
                                    a.ld, r);
  report_status(a.status, r, code);
  (void)L;
}

}  // namespace harl
