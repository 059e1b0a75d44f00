// K4/K5 on the 5th-gen tensor cores: the (128,128)-hidden rollout networks
// with tcgen05.mma kind::tf32 in 3xTF32 (a*b ~= ah*bh + ah*bl + al*bh, both
// halves pre-rounded to tf32, so the result is fp32-accurate: the
// north-star 1e-4 tolerance is met with ~40x margin, single-pass TF32 is
// not).
//
// Layout per CTA (persistent, one 128-row population tile at a time):
//   * weights: resident in shared memory as hi/lo tf32 in the K-major
//     no-swizzle canonical layout (B operand), staged once per CTA;
//   * activations: never leave the SM between layers -- each epilogue
//     thread owns one row (TMEM lane), rounds/splits its activations and
//     writes them back into TMEM with tcgen05.st, where the next layer's MMA
//     reads them as the A operand (the ".ts" form);
//   * accumulators: TMEM, read back with tcgen05.ld.
//
// k_trunk_tc   : F(<=64) -> 128 -> 128, tanh.  VALUE mode finishes
//                ValueNet (rlcore.py:161-178) with the 128->1 dot in the
//                epilogue; POLICY mode writes the trunk output (rlcore.py:
//                136-139) for the heads kernel.
// k_heads_tc   : the four linear heads (compact tiling head, rlcore.py:
//                140-146); sampling + walker follow in k_sample_rows.
#pragma once

#include "mlp_ffma.cuh"
#include "tc_common.cuh"

namespace harl {

constexpr int TC_H = 128;     // hidden width handled by the tensor-core path
constexpr int TC_K1 = 64;     // padded feature length

// stage W (row-major [K][N] fp32, global) as B operand hi/lo (N x Kpad,
// K-major core layout) in shared memory
__device__ inline void stage_weights(const float* __restrict__ W, int K, int N,
                                     int Kpad, int Npad, uint8_t* hi,
                                     uint8_t* lo) {
  for (int i = threadIdx.x; i < Kpad * Npad; i += blockDim.x) {
    const int k = i / Npad, nn = i % Npad;
    const float w = (k < K && nn < N) ? W[k * N + nn] : 0.f;
    float h, l;
    tc::split_tf32(w, h, l);
    const uint32_t off = tc::kmajor_off(nn, k, Kpad);
    *(float*)(hi + off) = h;
    *(float*)(lo + off) = l;
  }
}

__device__ inline void tc_sync() {
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
}

// issue D = A_hi B_hi + A_hi B_lo + A_lo B_hi over Kpad (thread 0 only)
__device__ inline void mma_3xtf32(uint32_t d, uint32_t a_hi, uint32_t a_lo,
                                  uint32_t b_hi_s, uint32_t b_lo_s, int Kpad,
                                  uint32_t idesc) {
  const uint32_t sbo = (uint32_t)(Kpad / 4 * 128);
  for (int s = 0; s < Kpad / 8; ++s) {
    const uint64_t bh = tc::sdesc(b_hi_s + 256 * s, 128, sbo);
    const uint64_t bl = tc::sdesc(b_lo_s + 256 * s, 128, sbo);
    tc::mma_tf32_ts(d, a_hi + 8 * s, bh, idesc, s > 0);
    tc::mma_tf32_ts(d, a_hi + 8 * s, bl, idesc, 1);
    tc::mma_tf32_ts(d, a_lo + 8 * s, bh, idesc, 1);
  }
}

// split 32 fp32 values and store hi/lo into TMEM at columns (c_hi, c_lo)
__device__ inline void store_split32(uint32_t taddr_hi, uint32_t taddr_lo,
                                     const float* v) {
  float h[32], l[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) tc::split_tf32(v[j], h[j], l[j]);
  tc::tmem_st32(taddr_hi, h);
  tc::tmem_st32(taddr_lo, l);
}

enum TrunkMode { TRUNK_VALUE = 0, TRUNK_POLICY = 1 };

struct TrunkArgs {
  const double* feat0;  // [n0][F]
  const double* feat1;  // [n1][F] (VALUE mode: X'), may be null
  int64_t n0, n1;
  int32_t F;
  float* out0;          // VALUE: v [n0]; POLICY: hid [n0][128]
  float* out1;          // VALUE: v [n1]
  const float* W1;      // [F][128]
  const float* b1;
  const float* W2;      // [128][128]
  const float* b2;
  const float* w3;      // [128] (VALUE)
  const float* b3;      // [1]
  const void* packed;   // optional pre-packed smem image (k_pack_trunk)
};

constexpr int TRUNK_SMEM = 2 * (TC_K1 * TC_H * 4) + 2 * (TC_H * TC_H * 4) +
                           3 * TC_H * 4 + 16;
constexpr int TRUNK_IMAGE = (TRUNK_SMEM + 15) / 16 * 16;

// The shared-memory image of the trunk weights (W1/W2 hi+lo in the
// K-major core layout, b1, b2, w3) built once per parameter update; the
// persistent kernels then pull it in with a few bulk copies instead of
// re-splitting ~25 K weights per CTA per launch.
__global__ void k_pack_trunk(TrunkArgs a, uint8_t* img, int value_mode) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  uint8_t* w1h = img;
  uint8_t* w1l = w1h + TC_K1 * TC_H * 4;
  uint8_t* w2h = w1l + TC_K1 * TC_H * 4;
  uint8_t* w2l = w2h + TC_H * TC_H * 4;
  float* b = (float*)(w2l + TC_H * TC_H * 4);
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nth = gridDim.x * blockDim.x;
  for (int i = tid; i < TC_K1 * TC_H; i += nth) {
    const int k = i / TC_H, nn = i % TC_H;
    const float w = k < a.F ? a.W1[k * TC_H + nn] : 0.f;
    float h, l;
    tc::split_tf32(w, h, l);
    *(float*)(w1h + tc::kmajor_off(nn, k, TC_K1)) = h;
    *(float*)(w1l + tc::kmajor_off(nn, k, TC_K1)) = l;
  }
  for (int i = tid; i < TC_H * TC_H; i += nth) {
    const int k = i / TC_H, nn = i % TC_H;
    float h, l;
    tc::split_tf32(a.W2[k * TC_H + nn], h, l);
    *(float*)(w2h + tc::kmajor_off(nn, k, TC_H)) = h;
    *(float*)(w2l + tc::kmajor_off(nn, k, TC_H)) = l;
  }
  for (int i = tid; i < TC_H; i += nth) {
    b[i] = a.b1[i];
    b[TC_H + i] = a.b2[i];
    b[2 * TC_H + i] = value_mode ? a.w3[i] : 0.f;
  }
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) k_trunk_tc(TrunkArgs a) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* w1h = sm;
  uint8_t* w1l = w1h + TC_K1 * TC_H * 4;
  uint8_t* w2h = w1l + TC_K1 * TC_H * 4;
  uint8_t* w2l = w2h + TC_H * TC_H * 4;
  float* sb1 = (float*)(w2l + TC_H * TC_H * 4);
  float* sb2 = sb1 + TC_H;
  float* sw3 = sb2 + TC_H;
  __shared__ uint64_t bar, wbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tc::tmem_alloc(&tbase, 512);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_init(&wbar, 1);
  }
  __syncthreads();
  if (a.packed) {
    if (tid == 0) tc::bulk_load(sm, a.packed, TRUNK_IMAGE - 16, &wbar);
    tc::mbar_wait(&wbar, 0);
  } else {
    stage_weights(a.W1, a.F, TC_H, TC_K1, TC_H, w1h, w1l);
    stage_weights(a.W2, TC_H, TC_H, TC_H, TC_H, w2h, w2l);
    for (int i = tid; i < TC_H; i += blockDim.x) {
      sb1[i] = a.b1[i];
      sb2[i] = a.b2[i];
      sw3[i] = MODE == TRUNK_VALUE ? a.w3[i] : 0.f;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  const float b3 = MODE == TRUNK_VALUE ? a.b3[0] : 0.f;
  tc_sync();
  const uint32_t tm = tbase;
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
  // TMEM columns: X hi [0,64) X lo [64,128) D [128,256) H hi [256,384)
  // H lo [384,512)
  const uint32_t cXh = 0, cXl = 64, cD = 128, cHh = 256, cHl = 384;
  const uint32_t idesc = tc::idesc_tf32(128, TC_H);
  const uint32_t s_w1h = tc::smem_u32(w1h), s_w1l = tc::smem_u32(w1l);
  const uint32_t s_w2h = tc::smem_u32(w2h), s_w2l = tc::smem_u32(w2l);
  const int64_t t0 = (a.n0 + 127) / 128;
  const int64_t t1 = (a.n1 + 127) / 128;
  uint32_t phase = 0;
  for (int64_t tile = blockIdx.x; tile < t0 + t1; tile += gridDim.x) {
    const bool second = tile >= t0;
    const double* feat = second ? a.feat1 : a.feat0;
    const int64_t n = second ? a.n1 : a.n0;
    const int64_t row = (second ? tile - t0 : tile) * 128 + tid;
    // ---- X row -> TMEM (hi/lo) ----
    {
      float v[32];
      for (int c0 = 0; c0 < TC_K1; c0 += 32) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int k = c0 + j;
          v[j] = (row < n && k < a.F) ? (float)feat[row * a.F + k] : 0.f;
        }
        store_split32(tm + lane_off + cXh + c0, tm + lane_off + cXl + c0, v);
      }
      tc::tmem_st_wait();
    }
    tc_sync();
    if (tid == 0) {
      mma_3xtf32(tm + cD, tm + cXh, tm + cXl, s_w1h, s_w1l, TC_K1, idesc);
      tc::mma_commit(&bar);
    }
    __syncwarp();
    tc::mbar_wait(&bar, phase);
    phase ^= 1;
    tc::fence_after();
    // ---- layer 1 epilogue: tanh(z + b1) -> H (hi/lo) ----
    for (int c0 = 0; c0 < TC_H; c0 += 32) {
      float v[32];
      tc::tmem_ld32(tm + lane_off + cD + c0, v);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = tanhf(v[j] + sb1[c0 + j]);
      store_split32(tm + lane_off + cHh + c0, tm + lane_off + cHl + c0, v);
    }
    tc::tmem_st_wait();
    tc_sync();
    if (tid == 0) {
      mma_3xtf32(tm + cD, tm + cHh, tm + cHl, s_w2h, s_w2l, TC_H, idesc);
      tc::mma_commit(&bar);
    }
    __syncwarp();
    tc::mbar_wait(&bar, phase);
    phase ^= 1;
    tc::fence_after();
    // ---- layer 2 epilogue ----
    float acc = 0.f;
    float* orow = nullptr;
    if (MODE == TRUNK_POLICY && row < n) orow = a.out0 + row * TC_H;
    for (int c0 = 0; c0 < TC_H; c0 += 32) {
      float v[32];
      tc::tmem_ld32(tm + lane_off + cD + c0, v);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float h = tanhf(v[j] + sb2[c0 + j]);
        if (MODE == TRUNK_VALUE) acc = fmaf(h, sw3[c0 + j], acc);
        v[j] = h;
      }
      if (MODE == TRUNK_POLICY && orow) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *(float4*)(orow + c0 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
    }
    if (MODE == TRUNK_VALUE && row < n) (second ? a.out1 : a.out0)[row] = acc + b3;
    tc_sync();  // all TMEM reads of D done before the next tile's MMA
  }
  if (warp == 0) tc::tmem_dealloc(tm, 512);
}

// ---------------------------------------------------------------------------
// heads: logits = hid . Wh + bh for a 128-row tile, written IN PLACE over
// the tile's trunk rows (row stride 128) for the sampling kernel, and
// optionally to logits_out [n][NH].

constexpr int HEADS_NMAX = 128;   // padded head columns handled here

struct HeadsArgs {
  float* hid;         // [n][128] trunk output in, logits out (in place)
  const float* Wh;    // [128][NH]
  const float* bh;    // [NH]
  float* logits_out;  // optional [n][NH]
  int64_t n;
  int32_t NH, NHP;    // real / padded (multiple of 16) head columns
  const void* packed; // optional pre-packed smem image (k_pack_heads)
};

__host__ __device__ inline int heads_image_bytes(int NHP) {
  return 2 * NHP * TC_H * 4 + HEADS_NMAX * 4;
}

__global__ void k_pack_heads(HeadsArgs h, uint8_t* img) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  const int NHP = h.NHP;
  uint8_t* whh = img;
  uint8_t* whl = whh + NHP * TC_H * 4;
  float* b = (float*)(whl + NHP * TC_H * 4);
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nth = gridDim.x * blockDim.x;
  for (int i = tid; i < TC_H * NHP; i += nth) {
    const int k = i / NHP, nn = i % NHP;
    const float w = nn < h.NH ? h.Wh[k * h.NH + nn] : 0.f;
    float hi, lo;
    tc::split_tf32(w, hi, lo);
    *(float*)(whh + tc::kmajor_off(nn, k, TC_H)) = hi;
    *(float*)(whl + tc::kmajor_off(nn, k, TC_H)) = lo;
  }
  for (int i = tid; i < HEADS_NMAX; i += nth) b[i] = i < h.NH ? h.bh[i] : 0.f;
}

__global__ void __launch_bounds__(128, 1) k_heads_tc(HeadsArgs h) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  extern __shared__ __align__(1024) uint8_t sm[];
  const int NHP = h.NHP;
  uint8_t* whh = sm;
  uint8_t* whl = whh + NHP * TC_H * 4;
  float* sbh = (float*)(whl + NHP * TC_H * 4);
  __shared__ uint64_t bar, wbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tc::tmem_alloc(&tbase, 512);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_init(&wbar, 1);
  }
  __syncthreads();
  if (h.packed) {
    if (tid == 0) tc::bulk_load(sm, h.packed, heads_image_bytes(NHP), &wbar);
    tc::mbar_wait(&wbar, 0);
  } else {
    stage_weights(h.Wh, TC_H, h.NH, TC_H, NHP, whh, whl);
    for (int i = tid; i < HEADS_NMAX; i += blockDim.x) sbh[i] = i < h.NH ? h.bh[i] : 0.f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  tc_sync();
  const uint32_t tm = tbase;
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
  const uint32_t cAh = 0, cAl = 128, cD = 256;
  const uint32_t idesc = tc::idesc_tf32(128, NHP);
  const uint32_t s_hh = tc::smem_u32(whh), s_hl = tc::smem_u32(whl);
  const int64_t tiles_n = (h.n + 127) / 128;
  uint32_t phase = 0;
  for (int64_t tile = blockIdx.x; tile < tiles_n; tile += gridDim.x) {
    const int64_t row = tile * 128 + tid;
    float* hrow = h.hid + row * TC_H;
    for (int c0 = 0; c0 < TC_H; c0 += 32) {
      float v[32];
      if (row < h.n) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const float4 q = *(const float4*)(hrow + c0 + j);
          v[j] = q.x;
          v[j + 1] = q.y;
          v[j + 2] = q.z;
          v[j + 3] = q.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.f;
      }
      store_split32(tm + lane_off + cAh + c0, tm + lane_off + cAl + c0, v);
    }
    tc::tmem_st_wait();
    tc_sync();
    if (tid == 0) {
      mma_3xtf32(tm + cD, tm + cAh, tm + cAl, s_hh, s_hl, TC_H, idesc);
      tc::mma_commit(&bar);
    }
    __syncwarp();
    tc::mbar_wait(&bar, phase);
    phase ^= 1;
    tc::fence_after();
    for (int c0 = 0; c0 < NHP; c0 += 32) {
      float v[32];
      tc::tmem_ld32(tm + lane_off + cD + c0, v);
      if (row < h.n) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int c = c0 + j;
          if (c < h.NH) {
            const float zc = v[j] + sbh[c];
            hrow[c] = zc;
            if (h.logits_out) h.logits_out[row * h.NH + c] = zc;
          }
        }
      }
    }
    tc_sync();
  }
  if (warp == 0) tc::tmem_dealloc(tm, 512);
}

}  // namespace harl
