// Wide-epilogue tcgen05 kernels for the (128,128)-hidden rollout networks.
//
// The first-generation kernels (mlp_tc.cuh) ran 4 warps per CTA, one TMEM
// lane (= population row) per thread, so each thread did all 128 columns of
// every epilogue (tanh, tf32 split, TMEM store) serially -- with one CTA
// per SM (the weights fill shared memory) that epilogue, not the MMAs, was
// the kernel.  Here 16 warps share the tile: warp w reads/writes TMEM lanes
// 32*(w%4).. (the hardware's lane-quarter rule) and owns the 32-column
// group w/4, so every epilogue is 4x shorter per thread.
//
// k_policy_tc fuses trunk and heads (rlcore.py:136-146): the trunk output
// never leaves TMEM; the heads' weight image is streamed into the shared
// memory W1 occupied, as soon as layer 1's MMA has consumed it, so its copy
// overlaps the layer-1/2 epilogues.  Shared memory:
//   regA: W1 hi|lo (64 KB), then the heads image (whh|whl|bh)
//   regB: W2 hi|lo (128 KB) | b1 | b2 | w3   (loaded once per CTA)
// TMEM (512 columns): X hi/lo [0,128), D [128,256), H hi/lo [256,512).
//
// k_value_tc: the same trunk for ValueNet (rlcore.py:161-178); the final
// 128->1 dot is summed per column group and the 4 partials added in group
// order.
#pragma once

#include "mlp_tc.cuh"
#include "sample_kernels.cuh"
#include "space_kernels.cuh"

namespace harl {

constexpr int TC2_THREADS = 512;
constexpr int TC2_W1 = 2 * TC_K1 * TC_H * 4;                 // 64 KB
constexpr int TC2_W2 = 2 * TC_H * TC_H * 4 + 3 * TC_H * 4;   // 128 KB + b1,b2,w3
constexpr int TC2_W2P = 2 * TC_H * TC_H * 4 + 2 * TC_H * 4;  // policy: no w3

constexpr int TC2_LG_LD = 132;   // padded row stride of the logits staging tile

__host__ __device__ inline int tc2_regA(int NHP) {
  const int h = NHP > 0 ? heads_image_bytes(NHP) : 0;
  int a = h > TC2_W1 ? h : TC2_W1;
  if (NHP > 0 && a < 128 * TC2_LG_LD * 4) a = 128 * TC2_LG_LD * 4;
  return (a + 127) / 128 * 128;
}
__host__ __device__ inline int tc2_smem(int NHP) { return tc2_regA(NHP) + TC2_W2P; }

// X row slice [16g, 16g+16) -> TMEM hi/lo (fp64 -> fp32 -> tf32 split)
__device__ inline void tc2_stage_x(const double* feat, int64_t row, int64_t n,
                                   int F, int g, uint32_t t_hi, uint32_t t_lo) {
  float v[16], h[16], l[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int k = 16 * g + j;
    v[j] = (row < n && k < F) ? (float)__ldg(feat + row * F + k) : 0.f;
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) tc::split_tf32(v[j], h[j], l[j]);
  tc::tmem_st16(t_hi, h);
  tc::tmem_st16(t_lo, l);
}

// tanh(D + b) for this thread's 32 columns, split into H hi/lo
__device__ inline void tc2_tanh_split(uint32_t t_d, uint32_t t_hi, uint32_t t_lo,
                                      const float* b) {
  float v[32];
  tc::tmem_ld32(t_d, v);
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = tanhf(v[j] + b[j]);
  store_split32(t_hi, t_lo, v);
}

// X tile (rows r0.., contiguous fp64 [rows][F]) -> shared memory
__device__ inline void tc2_bulk_x(void* dst, const double* feat, int64_t r0,
                                  int rows, int F, uint64_t* bar) {
  tc::bulk_f64((double*)dst, feat + r0 * F, (uint32_t)rows * F, bar);
}

// this thread's 16-column slice of its row, from the staged tile
__device__ inline void tc2_stage_x_smem(const double* xs, int lrow, int rows,
                                        int F, int g, uint32_t t_hi, uint32_t t_lo) {
  float h[16], l[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int k = 16 * g + j;
    const float v = (lrow < rows && k < F) ? (float)xs[lrow * F + k] : 0.f;
    tc::split_tf32(v, h[j], l[j]);
  }
  tc::tmem_st16(t_hi, h);
  tc::tmem_st16(t_lo, l);
}

// M = 64 tiles (n <= 148 * 64 rows per launch: twice the CTAs of 128-row
// tiles, half the epilogue per warp).  Warp w: lane quarter q = w % 4 holds
// tile rows 16 q .. 16 q + 15 (lanes 32 q .. 32 q + 15), column group
// g = w / 4.
__device__ inline void tc64_stage_x_smem(const double* xs, int q, int lane,
                                         int rows, int F, int g,
                                         uint32_t t_hi, uint32_t t_lo) {
  float h[8], l[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = 16 * q + tc::frag64_row(lane, i);
    const int k = 16 * g + tc::frag64_col(lane, i);
    const float v = (r < rows && k < F) ? (float)xs[r * F + k] : 0.f;
    tc::split_tf32(v, h[i], l[i]);
  }
  tc::tmem_st16x256_x2(t_hi, h);
  tc::tmem_st16x256_x2(t_lo, l);
}

__device__ inline void tc64_tanh_split(uint32_t t_d, uint32_t t_hi,
                                       uint32_t t_lo, const float* b,
                                       int lane) {
  float v[16], h[16], l[16];
  tc::tmem_ld16x256_x4(t_d, v);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float z = tanhf(v[i] + b[tc::frag64_col(lane, i)]);
    tc::split_tf32(z, h[i], l[i]);
  }
  tc::tmem_st16x256_x4(t_hi, h);
  tc::tmem_st16x256_x4(t_lo, l);
}

struct PolicyTcArgs {
  const double* feat;   // [n][F] (16-byte aligned)
  int64_t n;
  int32_t F, NH, NHP;
  int32_t regA;         // bytes of shared-memory region A (>= tc2_regA(NHP))
  float* logits;        // [n][128] (the sampler's input, row stride 128)
  float* logits_out;    // optional [n][NH]
  const void* trunk_img;  // k_pack_trunk image
  const void* heads_img;  // k_pack_heads image
};

// The rest of the rollout step, fused behind the heads (FUSED = true):
// the CTA samples and applies its 128 rows' actions straight from the
// logits staging tile (k_sample_rows' 8-lane groups, two passes), then
// featurizes the new states of the same rows into X' (k_featurize2's 4-part
// rows) -- the logits never reach HBM and two launches disappear.
struct StepFuseArgs {
  SampleArgs s;               // sampler outputs (logits field unused)
  u128 base_arg;
  const u128* base_dev;       // graph replay: the step's RNG base state
  const uint16_t* tiles;      // current state [slot][ld]
  const uint8_t* knobs;
  double* feat_new;           // X' [n][F]
};

static_assert(FEAT2_THREADS == TC2_THREADS, "fused featurize shares the CTA");

template <bool FUSED, int M = 128>
__device__ __forceinline__ void policy_tc_body(const PolicyTcArgs& a,
                                               const StepFuseArgs* f,
                                               const harl_sketch_desc* sk,
                                               const PcgJump* J) {
  dbg_ts(0);
  extern __shared__ __align__(128) uint8_t sm2[];
  uint8_t* sm = sm2;
  const int regA = a.regA;
  uint8_t* rA = sm;
  uint8_t* rB = sm + regA;
  const float* sb1 = (const float*)(rB + 2 * TC_H * TC_H * 4);
  const float* sb2 = sb1 + TC_H;
  const float* sbh = (const float*)(rA + 2 * a.NHP * TC_H * 4);
  float* stg = (float*)rA;  // logits staging [128][TC2_LG_LD] after the heads MMA
  __shared__ uint64_t bar, wbar1, wbar2, hbar, xbar;
  __shared__ uint32_t tbase;
  static_assert(M == 128 || (M == 64 && !FUSED), "tile rows");
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, g = warp >> 2;
  const int lrow = q * 32 + lane;   // M = 128: this thread's tile row
  if (warp == 0) tc::tmem_alloc(&tbase, 512);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_init(&wbar1, 1);
    tc::mbar_init(&wbar2, 1);
    tc::mbar_init(&hbar, 1);
    tc::mbar_init(&xbar, 1);
  }
  __syncthreads();
  const uint8_t* timg = (const uint8_t*)a.trunk_img;
  const int64_t tiles = (a.n + M - 1) / M;
  if (tid == 0 && blockIdx.x < tiles) {
    // first tile: X into regB (W2 follows once X is in TMEM), W1 into regA
    const int64_t r0 = (int64_t)blockIdx.x * M;
    tc2_bulk_x(rB, a.feat, r0, (int)min((int64_t)M, a.n - r0), a.F, &xbar);
    tc::bulk_load(rA, timg, TC2_W1, &wbar1);
  }
  tc_sync();
  dbg_ts(1);
  const uint32_t tm = tbase;
  const uint32_t lo = (uint32_t)(q * 32) << 16;
  const uint32_t cXh = 0, cXl = 64, cD = 128, cHh = 256, cHl = 384;
  const uint32_t id_h = tc::idesc_tf32(M, TC_H);
  const uint32_t id_o = tc::idesc_tf32(M, a.NHP);
  const uint32_t sA = tc::smem_u32(rA), sB = tc::smem_u32(rB);
  uint32_t ph = 0, pw1 = 0, ph_h = 0, px = 0;
  bool first = true;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t r0 = tile * M;
    const int rows = (int)min((int64_t)M, a.n - r0);
    if (!first && tid == 0) tc2_bulk_x(rA, a.feat, r0, rows, a.F, &xbar);
    tc::mbar_wait(&xbar, px);
    px ^= 1;
    const double* xs = (const double*)(first ? rB : rA);
    if (g < TC_K1 / 16) {
      if constexpr (M == 128)
        tc2_stage_x_smem(xs, lrow, rows, a.F, g, tm + lo + cXh + 16 * g, tm + lo + cXl + 16 * g);
      else
        tc64_stage_x_smem(xs, q, lane, rows, a.F, g, tm + lo + cXh + 16 * g, tm + lo + cXl + 16 * g);
    }
    tc::tmem_st_wait();
    tc_sync();
    dbg_ts(2);
    if (tid == 0) {
      // the staged X is dead: async-proxy writes may now reuse its bytes
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (first) tc::bulk_load(rB, timg + TC2_W1, TC2_W2P, &wbar2);
      else tc::bulk_load(rA, timg, TC2_W1, &wbar1);
      tc::mbar_wait(&wbar1, pw1);
      dbg_ts(3);
      mma_3xtf32(tm + cD, tm + cXh, tm + cXl, sA, sA + TC_K1 * TC_H * 4, TC_K1, id_h);
      tc::mma_commit(&bar);
    }
    pw1 ^= 1;
    tc::mbar_wait(&bar, ph);
    ph ^= 1;
    tc::fence_after();
    dbg_ts(4);
    // regA is free: stream the heads image in behind the epilogues
    if (tid == 0) tc::bulk_load(rA, a.heads_img, heads_image_bytes(a.NHP), &hbar);
    if (first) tc::mbar_wait(&wbar2, 0);
    if constexpr (M == 128)
      tc2_tanh_split(tm + lo + cD + 32 * g, tm + lo + cHh + 32 * g, tm + lo + cHl + 32 * g,
                     sb1 + 32 * g);
    else
      tc64_tanh_split(tm + lo + cD + 32 * g, tm + lo + cHh + 32 * g, tm + lo + cHl + 32 * g,
                      sb1 + 32 * g, lane);
    tc::tmem_st_wait();
    tc_sync();
    dbg_ts(5);
    if (tid == 0) {
      mma_3xtf32(tm + cD, tm + cHh, tm + cHl, sB, sB + TC_H * TC_H * 4, TC_H, id_h);
      tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, ph);
    ph ^= 1;
    tc::fence_after();
    dbg_ts(6);
    if constexpr (M == 128)
      tc2_tanh_split(tm + lo + cD + 32 * g, tm + lo + cHh + 32 * g, tm + lo + cHl + 32 * g,
                     sb2 + 32 * g);
    else
      tc64_tanh_split(tm + lo + cD + 32 * g, tm + lo + cHh + 32 * g, tm + lo + cHl + 32 * g,
                      sb2 + 32 * g, lane);
    tc::tmem_st_wait();
    tc_sync();
    dbg_ts(7);
    tc::mbar_wait(&hbar, ph_h);
    ph_h ^= 1;
    dbg_ts(8);
    if (tid == 0) {
      mma_3xtf32(tm + cD, tm + cHh, tm + cHl, sA, sA + a.NHP * TC_H * 4, TC_H, id_o);
      tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, ph);
    ph ^= 1;
    tc::fence_after();
    dbg_ts(9);
    // logits (+ bias) -> padded staging tile in regA -> coalesced rows.
    // The heads weights are dead; the bias sits above the staging tile.
    float v[32];
    const bool has = 32 * g < a.NHP;
    if constexpr (M == 128) {
      if (has) {
        tc::tmem_ld32(tm + lo + cD + 32 * g, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] += sbh[32 * g + j];
      }
    } else {
      if (has) {
        tc::tmem_ld16x256_x4(tm + lo + cD + 32 * g, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] += sbh[32 * g + tc::frag64_col(lane, i)];
      }
    }
    __syncthreads();  // every thread has read the bias before it may be overwritten
    if (has) {
      if constexpr (M == 128) {
        float* srow = stg + lrow * TC2_LG_LD + 32 * g;
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *(float4*)(srow + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      } else {
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
          const int r = 16 * q + tc::frag64_row(lane, i);
          *(float2*)(stg + r * TC2_LG_LD + 32 * g + tc::frag64_col(lane, i)) =
              make_float2(v[i], v[i + 1]);
        }
      }
    }
    __syncthreads();
    if (!FUSED) {
      const int c4n = a.NHP / 4;
      for (int i = tid; i < rows * c4n; i += TC2_THREADS) {
        const int rr = i / c4n, c4 = i % c4n;
        *(float4*)(a.logits + (r0 + rr) * TC_H + 4 * c4) =
            *(const float4*)(stg + rr * TC2_LG_LD + 4 * c4);
      }
    }
    if (a.logits_out)
      for (int i = tid; i < rows * a.NH; i += TC2_THREADS) {
        const int rr = i / a.NH, c = i % a.NH;
        a.logits_out[(r0 + rr) * a.NH + c] = stg[rr * TC2_LG_LD + c];
      }
    if (FUSED) {
      int16_t* s_src = (int16_t*)(rA + 128 * TC2_LG_LD * 4);
      int16_t* s_dst = s_src + HARL_MAX_HEAD0;
      for (int i = tid; i < sk->n_head0; i += TC2_THREADS) {
        s_src[i] = sk->head0_src[i];
        s_dst[i] = sk->head0_dst[i];
      }
      __syncthreads();
      dbg_ts(11);
#pragma unroll 1
      for (int pass = 0; pass < 128 / (TC2_THREADS / SG); ++pass) {
        const int lr = pass * (TC2_THREADS / SG) + tid / SG;
        sample_group(*sk, *J, f->base_arg, f->base_dev, f->tiles, f->knobs,
                     f->s, r0 + lr, stg + lr * TC2_LG_LD, s_src, s_dst);
      }
      __syncthreads();   // the tile's new states are written (and visible)
      dbg_ts(12);
      featurize_tile(*sk, f->s.tiles_out, f->s.knobs_out, a.n, f->s.ld, r0,
                     f->feat_new, rA);
      dbg_ts(13);
    }
    first = false;
    tc_sync();  // staging reads done before the next tile reuses regA
    dbg_ts(10);
  }
  if (warp == 0) tc::tmem_dealloc(tm, 512);
}

__global__ void __launch_bounds__(TC2_THREADS, 1) k_policy_tc(PolicyTcArgs a) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  policy_tc_body<false>(a, nullptr, nullptr, nullptr);
}

// 64-row tiles: for launches of <= 148 * 64 rows (the steps after a cull)
__global__ void __launch_bounds__(TC2_THREADS, 1) k_policy_tc64(PolicyTcArgs a) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  policy_tc_body<false, 64>(a, nullptr, nullptr, nullptr);
}

__global__ void __launch_bounds__(TC2_THREADS, 1)
k_policy_step_fused(PolicyTcArgs a, StepFuseArgs f,
                    const __grid_constant__ harl_sketch_desc sk,
                    const __grid_constant__ PcgJump J) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  policy_tc_body<true>(a, &f, &sk, &J);
}

// regA must also hold the sampler's column tables and the featurize
// staging of the fused step
__host__ __device__ inline int tc2_fused_regA_need(int F, int local_slots,
                                                   int max_extent) {
  const int samp = 128 * TC2_LG_LD * 4 + 4 * HARL_MAX_HEAD0;
  const int feat = (int)feat2_smem_bytes(F, local_slots, max_extent);
  return samp > feat ? samp : feat;
}

struct ValueTcArgs {
  const double* feat0;  // X  [n0][F] (16-byte aligned)
  const double* feat1;  // X' [n1][F] (may be null; 16-byte aligned)
  int64_t n0, n1;
  int32_t F;
  float* out0;          // v [n0]
  float* out1;          // v [n1]
  const float* b3;      // [1] device
  const void* trunk_img;
};

constexpr int TC2_VX = 64 * TC_K1 * 8;   // half-tile X staging (32 KB)

__host__ __device__ inline int tc2_value_smem() { return TC2_W1 + TC2_W2 + TC2_VX; }

// X rows are staged in two 64-row halves through a 32 KB buffer (the
// weights take the rest of shared memory); the next tile's first half is
// prefetched as soon as the current tile's X is in TMEM.
__global__ void __launch_bounds__(TC2_THREADS, 1) k_value_tc(ValueTcArgs a) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  extern __shared__ __align__(128) uint8_t sm3[];
  uint8_t* rA = sm3;
  uint8_t* rB = sm3 + TC2_W1;
  double* xs = (double*)(sm3 + TC2_W1 + TC2_W2);
  const float* sb1 = (const float*)(rB + 2 * TC_H * TC_H * 4);
  const float* sb2 = sb1 + TC_H;
  const float* sw3 = sb2 + TC_H;
  __shared__ uint64_t bar, wbar, xbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, g = warp >> 2;
  const int lrow = q * 32 + lane;
  const int64_t t0 = (a.n0 + 127) / 128, t1 = (a.n1 + 127) / 128;
  auto tile_src = [&](int64_t tile, const double*& f, int64_t& n, int64_t& r0) {
    const bool second = tile >= t0;
    f = second ? a.feat1 : a.feat0;
    n = second ? a.n1 : a.n0;
    r0 = (second ? tile - t0 : tile) * 128;
  };
  if (warp == 0) tc::tmem_alloc(&tbase, 512);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_init(&wbar, 1);
    tc::mbar_init(&xbar, 1);
  }
  __syncthreads();
  if (tid == 0 && blockIdx.x < t0 + t1) {
    const double* f;
    int64_t n, r0;
    tile_src(blockIdx.x, f, n, r0);
    tc2_bulk_x(xs, f, r0, (int)min((int64_t)64, n - r0), a.F, &xbar);
    tc::bulk_load(rA, a.trunk_img, TC2_W1 + TC2_W2, &wbar);
  }
  tc_sync();
  const uint32_t tm = tbase;
  const uint32_t lo = (uint32_t)(q * 32) << 16;
  const uint32_t cXh = 0, cXl = 64, cD = 128, cHh = 256, cHl = 384;
  const uint32_t id_h = tc::idesc_tf32(128, TC_H);
  const uint32_t sA = tc::smem_u32(rA), sB = tc::smem_u32(rB);
  const float b3 = __ldg(a.b3);
  uint32_t ph = 0, px = 0;
  bool first = true;
  for (int64_t tile = blockIdx.x; tile < t0 + t1; tile += gridDim.x) {
    const double* feat;
    int64_t n, r0;
    tile_src(tile, feat, n, r0);
    const bool second = tile >= t0;
    const int rows = (int)min((int64_t)128, n - r0);
    const int64_t row = r0 + lrow;
    // half 0 (prefetched), then half 1
    tc::mbar_wait(&xbar, px);
    px ^= 1;
    if (q < 2 && g < TC_K1 / 16)
      tc2_stage_x_smem(xs, lrow, min(rows, 64), a.F, g, tm + lo + cXh + 16 * g,
                       tm + lo + cXl + 16 * g);
    __syncthreads();
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (rows > 64) tc2_bulk_x(xs, feat, r0 + 64, rows - 64, a.F, &xbar);
      else asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(&xbar)) : "memory");
    }
    tc::mbar_wait(&xbar, px);
    px ^= 1;
    if (q >= 2 && g < TC_K1 / 16)
      tc2_stage_x_smem(xs, lrow - 64, rows - 64, a.F, g, tm + lo + cXh + 16 * g,
                       tm + lo + cXl + 16 * g);
    tc::tmem_st_wait();
    if (first) tc::mbar_wait(&wbar, 0);
    tc_sync();
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const int64_t nt = tile + gridDim.x;
      if (nt < t0 + t1) {   // prefetch the next tile's first half
        const double* f;
        int64_t nn, rr0;
        tile_src(nt, f, nn, rr0);
        tc2_bulk_x(xs, f, rr0, (int)min((int64_t)64, nn - rr0), a.F, &xbar);
      }
      mma_3xtf32(tm + cD, tm + cXh, tm + cXl, sA, sA + TC_K1 * TC_H * 4, TC_K1, id_h);
      tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, ph);
    ph ^= 1;
    tc::fence_after();
    tc2_tanh_split(tm + lo + cD + 32 * g, tm + lo + cHh + 32 * g, tm + lo + cHl + 32 * g,
                   sb1 + 32 * g);
    tc::tmem_st_wait();
    tc_sync();
    if (tid == 0) {
      mma_3xtf32(tm + cD, tm + cHh, tm + cHl, sB, sB + TC_H * TC_H * 4, TC_H, id_h);
      tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, ph);
    ph ^= 1;
    tc::fence_after();
    {
      float v[32];
      tc::tmem_ld32(tm + lo + cD + 32 * g, v);
      float acc = 0.f;
#pragma unroll
      for (int j = 0; j < 32; ++j) acc = fmaf(tanhf(v[j] + sb2[32 * g + j]), sw3[32 * g + j], acc);
      // park the group's partial dot in TMEM column cD+g (D is dead now)
      tc::tmem_st1(tm + lo + cD + g, acc);
      tc::tmem_st_wait();
    }
    tc_sync();
    if (g == 0) {
      float p4[4];
      tc::tmem_ld4(tm + lo + cD, p4);
      if (row < n) (second ? a.out1 : a.out0)[row] = ((p4[0] + p4[1]) + (p4[2] + p4[3])) + b3;
    }
    first = false;
    tc_sync();
  }
  if (warp == 0) tc::tmem_dealloc(tm, 512);
}

}  // namespace harl
