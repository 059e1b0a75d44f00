// Self-test of the tcgen05 building blocks used by mlp_tc.cuh: one
// M=128 x N=128 x K=64 kind::tf32 product with the accumulator in TMEM,
// A either from TMEM (mode 0, the ".ts" form the MLP kernels use) or from
// shared memory (mode 1), B from shared memory in the K-major no-swizzle
// canonical layout; operands are passed through unrounded so the caller can
// also see how the tensor core consumes fp32 bits (mode 2 = mode 0 without
// the host-side rounding contract).
#pragma once

#include "tc_common.cuh"

namespace harl {

constexpr int PROBE_M = 128, PROBE_N = 128, PROBE_K = 64;

__global__ void __launch_bounds__(128)
k_tc_probe(const float* A, const float* B, float* D, int mode) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  extern __shared__ __align__(1024) uint8_t sm[];
  if (mode >= 3) {   // M = 64 layout probes (tc_probe_m64 below)
    return;
  }
  float* sB = (float*)sm;                              // N x K (K-major)
  float* sA = (float*)(sm + PROBE_N * PROBE_K * 4);    // M x K (K-major)
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tc::tmem_alloc(&tbase, 256);
  if (tid == 0) tc::mbar_init(&bar, 1);
  // B[k][n] (row-major K x N) -> K-major core-matrix layout of B^T
  for (int i = tid; i < PROBE_K * PROBE_N; i += blockDim.x) {
    const int k = i / PROBE_N, n = i % PROBE_N;
    *(float*)((uint8_t*)sB + tc::kmajor_off(n, k, PROBE_K)) = B[i];
  }
  if (mode == 1) {
    for (int i = tid; i < PROBE_M * PROBE_K; i += blockDim.x) {
      const int m = i / PROBE_K, k = i % PROBE_K;
      *(float*)((uint8_t*)sA + tc::kmajor_off(m, k, PROBE_K)) = A[i];
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = tbase;
  const uint32_t d_col = 0, a_col = 128;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  if (mode != 1) {
    // row tid of A -> TMEM lane tid, columns a_col .. a_col+63
    float v[32];
    for (int c0 = 0; c0 < PROBE_K; c0 += 32) {
      for (int j = 0; j < 32; ++j) v[j] = A[tid * PROBE_K + c0 + j];
      tc::tmem_st32(tm + lane_base + a_col + c0, v);
    }
    tc::tmem_st_wait();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (tid == 0) {
    const uint32_t idesc = tc::idesc_tf32(PROBE_M, PROBE_N);
    const uint32_t sb = PROBE_K / 4 * 128;
    for (int s = 0; s < PROBE_K / 8; ++s) {
      const uint64_t bd = tc::sdesc(tc::smem_u32(sB) + 256 * s, 128, sb);
      if (mode == 1) {
        const uint64_t ad = tc::sdesc(tc::smem_u32(sA) + 256 * s, 128, sb);
        tc::mma_tf32_ss(tm + d_col, ad, bd, idesc, s > 0);
      } else {
        tc::mma_tf32_ts(tm + d_col, tm + a_col + 8 * s, bd, idesc, s > 0);
      }
    }
    tc::mma_commit(&bar);
  }
  __syncwarp();
  tc::mbar_wait(&bar, 0);
  tc::fence_after();
  float out[32];
  for (int c0 = 0; c0 < PROBE_N; c0 += 32) {
    tc::tmem_ld32(tm + lane_base + d_col + c0, out);
    for (int j = 0; j < 32; ++j) D[tid * PROBE_N + c0 + j] = out[j];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tm, 256);
}

// M = 64 probes.  mode 3: A (64 x 64) from shared memory; mode 4: A from
// TMEM, row r at lane (r % 16) + 32 (r / 16); both MMA M=64 N=128 K=64 and
// dump every TMEM lane (128) x 128 columns into D[lane][col].  mode 5: TMEM
// filled with lane * 1000 + col, read back with tcgen05.ld.16x256b.x1 at the
// warp's lane quarter (and +16): D[(w * 64 + half * 32 + t) * 4 + i].
__global__ void __launch_bounds__(128)
k_tc_probe_m64(const float* A, const float* B, float* D, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  float* sB = (float*)sm;                              // N x K (K-major)
  float* sA = (float*)(sm + PROBE_N * PROBE_K * 4);    // 64 x K (K-major)
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tc::tmem_alloc(&tbase, 256);
  if (tid == 0) tc::mbar_init(&bar, 1);
  for (int i = tid; i < PROBE_K * PROBE_N; i += blockDim.x) {
    const int k = i / PROBE_N, n = i % PROBE_N;
    *(float*)((uint8_t*)sB + tc::kmajor_off(n, k, PROBE_K)) = B[i];
  }
  for (int i = tid; i < 64 * PROBE_K; i += blockDim.x) {
    const int m = i / PROBE_K, k = i % PROBE_K;
    *(float*)((uint8_t*)sA + tc::kmajor_off(m, k, PROBE_K)) = A[i];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = tbase;
  const uint32_t d_col = 0, a_col = 128;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  {
    // clear D and A regions (all lanes)
    float z[32];
    for (int j = 0; j < 32; ++j) z[j] = mode == 5 ? (float)(tid * 1000 + j) : 0.f;
    for (int c0 = 0; c0 < 256; c0 += 32) {
      if (mode == 5)
        for (int j = 0; j < 32; ++j) z[j] = (float)(tid * 1000 + c0 + j);
      tc::tmem_st32(tm + lane_base + c0, z);
    }
    tc::tmem_st_wait();
  }
  if (mode == 4) {
    // row r (0..63) of A -> lane (r % 16) + 32 (r / 16): warp w's lanes 0-15
    const int r = 16 * warp + lane;
    float v[32];
    for (int c0 = 0; c0 < PROBE_K; c0 += 32) {
      for (int j = 0; j < 32; ++j) v[j] = lane < 16 ? A[r * PROBE_K + c0 + j] : 0.f;
      tc::tmem_st32(tm + lane_base + a_col + c0, v);
    }
    tc::tmem_st_wait();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (mode != 5) {
    if (tid == 0) {
      const uint32_t idesc = tc::idesc_tf32(64, PROBE_N);
      const uint32_t sb = PROBE_K / 4 * 128;
      for (int s = 0; s < PROBE_K / 8; ++s) {
        const uint64_t bd = tc::sdesc(tc::smem_u32(sB) + 256 * s, 128, sb);
        if (mode == 3) {
          const uint64_t ad = tc::sdesc(tc::smem_u32(sA) + 256 * s, 128, sb);
          tc::mma_tf32_ss(tm + d_col, ad, bd, idesc, s > 0);
        } else {
          tc::mma_tf32_ts(tm + d_col, tm + a_col + 8 * s, bd, idesc, s > 0);
        }
      }
      tc::mma_commit(&bar);
    }
    __syncwarp();
    tc::mbar_wait(&bar, 0);
    tc::fence_after();
    float out[32];
    for (int c0 = 0; c0 < PROBE_N; c0 += 32) {
      tc::tmem_ld32(tm + lane_base + d_col + c0, out);
      for (int j = 0; j < 32; ++j) D[tid * PROBE_N + c0 + j] = out[j];
    }
  } else {
    for (int half = 0; half < 2; ++half) {
      uint32_t r[4];
      const uint32_t addr = tm + ((uint32_t)(warp * 32 + 16 * half) << 16);
      asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int i = 0; i < 4; ++i)
        D[((warp * 2 + half) * 32 + lane) * 4 + i] = __uint_as_float(r[i]);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tm, 256);
}

// kind::f16 probes (fp16 operands, fp32 accumulate), M=128 N=128 K=64:
// mode 6: A from TMEM, two fp16 per 32-bit column, element k of a row at
// column k/2, even k in the low half; mode 7: A from shared memory in the
// 2-byte K-major core layout.  B from shared memory in the same layout.
// The operands arrive as fp32 values the host made fp16-exact.
__global__ void __launch_bounds__(128)
k_tc_probe_f16(const float* A, const float* B, float* D, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sB = sm;                                  // N x K fp16 (K-major)
  uint8_t* sA = sm + PROBE_N * PROBE_K * 2;          // M x K fp16
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tc::tmem_alloc(&tbase, 256);
  if (tid == 0) tc::mbar_init(&bar, 1);
  for (int i = tid; i < PROBE_K * PROBE_N; i += blockDim.x) {
    const int k = i / PROBE_N, n = i % PROBE_N;
    *(__half*)(sB + tc::kmajor16_off(n, k, PROBE_K)) = __float2half_rn(B[i]);
  }
  for (int i = tid; i < PROBE_M * PROBE_K; i += blockDim.x) {
    const int m = i / PROBE_K, k = i % PROBE_K;
    *(__half*)(sA + tc::kmajor16_off(m, k, PROBE_K)) = __float2half_rn(A[i]);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = tbase;
  const uint32_t d_col = 0, a_col = 128;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  if (mode == 6) {
    float v[32];
    for (int j = 0; j < 32; ++j)
      v[j] = __uint_as_float(tc::pack_half2(A[tid * PROBE_K + 2 * j],
                                            A[tid * PROBE_K + 2 * j + 1]));
    tc::tmem_st32(tm + lane_base + a_col, v);
    tc::tmem_st_wait();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (tid == 0) {
    const uint32_t idesc = tc::idesc_f16(PROBE_M, PROBE_N);
    const uint32_t sb = PROBE_K / 8 * 128;
    for (int s = 0; s < PROBE_K / 16; ++s) {
      const uint64_t bd = tc::sdesc(tc::smem_u32(sB) + 256 * s, 128, sb);
      if (mode == 7) {
        const uint64_t ad = tc::sdesc(tc::smem_u32(sA) + 256 * s, 128, sb);
        tc::mma_f16_ss(tm + d_col, ad, bd, idesc, s > 0);
      } else {
        tc::mma_f16_ts(tm + d_col, tm + a_col + 8 * s, bd, idesc, s > 0);
      }
    }
    tc::mma_commit(&bar);
  }
  __syncwarp();
  tc::mbar_wait(&bar, 0);
  tc::fence_after();
  float out[32];
  for (int c0 = 0; c0 < PROBE_N; c0 += 32) {
    tc::tmem_ld32(tm + lane_base + d_col + c0, out);
    for (int j = 0; j < 32; ++j) D[tid * PROBE_N + c0 + j] = out[j];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tm, 256);
}

}  // namespace harl
