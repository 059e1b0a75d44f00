// 3xFP16 rollout networks on tcgen05 kind::f16 (PolicyNet.forward,
// rlcore.py:136-146; ValueNet.estimate, rlcore.py:161-178).
//
// Precision: every fp32 operand x is split into hi = fp16(x) and lo =
// fp16(x - hi) (both 11-bit significands, like the 3xTF32 split of
// mlp_tc2.cuh) and a*b ~= ah*bh + ah*bl + al*bh is accumulated in fp32 in
// TMEM.  kind::f16 runs a K=16 step in the time kind::tf32 runs K=8, and
// fp16 operands take half the bytes, so:
//   * all weights stay resident in shared memory for the launch (W1, W2 and
//     the heads, hi+lo: 146 KB for the conv2d heads) -- no re-streaming per
//     tile;
//   * a tile's TMEM footprint is 256 columns (D: 128 fp32 columns; A: X or
//     H, hi and lo packed two fp16 per column), so TWO 128-row tiles are in
//     flight per CTA: while the CUDA cores run one tile's epilogue (tanh,
//     split, tcgen05.st) the tensor core runs the other tile's layer.
// Weights are scaled by a power of two per matrix (chosen at pack time from
// max|W|, kept by the Adam refresh) so their fp16 halves stay normal; the
// epilogue multiplies the accumulator back (exact).
//
// Thread layout (16 warps): warp w reads/writes TMEM lane quarter q = w % 4
// (rows 32q..32q+31 of the tile, the hardware's lane-quarter rule) and
// column group g = w / 4.
#pragma once

#include "mlp_tc2.cuh"
#include "episode_kernels.cuh"

namespace harl {

constexpr int F16_FLOATS = 2048;                  // bias / scale block (bytes)
constexpr int F16_W1 = TC_H * TC_K1 * 2;          // one half of W1 (16 KB)
constexpr int F16_W2 = TC_H * TC_H * 2;           // one half of W2 (32 KB)
constexpr int F16_NHP_MAX = 128;                  // heads D fits one slot
// float indices inside the bias block
constexpr int F16_B1 = 0, F16_B2 = 128, F16_B3 = 256, F16_SC = 384;

// image: [floats][W1 hi][W1 lo][W2 hi][W2 lo]([Wh hi][Wh lo])
__host__ __device__ constexpr int f16_off_w1() { return F16_FLOATS; }
__host__ __device__ constexpr int f16_off_w2() { return F16_FLOATS + 2 * F16_W1; }
__host__ __device__ constexpr int f16_off_wh() {
  return F16_FLOATS + 2 * F16_W1 + 2 * F16_W2;
}
__host__ __device__ inline int f16_image_bytes(int NHP) {
  return f16_off_wh() + 2 * NHP * TC_H * 2;
}

// accurate tanh with one MUFU op: e = exp(-2|x|) (ex2.approx, rel. err
// ~2^-22); r = 2/(1+e) = 1/d, d = (1+e)/2 in (1/2, 1], from the minimax
// quadratic seed (rel. err 1/99) and two Newton steps (rel. err 1e-8);
// tanh = sign(x)(1 - e r).  Absolute error <= 1.4e-7 over the whole range
// (tanhf issues two MUFU ops per element, which bound the epilogue).
// 12 instructions per element.
__device__ __forceinline__ float tanh_1mufu(float x) {
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(fabsf(x) * -2.8853900817779268f));
  const float d = fmaf(e, 0.5f, 0.5f);
  float r = fmaf(fmaf(2.5858586f, d, -5.8181818f), d, 4.2424242f);
  r = fmaf(r, fmaf(-d, r, 1.f), r);
  r = fmaf(r, fmaf(-d, r, 1.f), r);
  return copysignf(fmaf(-e, r, 1.f), x);
}

// tanh with two MUFU ops and three other instructions: e = 2^(2x log2 e),
// tanh = 1 - 2 / (e + 1) with rcp.approx (|error| <= ~3e-7, near x = 0
// from the cancellation; +-1 exactly for |x| > 44, NaN propagates).  The
// hidden epilogues alternate it with tanh_1mufu over their columns: one
// is bound by the MUFU pipe (16 ops/clk/SM), the other by issue slots,
// and the mix keeps both below the single-formula bound.
#ifndef HARL_TANH_MIX
#define HARL_TANH_MIX 1
#endif
__device__ __forceinline__ float tanh_2mufu(float x) {
  float e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x * 2.8853900817779268f));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(e + 1.0f));
  return fmaf(-2.0f, r, 1.0f);
}
template <int J>
__device__ __forceinline__ float tanh_mix(float x) {
  if (HARL_TANH_MIX && (J & 1) == 0) return tanh_2mufu(x);
  return tanh_1mufu(x);
}

// (x0, x1) -> fp16 hi/lo pair words for two consecutive K elements:
// hi = fp16(x) (RN), lo = fp16(x - hi) (x - hi is exact in fp32)
__device__ __forceinline__ void split16x2(float x0, float x1, uint32_t& hi,
                                          uint32_t& lo) {
  hi = tc::pack_half2(x0, x1);
  const float2 h = __half22float2(*reinterpret_cast<const __half2*>(&hi));
  lo = tc::pack_half2(x0 - h.x, x1 - h.y);
}

__device__ inline void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
      ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]),
        "r"(r[5]), "r"(r[6]), "r"(r[7])
      : "memory");
}

__device__ inline void tmem_st16u(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
      ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]),
        "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]),
        "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

// hidden epilogue: D cols 32g.. -> tanh(D/scale + b) -> H hi/lo (K = 128:
// hi at a_hi, lo at a_hi + 64), 16 columns at a time
__device__ __forceinline__ void f16_hidden(uint32_t t_d, uint32_t a_hi,
                                           const float* b, float inv, int g) {
#pragma unroll
  for (int hlf = 0; hlf < 2; ++hlf) {
    const int c0 = 32 * g + 16 * hlf;
    float v[16];
    tc::tmem_ld16(t_d + c0, v);
    const float4* b4 = (const float4*)(b + c0);
    uint32_t h[8], l[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 bb = b4[j];
      float z0, z1, z2, z3;
      if (j & 1) {
        z0 = tanh_mix<1>(fmaf(v[4 * j], inv, bb.x));
        z1 = tanh_mix<1>(fmaf(v[4 * j + 1], inv, bb.y));
        z2 = tanh_mix<1>(fmaf(v[4 * j + 2], inv, bb.z));
        z3 = tanh_mix<1>(fmaf(v[4 * j + 3], inv, bb.w));
      } else {
        z0 = tanh_mix<0>(fmaf(v[4 * j], inv, bb.x));
        z1 = tanh_mix<0>(fmaf(v[4 * j + 1], inv, bb.y));
        z2 = tanh_mix<0>(fmaf(v[4 * j + 2], inv, bb.z));
        z3 = tanh_mix<0>(fmaf(v[4 * j + 3], inv, bb.w));
      }
      split16x2(z0, z1, h[2 * j], l[2 * j]);
      split16x2(z2, z3, h[2 * j + 1], l[2 * j + 1]);
    }
    tmem_st8(a_hi + c0 / 2, h);
    tmem_st8(a_hi + 64 + c0 / 2, l);
  }
}

// D = A_hi B_hi + A_hi B_lo + A_lo B_hi over K (one thread): A in TMEM
// (hi at a_hi, lo at a_lo, 8 columns per K=16 step), B in shared memory
__device__ __forceinline__ void mma_3xf16(uint32_t d, uint32_t a_hi,
                                          uint32_t a_lo, uint32_t b_hi,
                                          uint32_t b_lo, int K,
                                          uint32_t idesc) {
  const uint32_t sbo = (uint32_t)(K / 8 * 128);
  for (int s = 0; s < K / 16; ++s) {
    const uint64_t bh = tc::sdesc(b_hi + 256 * s, 128, sbo);
    const uint64_t bl = tc::sdesc(b_lo + 256 * s, 128, sbo);
    tc::mma_f16_ts(d, a_hi + 8 * s, bh, idesc, s > 0);
    tc::mma_f16_ts(d, a_hi + 8 * s, bl, idesc, 1);
    tc::mma_f16_ts(d, a_lo + 8 * s, bh, idesc, 1);
  }
}

// the same with A in shared memory (layer 1: the X tile's fp16 halves)
__device__ __forceinline__ void mma_3xf16_ss(uint32_t d, uint32_t a_hi,
                                             uint32_t a_lo, uint32_t b_hi,
                                             uint32_t b_lo, int K,
                                             uint32_t idesc) {
  const uint32_t sbo = (uint32_t)(K / 8 * 128);
  for (int s = 0; s < K / 16; ++s) {
    const uint64_t ah = tc::sdesc(a_hi + 256 * s, 128, sbo);
    const uint64_t al = tc::sdesc(a_lo + 256 * s, 128, sbo);
    const uint64_t bh = tc::sdesc(b_hi + 256 * s, 128, sbo);
    const uint64_t bl = tc::sdesc(b_lo + 256 * s, 128, sbo);
    tc::mma_f16_ss(d, ah, bh, idesc, s > 0);
    tc::mma_f16_ss(d, ah, bl, idesc, 1);
    tc::mma_f16_ss(d, al, bh, idesc, 1);
  }
}

struct F16Args {
  const double* feat0;  // [n0][F] (policy: the only input)
  const double* feat1;  // value: X' [n1][F], may be null
  int64_t n0, n1;
  int32_t F, NH, NHP;
  int32_t nxb;          // X staging buffers in shared memory (1 or 2)
  float* logits;        // policy: [n][128] (the sampler's input)
  float* logits_out;    // policy: optional [n][NH]
  float* out0;          // value: v [n0]
  float* out1;          // value: v [n1]
  const float* b3;      // value: [1] device
  const uint8_t* img;   // f16 image (k_pack16)
  int32_t early_w;      // the image was not written by the previous launch:
                        // load it before the PDL wait
  int32_t pair;         // value: n0 == n1, CTA-local pairs (X tile p, X' tile p)
  int32_t fin;          // value: the step's finish bookkeeping in the epilogue
};

// warp roles: 16 epilogue warps (TMEM lane quarter w % 4, column group
// w / 4; they also convert the X tiles) and one MMA / copy issuing warp
constexpr int F16_EPI_WARPS = 16;
constexpr int F16_THREADS = 32 * (F16_EPI_WARPS + 1);

__host__ __device__ inline int f16_xbuf_bytes(int F) {
  return (128 * F * 8 + 127) / 128 * 128;
}
// dynamic shared memory: the image, nxb X staging tiles (fp64 rows as in
// global memory) and, for the value net, the per-group partial dots
__host__ __device__ inline int f16_smem_bytes(bool policy, int NHP, int F,
                                              int nxb) {
  return (policy ? f16_image_bytes(NHP) : f16_off_wh()) +
         nxb * f16_xbuf_bytes(F) + (policy ? 0 : 2 * 4 * 128 * 4);
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];"
               ::"r"(tc::smem_u32(bar)) : "memory");
}

// this thread's X row slice (K columns 16g .. 16g+15) from the staged fp64
// tile -> fp16 hi/lo into the slot's A region (hi at a_hi, lo at a_hi + 32)
__device__ __forceinline__ void f16_stage_x(const double* xs, int rows, int F,
                                            int lrow, int g, uint32_t a_hi) {
  const double* src = xs + lrow * F;
  const bool ok = lrow < rows;
  uint32_t h[8], l[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int k = 16 * g + 2 * j;
    const float x0 = (ok && k < F) ? (float)src[k] : 0.f;
    const float x1 = (ok && k + 1 < F) ? (float)src[k + 1] : 0.f;
    split16x2(x0, x1, h[j], l[j]);
  }
  tmem_st8(a_hi + 8 * g, h);
  tmem_st8(a_hi + 32 + 8 * g, l);
}

// POLICY: trunk + heads (3 layers), logits out.  VALUE: trunk + 128->1 dot.
//
// Two 128-row tiles in flight per CTA: my tiles alternate between TMEM
// slots s = tile parity (D at 256 s, A = X or H at 256 s + 128).  Events
// run in one global order shared by the epilogue warps and the MMA
// thread: event e belongs to slot e % 2, and slot 1 lags one stage, so the
// two slots' output stages (which also stage the next X tile) are evenly
// spaced.  Per event the epilogue waits done[s] (the slot's MMA commit),
// works, and arrives on ready[s]; the MMA thread waits ready[s] and issues
// the slot's next layer.  X tiles arrive in shared memory by bulk copy
// (xfull[b]), issued by the MMA thread as soon as a buffer's previous tile
// has been converted.
//
// VALUE with a.fin (the step's finish fused, k_gbt_finish's epilogue work:
// advantage/TD, replay push, entry log, Track.advance -- tuner.py:393-412,
// rlcore.py:231-265, stopping.py:45-53): with a.pair the CTA takes X tile p
// and X' tile p as its slot-0 / slot-1 tiles, so the thread that writes
// V(X')[r] wrote V(X)[r] one event earlier (same lane quarter, lane and
// column group) and runs finish_row for r right there; the other column
// groups copy the tile's pushed X / X' rows into their replay slots.
// Without a.pair (V(X) reused from the previous step: n0 = 0) V(X) comes
// from the earlier launch.
template <bool POLICY, bool FIN = false>
__global__ void __launch_bounds__(F16_THREADS, 1)
k_mlp_f16(F16Args a, const __grid_constant__ GbtFinishArgs fin) {
  extern __shared__ __align__(1024) uint8_t smf[];
  const float* fl = (const float*)smf;
  const int img_bytes = POLICY ? f16_image_bytes(a.NHP) : f16_off_wh();
  const int xbb = f16_xbuf_bytes(a.F);
  uint8_t* xsm = smf + img_bytes;
  float* part = (float*)(xsm + a.nxb * xbb);       // value: [2][4][128]
  __shared__ uint64_t wbar[3], done[2], ready[2], xfull[2];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int NL = POLICY ? 3 : 2;
  const int NXB = a.nxb;
  const int64_t t0 = (a.n0 + 127) / 128, t1 = (a.n1 + 127) / 128;
  const int64_t units = a.pair ? t1 : t0 + t1;   // pairs or tiles
  const int64_t mine_u = units > blockIdx.x ? (units - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t mine = a.pair ? 2 * mine_u : mine_u;
  const int64_t cnt0 = (mine + 1) / 2, cnt1 = mine / 2;   // tiles per slot
  // global event e -> slot s = e % 2, slot step k = e / 2 - s (slot 1 lags
  // one stage), tile k / NL, layer k % NL
  const int64_t n_ev = 2 * (NL * cnt0 + 1) + 2;
  if (POLICY) dbg_ts(0);
  if (warp == 0) tc::tmem_alloc(&tbase, 512);
  if (tid == 0) {
    for (int i = 0; i < 3; ++i) tc::mbar_init(&wbar[i], 1);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&done[i], 1);
      tc::mbar_init(&ready[i], F16_EPI_WARPS);
      tc::mbar_init(&xfull[i], 1);
    }
  }
  tc_sync();
  if (POLICY) dbg_ts(1);
  const uint32_t tm = tbase;
  const bool mma_thread = mine > 0 && warp == F16_EPI_WARPS && lane == 0;
  auto load_weights = [&]() {
    tc::bulk_load(smf, a.img, (uint32_t)f16_off_w2(), &wbar[0]);
    tc::bulk_load(smf + f16_off_w2(), a.img + f16_off_w2(), 2 * F16_W2, &wbar[1]);
    if (POLICY)
      tc::bulk_load(smf + f16_off_wh(), a.img + f16_off_wh(),
                    (uint32_t)(2 * a.NHP * TC_H * 2), &wbar[2]);
  };
  if (mma_thread && a.early_w) load_weights();
  griddep_wait();  // PDL: the feature rows (and unsettled weights) are ready
  auto tile_of = [&](int64_t j, const double*& f, int64_t& r0, int& rows,
                     bool& second) {
    int64_t t;
    if (a.pair) {
      t = blockIdx.x + (j >> 1) * gridDim.x;
      second = (j & 1) != 0;
    } else {
      t = blockIdx.x + j * gridDim.x;
      second = t >= t0;
      if (second) t -= t0;
    }
    f = second ? a.feat1 : a.feat0;
    const int64_t n = second ? a.n1 : a.n0;
    r0 = t * 128;
    rows = (int)min((int64_t)128, n - r0);
  };
  if (mine > 0 && warp < F16_EPI_WARPS) {
    // ---------------- epilogue warps ------------------------------------
    const int q = warp & 3, g = warp >> 2;
    const int lrow = q * 32 + lane;
    const uint32_t lq = (uint32_t)(q * 32) << 16;
    auto arrive = [&](int s) {
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ready[s]);
    };
    // tile jt's staged rows -> A region at a_hi
    auto stage_tile = [&](int64_t jt, uint32_t a_hi) {
      const double* f;
      int64_t r0;
      int rows;
      bool sec;
      tile_of(jt, f, r0, rows, sec);
      const int b = (int)(jt % NXB);
      tc::mbar_wait(&xfull[b], (uint32_t)((jt / NXB) & 1));
      f16_stage_x((const double*)(xsm + b * xbb), rows, a.F, lrow, g, a_hi);
    };
    for (int s = 0; s < 2 && s < mine; ++s) {
      stage_tile(s, tm + lq + 256 * s + 128);
      tc::tmem_st_wait();
      arrive(s);
    }
    if (POLICY) dbg_ts(2);
    tc::mbar_wait(&wbar[0], 0);           // biases and scales
    if (POLICY) dbg_ts(3);
    const float inv1 = fl[F16_SC + 4], inv2 = fl[F16_SC + 5];
    uint32_t ph = 0;                      // bit s: done[s] parity
    // phase accounting (harl_debug_timestamps(3): CTA 0, warp 0 -> slots
    // 32 wait, 33 hidden, 34 output + staging, 35 events, 38 total)
    const bool prof = g_dbg_on == 3 && blockIdx.x == 0 && warp == 0;
    unsigned long long c_wait = 0, c_hid = 0, c_out = 0, n_evt = 0;
    const unsigned long long c_start = clock64();
    int ev_l0 = 0, ev_l1 = 0;           // (policy: the event order walked
    int64_t ev_t0 = 0, ev_t1 = 0;       // with per-slot counters)
    for (int64_t e = 0; e < n_ev; ++e) {
      int s, l;
      int64_t st;
      if constexpr (POLICY) {
        s = (int)(e & 1);
        if (e == 1) continue;           // slot 1 lags one stage
        l = s ? ev_l1 : ev_l0;
        st = s ? ev_t1 : ev_t0;
        if (s) {
          if (++ev_l1 == NL) { ev_l1 = 0; ++ev_t1; }
        } else {
          if (++ev_l0 == NL) { ev_l0 = 0; ++ev_t0; }
        }
        if (st >= (s ? cnt1 : cnt0)) continue;
      } else {
        // (the value kernel keeps the division form: the counters' extra
        // live registers spill there)
        (void)ev_l0; (void)ev_l1; (void)ev_t0; (void)ev_t1;
        s = (int)(e & 1);
        const int64_t k = (e >> 1) - s;
        if (k < 0) continue;
        st = k / NL;
        l = (int)(k % NL);
        if (st >= (s ? cnt1 : cnt0)) continue;
      }
      const int64_t jt = 2 * st + s;
      const bool has_next = st + 1 < (s ? cnt1 : cnt0);
      const unsigned long long c0 = prof ? clock64() : 0;
      tc::mbar_wait(&done[s], (ph >> s) & 1u);
      if (POLICY && e == 0) dbg_ts(6);
      ph ^= 1u << s;
      tc::fence_after();
      const unsigned long long c1 = prof ? clock64() : 0;
      const uint32_t t_d = tm + lq + 256 * s;
      if (l < NL - 1) {
        f16_hidden(t_d, t_d + 128, fl + (l == 0 ? F16_B1 : F16_B2),
                   l == 0 ? inv1 : inv2, g);
      } else {
        const double* f;
        int64_t r0;
        int rows;
        bool sec;
        tile_of(jt, f, r0, rows, sec);
        if constexpr (POLICY) {
          if (32 * g < a.NHP) {
            float v[32];
            tc::tmem_ld32(t_d + 32 * g, v);
            const float inv = fl[F16_SC + 6];
            const float* bh = fl + F16_B3 + 32 * g;
#pragma unroll
            for (int c = 0; c < 32; ++c) v[c] = fmaf(v[c], inv, bh[c]);
            if (lrow < rows) {
              float* dst = a.logits + (r0 + lrow) * TC_H + 32 * g;
              const int cmax = a.NHP - 32 * g;   // NHP: multiple of 16
#pragma unroll
              for (int c = 0; c < 32; c += 4)
                if (c < cmax)
                  *(float4*)(dst + c) = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
              if (a.logits_out) {
#pragma unroll
                for (int c = 0; c < 32; ++c)
                  if (32 * g + c < a.NH)
                    a.logits_out[(r0 + lrow) * a.NH + 32 * g + c] = v[c];
              }
            }
          }
        } else {
          float v[32];
          tc::tmem_ld32(t_d + 32 * g, v);
          const float* b2 = fl + F16_B2 + 32 * g;
          const float* w3 = fl + F16_B3 + 32 * g;
          float acc = 0.f;
#pragma unroll
          for (int c = 0; c < 32; ++c)
            acc = fmaf((c & 4) ? tanh_mix<1>(fmaf(v[c], inv2, b2[c]))
                               : tanh_mix<0>(fmaf(v[c], inv2, b2[c])),
                       w3[c], acc);
          part[(s * 4 + g) * 128 + lrow] = acc;
          // the quarter's four column groups (warps q, q+4, q+8, q+12)
          asm volatile("bar.sync %0, 128;" ::"r"(1 + q) : "memory");
          if (g == 0 && lrow < rows) {
            const float* pp = part + s * 512;
            (sec ? a.out1 : a.out0)[r0 + lrow] =
                ((pp[lrow] + pp[128 + lrow]) + (pp[256 + lrow] + pp[384 + lrow])) +
                __ldg(a.b3);
          }
          if (FIN && sec) {     // X' tile: V(X) and V(X') of its rows are in
            const int64_t wpos = fin.wpos_dev ? *fin.wpos_dev : fin.a.wpos;
            if (g == 0) {       // memory, written by this thread or earlier
              if (lrow < rows)
                finish_row(fin.a, fin.io, fin.ring, fin.log, fin.ts, wpos, r0 + lrow);
            } else if (fin.a.rl) {
              const int64_t lo = r0 > fin.a.keep_from ? r0 : fin.a.keep_from;
              const int64_t hi = r0 + rows;
              if (lo < hi) {
                const int F = fin.a.F;
                const int total = (int)(hi - lo) * F;
                const double* __restrict__ sx = fin.io.feat + lo * F;
                const double* __restrict__ sxn = fin.io.feat_new + lo * F;
                // all loads of a batch before its stores (the ring could
                // alias the rows as far as the compiler knows)
                constexpr int U = 8;
                for (int e0 = (g - 1) * 128 + lrow; e0 < total; e0 += 384 * U) {
                  double vx[U], vxn[U];
#pragma unroll
                  for (int u = 0; u < U; ++u) {
                    const int e = e0 + u * 384;
                    vx[u] = e < total ? sx[e] : 0.0;
                    vxn[u] = e < total ? sxn[e] : 0.0;
                  }
#pragma unroll
                  for (int u = 0; u < U; ++u) {
                    const int e = e0 + u * 384;
                    if (e < total) {
                      const int rr = e / F, k = e - rr * F;
                      const int64_t slot = (wpos + lo + rr) % fin.ring.cap;
                      fin.ring.X[slot * F + k] = vx[u];
                      fin.ring.Xn[slot * F + k] = vxn[u];
                    }
                  }
                }
              }
            }
          }
        }
        // the slot's last layer is done with A: stage its next tile's X
        if (has_next) stage_tile(jt + 2, t_d + 128);
      }
      tc::tmem_st_wait();
      arrive(s);
      if (prof) {
        const unsigned long long c2 = clock64();
        c_wait += c1 - c0;
        (l < NL - 1 ? c_hid : c_out) += c2 - c1;
        ++n_evt;
      }
    }
    if (prof && lane == 0) {
      g_dbg_ts[32] = c_wait;
      g_dbg_ts[33] = c_hid;
      g_dbg_ts[34] = c_out;
      g_dbg_ts[35] = n_evt;
      g_dbg_ts[38] = clock64() - c_start;
    }
  } else if (mma_thread) {
    // ---------------- MMA / copy issuing thread --------------------------
    auto copy_x = [&](int64_t jt) {       // tile jt -> buffer jt % NXB
      if (jt >= mine) return;
      const double* f;
      int64_t r0;
      int rows;
      bool sec;
      tile_of(jt, f, r0, rows, sec);
      const int b = (int)(jt % NXB);
      tc::bulk_f64((double*)(xsm + b * xbb), f + r0 * a.F,
                   (uint32_t)rows * a.F, &xfull[b]);
    };
    // the first X tiles ahead of the weight image (the epilogue warps
    // convert them while the image streams in), then the image in three
    // pieces: W1 + biases, W2, heads -- each layer's first MMA waits for
    // its own piece only
    for (int64_t jt = 0; jt < NXB; ++jt) copy_x(jt);
    if (!a.early_w) load_weights();
    const uint32_t sw = tc::smem_u32(smf);
    const uint32_t id_h = tc::idesc_f16(128, TC_H);
    const uint32_t id_o = tc::idesc_f16(128, POLICY ? a.NHP : TC_H);
    uint32_t pr = 0;                      // bit s: ready[s] parity
    const bool prof = g_dbg_on == 3 && blockIdx.x == 0;   // slots 36/37
    unsigned long long c_wait = 0, c_iss = 0;
    auto wait_ready = [&](int s) {
      const unsigned long long c0 = prof ? clock64() : 0;
      tc::mbar_wait(&ready[s], (pr >> s) & 1u);
      pr ^= 1u << s;
      tc::fence_after();
      if (prof) c_wait += clock64() - c0;
    };
    auto issue = [&](int s, int l) {
      if (l > 0) tc::mbar_wait(&wbar[l], 0);   // that layer's weights (once
                                              // complete, an immediate test)
      const unsigned long long c0 = prof ? clock64() : 0;
      const uint32_t d = tm + 256 * s, ah = d + 128;
      if (l == 0)
        mma_3xf16(d, ah, ah + 32, sw + f16_off_w1(),
                  sw + f16_off_w1() + F16_W1, TC_K1, id_h);
      else if (l == 1)
        mma_3xf16(d, ah, ah + 64, sw + f16_off_w2(),
                  sw + f16_off_w2() + F16_W2, TC_H, id_h);
      else
        mma_3xf16(d, ah, ah + 64, sw + f16_off_wh(),
                  sw + f16_off_wh() + a.NHP * TC_H * 2, TC_H, id_o);
      tc::mma_commit(&done[s]);
      if (prof) c_iss += clock64() - c0;
    };
    tc::mbar_wait(&wbar[0], 0);
#ifdef HARL_PHASE_TS
    if (POLICY && blockIdx.x == 0 && g_dbg_on) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      g_dbg_ts[4] = t;
    }
#endif
    // prologue: the slots' first tiles are staged (tile s converted)
    for (int s = 0; s < 2 && s < mine; ++s) {
      wait_ready(s);
      copy_x(s + NXB);
      issue(s, 0);
    }
#ifdef HARL_PHASE_TS
    if (POLICY && blockIdx.x == 0 && g_dbg_on) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      g_dbg_ts[5] = t;
    }
#endif
    int ev_l0 = 0, ev_l1 = 0;           // (policy: the event order walked
    int64_t ev_t0 = 0, ev_t1 = 0;       // with per-slot counters)
    for (int64_t e = 0; e < n_ev; ++e) {
      int s, l;
      int64_t st;
      if constexpr (POLICY) {
        s = (int)(e & 1);
        if (e == 1) continue;           // slot 1 lags one stage
        l = s ? ev_l1 : ev_l0;
        st = s ? ev_t1 : ev_t0;
        if (s) {
          if (++ev_l1 == NL) { ev_l1 = 0; ++ev_t1; }
        } else {
          if (++ev_l0 == NL) { ev_l0 = 0; ++ev_t0; }
        }
        if (st >= (s ? cnt1 : cnt0)) continue;
      } else {
        // (the value kernel keeps the division form: the counters' extra
        // live registers spill there)
        (void)ev_l0; (void)ev_l1; (void)ev_t0; (void)ev_t1;
        s = (int)(e & 1);
        const int64_t k = (e >> 1) - s;
        if (k < 0) continue;
        st = k / NL;
        l = (int)(k % NL);
        if (st >= (s ? cnt1 : cnt0)) continue;
      }
      const int64_t jt = 2 * st + s;
      wait_ready(s);
      if (l < NL - 1) {
        issue(s, l + 1);
      } else if (st + 1 < (s ? cnt1 : cnt0)) {   // tile jt + 2 was staged
        copy_x(jt + 2 + NXB);
        issue(s, 0);
      }
    }
    if (prof) {
      g_dbg_ts[36] = c_wait;
      g_dbg_ts[37] = c_iss;
    }
  }
  if (POLICY) dbg_ts(9);
  griddep_trigger();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tm, 512);
  if (POLICY) dbg_ts(10);
}

// ---------------------------------------------------------------------------
// image packing: one CTA per matrix; max|W| -> power-of-two scale; hi/lo
// fp16 halves of W * scale in the 2-byte K-major core layout

struct Pack16Mat {
  const float* W;    // row-major [K][N] fp32
  int32_t K, N, Kpad, Npad;
  uint16_t* hi;
  uint16_t* lo;
  float* scale;      // [0] = forward scale, [4] = inverse (image floats)
};
struct Pack16Vec {
  const float* src;
  int32_t len, pad_to;
  float* dst;
};
struct Pack16Args {
  Pack16Mat m[3];
  Pack16Vec v[3];
  int32_t n_mat, n_vec;
};

__host__ __device__ inline float f16_scale_for(float amax) {
  if (!(amax > 0.f) || !(amax < 3.0e38f)) return 1.f;
  int e;
  frexpf(amax, &e);           // amax in [2^(e-1), 2^e)
  e = e < -40 ? -40 : (e > 40 ? 40 : e);
  return ldexpf(1.f, -e);     // amax * scale in [0.5, 1)
}

__global__ void __launch_bounds__(1024) k_pack16(Pack16Args a) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  __shared__ float red[32];
  const int tid = threadIdx.x;
  if ((int)blockIdx.x < a.n_mat) {
    const Pack16Mat& M = a.m[blockIdx.x];
    float amax = 0.f;
    for (int i = tid; i < M.K * M.N; i += blockDim.x) amax = fmaxf(amax, fabsf(M.W[i]));
    for (int o = 16; o; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if ((tid & 31) == 0) red[tid >> 5] = amax;
    __syncthreads();
    if (tid < 32) {
      amax = tid < (int)(blockDim.x >> 5) ? red[tid] : 0.f;
      for (int o = 16; o; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      if (tid == 0) red[0] = amax;
    }
    __syncthreads();
    const float sc = f16_scale_for(red[0]);
    for (int i = tid; i < M.Kpad * M.Npad; i += blockDim.x) {
      const int k = i / M.Npad, nn = i % M.Npad;
      const float w = (k < M.K && nn < M.N) ? M.W[k * M.N + nn] * sc : 0.f;
      tc::store_split_f16(w, M.hi, M.lo, tc::kmajor16_off(nn, k, M.Kpad));
    }
    if (tid == 0) {
      M.scale[0] = sc;
      M.scale[4] = 1.f / sc;   // exact: a power of two
    }
  }
  if (blockIdx.x == 0)
    for (int q = 0; q < a.n_vec; ++q)
      for (int i = tid; i < a.v[q].pad_to; i += blockDim.x)
        a.v[q].dst[i] = i < a.v[q].len ? a.v[q].src[i] : 0.f;
}

}  // namespace harl
