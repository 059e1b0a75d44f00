// Shared device helpers: error plumbing, numpy-PCG64 jump-ahead streams and
// a bit-faithful port of glibc 2.39's log/log10 (the reference's
// math.log10, schedspace.py:435-437).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/harl_b200.h"

namespace harl {

void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);

// Programmatic dependent launch (sm_90+; HARL_PDL=1 sets the launch
// attribute, without it all of these are no-ops).  Every kernel waits for
// its predecessor grid (completion + memory visibility) with griddep_wait()
// before it reads anything the predecessor may have written or writes
// anything the predecessor may read.  The step kernels let their dependents
// launch late, with griddep_trigger() once a CTA's main work is done (an
// early trigger lets waiting dependent CTAs take residency the primary's
// later CTAs need).  Since every trigger comes after its kernel's own
// griddep_wait, a kernel that starts has everything before its predecessor
// complete: its pre-wait prologue may read data written two launches back
// or earlier (weight images, forest, tables).  HARL_PDL_EARLY=1 restores
// the trigger at kernel start (griddep_launch) for A/B.
#ifndef HARL_PDL_EARLY
#define HARL_PDL_EARLY 0
#endif
__device__ __forceinline__ void griddep_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void griddep_launch() {
#if HARL_PDL_EARLY
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
__device__ __forceinline__ void griddep_trigger() {
#if !HARL_PDL_EARLY
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

// Launch accounting and the optional per-kernel timer (harl_profile_*).
// Every library launch is bracketed by HARL_PROF_BEGIN(stream) and
// HARL_CHECK_LAUNCH(name); with the timer on (and the stream not being
// captured) the pair becomes spin-kernel, event, <kernel>, event.
void prof_begin(cudaStream_t st);
void prof_end(const char* where);
void prof_units(long long units);

// phase timestamps of CTA 0 (debug: harl_debug_timestamps)
__device__ int g_dbg_on;
__device__ unsigned long long g_dbg_ts[64];
// (compiled in only with -DHARL_PHASE_TS: the check costs every thread of
// the hot kernels a few instructions per stamp, ~3 % of the sampler)
__device__ inline void dbg_ts(int i) {
#ifdef HARL_PHASE_TS
  if (blockIdx.x == 0 && threadIdx.x == 0 && g_dbg_on) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_dbg_ts[i] = t;
  }
#else
  (void)i;
#endif
}

// Ampere-style asynchronous 16-byte global->shared copies (no register
// staging, so the compiler cannot serialise them behind shared stores)
__device__ inline void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ inline void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// grid extent probe: earliest CTA start / latest CTA end of one kernel
// (slots 60/61; harl_debug_timestamps resets them with on=1)
__device__ inline void dbg_grid(bool end, int slot = 60) {
#ifndef HARL_PHASE_TS
  (void)end;
  (void)slot;
  return;
#endif
  if (threadIdx.x == 0 && g_dbg_on == 2) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (end) atomicMax(&g_dbg_ts[slot + 1], t);
    else atomicMin(&g_dbg_ts[slot], t);
  }
}

#define HARL_PROF_BEGIN(st) ::harl::prof_begin((cudaStream_t)(st))
// work units (rows) of the launch that follows, for the per-kernel timer
#define HARL_PROF_UNITS(u) ::harl::prof_units((long long)(u))

#define HARL_CHECK_LAUNCH(where)                                     \
  do {                                                               \
    cudaError_t _e = cudaGetLastError();                             \
    if (_e != cudaSuccess) return ::harl::cuda_status(_e, where);    \
    ::harl::prof_end(where);                                         \
  } while (0)

// ---------------------------------------------------------------------------
// 128-bit helpers and numpy's PCG64 (XSL-RR 128/64, default multiplier).
// numpy steps the LCG first and outputs from the new state, so the k-th
// draw (1-based) after state s is out(A^k s + C_k).

struct u128 {
  uint64_t hi, lo;
};

__host__ __device__ inline u128 add128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
  return r;
}

__device__ inline u128 mul128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
  return r;
}

__device__ inline uint64_t pcg_output(u128 s) {
  uint64_t x = s.hi ^ s.lo;
  unsigned rot = (unsigned)(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

// Jump table: JA[i] = A^(2^i), JC[i] = C_(2^i) for the stream increment;
// built on the host per increment and passed in constant/global memory.
struct PcgJump {
  u128 A[64];
  u128 C[64];
};

// state after k steps from s
__device__ inline u128 pcg_advance(const PcgJump& J, u128 s, uint64_t k) {
  int i = 0;
  while (k) {
    if (k & 1ull) s = add128(mul128(J.A[i], s), J.C[i]);
    k >>= 1;
    ++i;
  }
  return s;
}

// k-th 64-bit draw (k >= 1) after state s
__device__ inline uint64_t pcg_draw64(const PcgJump& J, u128 s, uint64_t k) {
  return pcg_output(pcg_advance(J, s, k));
}

// Byte-sliced jump table of one stream increment: entry [L][b] advances
// b * 256^L steps, so any k < 2^32 is at most four table jumps (loads
// independent of the state, issued up front) instead of one dependent
// multiply per set bit with lane-divergent table indices.  Lives in
// global memory (32 KB, built once per increment by the host library).
struct PcgTab {
  u128 A[4 * 256];
  u128 C[4 * 256];
};

__device__ inline u128 ldg_u128(const u128* p) {
  const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(p));
  u128 r;
  r.hi = v.x;
  r.lo = v.y;
  return r;
}

__device__ inline u128 pcg_advance_tab(const PcgTab* T, u128 s, uint32_t k) {
  // entry 0 of every level is the identity (A = 1, C = 0), so the four
  // steps run unconditionally and all eight loads issue before the chain
  u128 A[4], C[4];
#pragma unroll
  for (int L = 0; L < 4; ++L) {
    const uint32_t b = (k >> (8 * L)) & 255u;
    A[L] = ldg_u128(&T->A[L * 256 + b]);
    C[L] = ldg_u128(&T->C[L * 256 + b]);
  }
#pragma unroll
  for (int L = 0; L < 4; ++L) s = add128(mul128(A[L], s), C[L]);
  return s;
}

// k-th draw with the table when there is one (and k fits), else bitwise
// the table path split in two, so a caller can issue the eight loads early
// and run the multiply chain once the base state has arrived
__device__ inline void pcg_tab_load(const PcgTab* T, uint32_t k, u128* A,
                                    u128* C) {
#pragma unroll
  for (int L = 0; L < 4; ++L) {
    const uint32_t b = (k >> (8 * L)) & 255u;
    A[L] = ldg_u128(&T->A[L * 256 + b]);
    C[L] = ldg_u128(&T->C[L * 256 + b]);
  }
}
__device__ inline u128 pcg_tab_apply(u128 s, const u128* A, const u128* C) {
#pragma unroll
  for (int L = 0; L < 4; ++L) s = add128(mul128(A[L], s), C[L]);
  return s;
}

// (out of line: keeps the table path's callers compact in the i-cache)
__device__ __noinline__ uint64_t pcg_draw64_bitwise(const PcgJump& J, u128 s,
                                                    uint64_t k) {
  return pcg_output(pcg_advance(J, s, k));
}

__device__ inline uint64_t pcg_draw64t(const PcgTab* T, const PcgJump& J,
                                       u128 s, uint64_t k) {
  if (T && k < (1ull << 32)) return pcg_output(pcg_advance_tab(T, s, (uint32_t)k));
  return pcg_draw64_bitwise(J, s, k);
}

__device__ inline double u64_to_unit(uint64_t x) {
  return (double)(x >> 11) * (1.0 / 9007199254740992.0);
}

// j-th 32-bit word (0-based) of Generator's buffered uint32 stream that
// starts at (s, has_uint32, uinteger).
__device__ inline uint32_t pcg_word32(const PcgJump& J, u128 s, int has32,
                                      uint32_t buffered, uint64_t j) {
  if (has32) {
    if (j == 0) return buffered;
    j -= 1;
  }
  uint64_t x = pcg_draw64(J, s, j / 2 + 1);
  return (j & 1ull) ? (uint32_t)(x >> 32) : (uint32_t)(x & 0xffffffffull);
}

// ---------------------------------------------------------------------------
// glibc 2.39 log (FMA variant, sysdeps/ieee754/dbl-64/e_log.c as built for
// x86-64 with FMA) and log10 (e_log10.c, no contraction).  The 128-entry
// table and polynomial coefficients are extracted from the build host's
// libm.so.6 by build.py (glibc_log_data.inc) and re-verified against
// math.log10 on the GPU box by the parity tests.

struct GlibcLogData {
  double ln2hi, ln2lo;
  double A[5];
  double B[11];
  double invc[128];
  double logc[128];
};

// single translation unit (harl_b200.cu), so the table is defined here.
// The scalars are read from the constant bank (uniform across a warp); the
// per-lane table lookups go through a global copy and the L1 path, since
// divergent constant-bank reads serialise.
__constant__ GlibcLogData c_logdata = {
#include "glibc_log_data.inc"
};
__device__ GlibcLogData g_logdata = {
#include "glibc_log_data.inc"
};

__device__ inline uint64_t dbits(double x) { return (uint64_t)__double_as_longlong(x); }
__device__ inline double bitsd(uint64_t u) { return __longlong_as_double((long long)u); }

__device__ inline double glibc_log(double x) {
  const GlibcLogData& D = c_logdata;
  uint64_t ix = dbits(x);
  const uint64_t LO = 0x3FEE000000000000ull;   // asuint64(1.0 - 0x1p-4)
  const uint64_t HI = 0x3FF1090000000000ull;   // asuint64(1.0 + 0x1.09p-4)
  if (ix - LO < HI - LO) {
    if (ix == 0x3FF0000000000000ull) return 0.0;
    double r = __dsub_rn(x, 1.0);
    double r2 = __dmul_rn(r, r);
    double r3 = __dmul_rn(r, r2);
    double q3 = __fma_rn(r3, D.B[10], __fma_rn(r2, D.B[9], __fma_rn(r, D.B[8], D.B[7])));
    double q2 = __fma_rn(r3, q3, __fma_rn(r2, D.B[6], __fma_rn(r, D.B[5], D.B[4])));
    double q1 = __fma_rn(r3, q2, __fma_rn(r2, D.B[3], __fma_rn(r, D.B[2], D.B[1])));
    double w = __dmul_rn(r, 134217728.0);  // 0x1p27
    double rhi = __dsub_rn(__dadd_rn(r, w), w);
    double rlo = __dsub_rn(r, rhi);
    w = __dmul_rn(__dmul_rn(rhi, rhi), D.B[0]);
    double hi = __dadd_rn(r, w);
    double lo = __dadd_rn(__dsub_rn(r, hi), w);
    lo = __fma_rn(__dmul_rn(D.B[0], rlo), __dadd_rn(rhi, r), lo);
    return __dadd_rn(__fma_rn(r3, q1, lo), hi);
  }
  uint64_t tmp = ix - 0x3fe6000000000000ull;
  int i = (int)((tmp >> 45) & 127u);
  int64_t k = (int64_t)tmp >> 52;
  double z = bitsd(ix - (tmp & (0xfffull << 52)));
  double r = __fma_rn(z, __ldg(&g_logdata.invc[i]), -1.0);
  double kd = (double)k;
  double w = __fma_rn(kd, D.ln2hi, __ldg(&g_logdata.logc[i]));
  double hi = __dadd_rn(w, r);
  double lo = __fma_rn(kd, D.ln2lo, __dadd_rn(__dsub_rn(w, hi), r));
  double r2 = __dmul_rn(r, r);
  double q = __fma_rn(r2, __fma_rn(r, D.A[4], D.A[3]), __fma_rn(r, D.A[2], D.A[1]));
  return __dadd_rn(__fma_rn(__dmul_rn(r, r2), q, __fma_rn(r2, D.A[0], lo)), hi);
}

// log10 for finite x >= 1 (footprint and flop features are always >= 1).
__device__ inline double glibc_log10_ge1(double x) {
  uint64_t u = dbits(x);
  int32_t hx = (int32_t)(u >> 32);
  int32_t k = (hx >> 20) - 1023;
  int32_t i = (int32_t)(((uint32_t)k & 0x80000000u) >> 31);
  hx = (hx & 0x000fffff) | ((0x3ff - i) << 20);
  double y = (double)(k + i);
  double m = bitsd(((uint64_t)(uint32_t)hx << 32) | (u & 0xffffffffull));
  const double ivln10 = 0x1.bcb7b1526e50ep-2;     // 0x3FDBCB7B1526E50E
  const double log10_2hi = 0x1.34413509f6000p-2;  // 0x3FD34413509F6000
  const double log10_2lo = 0x1.9fef311f12b36p-42; // 0x3D59FEF311F12B36
  double z = __dadd_rn(__dmul_rn(y, log10_2lo), __dmul_rn(ivln10, glibc_log(m)));
  return __dadd_rn(z, __dmul_rn(y, log10_2hi));
}

}  // namespace harl
