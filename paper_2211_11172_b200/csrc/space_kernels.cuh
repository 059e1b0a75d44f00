// Schedule-space kernels: initial sampler (K1), legality/apply walker (K2),
// featurizer (K3).  Integer/byte work, HBM-bound; population is SoA
// (tiles u16 [slot][ld], knobs u8 [3][ld]) so every per-slot access of a
// warp is one coalesced 64-byte request.
#pragma once

#include "common.cuh"

namespace harl {

// ---------------------------------------------------------------------------
// K1: sample_initial_schedules (schedspace.py:165-178).
// Each track draws, in order, one Generator.integers per tiled dim, then
// compute-at, parallel, unroll.  integers(n) with n == 1 consumes nothing;
// otherwise it takes one 32-bit word (Lemire, numpy's
// buffered_bounded_lemire_uint32) unless the rare rejection branch fires.
// The optimistic pass assumes no rejection; the first rejecting track is
// reported through *first_bad and repaired sequentially by the host loop.

struct InitArgs {
  int64_t t0, count, ld;
  uint64_t j0;              // 32-bit word index of track t0's first draw
  int32_t per_track;        // consuming draws per track
  int32_t bounds[HARL_MAX_DIMS + 3];
  int32_t nbounds;
  u128 s;
  int32_t has32;
  uint32_t buffered;
};

__device__ inline bool lemire32(uint32_t w, uint32_t n, uint32_t* out) {
  uint64_t m = (uint64_t)w * (uint64_t)n;
  uint32_t left = (uint32_t)m;
  if (left < n) {
    uint32_t thr = (uint32_t)((0u - n) % n);  // (2^32 - n) % n
    if (left < thr) return false;
  }
  *out = (uint32_t)(m >> 32);
  return true;
}

__device__ inline void write_initial(const harl_sketch_desc& sk, int64_t t,
                                     int64_t ld, const uint32_t* v,
                                     uint16_t* tiles, uint8_t* knobs) {
  const int L = sk.levels;
  for (int d = 0; d < sk.ndims; ++d) {
    const uint16_t* row = sk.tiling_table + (int64_t)(sk.tiling_offsets[d] + v[d]) * L;
    for (int lv = 0; lv < L; ++lv) tiles[(int64_t)(d * L + lv) * ld + t] = row[lv];
  }
  knobs[t] = (uint8_t)v[sk.ndims];
  knobs[ld + t] = (uint8_t)v[sk.ndims + 1];
  knobs[2 * ld + t] = (uint8_t)v[sk.ndims + 2];
}

__global__ void k_init_sample(const __grid_constant__ harl_sketch_desc sk,
                              const __grid_constant__ PcgJump J,
                              const __grid_constant__ InitArgs a,
                              uint16_t* tiles, uint8_t* knobs,
                              unsigned long long* first_bad) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  int64_t t = a.t0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.count) return;
  uint64_t j = a.j0 + (uint64_t)(t - a.t0) * (uint64_t)a.per_track;
  uint32_t v[HARL_MAX_DIMS + 3];
  for (int k = 0; k < a.nbounds; ++k) {
    uint32_t n = (uint32_t)a.bounds[k];
    v[k] = 0;
    if (n > 1) {
      uint32_t w = pcg_word32(J, a.s, a.has32, a.buffered, j++);
      if (!lemire32(w, n, &v[k])) {
        atomicMin(first_bad, (unsigned long long)t);
        return;
      }
    }
  }
  write_initial(sk, t, a.ld, v, tiles, knobs);
}

// exact sequential version for one track (rejection loop); returns words
// used through *used
__global__ void k_init_one(const __grid_constant__ harl_sketch_desc sk,
                           const __grid_constant__ PcgJump J,
                           const __grid_constant__ InitArgs a, int64_t t,
                           uint16_t* tiles, uint8_t* knobs,
                           unsigned long long* used) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  uint64_t j = a.j0;
  uint32_t v[HARL_MAX_DIMS + 3];
  for (int k = 0; k < a.nbounds; ++k) {
    uint32_t n = (uint32_t)a.bounds[k];
    v[k] = 0;
    if (n > 1) {
      while (!lemire32(pcg_word32(J, a.s, a.has32, a.buffered, j++), n, &v[k])) {
      }
    }
  }
  write_initial(sk, t, a.ld, v, tiles, knobs);
  *used = j - a.j0;
}

// ---------------------------------------------------------------------------
// K3: featurize (schedspace.py:372-438).  Footprints are exact int64 (the
// host checked every value < 2^53), converted once to fp64 and passed to
// the glibc-faithful log10; tile logs come from a host-built LUT of
// math.log2(v)/10.  Rows are staged in shared memory so the [n][F] output
// is written with coalesced stores.

__device__ inline void footprint_l1l2(const harl_sketch_desc& sk,
                                      const int64_t* t1, const int64_t* t2,
                                      bool root, int64_t* l1o, int64_t* l2o) {
  int64_t l1 = 0, l2 = 0;
  for (int s = 0; s < sk.n_stages; ++s) {
    int64_t s1 = 0, s2 = 0, o1 = 0, o2 = 0;
    const int tf = sk.stage_first[s], tn = sk.stage_ntensors[s];
    for (int ti = tf; ti < tf + tn; ++ti) {
      int64_t e1 = 1, e2 = 1;
      const int f = sk.tensor_first[ti], nt = sk.tensor_nterms[ti];
      for (int q = f; q < f + nt; ++q) {
        const int gi = sk.term_gi[q];
        const int64_t sc = sk.term_sc[q], off = sk.term_off[q];
        e1 *= sc * t1[gi] + off;
        e2 *= sc * t2[gi] + off;
      }
      s1 += e1;
      s2 += e2;
      o1 = e1;
      o2 = e2;
    }
    const int64_t inter = sk.stage_inter[s], extra = sk.stage_extra[s];
    s1 += (inter + extra) * o1;
    s2 += extra * o2 + (root ? inter * o2 : 0);
    l1 += s1;
    l2 += s2;
  }
  *l1o = l1;
  *l2o = l2;
}

// one footprint level alone (level 1: t = innermost tiles, every stage
// adds (inter+extra)*last; level 2: t = product of the two innermost
// levels, inter only at the root) -- the same integer sums as
// footprint_l1l2, split so two threads can take one level each
__device__ inline int64_t footprint_level(const harl_sketch_desc& sk,
                                          const int64_t* t, bool level1,
                                          bool root) {
  int64_t l = 0;
  for (int s = 0; s < sk.n_stages; ++s) {
    int64_t sacc = 0, o = 0;
    const int tf = sk.stage_first[s], tn = sk.stage_ntensors[s];
    for (int ti = tf; ti < tf + tn; ++ti) {
      int64_t e = 1;
      const int f = sk.tensor_first[ti], nt = sk.tensor_nterms[ti];
      for (int q = f; q < f + nt; ++q) e *= (int64_t)sk.term_sc[q] * t[sk.term_gi[q]] + sk.term_off[q];
      sacc += e;
      o = e;
    }
    const int64_t inter = sk.stage_inter[s], extra = sk.stage_extra[s];
    sacc += level1 ? (inter + extra) * o : extra * o + (root ? inter * o : 0);
    l += sacc;
  }
  return l;
}

// one feature row into dst[0..F)
__device__ inline void featurize_row(const harl_sketch_desc& sk,
                                     const uint16_t* tiles,
                                     const uint8_t* knobs, int64_t ld,
                                     int64_t r, double* dst,
                                     const double* lut = nullptr) {
  if (!lut) lut = sk.log2_lut;
  const int L = sk.levels, F = sk.feature_len;
  for (int i = 0; i < F; ++i) dst[i] = 0.0;
  int64_t t1[HARL_MAX_DIMS], t2[HARL_MAX_DIMS];
  for (int d = 0; d < sk.ndims; ++d) {
    int64_t prod = 1;
    for (int lv = 0; lv < L; ++lv) {
      const int v = tiles[(int64_t)(d * L + lv) * ld + r];
      dst[d * L + lv] = lut[v];
      if (lv >= L - 2) prod *= v;
      if (lv == L - 1) t1[d] = v;
    }
    t2[d] = (L >= 2) ? prod : t1[d];
  }
  const int ca = knobs[r], par = knobs[ld + r], ur = knobs[2 * ld + r];
  int pos = sk.max_feature_dims * L;
  dst[pos] = sk.ncas > 1 ? __ddiv_rn((double)ca, (double)(sk.ncas - 1)) : 0.0;
  dst[pos + 1] = sk.max_fusible ? __ddiv_rn((double)par, (double)sk.max_fusible) : 0.0;
  dst[pos + 2 + ur] = 1.0;
  pos += 2 + sk.n_unroll;
  int64_t l1, l2;
  footprint_l1l2(sk, t1, t2, ca == 0, &l1, &l2);
  dst[pos] = __ddiv_rn(glibc_log10_ge1(__dadd_rn(1.0, (double)l1)), 6.0);
  dst[pos + 1] = __ddiv_rn(glibc_log10_ge1(__dadd_rn(1.0, (double)l2)), 6.0);
  dst[pos + 2] = sk.flops_feature;
}

constexpr int FEAT_THREADS = 128;

__global__ void __launch_bounds__(FEAT_THREADS)
k_featurize(const __grid_constant__ harl_sketch_desc sk, const uint16_t* tiles,
            const uint8_t* knobs, int64_t n, int64_t ld, double* feat) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  extern __shared__ double sfeat[];
  const int F = sk.feature_len;
  const int64_t r0 = (int64_t)blockIdx.x * FEAT_THREADS;
  const int64_t r = r0 + threadIdx.x;
  if (r < n) featurize_row(sk, tiles, knobs, ld, r, sfeat + threadIdx.x * F);
  __syncthreads();
  const int64_t rows = min((int64_t)FEAT_THREADS, n - r0);
  double* out = feat + r0 * F;
  for (int64_t i = threadIdx.x; i < rows * F; i += FEAT_THREADS) out[i] = sfeat[i];
}

// Staged variant: the CTA's tile/knob columns (coalesced along rows) and
// the log2 LUT are copied into shared memory with all loads in flight at
// once; each thread then featurizes its row from shared memory.
constexpr int FEAT2_ROWS = 128;
constexpr int FEAT2_PARTS = 4;     // threads per row
constexpr int FEAT2_THREADS = FEAT2_ROWS * FEAT2_PARTS;
constexpr int FEAT2_LUT_MAX = 4096;

__host__ __device__ inline size_t feat2_smem_bytes(int F, int local_slots,
                                                   int max_extent) {
  const size_t lut = (max_extent + 1 <= FEAT2_LUT_MAX) ? (size_t)((max_extent + 2) & ~1) * 8 : 0;
  return (size_t)FEAT2_ROWS * F * 8 + lut +
         (((size_t)FEAT2_ROWS * local_slots * 2 + FEAT2_ROWS * 3 + 15) & ~(size_t)15);
}

// Featurize rows [r0, r0 + 128) of a population (n rows, leading dim ld)
// with FEAT2_THREADS threads, staging through `fsm` (feat2_smem_bytes).
__device__ __forceinline__ void featurize_tile(
    const harl_sketch_desc& sk, const uint16_t* __restrict__ tiles,
    const uint8_t* __restrict__ knobs, int64_t n, int64_t ld, int64_t r0,
    double* __restrict__ feat, unsigned char* fsm) {
  const int F = sk.feature_len, S = sk.local_slots;
  double* sfeat = (double*)fsm;
  const bool slut = sk.max_extent + 1 <= FEAT2_LUT_MAX;
  double* lut = slut ? sfeat + FEAT2_ROWS * F : nullptr;
  uint16_t* stile = (uint16_t*)(sfeat + FEAT2_ROWS * F + (slut ? (sk.max_extent + 2) & ~1 : 0));
  uint8_t* sknob = (uint8_t*)(stile + FEAT2_ROWS * S);
  const int rows = (int)min((int64_t)FEAT2_ROWS, n - r0);
  const bool vec = (ld % 16) == 0 && (((uintptr_t)tiles | (uintptr_t)knobs |
                                       (uintptr_t)sk.log2_lut) & 15) == 0;
  if (vec) {
    // 16-byte async copies: slot segments (8 rows per chunk), knob rows
    // (16 rows per chunk) and the LUT; chunks past `rows` stay inside the
    // allocation because ld is a multiple of 16
    const int cs = (rows + 7) / 8, ck = (rows + 15) / 16;
    for (int i = threadIdx.x; i < S * cs; i += FEAT2_THREADS) {
      const int sl = i / cs, c = i % cs;
      cp_async16(stile + sl * FEAT2_ROWS + 8 * c, tiles + (int64_t)sl * ld + r0 + 8 * c);
    }
    for (int i = threadIdx.x; i < 3 * ck; i += FEAT2_THREADS) {
      const int k = i / ck, c = i % ck;
      cp_async16(sknob + k * FEAT2_ROWS + 16 * c, knobs + (int64_t)k * ld + r0 + 16 * c);
    }
    if (slut) {
      const int nl = sk.max_extent + 1;
      for (int i = threadIdx.x; i < nl / 2; i += FEAT2_THREADS)
        cp_async16(lut + 2 * i, sk.log2_lut + 2 * i);
      if ((nl & 1) && threadIdx.x == 0) lut[nl - 1] = sk.log2_lut[nl - 1];
    }
    cp_async_wait_all();
  } else {
    for (int i = threadIdx.x; i < S * FEAT2_ROWS; i += FEAT2_THREADS)
      if (i % FEAT2_ROWS < rows)
        stile[i] = tiles[(int64_t)(i / FEAT2_ROWS) * ld + r0 + i % FEAT2_ROWS];
    for (int i = threadIdx.x; i < 3 * FEAT2_ROWS; i += FEAT2_THREADS)
      if (i % FEAT2_ROWS < rows)
        sknob[i] = knobs[(int64_t)(i / FEAT2_ROWS) * ld + r0 + i % FEAT2_ROWS];
    if (slut)
      for (int i = threadIdx.x; i <= sk.max_extent; i += FEAT2_THREADS) lut[i] = sk.log2_lut[i];
  }
  __syncthreads();

  for (int i = threadIdx.x; i < rows * F; i += FEAT2_THREADS) sfeat[i] = 0.0;
  __syncthreads();
  {
    // part 0: tile logs + knob features; parts 1/2: one footprint level
    // and its log10 each; part 3: the flops feature
    const int part = threadIdx.x / FEAT2_ROWS, rl = threadIdx.x % FEAT2_ROWS;
    if (rl < rows) {
      const int L = sk.levels;
      double* dst = sfeat + rl * F;
      const int ca = sknob[rl];
      int pos = sk.max_feature_dims * L;
      if (part == 0) {
        for (int d = 0; d < sk.ndims; ++d)
          for (int lv = 0; lv < L; ++lv)
            dst[d * L + lv] = (slut ? lut : sk.log2_lut)[stile[(d * L + lv) * FEAT2_ROWS + rl]];
        const int par = sknob[FEAT2_ROWS + rl], ur = sknob[2 * FEAT2_ROWS + rl];
        dst[pos] = sk.ncas > 1 ? __ddiv_rn((double)ca, (double)(sk.ncas - 1)) : 0.0;
        dst[pos + 1] = sk.max_fusible ? __ddiv_rn((double)par, (double)sk.max_fusible) : 0.0;
        dst[pos + 2 + ur] = 1.0;
      } else if (part == 1 || part == 2) {
        int64_t t[HARL_MAX_DIMS];
        for (int d = 0; d < sk.ndims; ++d) {
          const int vl = stile[(d * L + L - 1) * FEAT2_ROWS + rl];
          t[d] = (part == 2 && L >= 2)
                     ? (int64_t)stile[(d * L + L - 2) * FEAT2_ROWS + rl] * vl : vl;
        }
        const int64_t l = footprint_level(sk, t, part == 1, ca == 0);
        pos += 2 + sk.n_unroll;
        dst[pos + part - 1] = __ddiv_rn(glibc_log10_ge1(__dadd_rn(1.0, (double)l)), 6.0);
      } else {
        dst[pos + 2 + sk.n_unroll + 2] = sk.flops_feature;
      }
    }
  }
  __syncthreads();

  double* out = feat + r0 * F;
  for (int i = threadIdx.x; i < rows * F; i += FEAT2_THREADS) out[i] = sfeat[i];

}

__global__ void __launch_bounds__(FEAT2_THREADS)
k_featurize2(const __grid_constant__ harl_sketch_desc sk,
             const uint16_t* __restrict__ tiles,
             const uint8_t* __restrict__ knobs, int64_t n, int64_t ld,
             double* __restrict__ feat) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  dbg_ts(32);
  extern __shared__ __align__(16) unsigned char fsm[];
  featurize_tile(sk, tiles, knobs, n, ld, (int64_t)blockIdx.x * FEAT2_ROWS, feat, fsm);
  griddep_trigger();
  dbg_ts(35);
}

// ---------------------------------------------------------------------------
// K2: legality and the walker (schedspace.py:196-301).

// movable-slot bitmask: bit s set iff slot s of this sketch has factor > 1
__device__ inline uint64_t movable_bits(const harl_sketch_desc& sk,
                                        const uint16_t* tiles, int64_t ld,
                                        int64_t r) {
  uint64_t m = 0;
  for (int s = 0; s < sk.local_slots; ++s)
    if (tiles[(int64_t)s * ld + r] > 1) m |= (1ull << s);
  return m;
}

// bits 0-2 compute-at [pos>0, 1, pos<top], 3-5 parallel, 6-8 unroll
__device__ inline uint32_t shift_bits_of(const harl_sketch_desc& sk, int ca,
                                         int par, int ur) {
  auto tri = [](int pos, int top) -> uint32_t {
    return (pos > 0 ? 1u : 0u) | 2u | (pos < top ? 4u : 0u);
  };
  return tri(ca, sk.ncas - 1) | (tri(par, sk.max_fusible) << 3) |
         (tri(ur, sk.n_unroll - 1) << 6);
}

__global__ void k_action_masks(const __grid_constant__ harl_sketch_desc sk,
                               const uint16_t* tiles, const uint8_t* knobs,
                               int64_t n, int64_t ld, uint8_t* tiling,
                               uint8_t* shift) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int S = sk.num_slots, L = sk.levels;
  const int64_t W = (int64_t)S * S + 1;
  const uint64_t mv = movable_bits(sk, tiles, ld, r);
  uint8_t* row = tiling + r * W;
  for (int64_t c = 0; c < W - 1; ++c) {
    const int src = (int)(c / S), dst = (int)(c % S);
    row[c] = (src < sk.local_slots && ((mv >> src) & 1ull) &&
              src / L == dst / L && src != dst) ? 1 : 0;
  }
  row[W - 1] = 1;
  const uint32_t sb = shift_bits_of(sk, knobs[r], knobs[ld + r], knobs[2 * ld + r]);
  for (int i = 0; i < 9; ++i) shift[r * 9 + i] = (sb >> i) & 1u;
}

// Apply one decoded action to row r; returns HARL_ST_* (first failing
// subspace in the reference's check order).  Writes the new state.
__device__ inline int apply_row(const harl_sketch_desc& sk,
                                const uint16_t* tiles, const uint8_t* knobs,
                                int64_t ld, int64_t r, int a0, int a1, int a2,
                                int a3, uint16_t* tiles_out,
                                uint8_t* knobs_out, int64_t ldo, int64_t ro) {
  const int S = sk.num_slots, L = sk.levels;
  int src = -1, dst = -1;
  if (a0 != S * S) {
    src = a0 / S;
    dst = a0 % S;
  }
  for (int s = 0; s < sk.local_slots; ++s)
    tiles_out[(int64_t)s * ldo + ro] = tiles[(int64_t)s * ld + r];
  if (src >= 0) {
    if (src >= sk.local_slots || dst >= sk.local_slots || dst < 0) return HARL_ST_TILING;
    if (src / L != dst / L) return HARL_ST_TILING;
    if (src == dst) return HARL_ST_TILING;
    const uint32_t f = tiles[(int64_t)src * ld + r];
    if (f <= 1) return HARL_ST_TILING;
    const uint32_t p = sk.spf_lut[f];
    tiles_out[(int64_t)src * ldo + ro] = (uint16_t)(f / p);
    tiles_out[(int64_t)dst * ldo + ro] = (uint16_t)(tiles[(int64_t)dst * ld + r] * p);
  }
  const int ca = (int)knobs[r] + (a1 - 1);
  if (ca < 0 || ca >= sk.ncas) return HARL_ST_COMPUTE_AT;
  const int par = (int)knobs[ld + r] + (a2 - 1);
  if (par < 0 || par > sk.max_fusible) return HARL_ST_PARALLEL;
  const int ur = (int)knobs[2 * ld + r] + (a3 - 1);
  if (ur < 0 || ur >= sk.n_unroll) return HARL_ST_UNROLL;
  knobs_out[ro] = (uint8_t)ca;
  knobs_out[ldo + ro] = (uint8_t)par;
  knobs_out[2 * ldo + ro] = (uint8_t)ur;
  return HARL_ST_OK;
}

__device__ inline void report_status(unsigned long long* status, int64_t row,
                                     int code) {
  if (code != HARL_ST_OK)
    atomicMin(status, (unsigned long long)(row * 16 + code));
}

__global__ void k_apply_actions(const __grid_constant__ harl_sketch_desc sk,
                                const uint16_t* tiles, const uint8_t* knobs,
                                int64_t n, int64_t ld, const int32_t* actions,
                                uint16_t* tiles_out, uint8_t* knobs_out,
                                unsigned long long* status) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int code = apply_row(sk, tiles, knobs, ld, r, actions[r], actions[n + r],
                             actions[2 * n + r], actions[3 * n + r], tiles_out,
                             knobs_out, ld, r);
  report_status(status, r, code);
}

}  // namespace harl

namespace harl {

// ---------------------------------------------------------------------------
// Uniform actions for the non-RL searchers (TuningSession._uniform_actions,
// tuner.py:341-348): for head h, row r (head-major) one
// Generator.integers(len(valid)) -- no draw when a single choice is valid --
// then the chosen index among the valid ones in increasing index order.

__device__ inline int head0_valid_count(const harl_sketch_desc& sk, uint64_t mv) {
  // every movable slot can move to the L-1 other slots of its dimension,
  // plus the always-valid no-op
  return __popcll(mv) * (sk.levels - 1) + 1;
}

struct UniformArgs {
  int64_t n, ld;
  u128 s;
  int32_t has32;
  uint32_t buffered;
};

// pass 1: per (h, r) choice count; consumes[i] = (count > 1)
__global__ void k_uniform_counts(const __grid_constant__ harl_sketch_desc sk,
                                 const uint16_t* tiles, const uint8_t* knobs,
                                 int64_t n, int64_t ld, int32_t* count) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const uint64_t mv = movable_bits(sk, tiles, ld, r);
  const uint32_t sb = shift_bits_of(sk, knobs[r], knobs[ld + r], knobs[2 * ld + r]);
  count[r] = head0_valid_count(sk, mv);
  for (int h = 1; h < 4; ++h) count[h * n + r] = __popc((sb >> (3 * (h - 1))) & 7u);
}

// single-CTA exclusive scan of (count > 1) over 4n entries -> word offsets
__global__ void k_uniform_scan(const int32_t* count, int64_t total,
                               int64_t* offset, int64_t* total_words) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  __shared__ int64_t carry;
  __shared__ int64_t warp_sums[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t base = 0; base < total; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    int64_t v = (i < total && count[i] > 1) ? 1 : 0;
    int64_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int64_t w = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t t = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += t;
      }
      warp_sums[lane] = w;
    }
    __syncthreads();
    const int64_t before = carry + (warp ? warp_sums[warp - 1] : 0) + x - v;
    if (i < total) offset[i] = before;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = before + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total_words = carry;
}

// value of the k-th valid tiling column (increasing full index)
__device__ inline int head0_kth_valid(const harl_sketch_desc& sk, uint64_t mv,
                                      int k) {
  const int S = sk.num_slots, L = sk.levels;
  for (int src = 0; src < sk.local_slots; ++src) {
    if (!((mv >> src) & 1ull)) continue;
    const int base = (src / L) * L;
    for (int dst = base; dst < base + L; ++dst) {
      if (dst == src) continue;
      if (k == 0) return src * S + dst;
      --k;
    }
  }
  return S * S;  // the no-op is the last valid index
}

// pass 2: draw and decode (optimistic: no rejection before element i0)
__global__ void k_uniform_draw(const __grid_constant__ harl_sketch_desc sk,
                               const __grid_constant__ PcgJump J,
                               const __grid_constant__ UniformArgs a,
                               int64_t i0, uint64_t j0, const uint16_t* tiles,
                               const uint8_t* knobs, const int32_t* count,
                               const int64_t* offset, int32_t* actions,
                               unsigned long long* first_bad) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  const int64_t i = i0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 4 * a.n) return;
  const int64_t h = i / a.n, r = i % a.n;
  const int c = count[i];
  uint32_t v = 0;
  if (c > 1) {
    const uint64_t j = j0 + (uint64_t)(offset[i] - offset[i0]);
    if (!lemire32(pcg_word32(J, a.s, a.has32, a.buffered, j), (uint32_t)c, &v)) {
      atomicMin(first_bad, (unsigned long long)i);
      return;
    }
  }
  if (h == 0) {
    actions[r] = head0_kth_valid(sk, movable_bits(sk, tiles, a.ld, r), (int)v);
  } else {
    const uint32_t sb = shift_bits_of(sk, knobs[r], knobs[a.ld + r], knobs[2 * a.ld + r]);
    const uint32_t m3 = (sb >> (3 * (h - 1))) & 7u;
    int k = (int)v, col = 0;
    for (int j = 0; j < 3; ++j)
      if ((m3 >> j) & 1u) {
        if (k == 0) { col = j; break; }
        --k;
      }
    actions[h * a.n + r] = col;
  }
}

// sequential repair of element i (rejection loop); words used -> *used
__global__ void k_uniform_one(const __grid_constant__ harl_sketch_desc sk,
                              const __grid_constant__ PcgJump J,
                              const __grid_constant__ UniformArgs a, int64_t i,
                              uint64_t j0, const uint16_t* tiles,
                              const uint8_t* knobs, const int32_t* count,
                              int32_t* actions, unsigned long long* used) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int64_t h = i / a.n, r = i % a.n;
  uint64_t j = j0;
  uint32_t v = 0;
  while (!lemire32(pcg_word32(J, a.s, a.has32, a.buffered, j++), (uint32_t)count[i], &v)) {
  }
  *used = j - j0;
  if (h == 0) {
    actions[r] = head0_kth_valid(sk, movable_bits(sk, tiles, a.ld, r), (int)v);
  } else {
    const uint32_t sb = shift_bits_of(sk, knobs[r], knobs[a.ld + r], knobs[2 * a.ld + r]);
    const uint32_t m3 = (sb >> (3 * (h - 1))) & 7u;
    int k = (int)v, col = 0;
    for (int q = 0; q < 3; ++q)
      if ((m3 >> q) & 1u) {
        if (k == 0) { col = q; break; }
        --k;
      }
    actions[h * a.n + r] = col;
  }
}

}  // namespace harl
