// rank_scores (costmodel.py:266-286) over the device entry log: the top k
// distinct, unmeasured visited states by (score desc, insertion order asc).
//
// The reference walks every CandidateEntry building a canonical string,
// dedups through a Python set, re-predicts the pool and sorts it.  Here:
//   (1) k_rank_insert  every item (excluded states first, then visits in
//       order) hashes its state into an open-addressing table; the slot
//       keeps the smallest item index (atomicMin) -> the slot's
//       representative is an excluded state if one hashed there, else the
//       first visit of that hash;
//   (2) k_rank_mark    a visit is kept when it is its slot's representative,
//       or when its state differs from the representative's (a 64-bit hash
//       collision: kept, counted, and the host's exact rank_scores pass
//       removes whatever such keeps duplicate); exact state compares only;
//   (3) k_rank_select  radix select of the k' = k + collisions largest
//       96-bit keys (score as ordered bits, then ~visit) over the kept
//       visits, 8 bits per pass, the last CTA of each pass picking the
//       digit (no host round trip);
//   (4) k_rank_emit    the kept visits at or above the threshold.
// The selection contains every true top-k entry at its first occurrence
// (DESIGN.md §8), so the reference's own rank_scores applied to it returns
// exactly what it returns on the full entry list.
#pragma once

#include "common.cuh"

namespace harl {

struct RankState {
  unsigned long long kept;        // visits kept by k_rank_mark
  unsigned long long collisions;  // kept for a hash collision
  unsigned long long k_target;    // k + collisions, capped at kept
  unsigned long long remaining;   // still to select inside the prefix
  unsigned long long prefix_hi;   // ordered score bits decided so far
  unsigned int prefix_lo;         // ~visit bits decided so far
  int done;                       // threshold final (prefix, low bits 0)
  unsigned int blocks_done;
  unsigned int out_count;
  unsigned int hist[256];
};

struct RankArgs {
  const uint16_t* tiles;    // [slots][ld] visits
  const uint8_t* knobs;     // [3][ld]
  const double* score;      // [ld]
  int64_t ld, V;
  const uint16_t* ex_tiles; // [slots][ex_ld] excluded states
  const uint8_t* ex_knobs;  // [3][ex_ld]
  int64_t ex_ld, E;
  int32_t slots;
  unsigned long long* keys; // [tsize], 0 = empty
  int32_t* reps;            // [tsize], INT_MAX = none
  int64_t tmask;
  uint8_t* keep;            // [V]
  RankState* st;
  int64_t k;
  int32_t* out_idx;         // [>= k + collisions]
  int64_t out_cap;
};

__device__ __forceinline__ unsigned long long rank_mix(unsigned long long h) {
  h ^= h >> 33;
  h *= 0xff51afd7ed558ccdull;
  h ^= h >> 33;
  h *= 0xc4ceb9fe1a85ec53ull;
  h ^= h >> 33;
  return h;
}

// state of item i (i < E: excluded state i, else visit i - E)
__device__ __forceinline__ void rank_src(const RankArgs& a, int64_t i,
                                         const uint16_t** t, const uint8_t** k,
                                         int64_t* col, int64_t* ld) {
  if (i < a.E) {
    *t = a.ex_tiles; *k = a.ex_knobs; *col = i; *ld = a.ex_ld;
  } else {
    *t = a.tiles; *k = a.knobs; *col = i - a.E; *ld = a.ld;
  }
}

__device__ __forceinline__ unsigned long long rank_hash(const RankArgs& a,
                                                        int64_t i) {
  const uint16_t* t; const uint8_t* kn; int64_t c, ld;
  rank_src(a, i, &t, &kn, &c, &ld);
  unsigned long long h = 0x9e3779b97f4a7c15ull;
  int s = 0;
  for (; s + 4 <= a.slots; s += 4) {
    unsigned long long w = (unsigned long long)t[(int64_t)s * ld + c] |
        ((unsigned long long)t[(int64_t)(s + 1) * ld + c] << 16) |
        ((unsigned long long)t[(int64_t)(s + 2) * ld + c] << 32) |
        ((unsigned long long)t[(int64_t)(s + 3) * ld + c] << 48);
    h = rank_mix(h ^ w);
  }
  unsigned long long w = 0;
  int sh = 0;
  for (; s < a.slots; ++s, sh += 16)
    w |= (unsigned long long)t[(int64_t)s * ld + c] << sh;
  w ^= ((unsigned long long)kn[c] | ((unsigned long long)kn[ld + c] << 8) |
        ((unsigned long long)kn[2 * ld + c] << 16)) << 40;
  h = rank_mix(h ^ w ^ 0x5bd1e995ull);
  return h ? h : 1ull;
}

__device__ __forceinline__ bool rank_same(const RankArgs& a, int64_t i,
                                          int64_t j) {
  const uint16_t *ti, *tj; const uint8_t *ki, *kj; int64_t ci, cj, li, lj;
  rank_src(a, i, &ti, &ki, &ci, &li);
  rank_src(a, j, &tj, &kj, &cj, &lj);
  for (int s = 0; s < a.slots; ++s)
    if (ti[(int64_t)s * li + ci] != tj[(int64_t)s * lj + cj]) return false;
  for (int q = 0; q < 3; ++q)
    if (ki[q * li + ci] != kj[q * lj + cj]) return false;
  return true;
}

__device__ __forceinline__ int64_t rank_find(const RankArgs& a,
                                             unsigned long long h) {
  int64_t pos = (int64_t)(h & (unsigned long long)a.tmask);
  while (a.keys[pos] != h) pos = (pos + 1) & a.tmask;
  return pos;
}

__global__ void k_rank_insert(RankArgs a) {
  griddep_wait();
  griddep_launch();
  const int64_t n = a.E + a.V;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long h = rank_hash(a, i);
    int64_t pos = (int64_t)(h & (unsigned long long)a.tmask);
    for (;;) {
      const unsigned long long prev = atomicCAS(a.keys + pos, 0ull, h);
      if (prev == 0ull || prev == h) break;
      pos = (pos + 1) & a.tmask;
    }
    atomicMin(a.reps + pos, (int32_t)i);
  }
}

__global__ void k_rank_mark(RankArgs a) {
  griddep_wait();
  griddep_launch();
  unsigned int kept = 0, coll = 0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < a.V;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = a.E + v;
    const int64_t rep = a.reps[rank_find(a, rank_hash(a, i))];
    uint8_t k = 1;
    if (rep != i) {
      if (rank_same(a, i, rep)) k = 0;
      else ++coll;
    }
    a.keep[v] = k;
    kept += k;
  }
  // warp then block aggregation of the two counters
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    kept += __shfl_xor_sync(0xffffffffu, kept, o);
    coll += __shfl_xor_sync(0xffffffffu, coll, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (kept) atomicAdd(&a.st->kept, (unsigned long long)kept);
    if (coll) atomicAdd(&a.st->collisions, (unsigned long long)coll);
  }
}

// ordered 64-bit image of a double (total order, larger = better)
__device__ __forceinline__ unsigned long long rank_okey(double s) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(s);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// digit d (0..11) of the 96-bit key (hi: ordered score, lo: ~visit)
__device__ __forceinline__ bool rank_match(unsigned long long hi,
                                           unsigned int lo, int d,
                                           const RankState& st,
                                           unsigned int* digit) {
  if (d < 8) {
    const int sh = 56 - 8 * d;
    if (d > 0 && (hi >> (sh + 8)) != (st.prefix_hi >> (sh + 8))) return false;
    *digit = (unsigned int)(hi >> sh) & 255u;
    return true;
  }
  if (hi != st.prefix_hi) return false;
  const int sh = 24 - 8 * (d - 8);
  if (d > 8 && (lo >> (sh + 8)) != (st.prefix_lo >> (sh + 8))) return false;
  *digit = (lo >> sh) & 255u;
  return true;
}

__global__ void k_rank_select(RankArgs a, int d) {
  griddep_wait();
  griddep_launch();
  __shared__ unsigned int hist[256];
  __shared__ bool last;
  RankState& st = *a.st;
  unsigned long long ktarget = a.k + st.collisions;
  if (ktarget > st.kept) ktarget = st.kept;
  const bool all = (ktarget == st.kept);
  if (st.done || all || ktarget == 0) {
    if (d == 0 && blockIdx.x == 0 && threadIdx.x == 0) {
      st.k_target = ktarget;
      st.done = 1;
      st.prefix_hi = 0ull;
      st.prefix_lo = 0u;
      if (ktarget == 0) st.prefix_hi = ~0ull, st.prefix_lo = ~0u;
    }
    return;
  }
  for (int t = threadIdx.x; t < 256; t += blockDim.x) hist[t] = 0;
  __syncthreads();
  // scores cluster (a GBT ensemble has few distinct values near the top),
  // so most lanes of a warp hit the same bin: one atomic per distinct
  // digit per warp (__match_any_sync), not one per item
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t vend = (a.V + 31) & ~(int64_t)31;   // whole warps iterate
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < vend;
       v += stride) {
    unsigned int dg = 0xffffffffu;
    if (v < a.V && a.keep[v]) {
      unsigned int t;
      if (rank_match(rank_okey(a.score[v]), ~(unsigned int)v, d, st, &t)) dg = t;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, dg);
    if (dg != 0xffffffffu && (threadIdx.x & 31) == __ffs(peers) - 1)
      atomicAdd(&hist[dg], (unsigned int)__popc(peers));
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 256; t += blockDim.x)
    if (hist[t]) atomicAdd(&st.hist[t], hist[t]);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0)
    last = (atomicAdd(&st.blocks_done, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  // the last CTA picks the digit: the 256 global bins into shared memory in
  // parallel, a suffix sum over them, the bin where the remaining count
  // falls
  __threadfence();
  __shared__ unsigned long long suf[256];
  __shared__ int s_b;
  unsigned int* hs = hist;   // reuse the CTA histogram for the totals
  for (int t = threadIdx.x; t < 256; t += blockDim.x)
    hs[t] = *(volatile unsigned int*)&st.hist[t];
  __syncthreads();
  for (int t = threadIdx.x; t < 256; t += blockDim.x) suf[t] = hs[t];
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {   // suf[t] = sum of bins >= t
    unsigned long long v = 0;
    for (int t = threadIdx.x; t < 256; t += blockDim.x)
      if (t + o < 256) v = suf[t + o];
    __syncthreads();
    for (int t = threadIdx.x; t < 256; t += blockDim.x)
      if (t + o < 256) suf[t] += v;
    __syncthreads();
  }
  const unsigned long long rem0 = (d == 0) ? ktarget : st.remaining;
  if (threadIdx.x == 0) s_b = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < 256; t += blockDim.x) {
    const unsigned long long above = t < 255 ? suf[t + 1] : 0ull;
    if (t > 0 && above < rem0 && rem0 <= suf[t]) s_b = t;   // unique
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int b = s_b;   // 0 when no higher bin reaches rem0
    const unsigned long long above = b < 255 ? suf[b + 1] : 0ull;
    const unsigned long long inb = hs[b];
    const unsigned long long rem = rem0 - above;
    if (d < 8) st.prefix_hi |= (unsigned long long)b << (56 - 8 * d);
    else st.prefix_lo |= (unsigned int)b << (24 - 8 * (d - 8));
    st.remaining = rem;
    if (d == 0) st.k_target = ktarget;
    if (inb == rem) st.done = 1;   // the whole bucket is selected
    st.blocks_done = 0;
  }
  for (int t = threadIdx.x; t < 256; t += blockDim.x) st.hist[t] = 0;
}

__global__ void k_rank_emit(RankArgs a) {
  griddep_wait();
  griddep_launch();
  const RankState& st = *a.st;
  if (st.k_target == 0) return;
  const unsigned long long ph = st.prefix_hi;
  const unsigned int pl = st.prefix_lo;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < a.V;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (!a.keep[v]) continue;
    const unsigned long long hi = rank_okey(a.score[v]);
    const unsigned int lo = ~(unsigned int)v;
    if (hi > ph || (hi == ph && lo >= pl)) {
      const unsigned int p = atomicAdd(&a.st->out_count, 1u);
      if ((int64_t)p < a.out_cap) a.out_idx[p] = (int32_t)v;
    }
  }
}

__global__ void k_rank_stats(RankArgs a, int64_t* stats) {
  griddep_wait();
  griddep_launch();
  const RankState& st = *a.st;
  stats[0] = st.out_count;
  stats[1] = (int64_t)st.kept;
  stats[2] = (int64_t)st.collisions;
  stats[3] = (int64_t)st.k_target;
}

}  // namespace harl
