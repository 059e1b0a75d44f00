// The analytic measurement model (measure.py:86-167) on the device:
// simulate_time for a population of states, and brute_force_best's
// exhaustive sweep over a sketch's whole space.  fp64 with the reference's
// operation order (no contraction):
//   per anchor stage: ((flops / peak) * miss(l1, l2)) * u / speedup,
//   miss = (1 + p1 * max(0, l1/c1 - 1)) * (1 + p2 * max(0, l2/c2 - 1)),
//   speedup = used * balance * (1 - overhead * (k - 1)) over the first k
//   levels of the spatial dims (k = parallel fuse count),
// then the non-anchor ("skipped") nodes' (flops / peak) * miss(l_full,
// l_full), summed in order.  Footprints are the exact integer per-stage
// sums of stage_footprints (schedspace.py:385-407).
#pragma once

#include "common.cuh"

namespace harl {

__device__ __forceinline__ double sim_miss(double l1, double l2,
                                           const harl_sim_desc& p) {
  double e1 = __dsub_rn(__ddiv_rn(l1, p.cap_l1), 1.0);
  double e2 = __dsub_rn(__ddiv_rn(l2, p.cap_l2), 1.0);
  e1 = e1 > 0.0 ? e1 : 0.0;
  e2 = e2 > 0.0 ? e2 : 0.0;
  const double m1 = __dadd_rn(1.0, __dmul_rn(p.miss_l1, e1));
  const double m2 = __dadd_rn(1.0, __dmul_rn(p.miss_l2, e2));
  return __dmul_rn(m1, m2);
}

// t: the state's tile factors [ndims * L] (local slot order)
__device__ inline double sim_time_state(const harl_sketch_desc& sk,
                                        const harl_sim_desc& p, const int* t,
                                        int ca, int par, int ur) {
  const int L = sk.levels;
  const double u = p.unroll_factor[ur];
  double total = 0.0;
  for (int s = 0; s < sk.n_stages; ++s) {
    // stage_footprints for this stage (exact integers)
    int64_t l1 = 0, l2 = 0, o1 = 0, o2 = 0;
    const int tf = sk.stage_first[s], tn = sk.stage_ntensors[s];
    for (int ti = tf; ti < tf + tn; ++ti) {
      int64_t e1 = 1, e2 = 1;
      const int f = sk.tensor_first[ti], nt = sk.tensor_nterms[ti];
      for (int q = f; q < f + nt; ++q) {
        const int gi = sk.term_gi[q];
        const int64_t v1 = t[gi * L + L - 1];
        const int64_t v2 = L >= 2 ? (int64_t)t[gi * L + L - 2] * v1 : v1;
        e1 *= (int64_t)sk.term_sc[q] * v1 + sk.term_off[q];
        e2 *= (int64_t)sk.term_sc[q] * v2 + sk.term_off[q];
      }
      l1 += e1;
      l2 += e2;
      o1 = e1;
      o2 = e2;
    }
    const int64_t inter = sk.stage_inter[s], extra = sk.stage_extra[s];
    l1 += (inter + extra) * o1;
    l2 += extra * o2;
    if (ca == 0) l2 += inter * o2;
    const double m = sim_miss((double)l1, (double)l2, p);
    // _parallel_speedup (measure.py:86-96)
    double spd = 1.0;
    const int nsp = p.stage_spatial_n[s];
    if (par > 0 && nsp > 0) {
      int64_t extent = 1;
      for (int i = 0; i < nsp; ++i) {
        const int gi = p.stage_spatial[s][i];
        for (int lv = 0; lv < par; ++lv) extent *= t[gi * L + lv];
      }
      const int64_t cores = p.cores;
      const int64_t used = extent < cores ? extent : cores;
      const double qd = __ddiv_rn((double)extent, (double)cores);
      const int64_t den = (int64_t)ceil(qd) * cores;
      const double balance = __ddiv_rn((double)extent, (double)den);
      spd = __dmul_rn(__dmul_rn((double)used, balance),
                      __dsub_rn(1.0, __dmul_rn(p.par_overhead, (double)(par - 1))));
    }
    const double term = __ddiv_rn(
        __dmul_rn(__dmul_rn(__ddiv_rn(p.stage_flops[s], p.peak_flops), m), u), spd);
    total = __dadd_rn(total, term);
  }
  for (int k = 0; k < p.n_skipped; ++k)
    total = __dadd_rn(total, __dmul_rn(__ddiv_rn(p.skipped_flops[k], p.peak_flops),
                                       sim_miss(p.skipped_l1[k], p.skipped_l2[k], p)));
  return total;
}

__global__ void k_sim_time(const __grid_constant__ harl_sketch_desc sk,
                           const __grid_constant__ harl_sim_desc p,
                           const uint16_t* tiles, const uint8_t* knobs,
                           int64_t n, int64_t ld, double* out) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    int t[HARL_MAX_SLOTS];
    for (int s = 0; s < sk.local_slots; ++s) t[s] = tiles[(int64_t)s * ld + r];
    out[r] = sim_time_state(sk, p, t, knobs[r], knobs[ld + r], knobs[2 * ld + r]);
  }
}

// state number x of the space: the tilings of dim 0 vary slowest
// (itertools.product), then compute-at, parallel, unroll (fastest)
__device__ __forceinline__ void sim_decode(const harl_sketch_desc& sk,
                                           uint64_t x, int* t, int* ca,
                                           int* par, int* ur) {
  const int L = sk.levels;
  *ur = (int)(x % (uint64_t)sk.n_unroll);
  x /= (uint64_t)sk.n_unroll;
  *par = (int)(x % (uint64_t)(sk.max_fusible + 1));
  x /= (uint64_t)(sk.max_fusible + 1);
  *ca = (int)(x % (uint64_t)sk.ncas);
  x /= (uint64_t)sk.ncas;
  for (int d = sk.ndims - 1; d >= 0; --d) {
    const uint64_t c = (uint64_t)sk.tiling_counts[d];
    const int64_t idx = (int64_t)(x % c);
    x /= c;
    const uint16_t* row = sk.tiling_table + (sk.tiling_offsets[d] + idx) * L;
    for (int lv = 0; lv < L; ++lv) t[d * L + lv] = row[lv];
  }
}

__device__ __forceinline__ unsigned long long sim_okey(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// pass 1: the minimum time over states [x0, x0 + count)
__global__ void k_brute_min(const __grid_constant__ harl_sketch_desc sk,
                            const __grid_constant__ harl_sim_desc p,
                            uint64_t x0, uint64_t count,
                            unsigned long long* best) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  unsigned long long mine = ~0ull;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x) {
    int t[HARL_MAX_SLOTS], ca, par, ur;
    sim_decode(sk, x0 + i, t, &ca, &par, &ur);
    const unsigned long long k = sim_okey(sim_time_state(sk, p, t, ca, par, ur));
    mine = k < mine ? k : mine;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xffffffffu, mine, o);
    mine = v < mine ? v : mine;
  }
  if ((threadIdx.x & 31) == 0 && mine != ~0ull) atomicMin(best, mine);
}

// ---- ties: brute_force_best keeps the tied state with the smallest
// canonical text (schedspace.py:117-120: "sk|t=a.b;c.d|ca=X|par=Y|ur=Z";
// the common "sk|t=" prefix is skipped).  Rendered per compare into local
// buffers, compared bytewise.

constexpr int CANON_MAX = 8 * HARL_MAX_SLOTS + 48;

__device__ __forceinline__ int canon_num(char* b, int p, int v) {
  char d[12];
  int n = 0;
  do {
    d[n++] = (char)('0' + v % 10);
    v /= 10;
  } while (v);
  while (n) b[p++] = d[--n];
  return p;
}

__device__ inline int canon_render(const harl_sketch_desc& sk, uint64_t x,
                                   char* b) {
  int t[HARL_MAX_SLOTS], ca, par, ur;
  sim_decode(sk, x, t, &ca, &par, &ur);
  const int L = sk.levels;
  int p = 0;
  for (int d = 0; d < sk.ndims; ++d) {
    if (d) b[p++] = ';';
    for (int lv = 0; lv < L; ++lv) {
      if (lv) b[p++] = '.';
      p = canon_num(b, p, t[d * L + lv]);
    }
  }
  b[p++] = '|'; b[p++] = 'c'; b[p++] = 'a'; b[p++] = '=';
  p = canon_num(b, p, ca);
  b[p++] = '|'; b[p++] = 'p'; b[p++] = 'a'; b[p++] = 'r'; b[p++] = '=';
  p = canon_num(b, p, par);
  b[p++] = '|'; b[p++] = 'u'; b[p++] = 'r'; b[p++] = '=';
  p = canon_num(b, p, ur);
  return p;
}

// canonical(x_a) < canonical(x_b) (Python str order = bytewise for ASCII)
__device__ inline bool canon_less(const harl_sketch_desc& sk, uint64_t xa,
                                  uint64_t xb) {
  if (xa == ~0ull) return false;
  if (xb == ~0ull) return true;
  char a[CANON_MAX], b[CANON_MAX];
  const int na = canon_render(sk, xa, a), nb = canon_render(sk, xb, b);
  const int n = na < nb ? na : nb;
  for (int i = 0; i < n; ++i)
    if (a[i] != b[i]) return (unsigned char)a[i] < (unsigned char)b[i];
  return na < nb;
}

__device__ inline uint64_t canon_warp_min(const harl_sketch_desc& sk,
                                          uint64_t x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const uint64_t y = __shfl_xor_sync(0xffffffffu, x, o);
    if (canon_less(sk, y, x)) x = y;
  }
  return x;
}

// pass 2: among the states attaining the minimum time, the one with the
// smallest canonical text -- per block into block_best[blockIdx]
__global__ void k_brute_ties(const __grid_constant__ harl_sketch_desc sk,
                             const __grid_constant__ harl_sim_desc p,
                             uint64_t x0, uint64_t count,
                             const unsigned long long* best,
                             unsigned long long* block_best) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  const unsigned long long b = *best;
  uint64_t mine = ~0ull;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x) {
    int t[HARL_MAX_SLOTS], ca, par, ur;
    sim_decode(sk, x0 + i, t, &ca, &par, &ur);
    if (sim_okey(sim_time_state(sk, p, t, ca, par, ur)) == b &&
        canon_less(sk, x0 + i, mine))
      mine = x0 + i;
  }
  mine = canon_warp_min(sk, mine);
  __shared__ uint64_t sw[32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sw[w] = mine;
  __syncthreads();
  if (w == 0) {
    uint64_t v = lane < (int)(blockDim.x >> 5) ? sw[lane] : ~0ull;
    v = canon_warp_min(sk, v);
    if (lane == 0) block_best[blockIdx.x] = v;
  }
}

// pass 3: one warp reduces the per-block winners
__global__ void k_brute_final(const __grid_constant__ harl_sketch_desc sk,
                              const unsigned long long* block_best, int n,
                              unsigned long long* out) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  uint64_t v = ~0ull;
  for (int i = threadIdx.x; i < n; i += 32)
    if (canon_less(sk, block_best[i], v)) v = block_best[i];
  v = canon_warp_min(sk, v);
  if (threadIdx.x == 0) *out = v;
}

}  // namespace harl
