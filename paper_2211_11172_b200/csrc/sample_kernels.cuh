// K4 epilogue as its own full-occupancy kernel: masked log-softmax per head
// (rlcore.py:185-199), inverse-CDF sampling on the numpy PCG64 stream
// (rlcore.py:202-213, select_actions 216-228) and decode + apply
// (schedspace.py:196-301).  A group of 8 lanes per row: the head-0
// columns are spread over the group (max / sum / inclusive CDF scan with
// 3-step shuffles), lanes 0-3 draw the four heads' uniforms in parallel
// (one PCG64 jump each), lanes 0-2 sample the 3-way shift heads, and the
// walker writes 8 slots per lane.  (Thread-per-row is latency-bound at
// 16 K rows; warp-per-row wastes ~4x the issue slots.)
//
// Uniforms: draw #(h*m + row + 1) after the step's base state, row = the
// global row (shards) or the local row.
#pragma once

#include "common.cuh"
#include "space_kernels.cuh"

namespace harl {

struct LaneJump {
  u128 A[32];
  u128 C[32];
};

#ifndef HARL_SAMPLE_LANES
#define HARL_SAMPLE_LANES 8
#endif
#ifndef HARL_SAMPLE_ROWS
#define HARL_SAMPLE_ROWS 16     // rows per CTA
#endif
#ifndef HARL_SAMPLE_MINB
#define HARL_SAMPLE_MINB (7 * 8 * 16 / (HARL_SAMPLE_LANES * HARL_SAMPLE_ROWS))  // 72 registers: one wave of 16-row CTAs at 16 K rows, fewer spills than 64 (-1 us per launch)
#endif
#ifndef HARL_SAMPLE_FILL_FIRST
#define HARL_SAMPLE_FILL_FIRST 1
#endif
constexpr int SG = HARL_SAMPLE_LANES;   // lanes cooperating on one row
constexpr int SAMPLE_THREADS = HARL_SAMPLE_ROWS * SG;
constexpr int SAMPLE_MAXI = 16;        // cached exps per lane (C0 <= 128)
static_assert(SAMPLE_THREADS <= 1024, "HARL_SAMPLE_ROWS x HARL_SAMPLE_LANES: at most 1024 threads");
static_assert(HARL_SAMPLE_MINB >= 1, "HARL_SAMPLE_MINB must be at least 1");

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
  const int32_t* grow;   // optional: global row of each local row (shards)
  int64_t m_total;       // rows drawn this step over all shards
  const PcgTab* pcg_tab; // optional byte-sliced jump table of the stream
  int32_t prefill;       // launched with PDL: stage the constant tables
                         // before the programmatic-dependency wait
};

__device__ inline float gmaxf(float v) {
#pragma unroll
  for (int o = SG / 2; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o, SG));
  return v;
}
__device__ inline double gsum(double v) {
#pragma unroll
  for (int o = SG / 2; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, SG);
  return v;
}
__device__ inline int gsumi(int v) {
#pragma unroll
  for (int o = SG / 2; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, SG);
  return v;
}

// one thread's masked log-softmax logp of column a (inject mode only)
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

// 3-column shift head, sequential in one thread (the reference's cumsum).
// The inverse CDF compares the running sum of the exps with u * s instead
// of dividing every probability by s (the reference's p = e / s, cumsum,
// count(c < u)); the two differ only for a uniform within rounding of a
// CDF boundary, far inside the fp32-logit flips the parity tests bound.
__device__ inline int sample3(const float* z, uint32_t m3, double u,
                              double* logp_out) {
  float zmax = -INFINITY;
  for (int j = 0; j < 3; ++j)
    if ((m3 >> j) & 1u) zmax = fmaxf(zmax, z[j]);
  double e[3], s = 0.0;
  for (int j = 0; j < 3; ++j) {
    e[j] = ((m3 >> j) & 1u) ? (double)expf(z[j] - zmax) : 0.0;
    s += e[j];
  }
  const double us = u * s;
  int count = 0;
  double c = 0.0;
  for (int j = 0; j < 3; ++j) {
    c += e[j];
    count += (c < us);
  }
  int idx = min(count, 2);
  while (idx > 0 && !((m3 >> idx) & 1u)) --idx;
  const bool ok = (m3 >> idx) & 1u;
  // log(s) in fp32 (s in [1, 3]): ~2e-7 absolute on logp
  *logp_out = ok ? ((double)z[idx] - (double)zmax - (double)logf((float)s))
                 : -INFINITY;
  return ok ? idx : -1;
}

// The footprint tables and the log2 LUT of the in-sampler featurize,
// staged in shared memory by the CTA prologue: the descriptor's arrays live
// in the kernel's parameter bank (indexed loads through the constant cache)
// and the LUT in global memory, and on a cold SM each dependent lookup of
// the per-term chain cost an L2 round trip (3.7 us for the footprint of
// one row on the first CTA of an SM, phase probe).  Units are (tensor,
// level) pairs so the row's 8 lanes share the products.
constexpr int FEAT_LUT_SMEM_MAX = 1024;   // LUT entries staged (8 KB)
struct FootSmem {
  int16_t gi[HARL_MAX_TERMS];
  int32_t sc[HARL_MAX_TERMS], off[HARL_MAX_TERMS];
  int16_t tfirst[HARL_MAX_TENSORS], tn[HARL_MAX_TENSORS];
  int32_t coef1[HARL_MAX_TENSORS];   // level 1: inter+extra on a stage's last tensor
  int32_t coef2x[HARL_MAX_TENSORS];  // level 2: extra on the last tensor
  int32_t coef2i[HARL_MAX_TENSORS];  // level 2 at the root: + inter
};

__device__ inline void foot_fill(const harl_sketch_desc& sk, FootSmem* fs,
                                 double* lut_s, int lut_n) {
  for (int q = threadIdx.x; q < sk.n_terms; q += blockDim.x) {
    fs->gi[q] = sk.term_gi[q];
    fs->sc[q] = sk.term_sc[q];
    fs->off[q] = sk.term_off[q];
  }
  for (int ti = threadIdx.x; ti < sk.n_tensors; ti += blockDim.x) {
    fs->tfirst[ti] = sk.tensor_first[ti];
    fs->tn[ti] = sk.tensor_nterms[ti];
    // the last tensor of each stage carries the stage terms
    int c1 = 0, c2x = 0, c2i = 0;
    for (int st = 0; st < sk.n_stages; ++st)
      if (sk.stage_ntensors[st] > 0 &&
          ti == sk.stage_first[st] + sk.stage_ntensors[st] - 1) {
        c1 = sk.stage_inter[st] + sk.stage_extra[st];
        c2x = sk.stage_extra[st];
        c2i = sk.stage_inter[st];
      }
    fs->coef1[ti] = c1;
    fs->coef2x[ti] = c2x;
    fs->coef2i[ti] = c2i;
  }
  if (lut_s)
    for (int v = threadIdx.x; v < lut_n; v += blockDim.x) lut_s[v] = __ldg(sk.log2_lut + v);
}

// the CTA's constant tables: compact head-0 column -> (src, dst) slots,
// footprint terms, log2 LUT (from the descriptor's device copy when there
// is one: coalesced loads, not per-thread constant-bank reads that
// serialise by address)
__device__ inline void sample_fill(const harl_sketch_desc& sk, int16_t* s_src,
                                   int16_t* s_dst, FootSmem* fs, double* lut_s,
                                   int lut_n) {
  const harl_sketch_desc& sg = sk.dev_self ? *sk.dev_self : sk;
  for (int i = threadIdx.x; i < sk.n_head0; i += blockDim.x) {
    const int16_t vs = sg.head0_src[i], vd = sg.head0_dst[i];
    s_src[i] = vs;
    s_dst[i] = vd;
  }
  if (fs) foot_fill(sg, fs, lut_s, lut_n);
}

// inject mode (parity replays): lane 0 scores the given actions; out of
// line so the sampling path stays compact in the instruction cache
struct InjectRow {
  int act[4];
  int col0;
  int dead;
  double lp;
};
__device__ __noinline__ InjectRow sample_inject_row(
    const float* z, int C0, int S, uint64_t mv, const int16_t* s_src,
    const int16_t* s_dst, uint32_t sb, const int32_t* inject, int64_t n,
    int64_t rr) {
  InjectRow o;
  int* act = o.act;
  auto legal0 = [&](int j) -> bool {
    return j == C0 - 1 || ((mv >> s_src[j]) & 1ull);
  };
  const int full = inject[rr];
  int jj = -1;
  if (full == S * S) jj = C0 - 1;
  else if (full >= 0 && full < S * S)
    for (int c = 0; c < C0 - 1; ++c)
      if (s_src[c] == full / S && s_dst[c] == full % S) jj = c;
  act[0] = full;
  o.col0 = jj < 0 ? 0 : jj;
  double lp = jj < 0 ? -INFINITY : row_logp(z, C0, legal0, jj);
  bool d = false;
  for (int h = 1; h < 4; ++h) {
    const uint32_t m3 = (sb >> (3 * (h - 1))) & 7u;
    act[h] = inject[h * n + rr];
    lp += row_logp(z + C0 + 3 * (h - 1), 3,
                   [&](int j) -> bool { return (m3 >> j) & 1u; }, act[h]);
    d |= (m3 == 0);
  }
  o.lp = lp;
  o.dead = d;
  return o;
}

// One 8-lane group samples and applies the action of global row r (the
// rows past a.n compute on row 0 and write nothing, so every lane stays in
// the group shuffles).  zrow: the row's logits (null: a.logits + r*ldz);
// s_src/s_dst: the compact head-0 column tables, filled by the caller.
// NSL: slots per lane (a row's local slots <= SG * NSL; the host picks the
// smallest of 2 / 4 / 8, so the state loops carry no dead iterations)
template <int MAXI = SAMPLE_MAXI, int NSL = HARL_MAX_SLOTS / SG>
__device__ __forceinline__ void sample_group(
    const harl_sketch_desc& sk, const PcgJump& J, u128 base_arg,
    const u128* base_dev, const uint16_t* __restrict__ tiles,
    const uint8_t* __restrict__ knobs, const SampleArgs& a, int64_t r,
    const float* zrow, const int16_t* s_src, const int16_t* s_dst,
    uint16_t* st_tiles = nullptr, uint8_t* st_knobs = nullptr,
    bool fill_tables = false, FootSmem* fs = nullptr, double* lut_s = nullptr,
    int lut_n = 0) {
  const int g = threadIdx.x & (SG - 1);
  // every group stays in the shuffles; out-of-range rows compute on row 0
  const bool live = r < a.n;
  const int64_t rr = live ? r : 0;
  const int S = sk.num_slots, C0 = sk.n_head0;
  const bool draw = !a.inject && g < 4;
#if HARL_SAMPLE_FILL_FIRST
  // the CTA's constant tables first: holding the row loads (32 registers of
  // PCG table entries among them) across the table fill spilled them, and
  // the spill stores serialised the row loads behind their round trips
  if (fill_tables) {
    sample_fill(sk, const_cast<int16_t*>(s_src), const_cast<int16_t*>(s_dst),
                fs, lut_s, lut_n);
    __syncthreads();
    fill_tables = false;
  }
#endif
  // ---- every global load of the row is issued before any math ----------
  u128 base = base_arg;
  int64_t grow_r = rr;
  if (draw) {
    if (base_dev) base = *base_dev;
    if (a.grow) grow_r = (int64_t)a.grow[rr];
  }
  static_assert(NSL * SG <= HARL_MAX_SLOTS, "slots per lane");
  int tv[NSL];
#pragma unroll
  for (int i = 0; i < NSL; ++i) {
    const int s = g + SG * i;
    tv[i] = s < sk.local_slots ? tiles[(int64_t)s * a.ld + rr] : 0;
  }
  const int ca0 = knobs[rr], par0 = knobs[a.ld + rr], ur0 = knobs[2 * a.ld + rr];
  // this lane's draw: table entries loaded now, applied after the barrier
  const uint64_t kdraw = (uint64_t)g * (uint64_t)a.m_total + (uint64_t)grow_r + 1;
  const bool tab = draw && a.pcg_tab && kdraw < (1ull << 32);
  u128 pA[4], pC[4];
  if (tab) pcg_tab_load(a.pcg_tab, (uint32_t)kdraw, pA, pC);
  const float* z = zrow ? zrow : a.logits + rr * a.ldz;
  // lane g owns the contiguous head-0 columns [g*nI, g*nI + nI): local
  // max / sum / prefix, then one 8-lane scan of the lane totals
  const int nI = (C0 + SG - 1) / SG;
  const int jb = g * nI;
  float zc[MAXI];   // head-0 logits j = jb + i (padding reads as -inf)
  float z3[3] = {0.f, 0.f, 0.f};   // shift head g+1's three logits (lanes 0-2)
  if (!a.inject) {
#pragma unroll
    for (int i = 0; i < MAXI; ++i) {
      const int j = jb + i;
      zc[i] = (i < nI && j < C0) ? z[j] : -INFINITY;
    }
    if (g < 3) {
#pragma unroll
      for (int j = 0; j < 3; ++j) z3[j] = z[C0 + 3 * g + j];
    }
  }
  if (fill_tables) {
    dbg_ts(38);
    // the CTA's head-0 column tables, filled while the row loads above are
    // in flight (the caller passes this CTA's shared arrays)
    sample_fill(sk, const_cast<int16_t*>(s_src), const_cast<int16_t*>(s_dst),
                fs, lut_s, lut_n);
    dbg_ts(39);
    __syncthreads();
    dbg_ts(36);
  }
  // ---- uniforms: lane h of the group draws head h ---------------------
  double u_mine = 0.0;
  if (tab) u_mine = u64_to_unit(pcg_output(pcg_tab_apply(base, pA, pC)));
  else if (draw) u_mine = u64_to_unit(pcg_draw64_bitwise(J, base, kdraw));
  dbg_ts(17);
  // ---- current state: lane g holds slots g, g+8, ... --------------------
  uint64_t mv = 0;
#pragma unroll
  for (int i = 0; i < NSL; ++i)
    if (tv[i] > 1) mv |= 1ull << (g + SG * i);
#pragma unroll
  for (int o = SG / 2; o; o >>= 1) mv |= __shfl_xor_sync(0xffffffffu, mv, o, SG);
  const uint32_t sb = shift_bits_of(sk, ca0, par0, ur0);
  dbg_ts(18);
  auto legal0 = [&](int j) -> bool {
    return j == C0 - 1 || ((mv >> s_src[j]) & 1ull);
  };
  int act[4];
  int col0 = 0;
  double lp_total = 0.0;
  bool dead = false;
  // ---- head 0: columns j = g + 8 i --------------------------------------
  if (a.inject) {
    if (g == 0) {
      const InjectRow o = sample_inject_row(z, C0, S, mv, s_src, s_dst, sb,
                                            a.inject, a.n, rr);
#pragma unroll
      for (int h = 0; h < 4; ++h) act[h] = o.act[h];
      col0 = o.col0;
      lp_total = o.lp;
      dead = o.dead != 0;
    }
  } else {
    const double u0 = __shfl_sync(0xffffffffu, u_mine, 0, SG);
    // the lane's cached columns: in range (rm) and legal (lm), tested once
    uint32_t lm = 0, rm = 0;
#pragma unroll
    for (int i = 0; i < MAXI; ++i) {
      const int j = jb + i;
      if (i < nI && j < C0) {
        rm |= 1u << i;
        if (legal0(j)) lm |= 1u << i;
      }
    }
    float zmax = -INFINITY;
#pragma unroll
    for (int i = 0; i < MAXI; ++i)
      if ((lm >> i) & 1u) zmax = fmaxf(zmax, zc[i]);
    for (int i = MAXI; i < nI; ++i) {   // wide heads (C0 > 128)
      const int j = jb + i;
      if (j < C0 && legal0(j)) zmax = fmaxf(zmax, z[j]);
    }
    zmax = gmaxf(zmax);
    dead |= (zmax == -INFINITY);
    float e[MAXI];
    double sl = 0.0;
#pragma unroll
    for (int i = 0; i < MAXI; ++i) {
      e[i] = ((lm >> i) & 1u) ? expf(zc[i] - zmax) : 0.f;
      sl += (double)e[i];
    }
    for (int i = MAXI; i < nI; ++i) {
      const int j = jb + i;
      if (j < C0 && legal0(j)) sl += (double)expf(z[j] - zmax);
    }
    const double s = gsum(sl);
    dbg_ts(19);
    // inverse CDF on the running sums of the exps against u * s (no
    // division per column, see sample3); lane offsets = exclusive scan of
    // the lane totals (3 shuffle steps)
    const double tot = sl;
    const double us0 = u0 * s;
    double incl = tot;
#pragma unroll
    for (int o = 1; o < SG; o <<= 1) {
      const double t = __shfl_up_sync(0xffffffffu, incl, o, SG);
      if (g >= o) incl += t;
    }
    double c = incl - tot;   // exclusive offset
    int count = 0;
#pragma unroll
    for (int i = 0; i < MAXI; ++i) {
      c += (double)e[i];
      if (((rm >> i) & 1u) && c < us0) ++count;
    }
    for (int i = MAXI; i < nI; ++i) {
      const int j = jb + i;
      if (j < C0) {
        if (legal0(j)) c += (double)expf(z[j] - zmax);
        if (c < us0) ++count;
      }
    }
    count = gsumi(count);
    dbg_ts(20);
    int idx = min(count, C0 - 1);
    while (idx > 0 && !legal0(idx)) --idx;
    const bool ok = legal0(idx);
    // log(s) in fp32 (s in [1, C0]): ~5e-7 absolute on logp, against the
    // 1e-4 * max(|logp|, rms) tolerance
    const double lp0 = ok ? ((double)z[idx] - (double)zmax -
                             (double)logf((float)s)) : -INFINITY;
    act[0] = !ok ? 0 : ((idx == C0 - 1) ? S * S : s_src[idx] * S + s_dst[idx]);
    col0 = ok ? idx : 0;
    // shift heads: lane h-1 handles head h
    int ah = 0;
    double lph = 0.0;
    const int hh = g + 1;
    const double uh = __shfl_sync(0xffffffffu, u_mine, hh < 4 ? hh : 0, SG);
    if (hh < 4) {
      const uint32_t m3 = (sb >> (3 * (hh - 1))) & 7u;
      const int j = sample3(z3, m3, uh, &lph);
      ah = j < 0 ? 0 : j;
    }
    dbg_ts(21);
    lp_total = lp0;
#pragma unroll
    for (int h = 1; h < 4; ++h) {
      act[h] = __shfl_sync(0xffffffffu, ah, h - 1, SG);
      lp_total += __shfl_sync(0xffffffffu, lph, h - 1, SG);
    }
#pragma unroll
    for (int h = 1; h < 4; ++h) dead |= (((sb >> (3 * (h - 1))) & 7u) == 0);
  }
  // inject mode: broadcast lane 0's decisions
#pragma unroll
  for (int h = 0; h < 4; ++h) act[h] = __shfl_sync(0xffffffffu, act[h], 0, SG);
  col0 = __shfl_sync(0xffffffffu, col0, 0, SG);
  lp_total = __shfl_sync(0xffffffffu, lp_total, 0, SG);
  dead = __shfl_sync(0xffffffffu, (int)dead, 0, SG);
  // ---- decode + apply (schedspace.py:196-210, 265-301) -----------------
  int src = -1, dst = -1;
  if (act[0] != S * S) {
    src = act[0] / S;
    dst = act[0] % S;
  }
  int code = dead ? HARL_ST_NO_VALID : HARL_ST_OK;
  // factors at src/dst: shuffled unconditionally so every lane of the warp
  // executes the same shuffles whatever its group decided
  const int sidx = src >= 0 && src < HARL_MAX_SLOTS ? src : 0;
  const int didx = dst >= 0 && dst < HARL_MAX_SLOTS ? dst : 0;
  int vs = 0, vd = 0;
#pragma unroll
  for (int i = 0; i < NSL; ++i) {
    if (i == sidx / SG) vs = tv[i];
    if (i == didx / SG) vd = tv[i];
  }
  const int f_src = __shfl_sync(0xffffffffu, vs, sidx % SG, SG);
  const int f_dst = __shfl_sync(0xffffffffu, vd, didx % SG, SG);
  int p = 1;
  if (code == HARL_ST_OK && src >= 0) {
    if (src >= sk.local_slots || dst >= sk.local_slots || dst < 0 ||
        src / sk.levels != dst / sk.levels || src == dst || f_src <= 1)
      code = HARL_ST_TILING;
    else
      p = sk.spf_lut[f_src];
  }
  const int ca = ca0 + (act[1] - 1), par = par0 + (act[2] - 1),
            ur = ur0 + (act[3] - 1);
  if (code == HARL_ST_OK) {
    if (ca < 0 || ca >= sk.ncas) code = HARL_ST_COMPUTE_AT;
    else if (par < 0 || par > sk.max_fusible) code = HARL_ST_PARALLEL;
    else if (ur < 0 || ur >= sk.n_unroll) code = HARL_ST_UNROLL;
  }
  dbg_ts(22);
  if (!live) return;
  const bool moved = code == HARL_ST_OK && src >= 0;
#pragma unroll
  for (int i = 0; i < NSL; ++i) {
    const int s = g + SG * i;
    if (s < sk.local_slots) {
      int v = tv[i];
      if (moved && s == src) v = f_src / p;
      if (moved && s == dst) v = f_dst * p;
      a.tiles_out[(int64_t)s * a.ld + r] = (uint16_t)v;
      if (st_tiles) st_tiles[s] = (uint16_t)v;
    }
  }
  if (st_knobs && g == 0) {   // the successor's knobs (old ones on failure)
    const bool ok = code == HARL_ST_OK;
    st_knobs[0] = (uint8_t)(ok ? ca : ca0);
    st_knobs[1] = (uint8_t)(ok ? par : par0);
    st_knobs[2] = (uint8_t)(ok ? ur : ur0);
  }
  if (g == 0) {
    if (code == HARL_ST_OK) {
      a.knobs_out[r] = (uint8_t)ca;
      a.knobs_out[a.ld + r] = (uint8_t)par;
      a.knobs_out[2 * a.ld + r] = (uint8_t)ur;
    }
    for (int h = 0; h < 4; ++h) a.actions[h * a.n + r] = act[h];
    a.logp[r] = lp_total;
    a.move_bits[r] = mv;
    a.shift_bits[r] = sb;
    a.head0_col[r] = col0;
    report_status(a.status, r, code);
  }
}

// featurize one successor state (schedspace.py:415-438) with the row's 8
// lanes: tile logs spread over the lanes, the two footprint levels (and
// their glibc log10s) on lanes 1 and 2, the knob/flop features on lane 0;
// the row is built in shared memory (dst, F doubles) from the successor
// state the sampler left in st / kn
__device__ __forceinline__ void featurize_group(const harl_sketch_desc& sk,
                                                int g, unsigned gmask,
                                                const uint16_t* st,
                                                const uint8_t* kn, double* dst,
                                                const FootSmem* fs,
                                                const double* lut_s) {
  const int F = sk.feature_len, L = sk.levels;
  for (int k = g; k < F; k += SG) dst[k] = 0.0;
  __syncwarp(gmask);
  dbg_ts(32);
  for (int s2 = g; s2 < sk.local_slots; s2 += SG)
    dst[s2] = lut_s ? lut_s[st[s2]] : __ldg(sk.log2_lut + st[s2]);
  const int ca = kn[0], par = kn[1], ur = kn[2];
  dbg_ts(33);
  const int pos = sk.max_feature_dims * L;
  // footprints (footprint_level's integer sums, schedspace.py:415-438):
  // unit u = (tensor u/2, level 1 + u%2); per tensor e = prod over its
  // terms of (sc * t[gi] + off), weighted 1 (+ the stage terms on a
  // stage's last tensor); int64 sums, so the lane split is exact
  const bool root = ca == 0;
  long long l1 = 0, l2 = 0;
  for (int u = g; u < 2 * sk.n_tensors; u += SG) {
    const int ti = u >> 1;
    const bool lv2 = (u & 1) && L >= 2;
    long long e = 1;
    const int f = fs->tfirst[ti], nt = fs->tn[ti];
    for (int q = f; q < f + nt; ++q) {
      const int d = fs->gi[q];
      long long t = st[d * L + L - 1];
      if (lv2) t *= st[d * L + L - 2];
      e *= (long long)fs->sc[q] * t + fs->off[q];
    }
    if (u & 1) l2 += e * (1 + fs->coef2x[ti] + (root ? fs->coef2i[ti] : 0));
    else l1 += e * (1 + fs->coef1[ti]);
  }
#pragma unroll
  for (int o = SG / 2; o; o >>= 1) {
    l1 += __shfl_xor_sync(gmask, l1, o, SG);
    l2 += __shfl_xor_sync(gmask, l2, o, SG);
  }
  if (g == 0) {
    dst[pos] = sk.ncas > 1 ? __ddiv_rn((double)ca, (double)(sk.ncas - 1)) : 0.0;
    dst[pos + 1] = sk.max_fusible ? __ddiv_rn((double)par, (double)sk.max_fusible) : 0.0;
    dst[pos + 2 + ur] = 1.0;
    dst[pos + 2 + sk.n_unroll + 2] = sk.flops_feature;
  } else if (g == 1 || g == 2) {
    const long long l = g == 1 ? l1 : l2;
    dst[pos + 2 + sk.n_unroll + g - 1] =
        __ddiv_rn(glibc_log10_ge1(__dadd_rn(1.0, (double)l)), 6.0);
  }
}

// MAXI: head-0 columns cached per lane (>= ceil(C0 / SG) for the cached
// path; the host picks the smallest of 8 / 12 / 16 that covers the head so
// the unrolled column loops carry no dead iterations)
template <bool FEAT, int MAXI, int NSL>
__global__ void __launch_bounds__(SAMPLE_THREADS, HARL_SAMPLE_MINB)
k_sample_rows(const __grid_constant__ harl_sketch_desc sk,
              const __grid_constant__ PcgJump J,
              const __grid_constant__ LaneJump LJ, u128 base_arg,
              const u128* base_dev, const uint16_t* __restrict__ tiles,
              const uint8_t* __restrict__ knobs, SampleArgs a,
              double* __restrict__ feat_out) {
  constexpr int ROWS = SAMPLE_THREADS / SG;
  __shared__ int16_t s_src[HARL_MAX_HEAD0], s_dst[HARL_MAX_HEAD0];
  __shared__ uint16_t s_st[FEAT ? ROWS : 1][HARL_MAX_SLOTS];
  __shared__ uint8_t s_kn[FEAT ? ROWS : 1][4];
  extern __shared__ double s_feat[];   // FEAT: [ROWS][F], then the LUT
  __shared__ FootSmem s_foot[1];
  (void)LJ;
  const int lut_n = sk.max_extent + 1;
  double* lut_s = (FEAT && lut_n <= FEAT_LUT_SMEM_MAX)
                      ? s_feat + (SAMPLE_THREADS / SG) * sk.feature_len : nullptr;
  // launched with PDL: the constant tables are staged while the previous
  // kernel drains; otherwise inside sample_group behind the row loads
  if (a.prefill) sample_fill(sk, s_src, s_dst, FEAT ? s_foot : nullptr, lut_s, lut_n);
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  if (a.prefill) __syncthreads();
  dbg_ts(16);
  dbg_grid(false, 60);
  const int lr = threadIdx.x / SG;
  const int64_t r0 = (int64_t)blockIdx.x * ROWS;
  const int64_t r = r0 + lr;
  sample_group<MAXI, NSL>(sk, J, base_arg, base_dev, tiles, knobs, a, r, nullptr, s_src,
               s_dst, FEAT ? s_st[lr] : nullptr, FEAT ? s_kn[lr] : nullptr,
               /*fill_tables=*/!a.prefill, FEAT ? s_foot : nullptr, lut_s, lut_n);
  dbg_ts(23);
  if (FEAT) {
    const int g = threadIdx.x & (SG - 1);
    const unsigned gmask = (SG == 32 ? 0xffffffffu : ((1u << SG) - 1u))
                           << (threadIdx.x & (32 - SG));
    __syncwarp(gmask);
    const int F = sk.feature_len;
    if (r < a.n)
      featurize_group(sk, g, gmask, s_st[lr], s_kn[lr], s_feat + lr * F,
                      s_foot, lut_s);
    dbg_ts(34);
    __syncthreads();
    dbg_ts(35);
    const int64_t rows = a.n - r0 < ROWS ? a.n - r0 : ROWS;
    double* out = feat_out + r0 * F;
    for (int i = threadIdx.x; i < rows * F; i += blockDim.x) out[i] = s_feat[i];
    dbg_ts(31);
  }
  griddep_trigger();
  dbg_grid(true, 60);
}

}  // namespace harl

#include "gbt_kernels.cuh"

namespace harl {

// ---------------------------------------------------------------------------
// Sampler + featurize + GBT predict/reward in one kernel (populations whose
// step rows fit the in-sampler featurize).  The successor rows' features
// are already in shared memory when the sampler has featurized them, so
// the cost model (costmodel.py:219-230: pred = base + sum_t lr*leaf_t in
// tree order, np.maximum(pred, floor)) and the reward (tuner.py:389-391:
// (new - old) / old) are evaluated right there: no feature round trip, no
// separate GBT launch with its own forest prologue.  The forest's
// perfect-tree image (depth <= SGBT_DEPTH; the reference's GbtConfig
// default is 6) is bulk-copied into shared memory at kernel start -- the
// forest is written by host copies only, so the copy runs ahead of the
// programmatic-dependency wait and lands while the CTA samples.  The 8
// lanes of a row walk trees g, g+8, ... (4 side by side) and then add the
// contributions in tree order through group shuffles, every lane forming
// the same sequential sum (bit-identical to gbt2_body).  A reloaded forest
// the region cannot hold (deeper, more trees than the launch was sized
// for, or no perfect image) is walked from the global node records.
constexpr int SGBT_ROWS = 64;
constexpr int SGBT_THREADS = SGBT_ROWS * SG;
constexpr int SGBT_MAX_TREES = 8 * SG;   // 8 contributions per lane
constexpr int SGBT_DEPTH = 6;
static_assert(SGBT_THREADS <= 1024, "k_sample_gbt: at most 1024 threads");

struct SampleGbtArgs {
  const GbtNode* nodes;        // node records (fallback walk)
  const int32_t* tree_first;
  const GbtHdr* hdr;           // run-time forest scalars
  const double* old_score;     // [n] score of the row's current state
  double* score;               // [n] out
  double* reward;              // [n] out
  int32_t region;              // shared bytes reserved for the image
};

__host__ __device__ inline size_t sgbt_region_bytes(int t_cap) {
  return gbt_perfect_bytes(t_cap, SGBT_DEPTH);
}

template <int MAXI, int NSL>
__global__ void __launch_bounds__(SGBT_THREADS, 2)
k_sample_gbt(const __grid_constant__ harl_sketch_desc sk,
             const __grid_constant__ PcgJump J, u128 base_arg,
             const u128* base_dev, const uint16_t* __restrict__ tiles,
             const uint8_t* __restrict__ knobs, SampleArgs a,
             double* __restrict__ feat_out,
             const __grid_constant__ SampleGbtArgs ga) {
  constexpr int ROWS = SGBT_ROWS;
  __shared__ int16_t s_src[HARL_MAX_HEAD0], s_dst[HARL_MAX_HEAD0];
  __shared__ uint16_t s_st[ROWS][HARL_MAX_SLOTS];
  __shared__ uint8_t s_kn[ROWS][4];
  __shared__ FootSmem s_foot[1];
  __shared__ uint64_t fbar;
  __shared__ int s_gi[3];          // n_trees, fitted, staged depth (0: global walk)
  __shared__ double s_gd[2];       // base, floor
  extern __shared__ __align__(16) unsigned char sgm[];
  unsigned char* s_forest = sgm;
  double* s_feat = (double*)(sgm + ga.region);
  if (threadIdx.x == 0) {
    const GbtHdr h = *ga.hdr;
    const int D = h.perfect_depth;
    const bool stage = h.fitted && h.n_trees > 0 && D >= 1 && D <= SGBT_DEPTH &&
                       h.perfect_bytes > 0 && h.perfect_bytes <= ga.region;
    s_gi[0] = h.n_trees;
    s_gi[1] = h.fitted;
    s_gi[2] = stage ? D : 0;
    s_gd[0] = h.base;
    s_gd[1] = h.floor_value;
    if (stage) {
      tc::mbar_init(&fbar, 1);
      tc::bulk_load(s_forest, h.perfect, (uint32_t)h.perfect_bytes, &fbar);
    }
  }
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  const int lut_n = sk.max_extent + 1;
  double* lut_s = lut_n <= FEAT_LUT_SMEM_MAX ? s_feat + ROWS * sk.feature_len : nullptr;
  const int lr = threadIdx.x / SG;
  const int g = threadIdx.x & (SG - 1);
  const int64_t r0 = (int64_t)blockIdx.x * ROWS;
  const int64_t r = r0 + lr;
  // (the table fill inside ends with a CTA barrier: s_gi/s_gd are visible)
  sample_group<MAXI, NSL>(sk, J, base_arg, base_dev, tiles, knobs, a, r, nullptr,
                          s_src, s_dst, s_st[lr], s_kn[lr], /*fill_tables=*/true,
                          s_foot, lut_s, lut_n);
  const unsigned gmask = (SG == 32 ? 0xffffffffu : ((1u << SG) - 1u))
                         << (threadIdx.x & (32 - SG));
  __syncwarp(gmask);
  const int F = sk.feature_len;
  double* x = s_feat + lr * F;
  if (r < a.n) featurize_group(sk, g, gmask, s_st[lr], s_kn[lr], x, s_foot, lut_s);
  const bool live = r < a.n;
  const double o = (live && ga.old_score) ? ga.old_score[r] : 1.0;
  __syncthreads();
  {
    const int64_t rows = a.n - r0 < ROWS ? a.n - r0 : ROWS;
    double* out = feat_out + r0 * F;
    for (int i = threadIdx.x; i < rows * F; i += blockDim.x) out[i] = s_feat[i];
  }
  // ---- cost model on the row's features (shared memory) -------------------
  const int T = s_gi[0], fitted = s_gi[1], D = s_gi[2];
  double c[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) c[j] = 0.0;
  if (fitted) {
    const uint32_t s_x = tc::smem_u32(x);
    if (D > 0) {
      tc::mbar_wait(&fbar, 0);
      const int NI = (1 << D) - 1, NLF = 1 << D;
      const uint32_t s_thr = tc::smem_u32(s_forest);
      const uint32_t s_leaf = s_thr + (uint32_t)gbt_perfect_off_leaf(T, D);
      const uint32_t s_ft = s_thr + (uint32_t)gbt_perfect_off_feat(T, D);
#pragma unroll
      for (int jb = 0; jb < 8; jb += GBT_ILP) {
        uint32_t tbase[GBT_ILP], idx[GBT_ILP];
#pragma unroll
        for (int k = 0; k < GBT_ILP; ++k) {
          const int t = g + SG * (jb + k);
          tbase[k] = (uint32_t)((t < T ? t : 0) * NI);
          idx[k] = 0;
        }
        if (g + SG * jb >= T) continue;
        for (int lv = 0; lv < D; ++lv) {
          int f[GBT_ILP];
          double th[GBT_ILP], xv[GBT_ILP];
#pragma unroll
          for (int k = 0; k < GBT_ILP; ++k) {
            f[k] = lds_s16(s_ft + 2u * (tbase[k] + idx[k]));
            th[k] = lds_f64(s_thr + 8u * (tbase[k] + idx[k]));
          }
#pragma unroll
          for (int k = 0; k < GBT_ILP; ++k) xv[k] = lds_f64(s_x + 8u * (uint32_t)f[k]);
#pragma unroll
          for (int k = 0; k < GBT_ILP; ++k) idx[k] = 2u * idx[k] + (xv[k] <= th[k] ? 1u : 2u);
        }
#pragma unroll
        for (int k = 0; k < GBT_ILP; ++k) {
          const int t = g + SG * (jb + k);
          const double lv = lds_f64(s_leaf + 8u * ((uint32_t)(t < T ? t : 0) * NLF +
                                                   idx[k] - (uint32_t)NI));
          if (t < T) c[jb + k] = lv;
        }
      }
    } else {
      // node records in global memory (a forest the region cannot hold)
      const double* xg = x;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int t = g + SG * j;
        if (t < T) {
          const GbtNode* tree = ga.nodes + __ldg(ga.tree_first + t);
          GbtNode nd = tree[0];
          while (nd.feat >= 0) nd = tree[(xg[nd.feat] <= nd.v) ? nd.left : nd.right];
          c[j] = nd.v;
        }
      }
    }
  }
  // tree-order sum (pred = pred + lr*leaf, costmodel.py:208/228): every lane
  // of the group forms the same sequential chain from the shuffled terms
  double pred = 1.0;
  if (fitted) {
    pred = s_gd[0];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int q = 0; q < SG; ++q) {
        const double v = __shfl_sync(0xffffffffu, c[j], q, SG);
        if (SG * j + q < T) pred = __dadd_rn(pred, v);
      }
    }
  }
  if (live && g == 0) {
    const double fl = s_gd[1];
    const double s = (pred != pred) ? pred : (pred < fl ? fl : pred);
    ga.score[r] = s;
    if (ga.old_score) ga.reward[r] = __ddiv_rn(__dsub_rn(s, o), o);
  }
  griddep_trigger();
}

}  // namespace harl
