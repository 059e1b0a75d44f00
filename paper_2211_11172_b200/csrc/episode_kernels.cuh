// K5 tail + K8: per-step bookkeeping of _run_episode (tuner.py:393-412):
// advantage/TD (rlcore.py:231-234, tuner.py:398), the replay push
// (rlcore.py:253-265: a FIFO holding the last `cap` transitions, pushed in
// row order), the visited-entry log (tuner.py:406-412) and Track.advance
// (stopping.py:45-53); plus the survivor compaction after a host cull.
#pragma once

#include "common.cuh"

namespace harl {

struct FinishArgs {
  int64_t n;            // rows this step (m)
  int64_t ld;           // leading dim of the population state arrays
  int64_t vbase;        // visit index of row 0 in the entry log
  int32_t local_slots;
  int32_t F;
  double discount;
  int32_t rl;           // value/advantage/replay only for RL searchers
  int64_t wpos;         // ring slot receiving row 0 (mod cap)
  int64_t keep_from;    // rows >= keep_from survive in the ring
};

constexpr int FIN_ROWS = 64;       // rows per CTA
constexpr int FIN_THREADS = 256;   // row work on the first 64, copy on all

__device__ inline void finish_row(const FinishArgs& a,
                                  const harl_step_buffers& io,
                                  const harl_replay_ring& ring,
                                  const harl_entry_log& log,
                                  const harl_track_stats& ts, int64_t wpos,
                                  int64_t r) {
  const int32_t* __restrict__ row_track = io.row_track;
  (void)FIN_THREADS;
  const uint16_t* __restrict__ tiles_new = io.tiles_new;
  const uint8_t* __restrict__ knobs_new = io.knobs_new;
  uint16_t* __restrict__ log_tiles = log.tiles;
  uint8_t* __restrict__ log_knobs = log.knobs;
  const double* new_score = io.new_score;
  const double* reward = io.reward;
  const float* v_cur = io.v_cur;
  const float* v_next = io.v_next;
  const int32_t* actions = io.actions;
  const int32_t* head0_col = io.head0_col;
  const double* logp = io.logp;
  const uint64_t* move_bits = io.move_bits;
  const uint32_t* shift_bits = io.shift_bits;
  double* adv_out = io.adv;
  const int64_t v = a.vbase + r;
  // every independent load of the row first (one memory round trip), then
  // the track-indexed ones (a second), then the stores
  const int32_t t = row_track[r];
  const double sc = new_score[r];
  const double rw = reward[r];
  uint8_t kn[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) kn[k] = knobs_new[(int64_t)k * a.ld + r];
  constexpr int TB = 32;
  uint16_t tl[TB];
#pragma unroll
  for (int q = 0; q < TB; ++q)
    tl[q] = (q < a.local_slots) ? tiles_new[(int64_t)q * a.ld + r] : 0;
  float vn32 = 0.f, vc32 = 0.f;
  double lp = 0.0;
  int32_t acts[4] = {0, 0, 0, 0};
  uint64_t mb = 0;
  uint32_t sb = 0;
  const bool push = a.rl && r >= a.keep_from;
  if (a.rl) {
    vn32 = v_next[r];
    vc32 = v_cur[r];
  }
  if (push) {
    acts[0] = head0_col[r];
#pragma unroll
    for (int h = 1; h < 4; ++h) acts[h] = actions[(int64_t)h * a.n + r];
    lp = logp[r];
    mb = move_bits[r];
    sb = shift_bits[r];
  }
  const int32_t st = ts.steps[t] + 1;
  const double best = ts.best_score[t];
#pragma unroll
  for (int q = 0; q < TB; ++q)
    if (q < a.local_slots) log_tiles[(int64_t)q * log.ld + v] = tl[q];
  for (int s0 = TB; s0 < a.local_slots; ++s0)
    log_tiles[(int64_t)s0 * log.ld + v] = tiles_new[(int64_t)s0 * a.ld + r];
#pragma unroll
  for (int k = 0; k < 3; ++k) log_knobs[(int64_t)k * log.ld + v] = kn[k];
  log.score[v] = sc;
  log.reward[v] = rw;
  log.track[v] = t;
  // Track.advance: steps += 1; best on strict improvement
  ts.steps[t] = st;
  if (sc > best) {
    ts.best_score[t] = sc;
    ts.best_step[t] = st;
  }
  if (!a.rl) return;
  // advantage(reward, v_next, v_cur) = reward + discount*v_next - v_cur
  const double tdv = __dadd_rn(rw, __dmul_rn(a.discount, (double)vn32));
  const double adv = __dsub_rn(tdv, (double)vc32);
  adv_out[r] = adv;
  if (!push) return;
  const int64_t slot = (wpos + r) % ring.cap;
  *(int4*)&ring.actions[slot * 4] = make_int4(acts[0], acts[1], acts[2], acts[3]);
  ring.scalars[slot * 4 + 0] = lp;
  ring.scalars[slot * 4 + 1] = rw;
  ring.scalars[slot * 4 + 2] = adv;
  ring.scalars[slot * 4 + 3] = tdv;
  ring.move_bits[slot] = mb;
  ring.shift_bits[slot] = sb;
}

// Per step: the row bookkeeping above for 64 rows, then the CTA copies the
// surviving rows' X and X' into their replay slots.  The rows' features are
// contiguous in both [n][F] arrays, so the loads are coalesced; slots are
// consecutive modulo cap.
__global__ void __launch_bounds__(FIN_THREADS)
k_finish_step(FinishArgs a, const __grid_constant__ harl_step_buffers io,
              const __grid_constant__ harl_replay_ring ring,
              const __grid_constant__ harl_entry_log log,
              const __grid_constant__ harl_track_stats ts,
              const int64_t* wpos_dev) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  const int64_t r0 = (int64_t)blockIdx.x * FIN_ROWS;
  const int64_t wpos = wpos_dev ? *wpos_dev : a.wpos;
  if (threadIdx.x < FIN_ROWS && r0 + threadIdx.x < a.n)
    finish_row(a, io, ring, log, ts, wpos, r0 + threadIdx.x);
  if (!a.rl) return;
  const int64_t lo = r0 > a.keep_from ? r0 : a.keep_from;
  const int64_t hi = r0 + FIN_ROWS < a.n ? r0 + FIN_ROWS : a.n;
  if (lo >= hi) return;
  const int F = a.F;
  const int total = (int)(hi - lo) * F;
  const double* sx = io.feat + lo * F;
  const double* sxn = io.feat_new + lo * F;
  constexpr int U = 8;
  for (int e0 = threadIdx.x; e0 < total; e0 += FIN_THREADS * U) {
    double vx[U], vxn[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * FIN_THREADS;
      vx[u] = e < total ? sx[e] : 0.0;
      vxn[u] = e < total ? sxn[e] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * FIN_THREADS;
      if (e < total) {
        const int rr = e / F, k = e - rr * F;
        const int64_t slot = (wpos + lo + rr) % ring.cap;
        ring.X[slot * F + k] = vx[u];
        ring.Xn[slot * F + k] = vxn[u];
      }
    }
  }
}

// GBT predict + reward + the finish bookkeeping in one persistent kernel
// (the value pass runs first, so v_cur/v_next are ready): after a tile's
// scores are written, group 1's 64 threads run finish_row for its rows and
// groups 2-7 copy the pushed rows' X / X' into their replay slots.
struct GbtFinishArgs {
  FinishArgs a;
  harl_step_buffers io;
  harl_replay_ring ring;
  harl_entry_log log;
  harl_track_stats ts;
  const int64_t* wpos_dev;
};

struct GbtFinishEpilogue {
  const GbtFinishArgs& f;
  __device__ void operator()(int64_t r0, int rows, int g, int rl) const {
    const int64_t wpos = f.wpos_dev ? *f.wpos_dev : f.a.wpos;
    if (g == 1) {
      if (rl < rows) finish_row(f.a, f.io, f.ring, f.log, f.ts, wpos, r0 + rl);
      return;
    }
    if (g < 2 || !f.a.rl) return;
    const int64_t lo = r0 > f.a.keep_from ? r0 : f.a.keep_from;
    const int64_t hi = r0 + rows;
    if (lo >= hi) return;
    const int F = f.a.F;
    const int total = (int)(hi - lo) * F;
    const double* sx = f.io.feat + lo * F;
    const double* sxn = f.io.feat_new + lo * F;
    const int nthr = (GBT2_GROUPS - 2) * GBT2_ROWS;
    const int tid = threadIdx.x - 2 * GBT2_ROWS;
    for (int e = tid; e < total; e += nthr) {
      const int rr = e / F, k = e - rr * F;
      const int64_t slot = (wpos + lo + rr) % f.ring.cap;
      f.ring.X[slot * F + k] = sx[e];
      f.ring.Xn[slot * F + k] = sxn[e];
    }
  }
};

template <bool SMEM_NODES>
__global__ void __launch_bounds__(GBT2_THREADS)
k_gbt_finish(const GbtNode* __restrict__ gnodes,
             const int32_t* __restrict__ tree_first, int32_t n_trees,
             int64_t n_nodes, int32_t fitted, double base, double floor_value,
             const double* __restrict__ feat, int64_t n, int32_t F,
             double* score, const double* old_score, double* reward,
             const GbtHdr* hdr, int32_t t_cap,
             const __grid_constant__ GbtFinishArgs fa) {
  // (gbt2_body waits for the predecessor after its forest prologue; the
  // epilogue reads the write position after that)
  const GbtFinishEpilogue epi{fa};
  gbt2_body<SMEM_NODES>(gnodes, tree_first, n_trees, n_nodes, fitted, base,
                        floor_value, feat, n, F, score, old_score, reward, hdr,
                        t_cap, epi);
}

// replay feature rows (X, X') of the surviving pushes: one warp per row,
// lanes over features (coalesced), 32-bit index math
__global__ void __launch_bounds__(256)
k_ring_rows(int64_t n, int64_t keep_from, int32_t F, int64_t wpos_arg,
            const int64_t* wpos_dev, const double* __restrict__ feat,
            const double* __restrict__ feat_new,
            const __grid_constant__ harl_replay_ring ring) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  const int lane = threadIdx.x & 31;
  const int64_t wpos = wpos_dev ? *wpos_dev : wpos_arg;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = keep_from + (int64_t)blockIdx.x * (blockDim.x >> 5) +
                   (threadIdx.x >> 5);
       r < n; r += warps) {
    const int64_t slot = (wpos + r) % ring.cap;
    const double* x = feat + r * F;
    const double* xn = feat_new + r * F;
    double* dx = ring.X + slot * F;
    double* dxn = ring.Xn + slot * F;
    for (int k = lane; k < F; k += 32) {
      dx[k] = x[k];
      dxn[k] = xn[k];
    }
  }
}

// Survivor compaction: dst row i <- src row idx[i] for the population state
struct GatherArgs {
  int64_t n_out, ld_src, ld_dst;
  int32_t local_slots, F;
};

__global__ void k_gather_rows(GatherArgs a, const int32_t* idx,
                              const uint16_t* tiles, const uint8_t* knobs,
                              const double* feat, const double* score,
                              const int32_t* row_track, uint16_t* tiles_o,
                              uint8_t* knobs_o, double* feat_o, double* score_o,
                              int32_t* row_track_o) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  // one thread per copied element (not per row: a row's ~80 dependent
  // load/store pairs had serialised on their round trips), elements
  // ordered so consecutive threads write consecutive addresses
  const int64_t n = a.n_out;
  const int S = a.local_slots, F = a.F;
  const int64_t n_st = n * (S + 3), n_f = n * F, n_sc = 2 * n;
  const int64_t total = n_st + n_f + n_sc;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (e < n_st) {                       // state: slot-major, row fastest
      const int64_t s = e / n, i = e - s * n;
      const int64_t r = __ldg(idx + i);
      if (s < S) tiles_o[s * a.ld_dst + i] = tiles[s * a.ld_src + r];
      else knobs_o[(s - S) * a.ld_dst + i] = knobs[(s - S) * a.ld_src + r];
    } else if (e < n_st + n_f) {          // features: row-major
      const int64_t f = e - n_st, i = f / F, k = f - i * F;
      const int64_t r = __ldg(idx + i);
      feat_o[f] = feat[r * F + k];
    } else {
      const int64_t f = e - n_st - n_f;
      const int64_t i = f < n ? f : f - n;
      const int64_t r = __ldg(idx + i);
      if (f < n) score_o[i] = score[r];
      else row_track_o[i] = row_track[r];
    }
  }
}

}  // namespace harl
