/*
 * harl_b200.h — C ABI of the B200-native HARL inner search step.
 *
 * The reference (arXiv 2211.11172 "schedtune", pure Python/numpy) has no
 * native boundary; the functions below are exactly what its Python API for
 * this path would bind through ctypes.  Each entry
 * names the reference function it replaces (paths relative to
 * /root/reference/pkg/src/schedtune).
 *
 * Conventions
 *   - Plain C types only; every array argument is a DEVICE pointer unless
 *     the parameter name ends in `_host`.  `stream` is a cudaStream_t passed
 *     as void*.  The library never allocates or frees caller memory; scratch
 *     space is passed in by the caller.
 *   - Return 0 on success, a negative HARL_E* code otherwise; the message is
 *     available from harl_last_error().  Per-candidate failures that the
 *     reference reports as Python exceptions (InvalidActionError with its
 *     subspace, RlDivergedError) come back through an int32 status array
 *     written on device (see HARL_ST_*), and the Python layer raises the same
 *     exception types.
 *   - Population arrays are structure-of-arrays: tiles are uint16
 *     [slot][ld] (slot-major, leading dimension `ld` >= n), knobs are uint8
 *     [3][ld] (compute-at index, parallel fuse count, unroll index),
 *     features are float64 row-major [n][F].
 */
#ifndef HARL_B200_H
#define HARL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HARL_ABI_VERSION 1

#define HARL_MAX_DIMS 16
#define HARL_MAX_LEVELS 8
#define HARL_MAX_SLOTS 64
#define HARL_MAX_STAGES 16
#define HARL_MAX_TENSORS 48
#define HARL_MAX_TERMS 160
#define HARL_MAX_HEAD0 512   /* compact tiling-head columns, S*(L-1)+1 */
#define HARL_MAX_LAYERS 4
#define HARL_MAX_HIDDEN 256
#define HARL_MAX_FEATURES 128

/* error codes */
#define HARL_OK 0
#define HARL_E_ARG (-1)
#define HARL_E_CUDA (-2)
#define HARL_E_LIMIT (-3)

/* per-candidate status (first failing row wins, like the reference's
 * sequential loop); code values */
#define HARL_ST_OK 0
#define HARL_ST_TILING 1        /* InvalidActionError("tiling", ...) */
#define HARL_ST_COMPUTE_AT 2    /* InvalidActionError("compute_at", ...) */
#define HARL_ST_PARALLEL 3      /* InvalidActionError("parallel", ...) */
#define HARL_ST_UNROLL 4        /* InvalidActionError("unroll", ...) */
#define HARL_ST_NO_VALID 5      /* RlDivergedError: all-masked row */
#define HARL_ST_NONFINITE 6     /* RlDivergedError: non-finite loss/grad */

/* Per-sketch constant tables.  Mirrors SketchContext.__init__
 * (schedspace.py:324-368) plus the sampler/lookup tables; built on the
 * host by paper_2211_11172_b200.space.SketchTables. */
typedef struct harl_sketch_desc {
  int32_t levels, ndims, local_slots, num_slots;
  int32_t ncas, max_fusible, n_unroll, max_feature_dims, feature_len;
  int32_t n_stages, n_tensors, n_terms, max_extent, n_head0;
  int32_t extents[HARL_MAX_DIMS];
  int32_t tiling_counts[HARL_MAX_DIMS];
  int32_t tiling_offsets[HARL_MAX_DIMS];
  int16_t term_gi[HARL_MAX_TERMS], term_sc[HARL_MAX_TERMS],
      term_off[HARL_MAX_TERMS];
  int16_t tensor_first[HARL_MAX_TENSORS], tensor_nterms[HARL_MAX_TENSORS];
  int16_t stage_first[HARL_MAX_STAGES], stage_ntensors[HARL_MAX_STAGES],
      stage_inter[HARL_MAX_STAGES], stage_extra[HARL_MAX_STAGES];
  int16_t head0_src[HARL_MAX_HEAD0], head0_dst[HARL_MAX_HEAD0];
  double flops_feature; /* log10(max(flops,1))/12, host libm */
  const double* log2_lut;       /* device [max_extent+1]: log2(v)/10 */
  const uint16_t* spf_lut;      /* device [max_extent+1] */
  const uint16_t* tiling_table; /* device [sum tiling_counts][levels] */
  /* optional device copy of this descriptor (NULL: none).  Kernels that
   * stage the per-column / per-term tables into shared memory read them
   * from it with coalesced global loads instead of thread-divergent
   * kernel-parameter (constant bank) reads, which serialise per address. */
  const struct harl_sketch_desc* dev_self;
} harl_sketch_desc;

/* numpy PCG64 bit-generator state (Generator.bit_generator.state). */
typedef struct harl_pcg64 {
  uint64_t state_hi, state_lo, inc_hi, inc_lo;
  int32_t has_uint32;
  uint32_t uinteger;
} harl_pcg64;

/* Fully connected tanh network in fp32 for the rollout (fp64 master params
 * live elsewhere).  Layer i maps dims[i] -> dims[i+1]; W row-major
 * [dims[i]][dims[i+1]].  Policy: trunk layers (all tanh, rlcore.py:95-103
 * plus the trunk tanh of rlcore.py:139) then four linear heads packed into
 * one matrix [hidden][n_head0 + 9] whose first n_head0 columns are the
 * compact tiling-head columns.  Value: hidden layers tanh, last linear to 1.*/
typedef struct harl_mlp_desc {
  int32_t n_layers;
  int32_t dims[HARL_MAX_LAYERS + 1];
  const float* W[HARL_MAX_LAYERS];
  const float* b[HARL_MAX_LAYERS];
  const float* head_W; /* policy only: [dims[n_layers]][n_head_cols] */
  const float* head_b;
  int32_t n_head_cols;
} harl_mlp_desc;

/* GBT ensemble (costmodel.py:59-78,219-230).  Nodes of all trees are
 * concatenated 16-byte records {double v; int16 feature, left, right, pad}
 * where v is the split threshold of an internal node (feature >= 0) or
 * learning_rate * value of a leaf (feature == -1; the reference's product,
 * computed on the host); children are tree-local indices. */
typedef struct harl_forest_desc {
  int32_t n_trees, fitted;
  double base, floor_value;
  const int32_t* tree_first;  /* [n_trees] first node of each tree */
  const void* nodes;          /* [n_nodes] records */
  int64_t n_nodes;
  /* Optional device header {int32 n_trees, int32 fitted, double base,
   * double floor_value, int64 n_nodes} read by the kernels at run time.
   * When set, the host fields above are CAPACITIES (shared-memory sizing
   * only), so a refitted ensemble can be loaded into the same buffers
   * without re-recording captured launches. */
  const void* dev_hdr;
} harl_forest_desc;

/* The analytic measurement model of one sketch (SimHwParams + the
 * SketchContext stage data the simulator reads, measure.py:41-122).
 * Anchor stages in the sketch descriptor's stage order. */
typedef struct harl_sim_desc {
  int32_t cores, n_skipped;
  double cap_l1, cap_l2, miss_l1, miss_l2, par_overhead, peak_flops;
  double unroll_factor[HARL_MAX_LEVELS];   /* per unroll index */
  double stage_flops[HARL_MAX_STAGES];
  int32_t stage_spatial_n[HARL_MAX_STAGES];
  int16_t stage_spatial[HARL_MAX_STAGES][HARL_MAX_DIMS];
  double skipped_flops[HARL_MAX_STAGES], skipped_l1[HARL_MAX_STAGES],
      skipped_l2[HARL_MAX_STAGES];
} harl_sim_desc;

int harl_abi_version(void);
/* One-time setup (kernel shared-memory limits, device queries) so that the
 * step entry points can be recorded into CUDA graphs. */
int harl_prepare(void);
const char* harl_last_error(void);
int harl_device_query(int device, int* sm_count_host, int* cc_major_host,
                      int* cc_minor_host);

/* sample_initial_schedules (schedspace.py:165-178): numpy Generator
 * .integers semantics (Lemire on 32-bit halves, buffered high half),
 * track-major.  Exact including rejection draws (repaired sequentially).
 * Writes the number of 32-bit words consumed to *u32_used_host.
 * scratch: >= 16 bytes device. */
/* Build (once per stream increment) the device jump table the samplers use
 * for numpy's PCG64 stream; call before capturing a graph that samples from
 * this generator (during capture a missing table falls back to the slower
 * bitwise jump -- same draws). */
int harl_rng_prepare(const harl_pcg64* rng);

int harl_init_population(const harl_sketch_desc* sk, const harl_pcg64* rng,
                         int64_t count, uint16_t* tiles, uint8_t* knobs,
                         int64_t ld, int64_t* u32_used_host, void* scratch,
                         void* stream);

/* TuningSession._uniform_actions (tuner.py:341-348) for the non-RL
 * searchers: head-major Generator.integers(len(valid)) per row (no draw when
 * one choice is valid), exact including rejections.  actions: int32 [4][n]
 * full head indices.  scratch >= harl_uniform_scratch_bytes(n). */
int64_t harl_uniform_scratch_bytes(int64_t n);
int harl_uniform_actions(const harl_sketch_desc* sk, const uint16_t* tiles,
                         const uint8_t* knobs, int64_t n, int64_t ld,
                         const harl_pcg64* rng, int32_t* actions,
                         void* scratch, int64_t* u32_used_host, void* stream);

/* SketchContext.featurize (schedspace.py:415-438) incl. exact footprints
 * (372-411) and glibc-2.39-faithful log10. feat: [n][feature_len]. */
int harl_featurize(const harl_sketch_desc* sk, const uint16_t* tiles,
                   const uint8_t* knobs, int64_t n, int64_t ld, double* feat,
                   void* stream);

/* action_mask (schedspace.py:226-262), materialized: tiling [n][S*S+1]
 * and shift [n][9] (compute-at, parallel, unroll triples) as uint8. */
int harl_action_masks(const harl_sketch_desc* sk, const uint16_t* tiles,
                      const uint8_t* knobs, int64_t n, int64_t ld,
                      uint8_t* tiling, uint8_t* shift, void* stream);

/* decode_action + apply_action (schedspace.py:196-210,265-301) for
 * injected actions int32 [4][n] (head-major).  *status (caller-initialised
 * to UINT64_MAX) receives row*16 + HARL_ST_* of the first failing row. */
int harl_apply_actions(const harl_sketch_desc* sk, const uint16_t* tiles,
                       const uint8_t* knobs, int64_t n, int64_t ld,
                       const int32_t* actions, uint16_t* tiles_out,
                       uint8_t* knobs_out, uint64_t* status, void* stream);

/* SurrogateModel.predict (costmodel.py:219-230), fp64 bit-exact; if
 * old_score != NULL also reward = (new-old)/old (tuner.py:389-391). */
int harl_gbt_predict(const harl_forest_desc* forest, const double* feat,
                     int64_t n, int32_t feature_len, double* score,
                     const double* old_score, double* reward, void* stream);

/* select_actions (rlcore.py:216-228) fused with the walker: policy MLP
 * (fp32), masked log-softmax, inverse-CDF sampling on the PCG64 stream
 * (uniform for head h, row r = double #(h*n + r) after `rng`), then
 * decode+apply (schedspace.py:196-301).  Outputs: actions int32 [4][n]
 * (full head indices), logp float64 [n], new state, mask bits per row
 * (uint64 movable-slot bits, uint32 shift-mask bits) for the replay
 * buffer, the compact tiling-head column taken (head0_col, int32 [n]),
 * optional logits float32 [n][n_head_cols] (NULL to skip).  *status as in
 * harl_apply_actions (HARL_ST_NO_VALID for an all-masked row).
 * If `inject` != NULL the actions are taken from it (int32 [4][n]) and the
 * uniforms are not used (parity replay of oracle actions).  Population
 * shards: grow (optional device int32 [n]) is each local row's global row
 * and m_total the step's global row count; the uniform of head h is then
 * draw #(h*m_total + grow[r] + 1) (NULL/0: local rows, m_total = n). */
int harl_policy_step(const harl_sketch_desc* sk, const harl_mlp_desc* pol,
                     const double* feat, const uint16_t* tiles,
                     const uint8_t* knobs, int64_t n, int64_t ld,
                     const harl_pcg64* rng, const int32_t* inject,
                     int32_t* actions, double* logp, uint16_t* tiles_out,
                     uint8_t* knobs_out, uint64_t* move_bits,
                     uint32_t* shift_bits, int32_t* head0_col,
                     float* logits_out, uint64_t* status,
                     const int32_t* grow, int64_t m_total, void* stream);

/* select_actions + walker as harl_policy_step, on the tcgen05 path when
 * the policy is the production shape (hidden (128,128), feature_len <= 64,
 * n_head0 + 9 <= 128): trunk and heads as 3xTF32 tcgen05 MMAs with TMEM
 * accumulators and TMEM-resident activations.  hid_scratch: float32
 * [n][128] device scratch.  rng_state_dev (optional, device {hi, lo}
 * u64 PCG64 state) overrides rng's state at execution time so the call can
 * be replayed from a CUDA graph (rng still supplies the increment).
 * feat_out (optional, f64 [n][F]): also featurize the new states
 * (schedspace.py:415-438) -- with the packed weight images this is one
 * fused kernel (policy -> sample/apply -> featurize per 128-row tile, the
 * logits never leave the SM); otherwise a separate featurize launch.  Not
 * a fallback: returns HARL_E_ARG if the shape is not eligible (the caller
 * then uses harl_policy_step).  flags: HARL_STEP_FUSED (the one fused
 * 3xTF32 kernel), HARL_WEIGHTS_SETTLED (no launch since the one before the
 * previous launch on the stream wrote the weight images: with HARL_PDL=1 the
 * kernel may load them before its programmatic-dependency wait). */
#define HARL_STEP_FUSED 1
#define HARL_WEIGHTS_SETTLED 2
/* split launches on the 3xFP16 path (HARL_E_LIMIT, nothing launched,
 * elsewhere): MLP_ONLY runs the policy network into hid_scratch and
 * returns (rng may be NULL); SAMPLE_ONLY runs the sampler on the logits a
 * previous MLP_ONLY call left in hid_scratch for the same rows.  The engine
 * uses them to run the next step's policy network beside this step's value
 * and GBT passes. */
#define HARL_STEP_MLP_ONLY 4
#define HARL_STEP_SAMPLE_ONLY 8
/* harl_value_pair_tc with n0 == n1: each CTA takes the X and X' tiles of
 * the same rows as its two in-flight tiles (half the CTAs of the default
 * tile order), leaving SMs to a concurrent launch */
#define HARL_VALUE_PAIRED 16
int harl_policy_step_tc(const harl_sketch_desc* sk, const harl_mlp_desc* pol,
                        const double* feat, const uint16_t* tiles,
                        const uint8_t* knobs, int64_t n, int64_t ld,
                        const harl_pcg64* rng, const int32_t* inject,
                        int32_t* actions, double* logp, uint16_t* tiles_out,
                        uint8_t* knobs_out, uint64_t* move_bits,
                        uint32_t* shift_bits, int32_t* head0_col,
                        float* logits_out, uint64_t* status,
                        float* hid_scratch, const uint64_t* rng_state_dev,
                        const void* packed_trunk, const void* packed_heads,
                        const int32_t* grow, int64_t m_total, double* feat_out,
                        int32_t flags, void* stream);

/* harl_policy_step_tc with SurrogateModel.predict + the reward
 * (costmodel.py:219-230, tuner.py:389-391) fused into the sampler: the
 * successor rows it featurizes into feat_out are scored by `forest` (a
 * reloadable forest: dev_hdr set, host fields are capacities, at most 64
 * trees) into score[n], and reward[n] = (score - old_score) / old_score
 * (old_score NULL: no reward).  Bit-identical to harl_gbt_predict /
 * harl_gbt_finish_step on the same rows.  Returns HARL_E_LIMIT, launching
 * nothing, when the step is not eligible (not the 3xFP16 path, more rows
 * than the in-sampler featurize takes, forest capacity or shared memory):
 * the caller then scores with harl_gbt_finish_step. */
int harl_policy_step_tc_gbt(const harl_sketch_desc* sk, const harl_mlp_desc* pol,
                            const double* feat, const uint16_t* tiles,
                            const uint8_t* knobs, int64_t n, int64_t ld,
                            const harl_pcg64* rng, const int32_t* inject,
                            int32_t* actions, double* logp, uint16_t* tiles_out,
                            uint8_t* knobs_out, uint64_t* move_bits,
                            uint32_t* shift_bits, int32_t* head0_col,
                            float* logits_out, uint64_t* status,
                            float* hid_scratch, const uint64_t* rng_state_dev,
                            const void* packed_trunk, const void* packed_heads,
                            const int32_t* grow, int64_t m_total, double* feat_out,
                            int32_t flags, const harl_forest_desc* forest,
                            const double* old_score, double* score, double* reward,
                            void* stream);

/* V(X) and V(X') in one launch (tuner.py:395-396) on the tcgen05 path
 * (hidden (128,128), feature_len <= 64); HARL_E_ARG if not eligible. */
int harl_value_pair_tc(const harl_mlp_desc* val, const double* feat0,
                       int64_t n0, const double* feat1, int64_t n1,
                       int32_t feature_len, float* v0, float* v1,
                       const void* packed, int32_t flags, void* stream);

/* Pre-pack the tcgen05 weight images (tf32 hi/lo in the UMMA K-major
 * layout + biases) after every parameter change; the tcgen05 entry points
 * then bulk-copy them (cp.async.bulk) instead of re-splitting the weights
 * in every CTA.  which: 0 = trunk image, 1 = heads image. */
int64_t harl_tc_packed_bytes(int32_t which, int32_t n_head_cols);
int harl_pack_tc_weights(const harl_mlp_desc* pol, const harl_mlp_desc* val,
                         int32_t feature_len, void* pol_trunk,
                         void* pol_heads, void* val_trunk, void* stream);

/* ValueNet.estimate (rlcore.py:173) on feat (fp64 rows, fp32 math). */
int harl_value_forward(const harl_mlp_desc* val, const double* feat,
                       int64_t n, int32_t feature_len, float* v_out,
                       void* stream);


/* ------------------------------------------------------------------------
 * Episode-level pieces of TuningSession._run_episode (tuner.py:350-440). */

/* Replay FIFO (rlcore.py:253-265) as a device ring of `cap` slots.  Head-0
 * actions are stored as compact tiling-head columns; masks as movable-slot
 * bits + shift bits (ActionMask is a pure function of the state). */
typedef struct harl_replay_ring {
  double* X;            /* [cap][F]  features */
  double* Xn;           /* [cap][F]  next features */
  int32_t* actions;     /* [cap][4] */
  double* scalars;      /* [cap][4]  logp, reward, advantage, td target */
  uint64_t* move_bits;  /* [cap] */
  uint32_t* shift_bits; /* [cap] */
  int64_t cap;
} harl_replay_ring;

/* Visited-candidate log (CandidateEntry, tuner.py:406-412), SoA by visit. */
typedef struct harl_entry_log {
  uint16_t* tiles;  /* [slot][ld] */
  uint8_t* knobs;   /* [3][ld] */
  double* score;    /* [ld] */
  double* reward;   /* [ld] */
  int32_t* track;   /* [ld] */
  int64_t ld;
} harl_entry_log;

/* Track.advance state (stopping.py:31-53) indexed by track id. */
typedef struct harl_track_stats {
  int32_t* steps;
  double* best_score;
  int32_t* best_step;
} harl_track_stats;

/* One step's device arrays (n rows, row r = live track row_track[r]). */
typedef struct harl_step_buffers {
  const int32_t* row_track;
  const uint16_t* tiles_new;
  const uint8_t* knobs_new;
  const double* feat;       /* X  [n][F] */
  const double* feat_new;   /* X' [n][F] */
  const double* new_score;
  const double* reward;
  const float* v_cur;
  const float* v_next;
  const int32_t* actions;   /* [4][n] full head indices */
  const int32_t* head0_col; /* [n] compact column */
  const double* logp;
  const uint64_t* move_bits;
  const uint32_t* shift_bits;
  double* adv;              /* out [n] */
} harl_step_buffers;

/* advantage + TD target (rlcore.py:231-234, tuner.py:395-398), replay push
 * of rows >= keep_from into slots (wpos + r) % cap, entry log at visit
 * vbase + r, Track.advance.  rl == 0 skips value/advantage/replay.
 * wpos_dev (optional device int64) overrides wpos at execution time. */
int harl_finish_step(const harl_step_buffers* io, int64_t n, int64_t ld,
                     int64_t vbase, int32_t local_slots, int32_t feature_len,
                     double discount, int32_t rl, const harl_replay_ring* ring,
                     int64_t wpos, int64_t keep_from, const harl_entry_log* log,
                     const harl_track_stats* ts, const int64_t* wpos_dev,
                     void* stream);

/* harl_value_pair_tc with the step's finish (harl_finish_step: advantage /
 * TD, replay push incl. the X / X' rows, entry log, Track.advance;
 * tuner.py:393-412) run in the value kernel's epilogue for the X' rows:
 * n1 = the step's rows, n0 = n1 (V(X) computed here, each CTA taking the X
 * and X' tiles of the same rows) or 0 (V(X) already in v0 from the
 * previous step).  io->feat / feat_new / v_cur / v_next must be feat0 /
 * feat1 / v0 / v1.  Bit-identical to harl_value_pair_tc followed by
 * harl_finish_step.  HARL_E_LIMIT (nothing launched) when the step is not
 * on the 3xFP16 path: the caller runs the two calls then. */
int harl_value_finish_tc(const harl_mlp_desc* val, const double* feat0,
                         int64_t n0, const double* feat1, int64_t n1,
                         int32_t feature_len, float* v0, float* v1,
                         const void* packed, int32_t flags,
                         const harl_step_buffers* io, int64_t ld, int64_t vbase,
                         int32_t local_slots, double discount, int32_t rl,
                         const harl_replay_ring* ring, int64_t wpos,
                         int64_t keep_from, const harl_entry_log* log,
                         const harl_track_stats* ts, const int64_t* wpos_dev,
                         void* stream);

/* Survivor compaction after a host cull (stopping.py:68-86): row i of the
 * destination population <- row idx[i] of the source. */
/* harl_gbt_predict + harl_finish_step as one persistent kernel: the GBT
 * scores of X' = io->feat_new are written to io->new_score, the rewards
 * against old_score to io->reward, then each tile's rows get the finish
 * bookkeeping (advantage needs io->v_cur / io->v_next: run the value pass
 * first).  HARL_E_LIMIT when the forest does not fit in shared memory (use
 * the two calls then). */
int harl_gbt_finish_step(const harl_forest_desc* forest, int32_t feature_len,
                         const double* old_score, const harl_step_buffers* io,
                         int64_t n, int64_t ld, int64_t vbase,
                         int32_t local_slots, double discount, int32_t rl,
                         const harl_replay_ring* ring, int64_t wpos,
                         int64_t keep_from, const harl_entry_log* log,
                         const harl_track_stats* ts, const int64_t* wpos_dev,
                         void* stream);
int harl_gather_rows(const int32_t* idx, int64_t n_out, int32_t local_slots,
                     int32_t feature_len, const uint16_t* tiles,
                     const uint8_t* knobs, const double* feat,
                     const double* score, const int32_t* row_track,
                     int64_t ld_src, uint16_t* tiles_o, uint8_t* knobs_o,
                     double* feat_o, double* score_o, int32_t* row_track_o,
                     int64_t ld_dst, void* stream);

/* Flat parameter layout of one network inside the fp64 master buffer (the
 * same offsets index the fp32 rollout copy, Adam m/v and the gradient),
 * plus per-row scratch offsets used by the PPO kernels. */
typedef struct harl_net_layout {
  int32_t n_layers;
  int32_t dims[HARL_MAX_LAYERS + 1];
  int64_t off_W[HARL_MAX_LAYERS], off_b[HARL_MAX_LAYERS];
  int64_t off_hW, off_hb; /* policy heads, packed [H][n_head_cols] */
  int32_t n_head_cols;
  int32_t row_act[HARL_MAX_LAYERS + 1];
  int32_t row_delta[HARL_MAX_LAYERS];
  int32_t row_head;
} harl_net_layout;

typedef struct harl_ppo_hyper {
  double clip_ratio, entropy_weight, value_loss_weight;
  double lr_actor, lr_critic;
  double b1t_pi, b2t_pi, b1t_v, b2t_v; /* 1 - beta^t per optimizer */
  double beta1, beta2, one_m_beta1, one_m_beta2, eps;
} harl_ppo_hyper;

/* ppo_update (rlcore.py:361-378) on B replay slots `idx` (device int32):
 * fp64 forward/backward of both nets, fixed-order reductions, finite
 * checks, Adam (rlcore.py:62-71) on params[0, n_pi) (policy) and
 * [n_pi, n_params) (value), fp32 copy refresh.  losses (device double[16]):
 * actor loss, value loss, policy loss, entropy, mean ratio.  *bad (device
 * int32, caller zeroes) != 0 when a loss or gradient was not finite, in
 * which case no parameter changed (RlDivergedError). scratch >=
 * harl_ppo_scratch_bytes(). head0_src: compact column -> source slot.
 * adam_dev (optional device double[4]: 1-b1^t, 1-b2^t for policy then
 * value) overrides hp's bias corrections at execution time (graph
 * replay).  No host<->device copies: legal inside stream capture.
 * *_img (optional, from harl_pack_tc_weights): the Adam pass also
 * refreshes these tcgen05 weight images in place.
 * Sharded updates (population split over ranks): B = this rank's rows of
 * the minibatch, B_norm = the global minibatch size; phase 1 computes this
 * rank's gradient and loss partial sums (grads, losses[5..8]); the caller
 * sum-all-reduces both; phase 2 finalises the losses, checks finiteness and
 * applies Adam.  phase 3 = both (single device). */
int64_t harl_ppo_scratch_bytes(int32_t B, int32_t row_stride,
                               int32_t n_jobs);
/* phase flag: gradients and Adam in one launch without a grid barrier --
 * each gradient tile's CTA steps its own parameters after saving their
 * pre-update values; params, adam_m, adam_v must be rows 0-2 of one
 * [6][n_params] block whose rows 3-5 receive that backup.  bad[0] is
 * flagged as before and bad[1] must be writable (a per-update snapshot);
 * when the update flags bad the caller restores rows 0-2 from rows 3-5
 * (and the derived copies) before raising, as ppo_update steps nothing
 * then (rlcore.py:368-375).  Single device (phase 3) only. */
#define HARL_PPO_SPECULATIVE 8
int harl_ppo_update(const harl_net_layout* pol, const harl_net_layout* val,
                    const harl_ppo_hyper* hp, const harl_replay_ring* ring,
                    const int32_t* idx, int32_t B, int32_t feature_len,
                    int32_t n_head0, const int16_t* head0_src_host,
                    int32_t row_stride, double* params, double* grads,
                    double* adam_m, double* adam_v, float* params32,
                    int64_t n_pi, int64_t n_params, double* losses,
                    int32_t* bad, void* scratch, const double* adam_dev,
                    void* pol_trunk_img, void* pol_heads_img,
                    void* val_trunk_img, double* wt_params, int32_t B_norm,
                    int32_t phase, void* stream);

/* fp64 transposed copies of the matrices the PPO backward pass reads
 * (policy heads, policy/value W[l] for l >= 1): size in doubles, and a
 * rebuild from the master parameters (after any host-side upload; the Adam
 * kernel keeps them current afterwards). */
int64_t harl_ppo_wt_doubles(const harl_net_layout* pol,
                            const harl_net_layout* val);
int harl_ppo_wt_fill(const harl_net_layout* pol, const harl_net_layout* val,
                     const double* params, double* wt, void* stream);

/* Diagnostic: one 128x128x64 kind::tf32 tcgen05 MMA (A [128][64], B
 * [64][128] row-major fp32, D [128][128]); mode 0 = A from TMEM, 1 = A
 * from shared memory.  Used by the GPU tests to pin the descriptor
 * layouts the MLP kernels rely on. */
int harl_selftest_tcgen05(const float* A, const float* B, float* D, int mode,
                          void* stream);

/* rank_scores (costmodel.py:266-286) over the entry log: the visits of the
 * top k distinct states by (score desc, visit asc), excluding n_excluded
 * states given SoA ([local_slots][ex_ld] tiles, [3][ex_ld] knobs; the
 * reference's exclude=measured, tuner.py:481-482).  Duplicates collapse to
 * their first visit.  Writes the selected visit indices (unordered, count
 * stats[0]) to out_idx; stats (device int64[4]) = {selected, distinct kept,
 * hash-collision keeps, k'}.  k' = k + collisions: a 64-bit hash collision
 * keeps the colliding visit (exact compares only), so the selection is a
 * superset on which the reference's rank_scores gives its exact answer.
 * out_cap >= k + n_visits is always enough. */
int64_t harl_rank_scratch_bytes(int64_t n_visits, int64_t n_excluded);
int harl_rank_topk(const harl_entry_log* log, int32_t local_slots,
                   int64_t n_visits, const uint16_t* ex_tiles,
                   const uint8_t* ex_knobs, int64_t ex_ld, int64_t n_excluded,
                   int64_t k, void* scratch, int64_t scratch_bytes,
                   int32_t* out_idx, int64_t out_cap, int64_t* stats,
                   void* stream);

/* GBT refit: SurrogateModel.fit_incremental + _fit_tree (costmodel.py:
 * 81-141, 190-212) on the device, bit-exact with the reference.  X [n][F]
 * and y [n] (renormalised targets) on the device; n <= 16384, max_depth <=
 * 12.  Trees come back in heap layout, K = 2^(max_depth+1) - 1 nodes per
 * tree (children of k: 2k+1, 2k+2): out_feat [n_trees][K] (>= 0 split
 * feature, -1 leaf, -2 no node), out_thr, out_val (the node mean) [n_trees]
 * [K]; out_pred [n] the final training predictions; out_base (device
 * double) y.mean(); out_ntrees (device int32) trees built before the
 * residual early stop.  The host renumbers nodes in the reference's
 * depth-first creation order.  n_dev (optional device int32): the row
 * count read at run time, n then being the capacity (X, y, out_pred and the
 * scratch sized for n) -- one captured graph of the launch sequence serves
 * every training-set size up to n. */
int64_t harl_gbt_fit_scratch_bytes(int32_t n, int32_t feature_len,
                                   int32_t max_depth);
int harl_gbt_fit(const double* X, const double* y, int32_t n,
                 int32_t feature_len, int32_t n_trees, int32_t max_depth,
                 double learning_rate, int32_t min_leaf, void* scratch,
                 int64_t scratch_bytes, int32_t* out_feat, double* out_thr,
                 double* out_val, double* out_pred, double* out_base,
                 int32_t* out_ntrees, const int32_t* n_dev, void* stream);

/* TrackSet.cull (stopping.py:68-86), host-side (no device pointers): the
 * n_elim live tracks with the lowest (advantage, -index) are eliminated
 * (NaN advantages order last).  adv/tracks: the cull step's m rows; alive:
 * per-track 0/1, updated; gone_out: eliminated track ids ascending;
 * keep_out/n_keep: surviving rows ascending. */
int harl_cull_select(const double* adv, const int32_t* tracks, int64_t m,
                     uint8_t* alive, int64_t n_tracks, int64_t n_elim,
                     int64_t* gone_out, int32_t* keep_out, int64_t* n_keep);

/* Host-side: Python float repr (float.__repr__, as json.dumps renders
 * floats; NaN / Infinity / -Infinity) of v[0..n) joined by ", " -- the body
 * of json.dumps(list) -- for the trajectory log's per-visit reward lists
 * (tuner.py:414-420).  Returns the bytes written to out, or -(bytes needed)
 * if cap is too small (40 * n suffices).  threads <= 0: all cores. */
long long harl_format_floats(const double* v, long long n, char* out,
                             long long cap, int threads);

/* simulate_time (measure.py:99-112) for n states (SoA, leading dim ld):
 * out[r] = the model's seconds, bit-exact with the reference. */
int harl_sim_time(const harl_sketch_desc* sk, const harl_sim_desc* sim,
                  const uint16_t* tiles, const uint8_t* knobs, int64_t n,
                  int64_t ld, double* out, void* stream);
/* brute_force_best's sweep (measure.py:135-167) over state numbers
 * [x0, x0 + count) (dim 0's tilings slowest, then compute-at, parallel,
 * unroll): best (device u64) = ordered bits of the minimum time; out
 * (device u64) = the state number attaining it with the smallest canonical
 * text (the reference's tie rule).  scratch: scratch_len device u64 (one
 * per CTA of the sweep; >= 148 * 16 uses the full grid). */
int harl_brute_force(const harl_sketch_desc* sk, const harl_sim_desc* sim,
                     uint64_t x0, uint64_t count, unsigned long long* best,
                     unsigned long long* out, unsigned long long* scratch,
                     int64_t scratch_len, void* stream);

/* Host-side: ScheduleState.canonical (schedspace.py:117-120) of n states
 * (tiles [n][slots] u16, `levels` factors per tiled dim; knobs [n][3] u8):
 * "<prefix>|t=a.b;c.d|ca=..|par=..|ur=.." per state, each NUL-terminated,
 * into out.  Returns the bytes written, or -(bytes needed) if cap is too
 * small.  The drop-in's CandidateEntry texts (tuner.py:406-412). */
long long harl_format_canonical(const uint16_t* tiles, const uint8_t* knobs,
                                long long n, int slots, int levels,
                                const char* prefix, long long prefix_len,
                                char* out, long long cap);

/* Host-side: harl_gbt_fit's heap-layout trees (host copies) -> the
 * reference's node numbering (_fit_tree, costmodel.py:86-141), K slots per
 * tree in and out; sizes[t] = nodes of tree t.  0 on success. */
int harl_heap_to_creation_order(const int32_t* feat_h, const double* thr_h,
                                const double* val_h, int K, int n_trees,
                                int64_t* feature, double* threshold,
                                int64_t* left, int64_t* right, double* value,
                                int32_t* sizes);

/* Host-side: a GBT ensemble (the reference's _Tree arrays per tree,
 * costmodel.py:59-78: int64 feature/left/right, f64 threshold/value,
 * concatenated over the trees, sizes[t] nodes each, child indices local to
 * their tree) -> the device layouts DeviceForest uploads: 16-byte node
 * records (inner: the threshold; leaf: learning_rate * value,
 * costmodel.py:224) into nodes_out,
 * each tree's first record into firsts_out and, when the forest depth is in
 * [1, perfect_max], the perfect-tree image (gbt_kernels.cuh) into
 * perfect_out (*perfect_bytes_out its size, 0 if none).  Returns the depth
 * (inner levels of the deepest tree) or -1 (deeper than the reference's
 * 64-step walk), -2 (empty tree / child index outside its tree), -3 (more
 * than 1024 trees or a tree beyond int16 indices), -4 (perfect_cap too
 * small).  Replaces the per-round numpy packing of the forest reload. */
/* Host-side: the agent's numpy arrays <-> the flat fp64 parameter layout
 * (DeviceAgent._views) in one call.  Each op moves rows x ncols doubles:
 * flat[off + r*flat_ld + c] <-> host[r*host_ld + (cols ? cols[c] : c)]
 * (cols: the tiling head's legal columns, else NULL).  to_host = 0 packs
 * the arrays into flat, 1 writes flat back into them, 2 only compares
 * (returns 1 at the first bitwise difference).  0, or -1 for a bad op.  Replaces the per-array numpy copies of DeviceAgent._pack /
 * _unpack_into (rlcore.py:50-160 state, tuner.py:350-440). */
typedef struct harl_copy_op {
  int64_t off, flat_ld;
  void* host;
  int64_t host_ld, rows, ncols;
  const int64_t* cols;
} harl_copy_op;
int harl_agent_copy(const harl_copy_op* ops, int32_t n_ops, double* flat,
                    int32_t to_host);

long long harl_forest_pack(int n_trees, const int64_t* sizes,
                           const int64_t* feature, const double* threshold,
                           const int64_t* left, const int64_t* right,
                           const double* value, double learning_rate,
                           void* nodes_out, int32_t* firsts_out,
                           int perfect_max, void* perfect_out,
                           long long perfect_cap,
                           long long* perfect_bytes_out);

/* Instrumentation (no reference counterpart; the reference has no device).
 * harl_launch_count: kernels this library has launched since load (graph
 * replays excluded -- they do not pass through the library).
 * harl_profile_set(on, spin_ns): while on, every non-captured launch is
 * preceded by a spin kernel of spin_ns ns (<0 keeps the current value) and
 * bracketed by CUDA events on its own stream.  harl_profile_read
 * synchronises the recorded events and writes, per distinct kernel (first
 * appearance order, at most max_kernels), its name (NUL-terminated in
 * name_cap-byte slots), summed milliseconds, launch count and summed work
 * units (the rows each launch processed as the entry point counted them;
 * -1 if any launch of that kernel did not report them); it returns the
 * number of distinct kernels. */
long long harl_launch_count(void);
/* Debug: enable (on=1) phase timestamps (globaltimer ns) written by CTA 0
 * of the wide tcgen05 kernels; copies the first n (<= 64) to out_host. */
int harl_debug_timestamps(int on, unsigned long long* out_host, int n);
int harl_profile_set(int on, long long spin_ns);
int harl_profile_reset(void);
int harl_profile_read(int max_kernels, char* names, int name_cap,
                      double* total_ms, long long* launches,
                      long long* units);

#ifdef __cplusplus
}
#endif
#endif /* HARL_B200_H */
