// C-ABI entry points (include/harl_b200.h).  Single translation unit: all
// kernels are included here so constant-memory tables need no -rdc.
#include <climits>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <utility>
#include <mutex>
#include <string>
#include <vector>
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "gbt_kernels.cuh"
#include "mlp_ffma.cuh"
#include "space_kernels.cuh"
#include "episode_kernels.cuh"
#include "ppo_kernels.cuh"
#include "ppo_cluster.cuh"
#include "tc_probe.cuh"
#include "mlp_tc.cuh"
#include "sample_kernels.cuh"
#include "mlp_tc2.cuh"
#include "mlp_f16.cuh"
#include "rank_kernels.cuh"
#include "gbt_fit_kernels.cuh"
#include "sim_kernels.cuh"

namespace harl {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* where) {
  set_error("%s: %s", where, cudaGetErrorString(e));
  return HARL_E_CUDA;
}

// ---------------------------------------------------------------------------
// launch counter and per-kernel timer.  The timer puts a short spin kernel
// in front of the timed launch so the GPU is still busy when the host
// enqueues (begin event, kernel, end event): the begin timestamp is then the
// kernel's start, not the moment an idle stream saw the event.

__global__ void k_spin(unsigned long long ns) {
  griddep_wait();  // PDL: predecessors complete and visible
  griddep_launch();
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

struct ProfRec {
  const char* name;
  cudaEvent_t e0, e1;
  long long units;   // work units (rows) the launch processed, -1 unknown
};

static std::mutex g_prof_mu;
static bool g_prof_on = false;
static unsigned long long g_spin_ns = 20000;
static std::vector<cudaEvent_t> g_ev_pool;
static std::vector<ProfRec> g_prof_recs;
static size_t g_ev_used = 0;
static thread_local cudaEvent_t t_pending = nullptr;
static thread_local cudaStream_t t_pending_st = nullptr;
static thread_local long long t_units = -1;
static std::atomic<long long> g_launches{0};
static const size_t PROF_MAX_EVENTS = 1 << 16;

static cudaEvent_t prof_event() {
  if (g_ev_used == g_ev_pool.size()) {
    if (g_ev_pool.size() >= PROF_MAX_EVENTS) return nullptr;
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    g_ev_pool.push_back(e);
  }
  return g_ev_pool[g_ev_used++];
}

void prof_begin(cudaStream_t st) {
  t_pending = nullptr;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (!g_prof_on) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess ||
      cs != cudaStreamCaptureStatusNone)
    return;
  cudaEvent_t e = prof_event();
  if (!e) return;
  k_spin<<<1, 32, 0, st>>>(g_spin_ns);
  cudaEventRecord(e, st);
  t_pending = e;
  t_pending_st = st;
}

void prof_units(long long units) { t_units = units; }

void prof_end(const char* where) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const long long units = t_units;
  t_units = -1;
  if (!t_pending) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  cudaEvent_t e1 = prof_event();
  if (e1) {
    cudaEventRecord(e1, t_pending_st);
    g_prof_recs.push_back({where, t_pending, e1, units});
  }
  t_pending = nullptr;
}

// ---------------------------------------------------------------------------
// host-side PCG64 jump tables

typedef unsigned __int128 h128;
static const h128 PCG_MULT =
    ((h128)0x2360ED051FC65DA4ull << 64) | (h128)0x4385DF649FCCF645ull;

static inline u128 to_u128(h128 x) {
  u128 r;
  r.hi = (uint64_t)(x >> 64);
  r.lo = (uint64_t)x;
  return r;
}

static void build_jump(const harl_pcg64& g, PcgJump* J) {
  const h128 inc = ((h128)g.inc_hi << 64) | (h128)g.inc_lo;
  h128 A = PCG_MULT, C = inc;  // one step: s -> A s + C
  for (int i = 0; i < 64; ++i) {
    J->A[i] = to_u128(A);
    J->C[i] = to_u128(C);
    C = A * C + C;  // compose (A,C) with itself
    A = A * A;
  }
}

// byte-sliced jump tables (PcgTab), one per stream increment, built on the
// host and uploaded once; never freed (captured graphs bake the pointer)
static std::mutex g_tab_mu;
static std::vector<std::pair<h128, PcgTab*>> g_tabs;

static h128 to_h128(u128 x) { return ((h128)x.hi << 64) | (h128)x.lo; }

static int build_pcg_tab(const harl_pcg64& g, PcgTab** out) {
  const h128 inc = ((h128)g.inc_hi << 64) | (h128)g.inc_lo;
  std::lock_guard<std::mutex> lk(g_tab_mu);
  for (auto& e : g_tabs)
    if (e.first == inc) {
      *out = e.second;
      return HARL_OK;
    }
  PcgJump J;
  build_jump(g, &J);
  std::vector<PcgTab> host(1);
  PcgTab& T = host[0];
  for (int L = 0; L < 4; ++L) {
    // one step of this level advances 256^L draws: (A, C) = J[8L]
    const h128 A1 = to_h128(J.A[8 * L]), C1 = to_h128(J.C[8 * L]);
    h128 A = 1, C = 0;
    for (int b = 0; b < 256; ++b) {
      T.A[L * 256 + b] = to_u128(A);
      T.C[L * 256 + b] = to_u128(C);
      C = A1 * C + C1;  // compose one more level step after (A, C)
      A = A1 * A;
    }
  }
  PcgTab* dev = nullptr;
  cudaError_t e = cudaMalloc(&dev, sizeof(PcgTab));
  if (e != cudaSuccess) return cuda_status(e, "pcg table alloc");
  e = cudaMemcpy(dev, &T, sizeof(PcgTab), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_status(e, "pcg table upload");
  g_tabs.push_back({inc, dev});
  *out = dev;
  return HARL_OK;
}

// the table of this stream if it exists or can be built now (not while the
// stream is being captured); null -> kernels use the bitwise jump
static const PcgTab* pcg_tab_for(const harl_pcg64* rng, cudaStream_t st) {
  if (!rng) return nullptr;
  const h128 inc = ((h128)rng->inc_hi << 64) | (h128)rng->inc_lo;
  {
    std::lock_guard<std::mutex> lk(g_tab_mu);
    for (auto& e : g_tabs)
      if (e.first == inc) return e.second;
  }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess ||
      cs != cudaStreamCaptureStatusNone)
    return nullptr;
  PcgTab* t = nullptr;
  return build_pcg_tab(*rng, &t) == HARL_OK ? t : nullptr;
}

static inline u128 state_of(const harl_pcg64& g) {
  u128 s;
  s.hi = g.state_hi;
  s.lo = g.state_lo;
  return s;
}

static int sm_count() {
  static int v = 0;
  if (!v) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  }
  return v;
}

// Every library kernel is launched through launch_k: with HARL_PDL=1 the
// launch carries the programmatic-stream-serialization attribute, so the
// next kernel's CTAs are scheduled (and run their pre-wait prologue) while
// the previous grid drains; griddep_wait() inside each kernel keeps the
// data dependency exact.
static bool use_pdl() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HARL_PDL");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

template <typename... KArgs, typename... Args>
static void launch_k_pdl(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block,
                         size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (pdl) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// HARL_PDL_SAMPLE=1: the sampler alone (right behind the policy kernel) is
// launched with PDL, its constant-table staging overlapping the policy
// kernel's drain -- measured no faster at C2 (segments before the cull
// 1.5 % faster, the post-cull segment 1 % slower), off by default
static bool use_pdl_sample() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HARL_PDL_SAMPLE");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

template <typename... KArgs, typename... Args>
static void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (use_pdl()) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// HARL_PPO_TC=1: the DMMA PPO rows kernel (8 rows per CTA) instead of the
// SIMT one (2 rows per CTA, split reductions) -- measured slower at C2
// (41 vs 29 us: 32 CTAs per chain and dependent 32-step MMA chains)
// HARL_PPO_CL=1: the thread-block-cluster rows kernel (ppo_cluster.cuh)
// for the production network shape -- parity-green, but measured slower
// than the SIMT rows kernel at B = 256 (C2 episode 5.42 vs 5.35 ms): its
// column-slice exchanges move 28 KB per CTA through distributed shared
// memory (~21 B/cycle per SM) six times per update, ~1.5 us each
static bool use_ppo_cl() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HARL_PPO_CL");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}
static bool ppo_cl_shape(const harl_net_layout& P, const harl_net_layout& V,
                         int F) {
  return P.n_layers == 2 && P.dims[1] == PCL_H && P.dims[2] == PCL_H &&
         F >= 1 && F <= PCL_KX && P.n_head_cols >= 1 &&
         P.n_head_cols <= PCL_H && V.n_layers == 3 && V.dims[1] == PCL_H &&
         V.dims[2] == PCL_H && V.dims[3] == 1;
}

static bool use_ppo_tc() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HARL_PPO_TC");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// HARL_TC64=0 disables the 64-row-tile tcgen05 kernels
static bool use_tc64() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HARL_TC64");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// HARL_TC_GEN1=1 selects the first-generation 4-warp tcgen05 kernels
// 3xFP16 kernels (mlp_f16.cuh): HARL_TC16=0 falls back to 3xTF32;
// HARL_TC16_MIN_ROWS: launches below this many rows keep the 3xTF32 path
// (read per call: the A/B tests switch it inside one process; launches
// inside captured graphs do not pass through here)
static bool use_tc16(int64_t n) {
  const char* e = getenv("HARL_TC16");
  if (e && e[0] == '0') return false;
  const char* m = getenv("HARL_TC16_MIN_ROWS");
  return !m || n >= atoll(m);
}

// CTAs for a ping-pong f16 launch: every CTA takes tiles in pairs when
// there are more tiles than SMs (HARL_TC16_GRID overrides)
static int tc16_grid(int64_t tiles) {
  static long long forced = -1;
  if (forced < 0) {
    const char* e = getenv("HARL_TC16_GRID");
    forced = e ? atoll(e) : 0;
  }
  int64_t g = tiles < sm_count() ? tiles : sm_count();
  if (forced > 0 && forced < g) g = forced;
  return (int)(g > 0 ? g : 1);
}

static bool use_tc2() {
  static int v = -1;
  if (v < 0) v = getenv("HARL_TC_GEN1") ? 0 : 1;
  return v == 1;
}

static int max_dyn_smem() {
  static int v = -1;
  if (v < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  return v;
}

// Raise a kernel's dynamic shared-memory limit once (not per call, so the
// entry points stay legal inside CUDA-graph stream capture).
template <typename K>
static int allow_smem(K kernel, size_t bytes, const char* name) {
  static std::mutex mu;
  static const void* keys[64];
  static size_t have[64];
  static int nkeys = 0;
  if ((int)bytes > max_dyn_smem()) {
    set_error("%s: needs %zu bytes of shared memory (max %d)", name, bytes,
              max_dyn_smem());
    return HARL_E_LIMIT;
  }
  std::lock_guard<std::mutex> lock(mu);
  int slot = -1;
  for (int i = 0; i < nkeys; ++i)
    if (keys[i] == (const void*)kernel) slot = i;
  if (slot >= 0 && have[slot] >= bytes) return HARL_OK;
  cudaError_t e = cudaFuncSetAttribute(
      kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return cuda_status(e, name);
  if (slot < 0 && nkeys < 64) slot = nkeys++;
  if (slot >= 0) {
    keys[slot] = (const void*)kernel;
    have[slot] = bytes;
  }
  return HARL_OK;
}

template <typename K>
static int allow_max_smem(K kernel, const char* name) {
  cudaFuncAttributes at;
  cudaError_t e = cudaFuncGetAttributes(&at, kernel);
  if (e != cudaSuccess) return cuda_status(e, name);
  return allow_smem(kernel, (size_t)max_dyn_smem() - at.sharedSizeBytes, name);
}

static int check_sketch(const harl_sketch_desc* sk) {
  if (!sk) {
    set_error("null sketch descriptor");
    return HARL_E_ARG;
  }
  if (sk->ndims < 0 || sk->ndims > HARL_MAX_DIMS || sk->levels < 1 ||
      sk->levels > HARL_MAX_LEVELS || sk->num_slots > HARL_MAX_SLOTS ||
      sk->local_slots != sk->ndims * sk->levels ||
      sk->num_slots < sk->local_slots || sk->feature_len > HARL_MAX_FEATURES ||
      sk->n_head0 < 1 || sk->n_head0 > HARL_MAX_HEAD0) {
    set_error("sketch descriptor out of range");
    return HARL_E_ARG;
  }
  return HARL_OK;
}

static int check_mlp(const harl_mlp_desc* m, bool policy) {
  if (!m || m->n_layers < 1 || m->n_layers > HARL_MAX_LAYERS) {
    set_error("bad mlp descriptor");
    return HARL_E_ARG;
  }
  for (int l = 0; l <= m->n_layers; ++l)
    if (m->dims[l] < 1 || m->dims[l] > HARL_MAX_HIDDEN + HARL_MAX_FEATURES) {
      set_error("mlp layer width out of range");
      return HARL_E_ARG;
    }
  if (policy && (m->n_head_cols < 10 || !m->head_W || !m->head_b)) {
    set_error("policy descriptor missing heads");
    return HARL_E_ARG;
  }
  return HARL_OK;
}

}  // namespace harl

using namespace harl;

extern "C" {

int harl_rng_prepare(const harl_pcg64* rng) {
  if (!rng) {
    set_error("harl_rng_prepare: null generator");
    return HARL_E_ARG;
  }
  PcgTab* t = nullptr;
  return build_pcg_tab(*rng, &t);
}


int harl_abi_version(void) { return HARL_ABI_VERSION; }

const char* harl_last_error(void) { return g_err; }

int harl_device_query(int device, int* sm_count, int* cc_major, int* cc_minor) {
  cudaDeviceProp p;
  cudaError_t e = cudaGetDeviceProperties(&p, device);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDeviceProperties");
  if (sm_count) *sm_count = p.multiProcessorCount;
  if (cc_major) *cc_major = p.major;
  if (cc_minor) *cc_minor = p.minor;
  return HARL_OK;
}

int harl_init_population(const harl_sketch_desc* sk, const harl_pcg64* rng,
                         int64_t count, uint16_t* tiles, uint8_t* knobs,
                         int64_t ld, int64_t* u32_used_host, void* scratch,
                         void* stream) {
  int rc = check_sketch(sk);
  if (rc) return rc;
  if (count < 0 || ld < count || !rng || !scratch || !u32_used_host) {
    set_error("harl_init_population: bad arguments");
    return HARL_E_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  PcgJump J;
  build_jump(*rng, &J);
  InitArgs a;
  memset(&a, 0, sizeof(a));
  a.count = count;
  a.ld = ld;
  a.s = state_of(*rng);
  a.has32 = rng->has_uint32;
  a.buffered = rng->uinteger;
  a.nbounds = sk->ndims + 3;
  for (int d = 0; d < sk->ndims; ++d) a.bounds[d] = sk->tiling_counts[d];
  a.bounds[sk->ndims] = sk->ncas;
  a.bounds[sk->ndims + 1] = sk->max_fusible + 1;
  a.bounds[sk->ndims + 2] = sk->n_unroll;
  for (int k = 0; k < a.nbounds; ++k) a.per_track += a.bounds[k] > 1;
  unsigned long long* bad = (unsigned long long*)scratch;
  unsigned long long* used = bad + 1;
  // pinned host words for the two read-backs (a pageable copy stages
  // through a driver buffer)
  static thread_local unsigned long long* hw = nullptr;
  if (!hw) {
    cudaError_t e = cudaHostAlloc((void**)&hw, 16, cudaHostAllocDefault);
    if (e != cudaSuccess) return cuda_status(e, "init pinned words");
  }
  a.t0 = 0;
  a.j0 = 0;
  while (a.t0 < count) {
    cudaError_t e = cudaMemsetAsync(bad, 0xff, 8, st);   // ULLONG_MAX
    if (e != cudaSuccess) return cuda_status(e, "init memset");
    const int64_t todo = count - a.t0;
    // 64-thread CTAs: one track per thread, and every SM gets tracks at
    // 16 K (256-thread CTAs left most SMs idle)
    const int threads = 64;
    HARL_PROF_BEGIN(st);
    launch_k(k_init_sample, dim3((unsigned)((todo + threads - 1) / threads)), dim3(threads), 0, st, 
        *sk, J, a, tiles, knobs, bad);
    HARL_CHECK_LAUNCH("k_init_sample");
    e = cudaMemcpyAsync(hw, bad, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_status(e, "init sync");
    const unsigned long long first = hw[0];
    if (first == ULLONG_MAX) {
      a.j0 += (uint64_t)todo * (uint64_t)a.per_track;
      a.t0 = count;
      break;
    }
    // tracks [t0, first) are exact; redo `first` sequentially
    InitArgs one = a;
    one.j0 = a.j0 + (uint64_t)(first - a.t0) * (uint64_t)a.per_track;
    HARL_PROF_BEGIN(st);
    launch_k(k_init_one, dim3(1), dim3(1), 0, st, *sk, J, one, (int64_t)first, tiles, knobs, used);
    HARL_CHECK_LAUNCH("k_init_one");
    e = cudaMemcpyAsync(hw + 1, used, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_status(e, "init sync");
    const unsigned long long u = hw[1];
    a.j0 = one.j0 + u;
    a.t0 = (int64_t)first + 1;
  }
  *u32_used_host = (int64_t)a.j0;
  return HARL_OK;
}

int64_t harl_uniform_scratch_bytes(int64_t n) {
  return 4 * n * 4 + 4 * n * 8 + 64;
}

int harl_uniform_actions(const harl_sketch_desc* sk, const uint16_t* tiles,
                         const uint8_t* knobs, int64_t n, int64_t ld,
                         const harl_pcg64* rng, int32_t* actions,
                         void* scratch, int64_t* u32_used_host, void* stream) {
  int rc = check_sketch(sk);
  if (rc) return rc;
  if (!rng || !scratch || !u32_used_host || n < 0) {
    set_error("harl_uniform_actions: bad arguments");
    return HARL_E_ARG;
  }
  *u32_used_host = 0;
  if (n == 0) return HARL_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int32_t* count = (int32_t*)scratch;
  int64_t* offset = (int64_t*)((char*)scratch + 4 * n * 4);
  unsigned long long* misc = (unsigned long long*)(offset + 4 * n);
  HARL_PROF_BEGIN(st);
  launch_k(k_uniform_counts, dim3((unsigned)((n + 127) / 128)), dim3(128), 0, st, *sk, tiles, knobs,
                                                                n, ld, count);
  HARL_CHECK_LAUNCH("k_uniform_counts");
  HARL_PROF_BEGIN(st);
  launch_k(k_uniform_scan, dim3(1), dim3(1024), 0, st, count, 4 * n, offset, (int64_t*)&misc[1]);
  HARL_CHECK_LAUNCH("k_uniform_scan");
  PcgJump J;
  build_jump(*rng, &J);
  UniformArgs a;
  memset(&a, 0, sizeof(a));
  a.n = n;
  a.ld = ld;
  a.s = state_of(*rng);
  a.has32 = rng->has_uint32;
  a.buffered = rng->uinteger;
  auto d2h = [&](const void* src, void* dst, size_t bytes) -> cudaError_t {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st);
    return e == cudaSuccess ? cudaStreamSynchronize(st) : e;
  };
  int64_t total_words = 0;
  cudaError_t e = d2h(&misc[1], &total_words, 8);
  if (e != cudaSuccess) return cuda_status(e, "uniform total");
  int64_t i0 = 0;
  uint64_t j0 = 0;  // word index of element i0's draw
  int64_t off_i0 = 0;
  for (;;) {
    const unsigned long long init = ULLONG_MAX;
    e = cudaMemcpyAsync(misc, &init, 8, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_status(e, "uniform memcpy");
    const int64_t todo = 4 * n - i0;
    HARL_PROF_BEGIN(st);
    launch_k(k_uniform_draw, dim3((unsigned)((todo + 127) / 128)), dim3(128), 0, st, 
        *sk, J, a, i0, j0, tiles, knobs, count, offset, actions, misc);
    HARL_CHECK_LAUNCH("k_uniform_draw");
    unsigned long long bad = 0;
    if ((e = d2h(misc, &bad, 8)) != cudaSuccess) return cuda_status(e, "uniform sync");
    if (bad == ULLONG_MAX) {
      *u32_used_host = (int64_t)j0 + (total_words - off_i0);
      return HARL_OK;
    }
    int64_t off_b = 0;
    if ((e = d2h(&offset[bad], &off_b, 8)) != cudaSuccess) return cuda_status(e, "uniform sync");
    const uint64_t jb = j0 + (uint64_t)(off_b - off_i0);
    HARL_PROF_BEGIN(st);
    launch_k(k_uniform_one, dim3(1), dim3(1), 0, st, *sk, J, a, (int64_t)bad, jb, tiles, knobs,
                                   count, actions, &misc[2]);
    HARL_CHECK_LAUNCH("k_uniform_one");
    unsigned long long used = 0;
    if ((e = d2h(&misc[2], &used, 8)) != cudaSuccess) return cuda_status(e, "uniform sync");
    i0 = (int64_t)bad + 1;
    j0 = jb + used;
    if (i0 >= 4 * n) {
      *u32_used_host = (int64_t)j0;
      return HARL_OK;
    }
    if ((e = d2h(&offset[i0], &off_i0, 8)) != cudaSuccess) return cuda_status(e, "uniform sync");
  }
}

int harl_featurize(const harl_sketch_desc* sk, const uint16_t* tiles,
                   const uint8_t* knobs, int64_t n, int64_t ld, double* feat,
                   void* stream) {
  int rc = check_sketch(sk);
  if (rc) return rc;
  if (n <= 0) return HARL_OK;
  const size_t smem2 = feat2_smem_bytes(sk->feature_len, sk->local_slots, sk->max_extent);
  if (smem2 <= (size_t)max_dyn_smem()) {
    if ((rc = allow_smem(k_featurize2, smem2, "k_featurize2"))) return rc;
    HARL_PROF_BEGIN((cudaStream_t)stream);
    launch_k(k_featurize2, dim3((unsigned)((n + FEAT2_ROWS - 1) / FEAT2_ROWS)), dim3(FEAT2_THREADS), smem2, (cudaStream_t)stream, *sk, tiles, knobs, n, ld, feat);
    HARL_PROF_UNITS(n);
    HARL_CHECK_LAUNCH("k_featurize2");
    return HARL_OK;
  }
  const size_t smem = sizeof(double) * FEAT_THREADS * sk->feature_len;
  if ((rc = allow_smem(k_featurize, smem, "k_featurize"))) return rc;
  HARL_PROF_BEGIN((cudaStream_t)stream);
  launch_k(k_featurize, dim3((unsigned)((n + FEAT_THREADS - 1) / FEAT_THREADS)), dim3(FEAT_THREADS), smem, (cudaStream_t)stream, *sk, tiles, knobs, n, ld, feat);
  HARL_PROF_UNITS(n);
  HARL_CHECK_LAUNCH("k_featurize");
  return HARL_OK;
}

int harl_action_masks(const harl_sketch_desc* sk, const uint16_t* tiles,
                      const uint8_t* knobs, int64_t n, int64_t ld,
                      uint8_t* tiling, uint8_t* shift, void* stream) {
  int rc = check_sketch(sk);
  if (rc) return rc;
  if (n <= 0) return HARL_OK;
  HARL_PROF_BEGIN((cudaStream_t)stream);
  launch_k(k_action_masks, dim3((unsigned)((n + 127) / 128)), dim3(128), 0, (cudaStream_t)stream, 
      *sk, tiles, knobs, n, ld, tiling, shift);
  HARL_CHECK_LAUNCH("k_action_masks");
  return HARL_OK;
}

int harl_apply_actions(const harl_sketch_desc* sk, const uint16_t* tiles,
                       const uint8_t* knobs, int64_t n, int64_t ld,
                       const int32_t* actions, uint16_t* tiles_out,
                       uint8_t* knobs_out, uint64_t* status, void* stream) {
  int rc = check_sketch(sk);
  if (rc) return rc;
  if (n <= 0) return HARL_OK;
  HARL_PROF_BEGIN((cudaStream_t)stream);
  launch_k(k_apply_actions, dim3((unsigned)((n + 127) / 128)), dim3(128), 0, (cudaStream_t)stream, 
      *sk, tiles, knobs, n, ld, actions, tiles_out, knobs_out,
      (unsigned long long*)status);
  HARL_CHECK_LAUNCH("k_apply_actions");
  return HARL_OK;
}

int harl_gbt_predict(const harl_forest_desc* forest, const double* feat,
                     int64_t n, int32_t feature_len, double* score,
                     const double* old_score, double* reward, void* stream) {
  if (!forest || forest->n_trees < 0 || forest->n_trees > 1024 ||
      (forest->n_trees > 0 && (!forest->nodes || !forest->tree_first))) {
    set_error("harl_gbt_predict: bad forest");
    return HARL_E_ARG;
  }
  if (n <= 0) return HARL_OK;
  const int T = forest->n_trees > 0 ? forest->n_trees : 1;
  const int F = feature_len;
  const size_t cap = (size_t)max_dyn_smem();
  const bool smem_nodes = gbt2_smem_bytes(true, forest->n_nodes, T, F) <= cap;
  const size_t smem = gbt2_smem_bytes(smem_nodes, forest->n_nodes, T, F);
  if (smem <= cap) {
    const int64_t tiles = (n + GBT2_ROWS - 1) / GBT2_ROWS;
    const int64_t grid = tiles < sm_count() ? tiles : sm_count();
    int rc = smem_nodes ? allow_smem(k_gbt_predict2<true>, smem, "k_gbt_predict2")
                        : allow_smem(k_gbt_predict2<false>, smem, "k_gbt_predict2");
    if (rc) return rc;
    HARL_PROF_BEGIN((cudaStream_t)stream);
    if (smem_nodes)
      launch_k(k_gbt_predict2<true>, dim3((unsigned)grid), dim3(GBT2_THREADS), smem, (cudaStream_t)stream, 
          (const GbtNode*)forest->nodes, forest->tree_first, forest->n_trees,
          forest->n_nodes, forest->fitted, forest->base, forest->floor_value, feat,
          n, F, score, old_score, reward, (const GbtHdr*)forest->dev_hdr, T);
    else
      launch_k(k_gbt_predict2<false>, dim3((unsigned)grid), dim3(GBT2_THREADS), smem, (cudaStream_t)stream, 
          (const GbtNode*)forest->nodes, forest->tree_first, forest->n_trees,
          forest->n_nodes, forest->fitted, forest->base, forest->floor_value, feat,
          n, F, score, old_score, reward, (const GbtHdr*)forest->dev_hdr, T);
    HARL_PROF_UNITS(n);
    HARL_CHECK_LAUNCH("k_gbt_predict2");
    return HARL_OK;
  }
  const int rows = T <= 192 ? GBT_THREADS / GBT_GROUPS : 4;
  const size_t smem1 = sizeof(double) * (size_t)rows * T;
  int rc = allow_smem(k_gbt_predict, smem1, "k_gbt_predict");
  if (rc) return rc;
  HARL_PROF_BEGIN((cudaStream_t)stream);
  launch_k(k_gbt_predict, dim3((unsigned)((n + rows - 1) / rows)), dim3(GBT_THREADS), smem1, (cudaStream_t)stream, 
      (const GbtNode*)forest->nodes, forest->tree_first, forest->n_trees,
      forest->fitted, forest->base, forest->floor_value, feat, n, feature_len,
      score, old_score, reward, rows, (const GbtHdr*)forest->dev_hdr);
  HARL_PROF_UNITS(n);
  HARL_CHECK_LAUNCH("k_gbt_predict");
  return HARL_OK;
}

int harl_policy_step(const harl_sketch_desc* sk, const harl_mlp_desc* pol,
                     const double* feat, const uint16_t* tiles,
                     const uint8_t* knobs, int64_t n, int64_t ld,
                     const harl_pcg64* rng, const int32_t* inject,
                     int32_t* actions, double* logp, uint16_t* tiles_out,
                     uint8_t* knobs_out, uint64_t* move_bits,
                     uint32_t* shift_bits, int32_t* head0_col,
                     float* logits_out, uint64_t* status,
                     const int32_t* grow, int64_t m_total, void* stream) {
  int rc = check_sketch(sk);
  if (rc) return rc;
  if ((rc = check_mlp(pol, true))) return rc;
  if (pol->n_head_cols != sk->n_head0 + 9 || pol->dims[0] != sk->feature_len) {
    set_error("policy descriptor does not match sketch");
    return HARL_E_ARG;
  }
  if (n <= 0) return HARL_OK;
  if (!rng && !inject) {
    set_error("harl_policy_step: need rng or injected actions");
    return HARL_E_ARG;
  }
  int ldbuf = pol->n_head_cols;
  for (int l = 0; l <= pol->n_layers; ++l) ldbuf = ldbuf > pol->dims[l] ? ldbuf : pol->dims[l];
  ldbuf += 1;  // bank-conflict padding
  const size_t smem = sizeof(float) * 2 * MLP_TM * (size_t)ldbuf;
  if ((rc = allow_smem(k_policy_step, smem, "k_policy_step"))) return rc;
  PcgJump J;
  StepRng sr;
  memset(&J, 0, sizeof(J));
  memset(&sr, 0, sizeof(sr));
  if (rng) {
    build_jump(*rng, &J);
    sr.s = state_of(*rng);
  }
  sr.grow = grow;
  sr.m_total = m_total;
  HARL_PROF_BEGIN((cudaStream_t)stream);
  launch_k(k_policy_step, dim3((unsigned)((n + MLP_TM - 1) / MLP_TM)), dim3(MLP_THREADS), smem, (cudaStream_t)stream, *sk, *pol, J, sr, feat, tiles, knobs, n,
                                          ld, inject, actions, logp, tiles_out,
                                          knobs_out, move_bits, shift_bits,
                                          head0_col, logits_out,
                                          (unsigned long long*)status, ldbuf);
  HARL_CHECK_LAUNCH("k_policy_step");
  return HARL_OK;
}

static void build_lane_jump(const harl_pcg64& g, LaneJump* LJ) {
  const h128 inc = ((h128)g.inc_hi << 64) | (h128)g.inc_lo;
  h128 A = 1, C = 0;  // l steps: s -> A s + C
  for (int l = 0; l < 32; ++l) {
    LJ->A[l] = to_u128(A);
    LJ->C[l] = to_u128(C);
    C = PCG_MULT * C + inc;
    A = PCG_MULT * A;
  }
}

static void sampler_setup(const harl_pcg64* rng, PcgJump* J, u128* base) {
  memset(J, 0, sizeof(*J));
  memset(base, 0, sizeof(*base));
  if (rng) {
    build_jump(*rng, J);
    *base = state_of(*rng);
  }
}

static SampleArgs sample_args(const float* logits, int ldz, int64_t n, int64_t ld,
                              const int32_t* inject, int32_t* actions, double* logp,
                              uint16_t* tiles_out, uint8_t* knobs_out,
                              uint64_t* move_bits, uint32_t* shift_bits,
                              int32_t* head0_col, uint64_t* status,
                              const int32_t* grow, int64_t m_total) {
  SampleArgs a;
  memset(&a, 0, sizeof(a));
  a.logits = logits;
  a.ldz = ldz;
  a.n = n;
  a.ld = ld;
  a.inject = inject;
  a.actions = actions;
  a.logp = logp;
  a.tiles_out = tiles_out;
  a.knobs_out = knobs_out;
  a.move_bits = move_bits;
  a.shift_bits = shift_bits;
  a.head0_col = head0_col;
  a.status = (unsigned long long*)status;
  a.grow = grow;
  a.m_total = m_total > 0 ? m_total : n;
  a.pcg_tab = nullptr;
  return a;
}

static int launch_sampler(const harl_sketch_desc* sk, const harl_pcg64* rng,
                          const uint64_t* rng_state_dev, const int32_t* grow,
                          int64_t m_total,
                          const float* logits, int ldz, int64_t n, int64_t ld,
                          const uint16_t* tiles, const uint8_t* knobs,
                          const int32_t* inject, int32_t* actions, double* logp,
                          uint16_t* tiles_out, uint8_t* knobs_out,
                          uint64_t* move_bits, uint32_t* shift_bits,
                          int32_t* head0_col, uint64_t* status,
                          cudaStream_t st, double* feat_out = nullptr,
                          const SampleGbtArgs* gf = nullptr,
                          bool after_policy = false) {
  PcgJump J;
  LaneJump LJ;
  u128 base;
  memset(&J, 0, sizeof(J));
  memset(&LJ, 0, sizeof(LJ));
  memset(&base, 0, sizeof(base));
  if (rng) {
    build_jump(*rng, &J);
    build_lane_jump(*rng, &LJ);
    base = state_of(*rng);
  }
  SampleArgs a;
  memset(&a, 0, sizeof(a));
  a.logits = logits;
  a.ldz = ldz;
  a.n = n;
  a.ld = ld;
  a.inject = inject;
  a.actions = actions;
  a.logp = logp;
  a.tiles_out = tiles_out;
  a.knobs_out = knobs_out;
  a.move_bits = move_bits;
  a.shift_bits = shift_bits;
  a.head0_col = head0_col;
  a.status = (unsigned long long*)status;
  a.grow = grow;
  a.m_total = m_total > 0 ? m_total : n;
  a.pcg_tab = pcg_tab_for(rng, st);
  // (PDL pays only right behind the policy kernel on the same stream; a
  // sampler behind a stream join, the forked-policy steps, gains nothing)
  const bool pdl = use_pdl() || (use_pdl_sample() && after_policy);
  a.prefill = pdl ? 1 : 0;
  const int rows_per_cta = SAMPLE_THREADS / SG;
  const dim3 grid((unsigned)((n + rows_per_cta - 1) / rows_per_cta));
  HARL_PROF_BEGIN(st);
  const int nI = (sk->n_head0 + SG - 1) / SG;
  auto go = [&](auto kfeat, auto kplain, auto kgbt) -> int {
    if (feat_out && gf) {   // + the cost model on the successor rows
      const size_t lut = sk->max_extent + 1 <= FEAT_LUT_SMEM_MAX
                             ? (size_t)(sk->max_extent + 1) * 8 : 0;
      const size_t smem = (size_t)gf->region + (size_t)SGBT_ROWS * sk->feature_len * 8 + lut;
      int rc = allow_smem(kgbt, smem, "k_sample_gbt");
      if (rc) return rc;
      const dim3 ggrid((unsigned)((n + SGBT_ROWS - 1) / SGBT_ROWS));
      launch_k(kgbt, ggrid, dim3(SGBT_THREADS), smem, st, *sk, J, base,
               (const u128*)rng_state_dev, tiles, knobs, a, feat_out, *gf);
    } else if (feat_out) {   // also featurize the successor states (schedspace.py:415)
      const size_t lut = sk->max_extent + 1 <= FEAT_LUT_SMEM_MAX
                             ? (size_t)(sk->max_extent + 1) * 8 : 0;
      const size_t smem = (size_t)rows_per_cta * sk->feature_len * 8 + lut;
      int rc = allow_smem(kfeat, smem, "k_sample_rows");
      if (rc) return rc;
      launch_k_pdl(pdl, kfeat, grid, dim3(SAMPLE_THREADS), smem, st, *sk, J, LJ, base,
                   (const u128*)rng_state_dev, tiles, knobs, a, feat_out);
    } else {
      launch_k_pdl(pdl, kplain, grid, dim3(SAMPLE_THREADS), 0, st, *sk, J, LJ, base,
                   (const u128*)rng_state_dev, tiles, knobs, a, (double*)nullptr);
    }
    return HARL_OK;
  };
  int grc;
  // instantiation: head-0 columns cached per lane (MAXI) x slots per lane
  const int nsl = sk->local_slots <= 2 * SG ? 2 : (sk->local_slots <= 4 * SG ? 4 : 8);
#define HARL_SAMPLER(MX, NS) \
  go(k_sample_rows<true, MX, NS>, k_sample_rows<false, MX, NS>, k_sample_gbt<MX, NS>)
#define HARL_SAMPLER_NSL(MX) \
  (nsl == 2 ? HARL_SAMPLER(MX, 2) : nsl == 4 ? HARL_SAMPLER(MX, 4) : HARL_SAMPLER(MX, 8))
  if (nI <= 8) grc = HARL_SAMPLER_NSL(8);
  else if (nI <= 12) grc = HARL_SAMPLER_NSL(12);
  else grc = HARL_SAMPLER_NSL(16);
#undef HARL_SAMPLER_NSL
#undef HARL_SAMPLER
  if (grc) return grc;
  HARL_PROF_UNITS(n);
  if (feat_out && gf) HARL_CHECK_LAUNCH("k_sample_gbt");
  else HARL_CHECK_LAUNCH("k_sample_rows");
  return HARL_OK;
}

// featurize inside the sampler up to this many rows per launch (measured:
// C2 16 K rows +4 % episode throughput; C3 at 32 K rows and the 1 M-row
// sweep faster with the separate featurizer)
#ifndef HARL_SAMPLE_FEAT_MAX_ROWS
#define HARL_SAMPLE_FEAT_MAX_ROWS 16384
#endif
static const int64_t SAMPLE_FEAT_MAX_ROWS = HARL_SAMPLE_FEAT_MAX_ROWS;

static bool tc_trunk_ok(const harl_mlp_desc* m, int F) {
  return m && m->n_layers >= 2 && m->dims[0] == F && F <= TC_K1 &&
         m->dims[1] == TC_H && m->dims[2] == TC_H;
}

static int policy_step_tc_impl(const harl_sketch_desc* sk, const harl_mlp_desc* pol,
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
                        int32_t flags, void* stream, const harl_forest_desc* forest,
                        const double* old_score, double* score, double* reward) {
  const int32_t fuse_tc = flags & HARL_STEP_FUSED;
  int rc = check_sketch(sk);
  if (rc) return rc;
  if ((rc = check_mlp(pol, true))) return rc;
  if (pol->n_layers != 2 || !tc_trunk_ok(pol, sk->feature_len) ||
      pol->n_head_cols != sk->n_head0 + 9 || pol->n_head_cols > HEADS_NMAX ||
      !hid_scratch) {
    set_error("harl_policy_step_tc: shape not eligible for the tcgen05 path");
    return HARL_E_ARG;
  }
  if (n <= 0) return HARL_OK;
  const bool mlp_only = (flags & HARL_STEP_MLP_ONLY) != 0;
  const bool sample_only = (flags & HARL_STEP_SAMPLE_ONLY) != 0;
  if (!rng && !inject && !mlp_only) {
    set_error("harl_policy_step_tc: need rng or injected actions");
    return HARL_E_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int NHP = (pol->n_head_cols + 15) / 16 * 16;
  const bool f16_path = !fuse_tc && packed_trunk && NHP <= F16_NHP_MAX && use_tc16(n) &&
      ((uintptr_t)feat & 15) == 0 &&
      (size_t)f16_smem_bytes(true, NHP, sk->feature_len, 1) <= (size_t)max_dyn_smem();
  if ((mlp_only || sample_only) && (!f16_path || (mlp_only && sample_only))) {
    set_error("harl_policy_step_tc: split launch not on the 3xFP16 path");
    return HARL_E_LIMIT;
  }
  // the cost model fused into the sampler: decided before anything launches
  SampleGbtArgs gf;
  memset(&gf, 0, sizeof(gf));
  if (forest) {
    const size_t lut = sk->max_extent + 1 <= FEAT_LUT_SMEM_MAX
                           ? (size_t)(sk->max_extent + 1) * 8 : 0;
    const size_t region = sgbt_region_bytes(forest->n_trees > 0 ? forest->n_trees : 1);
    if (!f16_path || !feat_out || n > SAMPLE_FEAT_MAX_ROWS || !forest->dev_hdr ||
        forest->n_trees > SGBT_MAX_TREES || !forest->tree_first || !forest->nodes ||
        !score || (size_t)region + (size_t)SGBT_ROWS * sk->feature_len * 8 + lut >
            (size_t)max_dyn_smem() / 2 - 16384) {
      set_error("harl_policy_step_tc_gbt: step not eligible for the fused cost model");
      return HARL_E_LIMIT;
    }
    gf.nodes = (const GbtNode*)forest->nodes;
    gf.tree_first = forest->tree_first;
    gf.hdr = (const GbtHdr*)forest->dev_hdr;
    gf.old_score = old_score;
    gf.score = score;
    gf.reward = reward;
    gf.region = (int32_t)region;
  }
  // 3xFP16 policy (trunk + heads, weights resident, two tiles in flight)
  if (f16_path && !sample_only) {
    const size_t smem = (size_t)f16_smem_bytes(true, NHP, sk->feature_len, 1);
    if ((rc = allow_smem(k_mlp_f16<true>, smem, "k_mlp_f16<policy>"))) return rc;
    F16Args fa;
    memset(&fa, 0, sizeof(fa));
    fa.nxb = 1;
    fa.feat0 = feat;
    fa.n0 = n;
    fa.F = sk->feature_len;
    fa.NH = pol->n_head_cols;
    fa.NHP = NHP;
    fa.logits = hid_scratch;
    fa.logits_out = logits_out;
    fa.img = (const uint8_t*)packed_trunk + TRUNK_IMAGE;
    fa.early_w = (flags & HARL_WEIGHTS_SETTLED) ? 1 : 0;
    HARL_PROF_BEGIN(st);
    GbtFinishArgs nofin;
    memset(&nofin, 0, sizeof(nofin));
    launch_k(k_mlp_f16<true>, dim3(tc16_grid((n + 127) / 128)), dim3(F16_THREADS),
             smem, st, fa, nofin);
    HARL_PROF_UNITS(n);
    HARL_CHECK_LAUNCH("k_mlp_f16<policy>");
    if (mlp_only) return HARL_OK;
  }
  if (f16_path) {
    const bool in_sampler = feat_out && n <= SAMPLE_FEAT_MAX_ROWS;
    rc = launch_sampler(sk, rng, rng_state_dev, grow, m_total, hid_scratch,
                        TC_H, n, ld, tiles, knobs, inject, actions, logp,
                        tiles_out, knobs_out, move_bits, shift_bits, head0_col,
                        status, st, in_sampler ? feat_out : nullptr,
                        forest ? &gf : nullptr, !sample_only);
    if (rc || !feat_out || in_sampler) return rc;
    return harl_featurize(sk, tiles_out, knobs_out, n, ld, feat_out, stream);
  }
  // fused step: policy -> sample/apply -> featurize in one kernel
  if (feat_out && fuse_tc && packed_trunk && packed_heads && use_tc2() &&
      ((uintptr_t)feat & 15) == 0) {
    int regA = tc2_regA(NHP);
    const int need = tc2_fused_regA_need(sk->feature_len, sk->local_slots, sk->max_extent);
    if (need > regA) regA = (need + 127) / 128 * 128;
    const size_t smem = (size_t)regA + TC2_W2P;
    if (smem <= (size_t)max_dyn_smem()) {
      if ((rc = allow_smem(k_policy_step_fused, smem, "k_policy_step_fused"))) return rc;
      PolicyTcArgs pa;
      memset(&pa, 0, sizeof(pa));
      pa.feat = feat;
      pa.n = n;
      pa.F = sk->feature_len;
      pa.NH = pol->n_head_cols;
      pa.NHP = NHP;
      pa.regA = regA;
      pa.logits = nullptr;
      pa.logits_out = logits_out;
      pa.trunk_img = packed_trunk;
      pa.heads_img = packed_heads;
      StepFuseArgs fa;
      memset(&fa, 0, sizeof(fa));
      PcgJump J;
      sampler_setup(rng, &J, &fa.base_arg);
      fa.base_dev = (const u128*)rng_state_dev;
      fa.s = sample_args(nullptr, TC2_LG_LD, n, ld, inject, actions, logp, tiles_out,
                         knobs_out, move_bits, shift_bits, head0_col, status, grow,
                         m_total);
      fa.s.pcg_tab = pcg_tab_for(rng, st);
      fa.tiles = tiles;
      fa.knobs = knobs;
      fa.feat_new = feat_out;
      const int64_t tiles_n = (n + 127) / 128;
      const int grid = (int)(tiles_n < sm_count() ? tiles_n : sm_count());
      HARL_PROF_BEGIN(st);
      launch_k(k_policy_step_fused, dim3(grid), dim3(TC2_THREADS), smem, st, pa, fa,
               *sk, J);
      HARL_PROF_UNITS(n);
      HARL_CHECK_LAUNCH("k_policy_step_fused");
      return HARL_OK;
    }
  }
  if (packed_trunk && packed_heads && use_tc2() && ((uintptr_t)feat & 15) == 0 &&
      (size_t)tc2_smem(NHP) <= (size_t)max_dyn_smem()) {
    if ((rc = allow_smem(k_policy_tc, (size_t)tc2_smem(NHP), "k_policy_tc"))) return rc;
    PolicyTcArgs pa;
    pa.feat = feat;
    pa.n = n;
    pa.F = sk->feature_len;
    pa.NH = pol->n_head_cols;
    pa.NHP = NHP;
    pa.regA = tc2_regA(NHP);
    pa.logits = hid_scratch;
    pa.logits_out = logits_out;
    pa.trunk_img = packed_trunk;
    pa.heads_img = packed_heads;
    // 64-row tiles when they still fit in one wave: twice the CTAs of
    // 128-row tiles, half the epilogue per warp (the post-cull steps)
    const int64_t tiles64 = (n + 63) / 64;
    if (use_tc64() && tiles64 <= sm_count()) {
      if ((rc = allow_smem(k_policy_tc64, (size_t)tc2_smem(NHP), "k_policy_tc64"))) return rc;
      HARL_PROF_BEGIN(st);
      launch_k(k_policy_tc64, dim3((unsigned)tiles64), dim3(TC2_THREADS), tc2_smem(NHP), st, pa);
      HARL_PROF_UNITS(n);
      HARL_CHECK_LAUNCH("k_policy_tc64");
    } else {
      const int64_t tiles_n = (n + 127) / 128;
      const int grid = (int)(tiles_n < sm_count() ? tiles_n : sm_count());
      HARL_PROF_BEGIN(st);
      launch_k(k_policy_tc, dim3(grid), dim3(TC2_THREADS), tc2_smem(NHP), st, pa);
      HARL_PROF_UNITS(n);
      HARL_CHECK_LAUNCH("k_policy_tc");
    }
    // small populations (latency-bound steps): the sampler featurizes the
    // successor states itself, one launch less; large ones (throughput-
    // bound): the 4-threads-per-row featurizer keeps every lane busy
    const bool in_sampler = feat_out && n <= SAMPLE_FEAT_MAX_ROWS;
    rc = launch_sampler(sk, rng, rng_state_dev, grow, m_total, hid_scratch,
                        TC_H, n, ld, tiles, knobs, inject, actions, logp,
                        tiles_out, knobs_out, move_bits, shift_bits, head0_col,
                        status, st, in_sampler ? feat_out : nullptr,
                        forest ? &gf : nullptr);
    if (rc || !feat_out || in_sampler) return rc;
    return harl_featurize(sk, tiles_out, knobs_out, n, ld, feat_out, stream);
  }
  if ((rc = allow_smem(k_trunk_tc<TRUNK_POLICY>, TRUNK_SMEM, "k_trunk_tc")))
    return rc;
  TrunkArgs ta;
  memset(&ta, 0, sizeof(ta));
  ta.feat0 = feat;
  ta.n0 = n;
  ta.F = sk->feature_len;
  ta.out0 = hid_scratch;
  ta.W1 = pol->W[0];
  ta.b1 = pol->b[0];
  ta.W2 = pol->W[1];
  ta.b2 = pol->b[1];
  ta.packed = packed_trunk;
  const int64_t tiles_n = (n + 127) / 128;
  const int grid = (int)(tiles_n < sm_count() ? tiles_n : sm_count());
  HARL_PROF_BEGIN(st);
  launch_k(k_trunk_tc<TRUNK_POLICY>, dim3(grid), dim3(128), TRUNK_SMEM, st, ta);
  HARL_CHECK_LAUNCH("k_trunk_tc<policy>");
  HeadsArgs ha;
  ha.hid = hid_scratch;
  ha.Wh = pol->head_W;
  ha.bh = pol->head_b;
  ha.logits_out = logits_out;
  ha.packed = packed_heads;
  ha.n = n;
  ha.NH = pol->n_head_cols;
  ha.NHP = (ha.NH + 15) / 16 * 16;
  const size_t smem = (size_t)2 * ha.NHP * TC_H * 4 + HEADS_NMAX * 4;
  if ((rc = allow_smem(k_heads_tc, smem, "k_heads_tc"))) return rc;
  HARL_PROF_BEGIN(st);
  launch_k(k_heads_tc, dim3(grid), dim3(128), smem, st, ha);
  HARL_CHECK_LAUNCH("k_heads_tc");
  rc = launch_sampler(sk, rng, rng_state_dev, grow, m_total, hid_scratch,
                        TC_H, n, ld,
                        tiles, knobs, inject,
                        actions, logp, tiles_out, knobs_out, move_bits,
                        shift_bits, head0_col, status, st);
    if (rc || !feat_out) return rc;
    return harl_featurize(sk, tiles_out, knobs_out, n, ld, feat_out, stream);
}

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
                        int32_t flags, void* stream) {
  return policy_step_tc_impl(sk, pol, feat, tiles, knobs, n, ld, rng, inject, actions,
                             logp, tiles_out, knobs_out, move_bits, shift_bits,
                             head0_col, logits_out, status, hid_scratch, rng_state_dev,
                             packed_trunk, packed_heads, grow, m_total, feat_out, flags,
                             stream, nullptr, nullptr, nullptr, nullptr);
}

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
                            void* stream) {
  if (!forest) {
    set_error("harl_policy_step_tc_gbt: forest required");
    return HARL_E_ARG;
  }
  return policy_step_tc_impl(sk, pol, feat, tiles, knobs, n, ld, rng, inject, actions,
                             logp, tiles_out, knobs_out, move_bits, shift_bits,
                             head0_col, logits_out, status, hid_scratch, rng_state_dev,
                             packed_trunk, packed_heads, grow, m_total, feat_out, flags,
                             stream, forest, old_score, score, reward);
}


static int value_pair_tc_impl(const harl_mlp_desc* val, const double* feat0,
                       int64_t n0, const double* feat1, int64_t n1,
                       int32_t feature_len, float* v0, float* v1,
                       const void* packed, int32_t flags, void* stream,
                       const GbtFinishArgs* fin) {
  int rc = check_mlp(val, false);
  if (rc) return rc;
  if (val->n_layers != 3 || !tc_trunk_ok(val, feature_len) ||
      val->dims[3] != 1) {
    set_error("harl_value_pair_tc: shape not eligible for the tcgen05 path");
    return HARL_E_ARG;
  }
  const bool f16_ok = packed && use_tc16(n0 + n1) && ((uintptr_t)feat0 & 15) == 0 &&
      ((uintptr_t)feat1 & 15) == 0 &&
      (size_t)f16_smem_bytes(false, 0, feature_len, 1) <= (size_t)max_dyn_smem();
  if (fin && (!f16_ok || !feat1 || n1 <= 0 || (n0 != 0 && n0 != n1) ||
              fin->a.n != n1)) {
    set_error("harl_value_finish_tc: step not eligible for the fused finish");
    return HARL_E_LIMIT;
  }
  if (n0 + n1 <= 0) return HARL_OK;
  if (f16_ok) {
    const int nxb = (size_t)f16_smem_bytes(false, 0, feature_len, 2) <=
                    (size_t)max_dyn_smem() ? 2 : 1;
    const size_t smem = (size_t)f16_smem_bytes(false, 0, feature_len, nxb);
    if ((rc = allow_smem(k_mlp_f16<false>, smem, "k_mlp_f16<value>"))) return rc;
    if ((rc = allow_smem(k_mlp_f16<false, true>, smem, "k_mlp_f16<value+finish>")))
      return rc;
    F16Args fa;
    memset(&fa, 0, sizeof(fa));
    fa.nxb = nxb;
    fa.feat0 = feat0;
    fa.feat1 = feat1;
    fa.n0 = n0;
    fa.n1 = feat1 ? n1 : 0;
    fa.F = feature_len;
    fa.out0 = v0;
    fa.out1 = v1;
    fa.b3 = val->b[2];
    fa.img = (const uint8_t*)packed + TRUNK_IMAGE;
    fa.early_w = (flags & HARL_WEIGHTS_SETTLED) ? 1 : 0;
    GbtFinishArgs nofin;
    memset(&nofin, 0, sizeof(nofin));
    fa.fin = fin ? 1 : 0;
    fa.pair = ((fin || (flags & HARL_VALUE_PAIRED)) && n0 == n1) ? 1 : 0;
    const int64_t tiles_n = fa.pair ? (n1 + 127) / 128
                                    : (n0 + 127) / 128 + (fa.n1 + 127) / 128;
    HARL_PROF_BEGIN((cudaStream_t)stream);
    if (fin)
      launch_k(k_mlp_f16<false, true>, dim3(tc16_grid(tiles_n)), dim3(F16_THREADS), smem,
               (cudaStream_t)stream, fa, *fin);
    else
      launch_k(k_mlp_f16<false, false>, dim3(tc16_grid(tiles_n)), dim3(F16_THREADS), smem,
               (cudaStream_t)stream, fa, nofin);
    HARL_PROF_UNITS(n0 + fa.n1);
    if (fin) HARL_CHECK_LAUNCH("k_mlp_f16<value+finish>");
    else HARL_CHECK_LAUNCH("k_mlp_f16<value>");
    return HARL_OK;
  }
  if (packed && use_tc2() && ((uintptr_t)feat0 & 15) == 0 &&
      ((uintptr_t)feat1 & 15) == 0) {
    const size_t smem = (size_t)tc2_value_smem();
    if ((rc = allow_smem(k_value_tc, smem, "k_value_tc"))) return rc;
    ValueTcArgs va;
    va.feat0 = feat0;
    va.feat1 = feat1;
    va.n0 = n0;
    va.n1 = feat1 ? n1 : 0;
    va.F = feature_len;
    va.out0 = v0;
    va.out1 = v1;
    va.b3 = val->b[2];
    va.trunk_img = packed;
    const int64_t tiles_n = (n0 + 127) / 128 + (va.n1 + 127) / 128;
    const int grid = (int)(tiles_n < sm_count() ? tiles_n : sm_count());
    HARL_PROF_BEGIN((cudaStream_t)stream);
    launch_k(k_value_tc, dim3(grid), dim3(TC2_THREADS), smem, (cudaStream_t)stream, va);
    HARL_PROF_UNITS(n0 + va.n1);
    HARL_CHECK_LAUNCH("k_value_tc");
    return HARL_OK;
  }
  if ((rc = allow_smem(k_trunk_tc<TRUNK_VALUE>, TRUNK_SMEM, "k_trunk_tc")))
    return rc;
  TrunkArgs ta;
  memset(&ta, 0, sizeof(ta));
  ta.feat0 = feat0;
  ta.feat1 = feat1;
  ta.n0 = n0;
  ta.n1 = feat1 ? n1 : 0;
  ta.F = feature_len;
  ta.out0 = v0;
  ta.out1 = v1;
  ta.W1 = val->W[0];
  ta.b1 = val->b[0];
  ta.W2 = val->W[1];
  ta.b2 = val->b[1];
  ta.w3 = val->W[2];
  ta.b3 = val->b[2];
  ta.packed = packed;
  const int64_t tiles_n = (n0 + 127) / 128 + (ta.n1 + 127) / 128;
  const int grid = (int)(tiles_n < sm_count() ? tiles_n : sm_count());
  HARL_PROF_BEGIN((cudaStream_t)stream);
  launch_k(k_trunk_tc<TRUNK_VALUE>, dim3(grid), dim3(128), TRUNK_SMEM, (cudaStream_t)stream, ta);
  HARL_CHECK_LAUNCH("k_trunk_tc<value>");
  return HARL_OK;
}

int harl_value_pair_tc(const harl_mlp_desc* val, const double* feat0,
                       int64_t n0, const double* feat1, int64_t n1,
                       int32_t feature_len, float* v0, float* v1,
                       const void* packed, int32_t flags, void* stream) {
  return value_pair_tc_impl(val, feat0, n0, feat1, n1, feature_len, v0, v1, packed,
                            flags, stream, nullptr);
}

int harl_value_finish_tc(const harl_mlp_desc* val, const double* feat0,
                         int64_t n0, const double* feat1, int64_t n1,
                         int32_t feature_len, float* v0, float* v1,
                         const void* packed, int32_t flags,
                         const harl_step_buffers* io, int64_t ld, int64_t vbase,
                         int32_t local_slots, double discount, int32_t rl,
                         const harl_replay_ring* ring, int64_t wpos,
                         int64_t keep_from, const harl_entry_log* log,
                         const harl_track_stats* ts, const int64_t* wpos_dev,
                         void* stream) {
  if (!io || !log || !ts || (rl && (!ring || ring->cap < 1)) ||
      io->v_cur != v0 || io->v_next != v1 || io->feat != feat0 || io->feat_new != feat1) {
    set_error("harl_value_finish_tc: bad arguments");
    return HARL_E_ARG;
  }
  GbtFinishArgs fa;
  memset(&fa, 0, sizeof(fa));
  fa.a.n = n1;
  fa.a.ld = ld;
  fa.a.vbase = vbase;
  fa.a.local_slots = local_slots;
  fa.a.F = feature_len;
  fa.a.discount = discount;
  fa.a.rl = rl;
  fa.a.wpos = wpos;
  fa.a.keep_from = keep_from;
  fa.io = *io;
  if (ring) fa.ring = *ring;
  if (fa.ring.cap < 1) fa.ring.cap = 1;
  fa.log = *log;
  fa.ts = *ts;
  fa.wpos_dev = wpos_dev;
  return value_pair_tc_impl(val, feat0, n0, feat1, n1, feature_len, v0, v1, packed,
                            flags, stream, &fa);
}

int harl_prepare(void) {
  // raise every kernel's dynamic shared-memory limit up front so that no
  // entry point needs cudaFuncSetAttribute while a stream is being captured
  int rc = 0;
  if ((rc = allow_max_smem(k_featurize, "k_featurize"))) return rc;
  if ((rc = allow_max_smem(k_featurize2, "k_featurize2"))) return rc;
  if ((rc = allow_max_smem(k_gbt_predict, "k_gbt_predict"))) return rc;
  if ((rc = allow_max_smem(k_gbt_predict2<true>, "k_gbt_predict2"))) return rc;
  if ((rc = allow_max_smem(k_gbt_predict2<false>, "k_gbt_predict2"))) return rc;
  if ((rc = allow_max_smem(k_policy_step, "k_policy_step"))) return rc;
  if ((rc = allow_max_smem(k_value_forward, "k_value_forward"))) return rc;
  if ((rc = allow_max_smem(k_trunk_tc<TRUNK_POLICY>, "k_trunk_tc"))) return rc;
  if ((rc = allow_max_smem(k_trunk_tc<TRUNK_VALUE>, "k_trunk_tc"))) return rc;
  if ((rc = allow_max_smem(k_heads_tc, "k_heads_tc"))) return rc;
  if ((rc = allow_max_smem(k_policy_tc, "k_policy_tc"))) return rc;
  if ((rc = allow_max_smem(k_policy_tc64, "k_policy_tc64"))) return rc;
  if ((rc = allow_max_smem(k_policy_step_fused, "k_policy_step_fused"))) return rc;
  if ((rc = allow_max_smem(k_value_tc, "k_value_tc"))) return rc;
  if ((rc = allow_max_smem(k_mlp_f16<true>, "k_mlp_f16<policy>"))) return rc;
  if ((rc = allow_max_smem(k_mlp_f16<false>, "k_mlp_f16<value>"))) return rc;
  if ((rc = allow_max_smem(k_ppo_rows, "k_ppo_rows"))) return rc;
  if ((rc = allow_max_smem(k_ppo_rows_tc, "k_ppo_rows_tc"))) return rc;
  // One shared-memory carveout for every kernel: the episode alternates
  // 230 KB-smem tcgen05 kernels with smem-light ones, and a carveout change
  // between consecutive kernels makes the SMs drain and reconfigure.
  // HARL_CARVEOUT=default keeps the driver's per-kernel choice.
  const char* cv = getenv("HARL_CARVEOUT");
  if (!cv || strcmp(cv, "default") != 0) {
    auto carve = [](auto kernel) {
      cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                           (int)cudaSharedmemCarveoutMaxShared);
    };
  carve(k_spin);
  carve(k_init_sample);
  carve(k_init_one);
  carve(k_uniform_counts);
  carve(k_uniform_scan);
  carve(k_uniform_draw);
  carve(k_uniform_one);
  carve(k_featurize);
  carve(k_featurize2);
  carve(k_action_masks);
  carve(k_apply_actions);
  carve(k_gbt_predict);
  carve(k_gbt_predict2<true>);
  carve(k_gbt_predict2<false>);
  carve(k_policy_step);
  carve(k_value_forward);
#define HARL_CARVE_SAMPLER(MX) \
  carve(k_sample_rows<false, MX, 2>); carve(k_sample_rows<true, MX, 2>); \
  carve(k_sample_rows<false, MX, 4>); carve(k_sample_rows<true, MX, 4>); \
  carve(k_sample_rows<false, MX, 8>); carve(k_sample_rows<true, MX, 8>);
  HARL_CARVE_SAMPLER(8)
  HARL_CARVE_SAMPLER(12)
  HARL_CARVE_SAMPLER(16)
#undef HARL_CARVE_SAMPLER
  carve(k_gbt_finish<true>);
  carve(k_gbt_finish<false>);
  carve(k_trunk_tc<TRUNK_POLICY>);
  carve(k_trunk_tc<TRUNK_VALUE>);
  carve(k_heads_tc);
  carve(k_pack_trunk);
  carve(k_pack_heads);
  carve(k_policy_tc);
  carve(k_policy_tc64);
  carve(k_policy_step_fused);
  carve(k_value_tc);
  carve(k_mlp_f16<true>);
  carve(k_mlp_f16<false>);
  carve(k_pack16);
  carve(k_finish_step);
  carve(k_ring_rows);
  carve(k_gather_rows);
  carve(k_ppo_rows);
  carve(k_ppo_rows_tc);
  carve(k_ppo_losses);
  carve(k_ppo_wgrad);
  carve(k_ppo_finalize);
  carve(k_ppo_adam);
  carve(k_ppo_wgrad_adam);
  carve(k_wt_fill);
  carve(k_tc_probe);
    cudaGetLastError();
  }
  (void)sm_count();
  return HARL_OK;
}

int64_t harl_tc_packed_bytes(int32_t which, int32_t n_head_cols) {
  // trunk images carry the 3xFP16 image (heads included) behind them
  if (which == 0)
    return TRUNK_IMAGE +
           f16_image_bytes(std::min((n_head_cols + 15) / 16 * 16, F16_NHP_MAX));
  return heads_image_bytes((n_head_cols + 15) / 16 * 16);
}

int harl_pack_tc_weights(const harl_mlp_desc* pol, const harl_mlp_desc* val,
                         int32_t feature_len, void* pol_trunk,
                         void* pol_heads, void* val_trunk, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (pol && pol_trunk) {
    if (!tc_trunk_ok(pol, feature_len) || pol->n_head_cols > HEADS_NMAX) {
      set_error("harl_pack_tc_weights: policy not eligible");
      return HARL_E_ARG;
    }
    TrunkArgs ta;
    memset(&ta, 0, sizeof(ta));
    ta.F = feature_len;
    ta.W1 = pol->W[0];
    ta.b1 = pol->b[0];
    ta.W2 = pol->W[1];
    ta.b2 = pol->b[1];
    HARL_PROF_BEGIN(st);
    launch_k(k_pack_trunk, dim3(64), dim3(256), 0, st, ta, (uint8_t*)pol_trunk, 0);
    HARL_CHECK_LAUNCH("k_pack_trunk<policy>");
    HeadsArgs ha;
    memset(&ha, 0, sizeof(ha));
    ha.Wh = pol->head_W;
    ha.bh = pol->head_b;
    ha.NH = pol->n_head_cols;
    ha.NHP = (ha.NH + 15) / 16 * 16;
    HARL_PROF_BEGIN(st);
    launch_k(k_pack_heads, dim3(64), dim3(256), 0, st, ha, (uint8_t*)pol_heads);
    HARL_CHECK_LAUNCH("k_pack_heads");
    if (ha.NHP <= F16_NHP_MAX) {
      uint8_t* f = (uint8_t*)pol_trunk + TRUNK_IMAGE;
      float* ff = (float*)f;
      uint16_t* h1 = (uint16_t*)(f + f16_off_w1());
      uint16_t* h2 = (uint16_t*)(f + f16_off_w2());
      uint16_t* hh = (uint16_t*)(f + f16_off_wh());
      Pack16Args pk;
      memset(&pk, 0, sizeof(pk));
      pk.m[0] = {pol->W[0], feature_len, TC_H, TC_K1, TC_H, h1, h1 + F16_W1 / 2, ff + F16_SC + 0};
      pk.m[1] = {pol->W[1], TC_H, TC_H, TC_H, TC_H, h2, h2 + F16_W2 / 2, ff + F16_SC + 1};
      pk.m[2] = {pol->head_W, TC_H, pol->n_head_cols, TC_H, ha.NHP, hh,
                 hh + ha.NHP * TC_H, ff + F16_SC + 2};
      pk.v[0] = {pol->b[0], TC_H, TC_H, ff + F16_B1};
      pk.v[1] = {pol->b[1], TC_H, TC_H, ff + F16_B2};
      pk.v[2] = {pol->head_b, pol->n_head_cols, TC_H, ff + F16_B3};
      pk.n_mat = 3;
      pk.n_vec = 3;
      HARL_PROF_BEGIN(st);
      launch_k(k_pack16, dim3(3), dim3(1024), 0, st, pk);
      HARL_CHECK_LAUNCH("k_pack16<policy>");
    }
  }
  if (val && val_trunk) {
    if (!tc_trunk_ok(val, feature_len)) {
      set_error("harl_pack_tc_weights: value net not eligible");
      return HARL_E_ARG;
    }
    TrunkArgs ta;
    memset(&ta, 0, sizeof(ta));
    ta.F = feature_len;
    ta.W1 = val->W[0];
    ta.b1 = val->b[0];
    ta.W2 = val->W[1];
    ta.b2 = val->b[1];
    ta.w3 = val->W[2];
    ta.b3 = val->b[2];
    HARL_PROF_BEGIN(st);
    launch_k(k_pack_trunk, dim3(64), dim3(256), 0, st, ta, (uint8_t*)val_trunk, 1);
    HARL_CHECK_LAUNCH("k_pack_trunk<value>");
    uint8_t* f = (uint8_t*)val_trunk + TRUNK_IMAGE;
    float* ff = (float*)f;
    uint16_t* h1 = (uint16_t*)(f + f16_off_w1());
    uint16_t* h2 = (uint16_t*)(f + f16_off_w2());
    Pack16Args pk;
    memset(&pk, 0, sizeof(pk));
    pk.m[0] = {val->W[0], feature_len, TC_H, TC_K1, TC_H, h1, h1 + F16_W1 / 2, ff + F16_SC + 0};
    pk.m[1] = {val->W[1], TC_H, TC_H, TC_H, TC_H, h2, h2 + F16_W2 / 2, ff + F16_SC + 1};
    pk.v[0] = {val->b[0], TC_H, TC_H, ff + F16_B1};
    pk.v[1] = {val->b[1], TC_H, TC_H, ff + F16_B2};
    pk.v[2] = {val->W[2], TC_H, TC_H, ff + F16_B3};
    pk.n_mat = 2;
    pk.n_vec = 3;
    HARL_PROF_BEGIN(st);
    launch_k(k_pack16, dim3(2), dim3(1024), 0, st, pk);
    HARL_CHECK_LAUNCH("k_pack16<value>");
  }
  return HARL_OK;
}

int harl_value_forward(const harl_mlp_desc* val, const double* feat, int64_t n,
                       int32_t feature_len, float* v_out, void* stream) {
  int rc = check_mlp(val, false);
  if (rc) return rc;
  if (val->dims[0] != feature_len || val->dims[val->n_layers] != 1 ||
      val->n_layers < 2) {
    set_error("value descriptor does not match");
    return HARL_E_ARG;
  }
  if (n <= 0) return HARL_OK;
  int ldbuf = 0;
  for (int l = 0; l <= val->n_layers; ++l) ldbuf = ldbuf > val->dims[l] ? ldbuf : val->dims[l];
  ldbuf += 1;
  const size_t smem = sizeof(float) * 2 * MLP_TM * (size_t)ldbuf;
  if ((rc = allow_smem(k_value_forward, smem, "k_value_forward"))) return rc;
  HARL_PROF_BEGIN((cudaStream_t)stream);
  launch_k(k_value_forward, dim3((unsigned)((n + MLP_TM - 1) / MLP_TM)), dim3(MLP_THREADS), smem, (cudaStream_t)stream, *val, feat, n, feature_len, v_out, ldbuf);
  HARL_CHECK_LAUNCH("k_value_forward");
  return HARL_OK;
}

int harl_gbt_finish_step(const harl_forest_desc* forest, int32_t feature_len,
                         const double* old_score, const harl_step_buffers* io, int64_t n, int64_t ld,
                         int64_t vbase, int32_t local_slots, double discount,
                         int32_t rl, const harl_replay_ring* ring, int64_t wpos,
                         int64_t keep_from, const harl_entry_log* log,
                         const harl_track_stats* ts, const int64_t* wpos_dev,
                         void* stream) {
  if (!forest || forest->n_trees < 0 || forest->n_trees > 1024 ||
      (forest->n_trees > 0 && (!forest->nodes || !forest->tree_first)) || !io ||
      !log || !ts || (rl && (!ring || ring->cap < 1))) {
    set_error("harl_gbt_finish_step: bad arguments");
    return HARL_E_ARG;
  }
  if (n <= 0) return HARL_OK;
  const int T = forest->n_trees > 0 ? forest->n_trees : 1;
  const int F = feature_len;
  const size_t cap = (size_t)max_dyn_smem();
  const bool smem_nodes = gbt2_smem_bytes(true, forest->n_nodes, T, F) <= cap;
  const size_t smem = gbt2_smem_bytes(smem_nodes, forest->n_nodes, T, F);
  if (smem > cap) {   // forest too large for the persistent kernel
    set_error("harl_gbt_finish_step: forest too large; use harl_gbt_predict + "
              "harl_finish_step");
    return HARL_E_LIMIT;
  }
  double* score = const_cast<double*>(io->new_score);
  double* reward = const_cast<double*>(io->reward);
  GbtFinishArgs fa;
  memset(&fa, 0, sizeof(fa));
  fa.a.n = n;
  fa.a.ld = ld;
  fa.a.vbase = vbase;
  fa.a.local_slots = local_slots;
  fa.a.F = F;
  fa.a.discount = discount;
  fa.a.rl = rl;
  fa.a.wpos = wpos;
  fa.a.keep_from = keep_from;
  fa.io = *io;
  if (ring) fa.ring = *ring;
  if (fa.ring.cap < 1) fa.ring.cap = 1;
  fa.log = *log;
  fa.ts = *ts;
  fa.wpos_dev = wpos_dev;
  const int64_t tiles = (n + GBT2_ROWS - 1) / GBT2_ROWS;
  const int64_t grid = tiles < sm_count() ? tiles : sm_count();
  int rc = smem_nodes ? allow_smem(k_gbt_finish<true>, smem, "k_gbt_finish")
                      : allow_smem(k_gbt_finish<false>, smem, "k_gbt_finish");
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  HARL_PROF_BEGIN(st);
  if (smem_nodes)
    launch_k(k_gbt_finish<true>, dim3((unsigned)grid), dim3(GBT2_THREADS), smem, st,
             (const GbtNode*)forest->nodes, forest->tree_first, forest->n_trees,
             forest->n_nodes, forest->fitted, forest->base, forest->floor_value,
             io->feat_new, n, F, score, old_score, reward,
             (const GbtHdr*)forest->dev_hdr, T, fa);
  else
    launch_k(k_gbt_finish<false>, dim3((unsigned)grid), dim3(GBT2_THREADS), smem, st,
             (const GbtNode*)forest->nodes, forest->tree_first, forest->n_trees,
             forest->n_nodes, forest->fitted, forest->base, forest->floor_value,
             io->feat_new, n, F, score, old_score, reward,
             (const GbtHdr*)forest->dev_hdr, T, fa);
  HARL_PROF_UNITS(n);
  HARL_CHECK_LAUNCH("k_gbt_finish");
  return HARL_OK;
}

int harl_finish_step(const harl_step_buffers* io, int64_t n, int64_t ld,
                     int64_t vbase, int32_t local_slots, int32_t feature_len,
                     double discount, int32_t rl, const harl_replay_ring* ring,
                     int64_t wpos, int64_t keep_from, const harl_entry_log* log,
                     const harl_track_stats* ts, const int64_t* wpos_dev,
                     void* stream) {
  if (!io || !log || !ts || (rl && (!ring || ring->cap < 1))) {
    set_error("harl_finish_step: bad arguments");
    return HARL_E_ARG;
  }
  if (n <= 0) return HARL_OK;
  FinishArgs a;
  memset(&a, 0, sizeof(a));
  a.n = n;
  a.ld = ld;
  a.vbase = vbase;
  a.local_slots = local_slots;
  a.F = feature_len;
  a.discount = discount;
  a.rl = rl;
  a.wpos = wpos;
  a.keep_from = keep_from;
  harl_replay_ring rg;
  memset(&rg, 0, sizeof(rg));
  if (ring) rg = *ring;
  if (rg.cap < 1) rg.cap = 1;
  HARL_PROF_BEGIN((cudaStream_t)stream);
  launch_k(k_finish_step, dim3((unsigned)((n + FIN_ROWS - 1) / FIN_ROWS)), dim3(FIN_THREADS),
           0, (cudaStream_t)stream, a, *io, rg, *log, *ts, wpos_dev);
  HARL_CHECK_LAUNCH("k_finish_step");
  return HARL_OK;
}

int harl_gather_rows(const int32_t* idx, int64_t n_out, int32_t local_slots,
                     int32_t feature_len, const uint16_t* tiles,
                     const uint8_t* knobs, const double* feat,
                     const double* score, const int32_t* row_track,
                     int64_t ld_src, uint16_t* tiles_o, uint8_t* knobs_o,
                     double* feat_o, double* score_o, int32_t* row_track_o,
                     int64_t ld_dst, void* stream) {
  if (n_out <= 0) return HARL_OK;
  GatherArgs a;
  a.n_out = n_out;
  a.ld_src = ld_src;
  a.ld_dst = ld_dst;
  a.local_slots = local_slots;
  a.F = feature_len;
  HARL_PROF_BEGIN((cudaStream_t)stream);
  const int64_t elems = n_out * (local_slots + 3 + feature_len + 2);
  int64_t gblocks = (elems + 255) / 256;
  if (gblocks > 8 * sm_count()) gblocks = 8 * sm_count();
  launch_k(k_gather_rows, dim3((unsigned)gblocks), dim3(256), 0, (cudaStream_t)stream, 
      a, idx, tiles, knobs, feat, score, row_track, tiles_o, knobs_o, feat_o,
      score_o, row_track_o);
  HARL_CHECK_LAUNCH("k_gather_rows");
  return HARL_OK;
}

// ---------------------------------------------------------------------------
// rank_scores on the entry log (rank_kernels.cuh)

static int64_t rank_table_size(int64_t items) {
  int64_t t = 1024;
  while (t < 2 * items) t <<= 1;
  return t;
}

static int64_t align256(int64_t x) { return (x + 255) & ~(int64_t)255; }

int64_t harl_rank_scratch_bytes(int64_t n_visits, int64_t n_excluded) {
  if (n_visits < 0 || n_excluded < 0) return -1;
  const int64_t T = rank_table_size(n_visits + n_excluded);
  return align256((int64_t)sizeof(RankState)) + align256(T * 8) +
         align256(T * 4) + align256(n_visits > 0 ? n_visits : 1);
}

int harl_rank_topk(const harl_entry_log* log, int32_t local_slots,
                   int64_t n_visits, const uint16_t* ex_tiles,
                   const uint8_t* ex_knobs, int64_t ex_ld, int64_t n_excluded,
                   int64_t k, void* scratch, int64_t scratch_bytes,
                   int32_t* out_idx, int64_t out_cap, int64_t* stats,
                   void* stream) {
  if (!log || !scratch || !out_idx || !stats || n_visits < 0 ||
      n_excluded < 0 || k < 0 || local_slots < 0) {
    set_error("harl_rank_topk: bad arguments");
    return HARL_E_ARG;
  }
  if (n_visits + n_excluded >= (int64_t)INT_MAX) {
    set_error("harl_rank_topk: %lld items exceed the int32 index range",
              (long long)(n_visits + n_excluded));
    return HARL_E_ARG;
  }
  if (n_excluded > 0 && (!ex_tiles && local_slots > 0 || !ex_knobs)) {
    set_error("harl_rank_topk: excluded states without arrays");
    return HARL_E_ARG;
  }
  if (scratch_bytes < harl_rank_scratch_bytes(n_visits, n_excluded)) {
    set_error("harl_rank_topk: scratch too small");
    return HARL_E_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t T = rank_table_size(n_visits + n_excluded);
  char* p = (char*)scratch;
  RankArgs a;
  memset(&a, 0, sizeof(a));
  a.st = (RankState*)p;
  p += align256((int64_t)sizeof(RankState));
  a.keys = (unsigned long long*)p;
  p += align256(T * 8);
  a.reps = (int32_t*)p;
  p += align256(T * 4);
  a.keep = (uint8_t*)p;
  a.tiles = log->tiles;
  a.knobs = log->knobs;
  a.score = log->score;
  a.ld = log->ld;
  a.V = n_visits;
  a.ex_tiles = ex_tiles;
  a.ex_knobs = ex_knobs;
  a.ex_ld = ex_ld;
  a.E = n_excluded;
  a.slots = local_slots;
  a.tmask = T - 1;
  a.k = k;
  a.out_idx = out_idx;
  a.out_cap = out_cap;
  cudaError_t e;
  if ((e = cudaMemsetAsync(a.st, 0, sizeof(RankState), st)) != cudaSuccess ||
      (e = cudaMemsetAsync(a.keys, 0, (size_t)T * 8, st)) != cudaSuccess ||
      (e = cudaMemsetAsync(a.reps, 0x7f, (size_t)T * 4, st)) != cudaSuccess)
    return cuda_status(e, "harl_rank_topk memset");
  const int64_t items = n_visits + n_excluded;
  const int cap = sm_count() * 8;
  auto grid = [&](int64_t n) {
    int64_t g = (n + 255) / 256;
    return (unsigned)(g < 1 ? 1 : (g > cap ? cap : g));
  };
  if (items > 0) {
    HARL_PROF_BEGIN(st);
    launch_k(k_rank_insert, dim3(grid(items)), dim3(256), 0, st, a);
    HARL_CHECK_LAUNCH("k_rank_insert");
  }
  if (n_visits > 0) {
    HARL_PROF_BEGIN(st);
    launch_k(k_rank_mark, dim3(grid(n_visits)), dim3(256), 0, st, a);
    HARL_CHECK_LAUNCH("k_rank_mark");
  }
  for (int d = 0; d < 12; ++d) {
    HARL_PROF_BEGIN(st);
    launch_k(k_rank_select, dim3(grid(n_visits)), dim3(256), 0, st, a, d);
    HARL_CHECK_LAUNCH("k_rank_select");
  }
  if (n_visits > 0) {
    HARL_PROF_BEGIN(st);
    launch_k(k_rank_emit, dim3(grid(n_visits)), dim3(256), 0, st, a);
    HARL_CHECK_LAUNCH("k_rank_emit");
  }
  HARL_PROF_BEGIN(st);
  launch_k(k_rank_stats, dim3(1), dim3(1), 0, st, a, stats);
  HARL_CHECK_LAUNCH("k_rank_stats");
  return HARL_OK;
}

// ---------------------------------------------------------------------------
// GBT refit (gbt_fit_kernels.cuh)

struct FitLayout {
  int64_t pred, resid, sorted_all, ord0, ord1, srt0, srt1, node_of, goleft,
      seg_start, seg_count, state, nleft, feat, thr, total, bgain, bpos, ctl,
      bytes;
};

static FitLayout fit_layout(int64_t n, int64_t F, int max_depth) {
  FitLayout L;
  const int64_t K = ((int64_t)1 << (max_depth + 1)) - 1;
  const int64_t NL = (int64_t)1 << max_depth;
  int64_t o = 0;
  auto take = [&](int64_t bytes) { int64_t r = o; o += align256(bytes); return r; };
  L.pred = take(n * 8);
  L.resid = take(n * 8);
  L.sorted_all = take(F * n * 4);
  L.ord0 = take(n * 4);
  L.ord1 = take(n * 4);
  L.srt0 = take(F * n * 4);
  L.srt1 = take(F * n * 4);
  L.node_of = take(n * 4);
  L.goleft = take(n * 4);
  L.seg_start = take(K * 4);
  L.seg_count = take(K * 4);
  L.state = take(K * 4);
  L.nleft = take(K * 4);
  L.feat = take(K * 4);
  L.thr = take(K * 8);
  L.total = take(K * 8);
  L.bgain = take(NL * F * 8);
  L.bpos = take(NL * F * 4);
  L.ctl = take((int64_t)sizeof(FitCtl));
  L.bytes = o;
  return L;
}

static int build_grad_jobs(const harl_net_layout& P, const harl_net_layout& V,
                           GradJob* jobs, int* n_jobs, int* n_tiles) {
  int nj = 0, tiles = 0;
  auto add = [&](int a_off, int ni, int d_off, int njj, int64_t g_off) {
    GradJob& j = jobs[nj++];
    j.a_off = a_off;
    j.ni = ni;
    j.d_off = d_off;
    j.nj = njj;
    j.g_off = g_off;
    j.tile_first = tiles;
    const int ti = ni == 0 ? 1 : (ni + WG_T - 1) / WG_T;
    tiles += ti * ((njj + WG_T - 1) / WG_T);
  };
  for (int l = 0; l < P.n_layers; ++l) {
    add(P.row_act[l], P.dims[l], P.row_delta[l], P.dims[l + 1], P.off_W[l]);
    add(0, 0, P.row_delta[l], P.dims[l + 1], P.off_b[l]);
  }
  add(P.row_act[P.n_layers], P.dims[P.n_layers], P.row_head, P.n_head_cols, P.off_hW);
  add(0, 0, P.row_head, P.n_head_cols, P.off_hb);
  for (int l = 0; l < V.n_layers; ++l) {
    add(V.row_act[l], V.dims[l], V.row_delta[l], V.dims[l + 1], V.off_W[l]);
    add(0, 0, V.row_delta[l], V.dims[l + 1], V.off_b[l]);
  }
  *n_jobs = nj;
  *n_tiles = tiles;
  return HARL_OK;
}

int harl_selftest_tcgen05(const float* A, const float* B, float* D, int mode,
                          void* stream) {
  const size_t smem = (PROBE_N + PROBE_M) * PROBE_K * 4 + 1024;
  if (mode >= 6) {
    int rc = allow_smem(k_tc_probe_f16, smem, "k_tc_probe_f16");
    if (rc) return rc;
    HARL_PROF_BEGIN((cudaStream_t)stream);
    launch_k(k_tc_probe_f16, dim3(1), dim3(128), smem, (cudaStream_t)stream, A, B, D, mode);
    HARL_CHECK_LAUNCH("k_tc_probe_f16");
    return HARL_OK;
  }
  if (mode >= 3) {
    int rc = allow_smem(k_tc_probe_m64, smem, "k_tc_probe_m64");
    if (rc) return rc;
    HARL_PROF_BEGIN((cudaStream_t)stream);
    launch_k(k_tc_probe_m64, dim3(1), dim3(128), smem, (cudaStream_t)stream, A, B, D, mode);
    HARL_CHECK_LAUNCH("k_tc_probe_m64");
    return HARL_OK;
  }
  int rc = allow_smem(k_tc_probe, smem, "k_tc_probe");
  if (rc) return rc;
  HARL_PROF_BEGIN((cudaStream_t)stream);
  launch_k(k_tc_probe, dim3(1), dim3(128), smem, (cudaStream_t)stream, A, B, D, mode);
  HARL_CHECK_LAUNCH("k_tc_probe");
  return HARL_OK;
}

static void build_trans_plan(const harl_net_layout& P, const harl_net_layout& V,
                             TransPlan* tp, PpoArgs* a) {
  memset(tp, 0, sizeof(*tp));
  int64_t dst = 0;
  auto add = [&](int64_t off, int K, int N) -> int64_t {
    const int64_t d = dst;
    tp->m[tp->n++] = {off, d, K, N};
    dst += (int64_t)K * N;
    return d;
  };
  const int H = P.dims[P.n_layers];
  const int64_t h = add(P.off_hW, H, P.n_head_cols);
  if (a) a->wt_head = h;
  for (int l = 1; l < P.n_layers; ++l) {
    const int64_t d = add(P.off_W[l], P.dims[l], P.dims[l + 1]);
    if (a) a->wt_P[l] = d;
  }
  for (int l = 1; l < V.n_layers; ++l) {
    const int64_t d = add(V.off_W[l], V.dims[l], V.dims[l + 1]);
    if (a) a->wt_V[l] = d;
  }
  tp->total = dst;
}

int64_t harl_ppo_wt_doubles(const harl_net_layout* pol, const harl_net_layout* val) {
  if (!pol || !val) return 0;
  TransPlan tp;
  build_trans_plan(*pol, *val, &tp, nullptr);
  return tp.total;
}

int harl_ppo_wt_fill(const harl_net_layout* pol, const harl_net_layout* val,
                     const double* params, double* wt, void* stream) {
  if (!pol || !val || !params || !wt) {
    set_error("harl_ppo_wt_fill: null argument");
    return HARL_E_ARG;
  }
  TransPlan tp;
  build_trans_plan(*pol, *val, &tp, nullptr);
  HARL_PROF_BEGIN((cudaStream_t)stream);
  launch_k(k_wt_fill, dim3(148), dim3(256), 0, (cudaStream_t)stream, tp, params, wt);
  HARL_CHECK_LAUNCH("k_wt_fill");
  return HARL_OK;
}

int64_t harl_ppo_scratch_bytes(int32_t B, int32_t row_stride, int32_t n_jobs) {
  (void)n_jobs;
  return (int64_t)B * row_stride * 8 + (int64_t)B * 4 * 8 +
         (int64_t)sizeof(GradJob) * 4 * (HARL_MAX_LAYERS + 2) + 256;
}

// HARL_PPO_FUSED_ADAM=1: k_ppo_wgrad + k_ppo_adam as one cooperative
// kernel (its whole grid co-resident, a grid barrier between gradients and
// Adam).  Bit-identical; the kernel itself is shorter (19.3 us live vs
// 13.1 + 9.3) but the C2 episode measured slower (5.83-5.94 vs 5.79 ms):
// the cooperative node costs more in the graph than the launch it saves.
static bool fused_wgrad_adam_ok(int grid) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("HARL_PPO_FUSED_ADAM");
    env = (e && e[0] == '1') ? 1 : 0;
  }
  if (!env || use_pdl()) return false;
  static int per_sm = -1;
  if (per_sm < 0) {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_ppo_wgrad_adam, 256, 0) !=
        cudaSuccess)
      nb = 0;
    per_sm = nb;
  }
  return (int64_t)per_sm * sm_count() >= grid;
}

// the grid barrier's {arrival count, generation} words (zeroed once)
static int ppo_barrier_words(unsigned int** out) {
  static unsigned int* words = nullptr;
  std::lock_guard<std::mutex> lk(g_tab_mu);
  if (!words) {
    cudaError_t e = cudaMalloc(&words, 2 * sizeof(unsigned int));
    if (e == cudaSuccess) e = cudaMemset(words, 0, 2 * sizeof(unsigned int));
    if (e != cudaSuccess) {
      words = nullptr;
      return cuda_status(e, "ppo barrier alloc");
    }
  }
  *out = words;
  return HARL_OK;
}

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
                    int32_t phase, void* stream) {
  if (B_norm <= 0) B_norm = B;
  // HARL_PPO_SPECULATIVE: gradients + Adam in one launch (k_ppo_wgrad_spec);
  // the pre-update values go to the backup block behind params/m/v
  const bool spec = (phase & HARL_PPO_SPECULATIVE) != 0;
  phase &= 3;
  if (phase < 1 || phase > 3) phase = 3;
  if (spec && phase != 3) {
    set_error("harl_ppo_update: the speculative update is single-device (phase 3)");
    return HARL_E_ARG;
  }
  if (spec && (adam_m != params + n_params || adam_v != params + 2 * n_params)) {
    set_error("harl_ppo_update: the speculative update needs params, m, v and "
              "the backup as consecutive [n_params] rows of one block");
    return HARL_E_ARG;
  }
  if (!pol || !val || !hp || !ring || B < 0 || n_head0 < 1 ||
      n_head0 > HARL_MAX_HEAD0 || pol->n_layers < 1 ||
      pol->n_layers > HARL_MAX_LAYERS || val->n_layers < 2 ||
      val->n_layers > HARL_MAX_LAYERS) {
    set_error("harl_ppo_update: bad arguments");
    return HARL_E_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  char* sc = (char*)scratch;
  double* rows = (double*)sc;
  double* rowout = rows + (int64_t)B * row_stride;
  GradJob jobs[4 * (HARL_MAX_LAYERS + 2)];
  int n_jobs = 0, n_tiles = 0;
  build_grad_jobs(*pol, *val, jobs, &n_jobs, &n_tiles);
  // the job table is passed by value (no host->device copy: the call is
  // legal inside CUDA-graph capture)
  PpoArgs a;
  memset(&a, 0, sizeof(a));
  a.B = B;
  a.F = feature_len;
  a.C0 = n_head0;
  a.row_stride = row_stride;
  a.B_norm = B_norm;
  a.clip_lo = 1.0 - hp->clip_ratio;
  a.clip_hi = 1.0 + hp->clip_ratio;
  a.w_ent = hp->entropy_weight;
  a.w_val = hp->value_loss_weight;
  a.bad = spec ? bad : nullptr;
  for (int j = 0; j < n_head0; ++j) a.head0_src[j] = head0_src_host[j];
  TransPlan tplan;
  build_trans_plan(*pol, *val, &tplan, &a);
  if (!wt_params) {
    set_error("harl_ppo_update: wt_params (transposed weights) required");
    return HARL_E_ARG;
  }
  int wmax = 0;
  for (int l = 0; l <= pol->n_layers; ++l) wmax = wmax > pol->dims[l] ? wmax : pol->dims[l];
  for (int l = 0; l <= val->n_layers; ++l) wmax = wmax > val->dims[l] ? wmax : val->dims[l];
  wmax = wmax > pol->n_head_cols ? wmax : pol->n_head_cols;
  // rows + the split-reduction partials (PPO_SPLIT x PPO_TM x widest layer)
  const size_t rsmem = sizeof(double) * (PPO_TM * (size_t)row_stride + 8 +
                                         (size_t)PPO_SPLIT * PPO_TM * wmax);
  AdamArgs ad;
  memset(&ad, 0, sizeof(ad));
  ad.n_pi = n_pi;
  ad.n = n_params;
  ad.h = *hp;
  // images as built by k_pack_trunk / k_pack_heads (mlp_tc.cuh)
  // ... and, behind each trunk image, the 3xFP16 image (mlp_f16.cuh)
  auto add_trunk = [&](const harl_net_layout& L, uint8_t* img, bool value) {
    const int H = TC_H;
    float* w1h = (float*)img;
    float* w1l = w1h + TC_K1 * H;
    float* w2h = w1l + TC_K1 * H;
    float* w2l = w2h + H * H;
    float* bb = w2l + H * H;
    uint8_t* f = img + TRUNK_IMAGE;
    float* ff = (float*)f;
    uint16_t* h1 = (uint16_t*)(f + f16_off_w1());
    uint16_t* h2 = (uint16_t*)(f + f16_off_w2());
    ad.pk.mat[ad.pk.n_mat++] = {L.off_W[0], L.dims[0], H, TC_K1, w1h, w1l,
                                h1, h1 + F16_W1 / 2, ff + F16_SC + 0};
    ad.pk.mat[ad.pk.n_mat++] = {L.off_W[1], H, H, H, w2h, w2l,
                                h2, h2 + F16_W2 / 2, ff + F16_SC + 1};
    ad.pk.vec[ad.pk.n_vec++] = {L.off_b[0], H, bb};
    ad.pk.vec[ad.pk.n_vec++] = {L.off_b[1], H, bb + H};
    ad.pk.vec[ad.pk.n_vec++] = {L.off_b[0], H, ff + F16_B1};
    ad.pk.vec[ad.pk.n_vec++] = {L.off_b[1], H, ff + F16_B2};
    if (value) {
      ad.pk.vec[ad.pk.n_vec++] = {L.off_W[2], H, bb + 2 * H};
      ad.pk.vec[ad.pk.n_vec++] = {L.off_W[2], H, ff + F16_B3};
    }
  };
  if (pol_trunk_img && pol_heads_img) {
    add_trunk(*pol, (uint8_t*)pol_trunk_img, false);
    const int NHP = (pol->n_head_cols + 15) / 16 * 16;
    float* whh = (float*)pol_heads_img;
    float* whl = whh + NHP * TC_H;
    uint8_t* f = (uint8_t*)pol_trunk_img + TRUNK_IMAGE;
    uint16_t* hh = (uint16_t*)(f + f16_off_wh());
    const bool f16 = NHP <= F16_NHP_MAX;
    ad.pk.mat[ad.pk.n_mat++] = {pol->off_hW, TC_H, pol->n_head_cols, TC_H,
                                whh, whl, f16 ? hh : nullptr,
                                hh + NHP * TC_H, (float*)f + F16_SC + 2};
    ad.pk.vec[ad.pk.n_vec++] = {pol->off_hb, pol->n_head_cols, whl + NHP * TC_H};
    if (f16)
      ad.pk.vec[ad.pk.n_vec++] = {pol->off_hb, pol->n_head_cols,
                                  (float*)f + F16_B3};
  }
  if (val_trunk_img) add_trunk(*val, (uint8_t*)val_trunk_img, true);
  ad.tp = tplan;
  ad.wt = wt_params;
  if (phase & 1) {
  if (use_ppo_cl() && ppo_cl_shape(*pol, *val, feature_len)) {
    // thread-block clusters: 8 CTAs x 32 rows, weight slices in shared
    // memory, activations exchanged through distributed shared memory
    const size_t csmem = pcl_smem_bytes(feature_len);
    int rc2 = allow_smem(k_ppo_rows_cl, csmem, "k_ppo_rows_cl");
    if (rc2) return rc2;
    if (B > 0) {
      HARL_PROF_BEGIN(st);
      launch_k(k_ppo_rows_cl, dim3((unsigned)((B + PCL_R - 1) / PCL_R * PCL_CTAS), 2),
               dim3(PCL_THREADS), csmem, st, a, *pol, *val, *ring, idx, params,
               rows, rowout);
      HARL_PROF_UNITS(B);
      HARL_CHECK_LAUNCH("k_ppo_rows_cl");
    }
  } else if (use_ppo_tc()) {
    // fp64 tensor-core rows kernel: 8 rows per CTA in shared memory
    const size_t tsmem = sizeof(double) * (size_t)PPO8_ROWS * row_stride;
    int rc2 = allow_smem(k_ppo_rows_tc, tsmem, "k_ppo_rows_tc");
    if (rc2) return rc2;
    if (B > 0) {
      HARL_PROF_BEGIN(st);
      launch_k(k_ppo_rows_tc, dim3((unsigned)((B + PPO8_ROWS - 1) / PPO8_ROWS), 2),
               dim3(PPO8_THREADS), tsmem, st, a, *pol, *val, *ring, idx, params,
               wt_params, rows, rowout);
      HARL_PROF_UNITS(B);
      HARL_CHECK_LAUNCH("k_ppo_rows_tc");
    }
  } else {
    int rc2 = allow_smem(k_ppo_rows, rsmem, "k_ppo_rows");
    if (rc2) return rc2;
    if (B > 0) {
      HARL_PROF_BEGIN(st);
      launch_k(k_ppo_rows, dim3((unsigned)((B + PPO_TM - 1) / PPO_TM), 2), dim3(PPO_THREADS), rsmem, st, 
          a, *pol, *val, *ring, idx, params, wt_params, rows, rowout);
      HARL_PROF_UNITS(B);
      HARL_CHECK_LAUNCH("k_ppo_rows");
    }
  }
  GradJobs jt;
  memset(&jt, 0, sizeof(jt));
  for (int j = 0; j < n_jobs; ++j) jt.j[j] = jobs[j];
  jt.n = n_jobs;
  // one extra CTA sums the per-row loss terms (and, on a single device,
  // forms the means and checks them) alongside the gradient tiles
  if (spec) {
    HARL_PROF_BEGIN(st);
    launch_k(k_ppo_wgrad_spec, dim3((unsigned)n_tiles + 1), dim3(256), 0, st, jt, B,
             row_stride, (const double*)rows, grads, bad, (const double*)rowout, losses,
             B_norm, hp->entropy_weight, hp->value_loss_weight, ad, adam_dev, params,
             adam_m, adam_v, params32, params + 3 * n_params);
    HARL_PROF_UNITS(B);
    HARL_CHECK_LAUNCH("k_ppo_wgrad_spec");
    return HARL_OK;
  }
  if (phase == 3 && fused_wgrad_adam_ok(n_tiles + 1)) {
    // gradients and Adam in one cooperative launch (grid barrier between)
    unsigned int* barw = nullptr;
    int rcb = ppo_barrier_words(&barw);
    if (rcb) return rcb;
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3((unsigned)n_tiles + 1);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    HARL_PROF_BEGIN(st);
    cudaLaunchKernelEx(&cfg, k_ppo_wgrad_adam, jt, B, row_stride,
                       (const double*)rows, grads, bad, (const double*)rowout,
                       losses, B_norm, hp->entropy_weight,
                       hp->value_loss_weight, ad, adam_dev, params, adam_m,
                       adam_v, params32, barw);
    HARL_CHECK_LAUNCH("k_ppo_wgrad_adam");
    return HARL_OK;
  }
  HARL_PROF_BEGIN(st);
  launch_k(k_ppo_wgrad, dim3((unsigned)n_tiles + 1), dim3(256), 0, st, jt, B, row_stride,
           rows, grads, bad, phase == 3 ? 1 : 0, (const double*)rowout, losses,
           phase == 3 ? B_norm : 0, hp->entropy_weight, hp->value_loss_weight);
  HARL_PROF_UNITS(B);
  HARL_CHECK_LAUNCH("k_ppo_wgrad");
  }
  if (!(phase & 2)) return HARL_OK;
  if (phase == 2) {   // sharded: means and checks over the all-reduced sums
    HARL_PROF_BEGIN(st);
    launch_k(k_ppo_finalize, dim3(148), dim3(256), 0, st, B_norm, hp->entropy_weight,
                                        hp->value_loss_weight, losses, grads,
                                        n_params, bad);
    HARL_CHECK_LAUNCH("k_ppo_finalize");
  }
  HARL_PROF_BEGIN(st);
  launch_k(k_ppo_adam, dim3(296), dim3(256), 0, st, ad, adam_dev, bad, grads, params, adam_m,
                                   adam_v, params32);
  HARL_CHECK_LAUNCH("k_ppo_adam");
  return HARL_OK;
}

// -- launch counter / per-kernel timer ----------------------------------------

long long harl_launch_count(void) { return g_launches.load(); }

int harl_debug_timestamps(int on, unsigned long long* out_host, int n) {
  if (on) {
    unsigned long long init[4] = {~0ull, 0ull, 0ull, 0ull};
    cudaError_t e0 = cudaMemcpyToSymbol(g_dbg_ts, init, sizeof(init),
                                        60 * sizeof(unsigned long long));
    if (e0 != cudaSuccess) return cuda_status(e0, "harl_debug_timestamps");
  }
  cudaError_t e = cudaMemcpyToSymbol(g_dbg_on, &on, sizeof(int));
  if (e != cudaSuccess) return cuda_status(e, "harl_debug_timestamps");
  if (out_host && n > 0) {
    e = cudaMemcpyFromSymbol(out_host, g_dbg_ts,
                             sizeof(unsigned long long) * (n < 64 ? n : 64));
    if (e != cudaSuccess) return cuda_status(e, "harl_debug_timestamps");
  }
  return HARL_OK;
}

int harl_profile_set(int on, long long spin_ns) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_on = on != 0;
  if (spin_ns >= 0) g_spin_ns = (unsigned long long)spin_ns;
  return HARL_OK;
}

int harl_profile_reset(void) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_recs.clear();
  g_ev_used = 0;
  return HARL_OK;
}

int harl_profile_read(int max_kernels, char* names, int name_cap,
                      double* total_ms, long long* launches,
                      long long* units) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  std::vector<std::string> keys;
  std::vector<double> ms;
  std::vector<long long> cnt, un;
  for (const ProfRec& r : g_prof_recs) {
    cudaError_t e = cudaEventSynchronize(r.e1);
    if (e != cudaSuccess) return cuda_status(e, "harl_profile_read");
    float t = 0.f;
    e = cudaEventElapsedTime(&t, r.e0, r.e1);
    if (e != cudaSuccess) return cuda_status(e, "harl_profile_read");
    size_t k = 0;
    while (k < keys.size() && keys[k] != r.name) ++k;
    if (k == keys.size()) {
      keys.push_back(r.name);
      ms.push_back(0.0);
      cnt.push_back(0);
      un.push_back(0);
    }
    ms[k] += t;
    cnt[k] += 1;
    // a launch whose units are unknown poisons the kernel's total
    if (un[k] >= 0) un[k] = r.units >= 0 ? un[k] + r.units : -1;
  }
  const int n = (int)keys.size();
  for (int k = 0; k < n && k < max_kernels; ++k) {
    if (names && name_cap > 0) {
      snprintf(names + (size_t)k * name_cap, (size_t)name_cap, "%s",
               keys[k].c_str());
    }
    if (total_ms) total_ms[k] = ms[k];
    if (launches) launches[k] = cnt[k];
    if (units) units[k] = un[k];
  }
  return n;
}


int64_t harl_gbt_fit_scratch_bytes(int32_t n, int32_t feature_len,
                                   int32_t max_depth) {
  if (n < 1 || feature_len < 1 || max_depth < 0 || max_depth > FIT_MAX_DEPTH)
    return -1;
  return fit_layout(n, feature_len, max_depth).bytes;
}

int harl_gbt_fit(const double* X, const double* y, int32_t n,
                 int32_t feature_len, int32_t n_trees, int32_t max_depth,
                 double learning_rate, int32_t min_leaf, void* scratch,
                 int64_t scratch_bytes, int32_t* out_feat, double* out_thr,
                 double* out_val, double* out_pred, double* out_base,
                 int32_t* out_ntrees, const int32_t* n_dev, void* stream) {
  if (!X || !y || n < 1 || feature_len < 1 || n_trees < 0 || max_depth < 0 ||
      min_leaf < 1 || !scratch || !out_feat || !out_thr || !out_val ||
      !out_pred || !out_base || !out_ntrees) {
    set_error("harl_gbt_fit: bad arguments");
    return HARL_E_ARG;
  }
  if (n > FIT_MAX_N || max_depth > FIT_MAX_DEPTH) {
    set_error("harl_gbt_fit: n %d > %d or depth %d > %d", n, FIT_MAX_N,
              max_depth, FIT_MAX_DEPTH);
    return HARL_E_LIMIT;
  }
  const FitLayout L = fit_layout(n, feature_len, max_depth);
  if (scratch_bytes < L.bytes) {
    set_error("harl_gbt_fit: scratch too small");
    return HARL_E_ARG;
  }
  char* p = (char*)scratch;
  FitArgs a;
  memset(&a, 0, sizeof(a));
  a.X = X;
  a.y = y;
  a.n = n;
  a.ncap = n;
  a.n_dev = n_dev;
  a.F = feature_len;
  a.K = (1 << (max_depth + 1)) - 1;
  a.max_depth = max_depth;
  a.min_leaf = min_leaf;
  a.lr = learning_rate;
  a.pred = out_pred;   // the running prediction lives in the output
  a.resid = (double*)(p + L.resid);
  a.sorted_all = (const int32_t*)(p + L.sorted_all);
  a.ord[0] = (int32_t*)(p + L.ord0);
  a.ord[1] = (int32_t*)(p + L.ord1);
  a.srt[0] = (int32_t*)(p + L.srt0);
  a.srt[1] = (int32_t*)(p + L.srt1);
  a.node_of = (int32_t*)(p + L.node_of);
  a.goleft = (int32_t*)(p + L.goleft);
  a.seg_start = (int32_t*)(p + L.seg_start);
  a.seg_count = (int32_t*)(p + L.seg_count);
  a.state = (int32_t*)(p + L.state);
  a.nleft = (int32_t*)(p + L.nleft);
  a.feat = (int32_t*)(p + L.feat);
  a.thr = (double*)(p + L.thr);
  a.total = (double*)(p + L.total);
  a.bgain = (double*)(p + L.bgain);
  a.bpos = (int32_t*)(p + L.bpos);
  a.ctl = (FitCtl*)(p + L.ctl);
  a.out_feat = out_feat;
  a.out_thr = out_thr;
  a.out_val = out_val;
  cudaStream_t st = (cudaStream_t)stream;
  int P2 = 1;
  while (P2 < n) P2 <<= 1;
  const size_t ssmem = (size_t)P2 * 12;
  int rc = allow_smem(k_fit_presort, ssmem, "k_fit_presort");
  if (rc) return rc;
  const unsigned gn = (unsigned)((n + 255) / 256 < sm_count() * 4 ? (n + 255) / 256 : sm_count() * 4);
  HARL_PROF_BEGIN(st);
  launch_k(k_fit_presort, dim3(feature_len), dim3(1024), ssmem, st, X, (int)n,
           n_dev, (int)feature_len, P2, (int)n, (int32_t*)a.sorted_all);
  HARL_CHECK_LAUNCH("k_fit_presort");
  HARL_PROF_BEGIN(st);
  launch_k(k_fit_iota, dim3(gn), dim3(256), 0, st, a.ord[0], (int)n, n_dev);
  HARL_CHECK_LAUNCH("k_fit_iota");
  HARL_PROF_BEGIN(st);
  launch_k(k_fit_base, dim3(1), dim3(256), 0, st, a);
  HARL_CHECK_LAUNCH("k_fit_base");
  const unsigned ginit = (unsigned)sm_count() * 4;
  for (int t = 0; t < n_trees; ++t) {
    HARL_PROF_BEGIN(st);
    launch_k(k_fit_tree_init, dim3(ginit), dim3(256), 0, st, a);
    HARL_CHECK_LAUNCH("k_fit_tree_init");
    HARL_PROF_BEGIN(st);
    launch_k(k_fit_tree_check, dim3(1), dim3(1), 0, st, a, t);
    HARL_CHECK_LAUNCH("k_fit_tree_check");
    for (int d = 0; d <= max_depth; ++d) {
      const int nl = 1 << d, lists = d & 1;
      HARL_PROF_BEGIN(st);
      launch_k(k_fit_stats, dim3(nl), dim3(128), 0, st, a, d, t, lists);
      HARL_CHECK_LAUNCH("k_fit_stats");
      if (d == max_depth) break;
      const int64_t wb = (int64_t)nl * feature_len * 32;
      HARL_PROF_BEGIN(st);
      launch_k(k_fit_best, dim3((unsigned)((wb + 255) / 256)), dim3(256), 0, st, a, d, lists);
      HARL_CHECK_LAUNCH("k_fit_best");
      HARL_PROF_BEGIN(st);
      launch_k(k_fit_split, dim3((unsigned)((nl + 127) / 128)), dim3(128), 0, st, a, d, lists);
      HARL_CHECK_LAUNCH("k_fit_split");
      HARL_PROF_BEGIN(st);
      launch_k(k_fit_route, dim3(gn), dim3(256), 0, st, a);
      HARL_CHECK_LAUNCH("k_fit_route");
      HARL_PROF_BEGIN(st);
      launch_k(k_fit_commit, dim3((unsigned)((nl + 127) / 128)), dim3(128), 0, st, a, d, t);
      HARL_CHECK_LAUNCH("k_fit_commit");
      const int64_t wp = (int64_t)nl * (feature_len + 1) * 32;
      HARL_PROF_BEGIN(st);
      launch_k(k_fit_partition, dim3((unsigned)((wp + 255) / 256)), dim3(256), 0, st, a, d, lists);
      HARL_CHECK_LAUNCH("k_fit_partition");
    }
    HARL_PROF_BEGIN(st);
    launch_k(k_fit_pred, dim3(gn), dim3(256), 0, st, a, t);
    HARL_CHECK_LAUNCH("k_fit_pred");
  }
  cudaError_t e;
  if ((e = cudaMemcpyAsync(out_base, &a.ctl->base, 8, cudaMemcpyDeviceToDevice, st)) != cudaSuccess ||
      (e = cudaMemcpyAsync(out_ntrees, &a.ctl->n_built, 4, cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
    return cuda_status(e, "harl_gbt_fit outputs");
  return HARL_OK;
}


// TrackSet.cull (stopping.py:68-86) on the host: the n_elim live tracks
// with the lowest (advantage, -index) go, for finite advantages (the
// engine routes a step with a NaN advantage to shard.eliminated, which runs
// the reference's own comparison sort; here NaN keys would order last; -0.0
// ties with +0.0 as in Python's comparisons).  rows: the cull step's m rows (row r = track
// tracks[r], advantage adv[r]); alive (per track, 0/1) is updated; gone_out
// gets the eliminated track ids ascending, keep_out the surviving rows
// ascending (the survivor gather's index list).
int harl_cull_select(const double* adv, const int32_t* tracks, int64_t m,
                     uint8_t* alive, int64_t n_tracks, int64_t n_elim,
                     int64_t* gone_out, int32_t* keep_out, int64_t* n_keep) {
  if (!adv || !tracks || !alive || m < 0 || n_elim < 0 || n_elim > m ||
      (n_elim && !gone_out) || !keep_out || !n_keep) {
    set_error("harl_cull_select: bad arguments");
    return HARL_E_ARG;
  }
  for (int64_t r = 0; r < m; ++r)
    if (tracks[r] < 0 || tracks[r] >= n_tracks || !alive[tracks[r]]) {
      set_error("harl_cull_select: row %lld is not a live track", (long long)r);
      return HARL_E_ARG;
    }
  if (n_elim > 0) {
    // ordered 64-bit keys (NaN last); the cut = the n_elim-th smallest key,
    // found by an MSB radix select (11-bit digits, each pass over the rows
    // still in the cut's bucket); everything below goes, ties at the cut go
    // by descending track index
    static thread_local std::vector<uint64_t> key, cand;
    key.resize((size_t)m);
    cand.resize((size_t)m);
    const uint64_t* bits = reinterpret_cast<const uint64_t*>(adv);
    for (int64_t r = 0; r < m; ++r) {
      uint64_t b = bits[r];
      if (b == 0x8000000000000000ull) b = 0;   // -0.0 ties with +0.0
      const bool nan = (b & 0x7fffffffffffffffull) > 0x7ff0000000000000ull;
      key[r] = nan ? ~0ull : ((b >> 63) ? ~b : (b | 0x8000000000000000ull));
    }
    uint64_t rank = (uint64_t)(n_elim - 1), prefix = 0;
    const uint64_t* src = key.data();
    int64_t n = m;
    uint32_t hist[2048];
    static const int kShift[6] = {53, 42, 31, 20, 9, 0};   // 5 x 11 + 9 bits
    for (int pass = 0; pass < 6; ++pass) {
      const int shift = kShift[pass], width = pass < 5 ? 11 : 9;
      const uint64_t dmask = (1ull << width) - 1;
      memset(hist, 0, sizeof(uint32_t) << width);
      for (int64_t i = 0; i < n; ++i) ++hist[(src[i] >> shift) & dmask];
      uint64_t d = 0, below = 0;
      while (below + hist[d] <= rank) below += hist[d++];
      rank -= below;
      prefix |= d << shift;
      // keep the bucket's keys
      int64_t c = 0;
      for (int64_t i = 0; i < n; ++i)
        if (((src[i] >> shift) & dmask) == d) cand[c++] = src[i];
      src = cand.data();
      n = c;
      if (n == 1) {
        prefix = cand[0];
        break;
      }
    }
    const uint64_t cut = prefix;
    static thread_local std::vector<int32_t> tied;
    static thread_local std::vector<uint64_t> elim;   // eliminated-track bitmap
    tied.clear();
    elim.assign((size_t)((n_tracks + 63) / 64), 0ull);
    // one marking pass (branch-free: the keep/go outcome is a coin flip per
    // row); the ties at the cut are rare and collected on the side
    int64_t below = 0;
    for (int64_t r = 0; r < m; ++r) {
      const uint64_t kk = key[r];
      const int32_t t = tracks[r];
      const uint64_t lt = kk < cut;
      elim[t >> 6] |= lt << (t & 63);
      below += (int64_t)lt;
      if (kk == cut) tied.push_back(t);
    }
    const int64_t need = n_elim - below;
    // the `need` highest track indices among the ties (a set: no full sort)
    if (need > 0 && need < (int64_t)tied.size())
      std::nth_element(tied.begin(), tied.begin() + (need - 1), tied.end(),
                       [](int32_t a, int32_t b) { return a > b; });
    for (int64_t i = 0; i < need; ++i) elim[tied[i] >> 6] |= 1ull << (tied[i] & 63);
    // eliminated tracks ascending straight from the bitmap
    int64_t g = 0;
    for (size_t w = 0; w < elim.size(); ++w)
      for (uint64_t bw = elim[w]; bw; bw &= bw - 1) {
        const int64_t t = (int64_t)w * 64 + __builtin_ctzll(bw);
        if (g < n_elim) gone_out[g] = t;
        ++g;
        alive[t] = 0;
      }
    int64_t k = 0;
    for (int64_t r = 0; r < m; ++r) {
      const int32_t t = tracks[r];
      keep_out[k] = (int32_t)r;
      k += (int64_t)(((elim[t >> 6] >> (t & 63)) & 1ull) ^ 1ull);
    }
    *n_keep = k;
    return HARL_OK;
  }
  int64_t k = 0;
  for (int64_t r = 0; r < m; ++r) {
    keep_out[k] = (int32_t)r;
    k += alive[tracks[r]] != 0;
  }
  *n_keep = k;
  return HARL_OK;
}


int harl_sim_time(const harl_sketch_desc* sk, const harl_sim_desc* sim,
                  const uint16_t* tiles, const uint8_t* knobs, int64_t n,
                  int64_t ld, double* out, void* stream) {
  if (!sk || !sim || !knobs || !out || n < 0 || sim->n_skipped < 0 ||
      sim->n_skipped > HARL_MAX_STAGES || sk->n_unroll > HARL_MAX_LEVELS) {
    set_error("harl_sim_time: bad arguments");
    return HARL_E_ARG;
  }
  if (n == 0) return HARL_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t g = (n + 127) / 128;
  const unsigned grid = (unsigned)(g < sm_count() * 8 ? g : sm_count() * 8);
  HARL_PROF_BEGIN(st);
  launch_k(k_sim_time, dim3(grid), dim3(128), 0, st, *sk, *sim, tiles, knobs, n, ld, out);
  HARL_CHECK_LAUNCH("k_sim_time");
  return HARL_OK;
}

int harl_brute_force(const harl_sketch_desc* sk, const harl_sim_desc* sim,
                     uint64_t x0, uint64_t count, unsigned long long* best,
                     unsigned long long* out, unsigned long long* scratch,
                     int64_t scratch_len, void* stream) {
  if (!sk || !sim || !best || !out || !scratch || sk->ncas < 1 ||
      sk->n_unroll < 1 || sk->n_unroll > HARL_MAX_LEVELS) {
    set_error("harl_brute_force: bad arguments");
    return HARL_E_ARG;
  }
  if (count == 0) return HARL_OK;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  if ((e = cudaMemsetAsync(best, 0xff, 8, st)) != cudaSuccess)
    return cuda_status(e, "harl_brute_force memset");
  const uint64_t g = (count + 255) / 256;
  uint64_t gmax = (uint64_t)sm_count() * 16;
  if (gmax > (uint64_t)scratch_len) gmax = (uint64_t)scratch_len;
  const unsigned grid = (unsigned)(g < gmax ? g : gmax);
  HARL_PROF_BEGIN(st);
  launch_k(k_brute_min, dim3(grid), dim3(256), 0, st, *sk, *sim, x0, count, best);
  HARL_CHECK_LAUNCH("k_brute_min");
  HARL_PROF_BEGIN(st);
  launch_k(k_brute_ties, dim3(grid), dim3(256), 0, st, *sk, *sim, x0, count,
           (const unsigned long long*)best, scratch);
  HARL_CHECK_LAUNCH("k_brute_ties");
  HARL_PROF_BEGIN(st);
  launch_k(k_brute_final, dim3(1), dim3(32), 0, st, *sk,
           (const unsigned long long*)scratch, (int)grid, out);
  HARL_CHECK_LAUNCH("k_brute_final");
  return HARL_OK;
}

}  // extern "C"
