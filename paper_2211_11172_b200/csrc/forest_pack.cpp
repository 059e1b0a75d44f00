// GBT ensemble -> the device layouts (host C++).
//
// The drop-in reloads the session's surrogate (costmodel.py:59-78, _Tree
// arrays per tree) onto the device before every episode, since run_round
// refits it after every round's measurements (tuner.py:480-520,
// fit_round -> fit_incremental, costmodel.py:190-212).  This file builds, in
// one pass over the trees, everything device.DeviceForest writes:
//   * 16-byte node records {v, feat, left, right, pad} (v = the threshold of
//     an inner node, learning_rate * value of a leaf -- the reference's fp64
//     product, costmodel.py:224),
//   * each tree's first record,
//   * the forest depth (internal levels of the deepest tree, with the
//     reference's 64-step walk bound, costmodel.py:67-78),
//   * for depth <= perfect_max the perfect-tree image the GBT kernels walk
//     (gbt_kernels.cuh: thresholds [T][2^D-1] f64, leaf values [T][2^D] f64,
//     features [T][2^D-1] i16, sections 16-byte aligned; a leaf above the
//     last level becomes pass-through slots, feature 0 / threshold +inf,
//     whose subtree repeats its value).
// tests/test_forest_records.py checks it byte for byte against the numpy
// restatement in device.py.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <vector>

namespace {

struct NodeRec {
  double v;
  int16_t feat, left, right, pad;
};
static_assert(sizeof(NodeRec) == 16, "node record is 16 bytes");

constexpr int kWalk = 63;        // inner levels the reference's 64-step walk finishes

// internal levels below node n (0 for a leaf); -1: deeper than the walk
// bound, -2: a child index outside the tree
int levels(const int64_t* feat, const int64_t* left, const int64_t* right,
           int64_t size, int64_t n, int budget, std::vector<int8_t>& memo) {
  if (n < 0 || n >= size) return -2;
  if (feat[n] < 0) return 0;
  if (memo[n] >= 0) return memo[n];
  if (budget == 0) return -1;
  const int a = levels(feat, left, right, size, left[n], budget - 1, memo);
  if (a < 0) return a;
  const int b = levels(feat, left, right, size, right[n], budget - 1, memo);
  if (b < 0) return b;
  const int d = 1 + (a > b ? a : b);
  memo[n] = (int8_t)d;
  return d;
}

}  // namespace

extern "C" {

// Returns the forest depth (>= 0) or an error: -1 a tree deeper than the
// reference's 64-step walk, -2 an empty tree or a child index outside it,
// -3 more than 1024 trees or a tree beyond int16 node indices, -4
// perfect_cap too small.
// The trees' arrays are concatenated (tree t's nodes follow tree t-1's;
// child indices local to the tree).  nodes_out: 16 * sum(sizes) bytes;
// firsts_out: n_trees int32;
// perfect_out / perfect_cap: the image buffer (may be null when depth >
// perfect_max); *perfect_bytes_out: bytes of the image written (0: none).
long long harl_forest_pack(int n_trees, const int64_t* sizes,
                           const int64_t* feature, const double* threshold,
                           const int64_t* left, const int64_t* right,
                           const double* value, double learning_rate,
                           void* nodes_out, int32_t* firsts_out,
                           int perfect_max, void* perfect_out,
                           long long perfect_cap,
                           long long* perfect_bytes_out) {
  *perfect_bytes_out = 0;
  if (n_trees > 1024) return -3;
  NodeRec* rec = static_cast<NodeRec*>(nodes_out);
  int depth = 0;
  int64_t first = 0;
  std::vector<int8_t> memo;
  for (int t = 0; t < n_trees; ++t) {
    const int64_t sz = sizes[t];
    if (sz > 32767) return -3;
    firsts_out[t] = (int32_t)first;
    memo.assign((size_t)sz, -1);
    const int64_t *ft = feature + first, *lt = left + first,
                  *rt = right + first;
    const int d = levels(ft, lt, rt, sz, 0, kWalk, memo);
    if (d < 0) return d;
    if (d > depth) depth = d;
    for (int64_t i = 0; i < sz; ++i) {
      NodeRec& r = rec[first + i];
      const bool leaf = ft[i] < 0;
      r.v = leaf ? learning_rate * value[first + i] : threshold[first + i];
      r.feat = (int16_t)ft[i];
      r.left = leaf ? 0 : (int16_t)lt[i];
      r.right = leaf ? 0 : (int16_t)rt[i];
      r.pad = 0;
    }
    first += sz;
  }
  if (n_trees == 0 || depth == 0 || depth > perfect_max || !perfect_out)
    return depth;
  const int D = depth;
  const int64_t T = n_trees, NI = (1 << D) - 1, NL = 1 << D;
  const int64_t b_leaf = (T * NI * 8 + 15) & ~(int64_t)15;
  const int64_t b_feat = b_leaf + T * NL * 8;
  const int64_t bytes = (b_feat + T * NI * 2 + 15) & ~(int64_t)15;
  if (bytes > perfect_cap) return -4;
  uint8_t* img = static_cast<uint8_t*>(perfect_out);
  memset(img, 0, (size_t)bytes);
  double* thr_p = reinterpret_cast<double*>(img);
  double* leaf_p = reinterpret_cast<double*>(img + b_leaf);
  int16_t* feat_p = reinterpret_cast<int16_t*>(img + b_feat);
  const double inf = std::numeric_limits<double>::infinity();
  std::vector<int64_t> cur(NL), nxt(NL);
  for (int64_t t = 0; t < T; ++t) {
    const NodeRec* tr = rec + firsts_out[t];
    cur[0] = 0;
    for (int d = 0; d < D; ++d) {
      const int64_t lo = (1 << d) - 1, w = 1 << d;
      for (int64_t i = 0; i < w; ++i) {
        const NodeRec& r = tr[cur[i]];
        const bool leaf = r.feat < 0;
        thr_p[t * NI + lo + i] = leaf ? inf : r.v;
        feat_p[t * NI + lo + i] = leaf ? 0 : r.feat;
        nxt[2 * i] = leaf ? cur[i] : r.left;
        nxt[2 * i + 1] = leaf ? cur[i] : r.right;
      }
      cur.swap(nxt);
    }
    for (int64_t i = 0; i < NL; ++i) leaf_p[t * NL + i] = tr[cur[i]].v;
  }
  *perfect_bytes_out = bytes;
  return depth;
}

}  // extern "C"
