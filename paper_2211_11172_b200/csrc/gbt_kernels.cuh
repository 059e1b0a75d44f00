// K6: GBT cost-model inference + reward (costmodel.py:67-78,219-237,
// tuner.py:389-391).  fp64 and bit-exact: the walk is a chain of exact
// comparisons, each tree's leaf contribution is the host-computed product
// learning_rate*leaf_value, and the contributions are added to the base in
// tree order with explicit round-to-nearest adds -- exactly the
// reference's ``pred = pred + lr * tree.predict(X)`` loop.
//
// Parallelism is (row x tree-group): G threads share a row, each walks
// every G-th tree and parks its leaf contributions in shared memory; one
// thread per row then sums them in tree order.  Nodes are 16-byte records
// read through the read-only/L1 path (the whole forest, ~100-150 KB, stays
// L1/L2-resident), so many CTAs fit per SM to hide the dependent-load
// latency of the walk.
#pragma once

#include "common.cuh"

namespace harl {

struct __align__(16) GbtNode {
  double v;        // split threshold (internal) / lr*value (leaf)
  int16_t feat;    // -1 for a leaf
  int16_t left, right, pad;
};

constexpr int GBT_GROUPS = 8;      // threads per row
constexpr int GBT_THREADS = 256;   // 32 rows per CTA

__global__ void __launch_bounds__(GBT_THREADS)
k_gbt_predict(const GbtNode* __restrict__ nodes,
              const int32_t* __restrict__ tree_first, int32_t n_trees,
              int32_t fitted, double base, double floor_value,
              const double* __restrict__ feat, int64_t n, int32_t F,
              double* score, const double* old_score, double* reward,
              int32_t rows_per_cta) {
  extern __shared__ double contrib[];  // [rows_per_cta][n_trees]
  const int g = threadIdx.x % GBT_GROUPS;
  const int rl = threadIdx.x / GBT_GROUPS;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r = r0 + rl;
  if (fitted && rl < rows_per_cta && r < n) {
    const double* x = feat + r * F;
    for (int t = g; t < n_trees; t += GBT_GROUPS) {
      const GbtNode* tree = nodes + tree_first[t];
      GbtNode nd = tree[0];
      // same 64-step cap as the reference's walk (trees are checked to be
      // shallower on the host)
      while (nd.feat >= 0) nd = tree[(__ldg(x + nd.feat) <= nd.v) ? nd.left : nd.right];
      contrib[rl * n_trees + t] = nd.v;
    }
  }
  __syncthreads();
  if (g != 0 || rl >= rows_per_cta || r >= n) return;
  double pred = 1.0;
  if (fitted) {
    pred = base;
    const double* c = contrib + rl * n_trees;
    for (int t = 0; t < n_trees; ++t) pred = __dadd_rn(pred, c[t]);
  }
  // np.maximum(pred, floor): NaN propagates
  const double s = (pred != pred) ? pred : (pred < floor_value ? floor_value : pred);
  score[r] = s;
  if (old_score) {
    const double o = old_score[r];
    reward[r] = __ddiv_rn(__dsub_rn(s, o), o);
  }
}

}  // namespace harl
