// K6: GBT cost-model inference + reward (costmodel.py:67-78,219-237,
// tuner.py:389-391).  fp64 and bit-exact: the walk is a chain of exact
// comparisons, and each tree adds the host-computed product
// learning_rate*leaf_value with one explicit round-to-nearest add, exactly
// the reference's ``pred = pred + lr * tree.predict(X)``.  The forest is
// staged once per CTA into shared memory (node = 24 bytes).
#pragma once

#include "common.cuh"

namespace harl {

struct __align__(8) GbtNode {
  double thr;      // split threshold (internal) / lr*value (leaf)
  int16_t feat;    // -1 for a leaf
  int16_t left, right, pad;
};

constexpr int GBT_THREADS = 512;

__global__ void __launch_bounds__(GBT_THREADS)
k_gbt_predict(const __grid_constant__ harl_forest_desc fo, const double* feat,
              int64_t n, int32_t F, double* score, const double* old_score,
              double* reward, int32_t n_nodes) {
  extern __shared__ GbtNode snodes[];
  __shared__ int32_t sfirst[1024];
  for (int i = threadIdx.x; i < n_nodes; i += blockDim.x) {
    GbtNode g;
    g.feat = fo.feature[i];
    g.left = fo.left[i];
    g.right = fo.right[i];
    g.pad = 0;
    g.thr = g.feat >= 0 ? fo.threshold[i] : fo.leaf_contrib[i];
    snodes[i] = g;
  }
  for (int i = threadIdx.x; i < fo.n_trees; i += blockDim.x) sfirst[i] = fo.tree_first[i];
  __syncthreads();
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    double pred;
    if (!fo.fitted) {
      pred = 1.0;
    } else {
      const double* x = feat + r * F;
      pred = fo.base;
      for (int t = 0; t < fo.n_trees; ++t) {
        const GbtNode* tree = snodes + sfirst[t];
        int node = 0;
        GbtNode g = tree[0];
        while (g.feat >= 0) {
          node = (x[g.feat] <= g.thr) ? g.left : g.right;
          g = tree[node];
        }
        pred = __dadd_rn(pred, g.thr);
      }
    }
    // np.maximum(pred, floor): NaN propagates
    const double s = (pred != pred) ? pred : (pred < fo.floor_value ? fo.floor_value : pred);
    score[r] = s;
    if (old_score) {
      const double o = old_score[r];
      reward[r] = __ddiv_rn(__dsub_rn(s, o), o);
    }
  }
}

}  // namespace harl
