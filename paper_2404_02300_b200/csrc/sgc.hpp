#pragma once

#include <vector>

#include "common.hpp"

namespace catgnn {

struct SgcReplicaHost {
  const float* x;        // device rows x ld (propagated features)
  uint32_t ld;
  const int32_t* labels; // device
  const uint32_t* order; // device n_epochs x n_train
  uint64_t n_train;
  float* W;              // device dim x C
  float* b;              // device C
  float* gW = nullptr;   // gradient-only mode
  float* gb = nullptr;
};

// train_epochs for several replicas in one launch (one CTA per replica).
void sgc_train(catgnn_ctx ctx, const std::vector<SgcReplicaHost>& reps, uint32_t dim, uint32_t C,
               float lr, uint32_t batch, uint32_t n_epochs, bool grad_only);
// evaluate_micro_f1 / softmax_loss support: correct-prediction count and
// per-row cross-entropy over the mask rows.
void sgc_eval(catgnn_ctx ctx, const float* x, uint32_t ld, uint32_t dim, const float* W,
              const float* b, uint32_t C, const int32_t* labels, const uint32_t* mask,
              uint64_t n_mask, unsigned long long* correct, double* row_loss);
// out[j] = sum_i alpha_i * src_i[j] in partition order, f64 accumulation.
void average_params(catgnn_ctx ctx, const std::vector<const float*>& d_src,
                    const std::vector<double>& alpha, uint64_t count, float* d_out);

}  // namespace catgnn
