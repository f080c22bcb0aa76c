// GNN replica state shared by gnn.cu (layers, forward / backward, optimizer)
// and gnn_train.cu (the partition-parallel training loop behind
// catgnn_gnn_distributed_train).
#pragma once

#include <string>
#include <vector>

#include "common.hpp"
#include "shard.hpp"

namespace catgnn {

struct Layer {
  uint32_t d_in = 0, d_out = 0;
  uint32_t K_in = 0;    // round4(d_in): activation row stride of the input
  uint32_t D_out = 0;   // round4(d_out)
  uint32_t ld_act = 0;  // row stride of this layer's output activations (>= D_out)
  bool out_in_next_mid = false;  // output written straight into the next (SAGE aggregate-first) layer's [h | mean]
  bool agg_first = false;
  // internal weight matrix (GEMM B operand): w_rows x w_cols
  uint32_t w_rows = 0, w_cols = 0;
  uint64_t off_w = 0, off_b = 0;
  // logical (exported) weight shape
  uint32_t lw_rows = 0, lw_cols = 0;
  uint32_t gemm_n = 0;   // forward GEMM N (transform-first SAGE: D_out + d_out)
};

}  // namespace catgnn

struct catgnn_model_s {
  catgnn_ctx ctx = nullptr;
  catgnn_model_config cfg{};
  std::vector<catgnn::Layer> layers;
  uint64_t n_params = 0;
  catgnn::DevBuf<float> params, grads, m, v;
  uint64_t step = 0;                       // updates issued (host count)
  catgnn::DevBuf<unsigned long long> step_dev;     // [completed updates, block ticket] (Adam bias correction)
  uint64_t last_rows = 0;
  catgnn_shard last_shard = nullptr;
  double last_loss = 0.0;
  catgnn::DevBuf<double> loss_dev;  // sum of the last step's per-row losses (read lazily)
  uint64_t loss_rows = 0;   // train rows of that step
  // bf16x3 copies of the weights (hi / lo per layer at ws_off, rows of round8(w_cols))
  catgnn::DevBuf<uint16_t> ws_hi, ws_lo;
  std::vector<uint64_t> ws_off;
  bool act_f16 = true;  // fp16 K2 inputs where safe (catgnn_model_set_act_f16; gnn.cu f16_bwd)
  std::vector<bool> h_split_only;  // layer outputs the last forward kept only as bf16x3 pairs
  // dZ_l of the last backward held only as fp16 rows rs[r] * dZ * scale (the
  // fp16 K2 inputs; catgnn_model_export converts back)
  struct DzF16 {
    bool on = false;
    const float* rs = nullptr;
    float scale = 1.0f;
    uint32_t ld = 0;
  };
  std::vector<DzF16> dz_f16;
  const float* dz_last = nullptr;  // where the last backward kept the last layer's dZ (may alias its T)
  std::vector<const float*> dz_ptr;  // per layer: the last backward's fp32 dZ buffer (lean aliasing)
};

namespace catgnn {

// One local iteration (forward + loss + backward + optimizer) with no host
// synchronisation; the loss sum stays on the device (m->loss_dev).
void model_train_step(catgnn_model m, catgnn_shard s);
// dst = sum_i alpha_i src_i (f64 accumulation in list order, from zero):
// model_average with caller-supplied weights (train.cpp:164-169).
void model_weighted_sum(const std::vector<catgnn_model>& src, const std::vector<double>& alpha,
                        catgnn_model dst);
// *acc += weight * (m's last loss sum), on m's stream (no host sync).
void model_accumulate_loss(catgnn_model m, double weight, double* acc);

}  // namespace catgnn
