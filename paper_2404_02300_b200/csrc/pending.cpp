// Temporary: entry points whose kernels land in the next commit.
#include "common.hpp"
using namespace catgnn;
#define PENDING { return guarded([&] { throw ConfigError("not implemented yet"); }); }
extern "C" {
int catgnn_model_create(catgnn_ctx, const catgnn_model_config*, catgnn_model*) PENDING
int catgnn_model_destroy(catgnn_model) PENDING
uint64_t catgnn_model_num_params(catgnn_model) { return 0; }
int catgnn_model_layer_shape(catgnn_model, uint32_t, uint32_t*, uint32_t*, uint64_t*, uint64_t*) PENDING
int catgnn_model_get_params(catgnn_model, float*) PENDING
int catgnn_model_set_params(catgnn_model, const float*) PENDING
int catgnn_model_copy_params(catgnn_model, catgnn_model) PENDING
int catgnn_model_get_grads(catgnn_model, float*) PENDING
int catgnn_model_train_step(catgnn_model, catgnn_shard, double*) PENDING
int catgnn_model_forward_backward(catgnn_model, catgnn_shard, double*) PENDING
int catgnn_model_forward(catgnn_model, catgnn_shard, float*, int, double*) PENDING
int catgnn_model_export(catgnn_model, uint32_t, int, float*, uint32_t*) PENDING
int catgnn_model_average(uint32_t, const catgnn_model*, const uint64_t*, catgnn_model) PENDING
int catgnn_comm_unique_id(char*) PENDING
int catgnn_comm_create(catgnn_ctx, int, int, const char*, catgnn_comm*) PENDING
int catgnn_comm_destroy(catgnn_comm) PENDING
int catgnn_model_scale(catgnn_model, double) PENDING
int catgnn_model_allreduce(catgnn_model, catgnn_comm) PENDING
}
