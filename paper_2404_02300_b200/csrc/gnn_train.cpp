// catgnn_gnn_distributed_train: the partition-parallel GNN training loop —
// distributed_train (/root/reference/proj/src/train.cpp:289-340) with the
// north-star models in place of the SGC softmax regression.
//
//   validate q / p / s as the reference (train.cpp:291-295)
//   alpha = sync_weights(owner && train counts of ALL partitions) (:139-152, :302)
//   shared = init (seeded Glorot; zero for the SGC kind, zero_params :67-72)
//   while done < epochs:
//     chunk = min(s, epochs - done)                               (:315)
//     replicas restart from shared                                (:316-317)
//     chunk local iterations per replica (full-batch step)
//     shared = sum_i alpha_i replica_i over all partitions       (:322, :154-172)
//     val / test micro-F1 of shared on the global graph          (:324-335)
//
// Everything between two averages is enqueued without a host synchronisation:
// each step's loss stays on the device and is folded into a per-iteration
// accumulator (alpha_i * mean CE_i), read once at the end.  With a
// communicator, rank r trains partitions r, r + N, ...; its
// share sum_{i in r} alpha_i theta_i is all-reduced over NVLink (NCCL sum) —
// the only exchange on the path.
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "artifact.hpp"
#include "comm.hpp"
#include "model.hpp"
#include "shard.hpp"

using namespace catgnn;

namespace {

void rc_check(int rc) {
  if (rc == CATGNN_OK) return;
  const std::string msg = catgnn_last_error();
  if (rc == CATGNN_ECONFIG) throw ConfigError(msg);
  if (rc == CATGNN_EDATA) throw DataError(msg);
  throw InternalError(msg);
}

struct ShardHandle {
  catgnn_shard s = nullptr;
  ~ShardHandle() {
    if (s) catgnn_shard_destroy(s);
  }
};
struct ModelHandle {
  catgnn_model m = nullptr;
  ~ModelHandle() {
    if (m) catgnn_model_destroy(m);
  }
};

std::vector<double> global_alpha(const std::vector<uint64_t>& counts) {
  uint64_t total = 0;
  for (uint64_t c : counts) total += c;
  if (counts.empty() || total == 0) throw DataError("model averaging requires a nonzero training-node count");
  std::vector<double> alpha(counts.size());
  double partial = 0.0;
  for (size_t i = 0; i + 1 < counts.size(); ++i) {
    alpha[i] = (double)counts[i] / (double)total;
    partial += alpha[i];
  }
  alpha.back() = 1.0 - partial;
  return alpha;
}

double role_f1(catgnn_model m, catgnn_shard g, int role, bool present) {
  if (!present) return 0.0;
  double f1 = 0.0;
  rc_check(catgnn_model_forward(m, g, nullptr, role, &f1));
  return f1;
}

}  // namespace

extern "C" int catgnn_gnn_distributed_train(catgnn_ctx ctx, const char* artifact_dir, const char* input,
                                            const char* features, const catgnn_gnn_train_config* cfg,
                                            catgnn_comm comm, catgnn_gnn_result* result) {
  return guarded([&] {
    if (!ctx || !artifact_dir || !cfg || !result) throw ConfigError("null argument");
    CG_CUDA(cudaSetDevice(ctx->device));
    catgnn_artifact a_handle = nullptr;
    rc_check(catgnn_artifact_open(artifact_dir, &a_handle));
    struct ArtClose {
      catgnn_artifact a;
      ~ArtClose() { catgnn_artifact_close(a); }
    } art_close{a_handle};
    const catgnn_artifact_s& art = *a_handle;
    const uint32_t p = art.num_partitions;
    // train.cpp:291-295
    if (cfg->workers == 0 || p == 0) throw ConfigError("need at least one worker and one partition");
    if (p % cfg->workers != 0) throw ConfigError("partition count must be a multiple of the worker count");
    if (cfg->sync_interval == 0) throw ConfigError("sync interval must be >= 1");
    if (!art.has_meta) throw DataError("artifact has no labels; partition with --nodes to enable training");
    const int nranks = comm ? comm->nranks : 1, rank = comm ? comm->rank : 0;
    if (comm && comm->ctx->device != ctx->device) throw ConfigError("communicator is on another device");
    if (p % (uint32_t)nranks != 0) throw ConfigError("partition count must be a multiple of the rank count");

    // alpha over ALL partitions from the node tables (owner && role == train,
    // train.cpp:266), so every rank holds the same weights without loading
    // the other ranks' shards
    std::vector<uint64_t> counts(p, 0);
    for (uint32_t s = 0; s < p; ++s)
      for (size_t i = 0; i < art.parts[s].ext.size(); ++i)
        counts[s] += art.parts[s].owner[i] && art.parts[s].role[i] == 1;
    const std::vector<double> alpha = global_alpha(counts);

    std::vector<uint32_t> mine;
    for (uint32_t s = (uint32_t)rank; s < p; s += (uint32_t)nranks) mine.push_back(s);
    std::vector<ShardHandle> shards(mine.size());
    for (size_t i = 0; i < mine.size(); ++i)
      rc_check(catgnn_shard_load(ctx, a_handle, (int32_t)mine[i], input, features, &shards[i].s));
    ShardHandle global;
    if (cfg->eval_global) rc_check(catgnn_shard_load(ctx, a_handle, -1, input, features, &global.s));

    catgnn_model_config mc = cfg->model;
    if (mc.in_dim == 0) {
      if (shards.empty()) throw DataError("no partition to train");
      mc.in_dim = shards[0].s->dim;
    }
    if (mc.classes == 0) {  // train.cpp:307-309: max label + 1 over the graph
      int32_t mx = 0;
      for (const auto& m : art.meta) mx = std::max(mx, m.label);
      mc.classes = (uint32_t)std::max(1, mx + 1);
    }
    ModelHandle shared;
    rc_check(catgnn_model_create(ctx, &mc, &shared.m));
    std::vector<ModelHandle> reps(mine.size());
    std::vector<catgnn_model> rep_ptrs(mine.size());
    std::vector<double> my_alpha(mine.size());
    for (size_t i = 0; i < mine.size(); ++i) {
      rc_check(catgnn_model_create(ctx, &mc, &reps[i].m));
      rep_ptrs[i] = reps[i].m;
      my_alpha[i] = alpha[mine[i]];
    }

    const uint64_t epochs = cfg->epochs;
    DevBuf<double> loss_acc;
    loss_acc.alloc(std::max<uint64_t>(1, epochs));
    CG_CUDA(cudaMemsetAsync(loss_acc.p, 0, std::max<uint64_t>(1, epochs) * 8, ctx->stream));

    uint64_t done = 0, ops = 0;
    result->n_hist = 0;
    while (done < epochs) {
      const uint64_t chunk = std::min<uint64_t>(cfg->sync_interval, epochs - done);
      for (auto& r : reps) rc_check(catgnn_model_copy_params(r.m, shared.m));
      for (uint64_t it = 0; it < chunk; ++it)
        for (size_t i = 0; i < reps.size(); ++i) {
          model_train_step(reps[i].m, shards[i].s);
          model_accumulate_loss(reps[i].m, my_alpha[i], loss_acc.p + done + it);
        }
      if (reps.empty()) CG_CUDA(cudaMemsetAsync(shared.m->params.p, 0, shared.m->n_params * 4, ctx->stream));
      else model_weighted_sum(rep_ptrs, my_alpha, shared.m);
      if (comm) rc_check(catgnn_model_allreduce(shared.m, comm));
      done += chunk;
      ops++;
      if (cfg->eval_global) {
        const double vf = role_f1(shared.m, global.s, 2, !global.s->h_val.empty());
        const double tf = role_f1(shared.m, global.s, 3, !global.s->h_test.empty());
        if (result->n_hist < result->hist_capacity) {
          const uint64_t k = result->n_hist;
          if (result->hist_epoch) result->hist_epoch[k] = done;
          if (result->hist_syncs) result->hist_syncs[k] = ops;
          if (result->hist_val) result->hist_val[k] = vf;
          if (result->hist_test) result->hist_test[k] = tf;
        }
        result->n_hist++;
      }
    }
    // losses: this rank's partitions' share, summed over ranks
    if (comm && epochs) {
      ncclResult_t r = ncclAllReduce(loss_acc.p, loss_acc.p, epochs, ncclFloat64, ncclSum, comm->comm, ctx->stream);
      if (r != ncclSuccess) throw InternalError(std::string("ncclAllReduce: ") + ncclGetErrorString(r));
    }
    std::vector<double> losses(epochs);
    if (epochs) CG_CUDA(cudaMemcpyAsync(losses.data(), loss_acc.p, epochs * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CG_CUDA(cudaStreamSynchronize(ctx->stream));
    result->n_losses = epochs;
    if (result->losses)
      std::copy(losses.begin(), losses.begin() + std::min<uint64_t>(epochs, result->loss_capacity), result->losses);
    result->num_params = catgnn_model_num_params(shared.m);
    result->averaging_ops = ops;
    result->in_dim = mc.in_dim;
    result->classes = mc.classes;
    if (result->params) {
      if (result->params_capacity < result->num_params) throw ConfigError("params buffer too small");
      rc_check(catgnn_model_get_params(shared.m, result->params));
    }
    if (result->model_out) {
      *result->model_out = shared.m;
      shared.m = nullptr;
    }
  });
}
