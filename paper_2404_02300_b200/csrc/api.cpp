// C ABI (include/catgnn.h): context, artifact, shards and the SGC path.
// Every entry point cites the reference function it replaces.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <numeric>
#include <random>
#include <filesystem>
#include <unordered_map>

#include "artifact.hpp"
#include "sgc.hpp"
#include "shard.hpp"

using namespace catgnn;

namespace catgnn {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace catgnn

// ------------------------------------------------------------------ context
cudaEvent_t catgnn_ctx_s::take_event() {
  if (!event_pool.empty()) {
    cudaEvent_t e = event_pool.back();
    event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  CG_CUDA(cudaEventCreate(&e));
  return e;
}
void catgnn_ctx_s::wait_for(const catgnn_ctx_s* other) {
  if (!other || other->stream == stream) return;
  // a small ring of timing-disabled events recorded on the other stream; an
  // event may be re-recorded once the wait that used it has been enqueued
  if (order_events.empty()) {
    order_events.resize(64);
    for (auto& e : order_events) CG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  cudaEvent_t e = order_events[order_next++ % order_events.size()];
  CG_CUDA(cudaEventRecord(e, other->stream));
  CG_CUDA(cudaStreamWaitEvent(stream, e, 0));
}

// Under stream capture the timing events become event-record nodes of the
// graph (cudaEventRecordExternal), re-recorded by every replay.
static void record_timing_event(cudaEvent_t e, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CG_CUDA(cudaStreamIsCapturing(st, &cs));
  if (cs == cudaStreamCaptureStatusActive) CG_CUDA(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal));
  else CG_CUDA(cudaEventRecord(e, st));
}
int catgnn_ctx_s::begin_timed(int kind, std::string label) {
  if (!timing) return -1;
  Pending p{take_event(), take_event(), kind, std::move(label)};
  record_timing_event(p.a, stream);
  pending.push_back(p);
  return (int)pending.size() - 1;
}
void catgnn_ctx_s::end_timed(int idx) {
  if (idx < 0) return;
  record_timing_event(pending[idx].b, stream);
}
void catgnn_ctx_s::drain_timing() {
  for (auto& p : pending) {
    CG_CUDA(cudaEventSynchronize(p.b));
    float ms = 0;
    CG_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
    if (p.kind == 0) { agg_ms += ms; agg_n++; }
    else if (p.kind == 1) { gemm_ms += ms; gemm_n++; }
    if (!p.label.empty()) {
      auto& l = by_label[p.label];
      l.first += ms;
      l.second++;
    }
    event_pool.push_back(p.a);
    event_pool.push_back(p.b);
  }
  pending.clear();
}
catgnn_ctx_s::~catgnn_ctx_s() {
  for (auto& p : pending) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
  for (auto e : event_pool) cudaEventDestroy(e);
  for (auto e : order_events) cudaEventDestroy(e);
  scratch.clear();
  if (own_stream && stream) cudaStreamDestroy(stream);
}

namespace {

void check_ctx(catgnn_ctx c) {
  if (!c) throw ConfigError("null context");
  CG_CUDA(cudaSetDevice(c->device));
}
void check_shard(catgnn_shard s) {
  if (!s) throw ConfigError("null shard");
  check_ctx(s->ctx);
}

template <typename T>
void h2d(T* dst, const T* src, size_t n, cudaStream_t st) {
  if (n) CG_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyHostToDevice, st));
}

// Host rows x dim -> device rows x ld.  One contiguous H2D copy (full PCIe /
// C2C bandwidth from pinned memory; a pitched host copy with 2408-byte rows
// runs at a fraction of it), then an on-device re-pitch when dim % 4 != 0.
void copy_features_in(catgnn_shard_s* s, const float* feats, uint32_t dim) {
  cudaStream_t st = s->ctx->stream;
  s->x_version++;  // the bf16x3 copy (gnn.cu) is re-split on next use
  s->x_fp32_valid = true;
  const size_t bytes = s->rows * (size_t)dim * sizeof(float);
  if (s->ld == dim) {
    CG_CUDA(cudaMemcpyAsync(s->x.p, feats, bytes, cudaMemcpyHostToDevice, st));
    return;
  }
  float* stage = s->ctx->scratch_buf<float>("feat_stage", s->rows * (size_t)dim);
  CG_CUDA(cudaMemcpyAsync(stage, feats, bytes, cudaMemcpyHostToDevice, st));
  CG_CUDA(cudaMemcpy2DAsync(s->x.p, s->ld * sizeof(float), stage, dim * sizeof(float), dim * sizeof(float),
                            s->rows, cudaMemcpyDeviceToDevice, st));
}

void upload_features(catgnn_shard_s* s, const float* feats, uint32_t dim) {
  s->dim = dim;
  s->ld = round_up(std::max<uint32_t>(dim, 1), 4);
  s->x.alloc(std::max<uint64_t>(1, s->rows) * s->ld);
  s->x_version++;
  s->x_fp32_valid = true;
  s->xprop.release();
  if (s->rows == 0 || dim == 0) return;
  if (s->ld != dim) CG_CUDA(cudaMemsetAsync(s->x.p, 0, s->x.bytes(), s->ctx->stream));
  if (feats) copy_features_in(s, feats, dim);
}

void set_labels(catgnn_shard_s* s, const int32_t* labels, const uint32_t* tr, uint64_t ntr,
                const uint32_t* va, uint64_t nva, const uint32_t* te, uint64_t nte) {
  cudaStream_t st = s->ctx->stream;
  s->h_labels.assign(labels ? labels : nullptr, labels ? labels + s->rows : nullptr);
  if (!labels) s->h_labels.assign(s->rows, 0);
  s->h_train.assign(tr, tr + ntr);
  s->train_sub.reset();  // train-row views of the old roles (csr.cu)
  s->train_nbr.reset();
  s->h_val.assign(va, va + nva);
  s->h_test.assign(te, te + nte);
  for (auto* v : {&s->h_train, &s->h_val, &s->h_test})
    for (uint32_t r : *v)
      if (r >= s->rows) throw DataError("role row outside the shard");
  int32_t mx = 0;
  for (int32_t l : s->h_labels) mx = std::max(mx, l);
  s->train_label_min = 0;
  s->train_label_max = -1;
  for (size_t i = 0; i < s->h_train.size(); ++i) {
    const int32_t l = s->h_labels[s->h_train[i]];
    s->train_label_min = i ? std::min(s->train_label_min, l) : l;
    s->train_label_max = i ? std::max(s->train_label_max, l) : l;
  }
  s->classes = (uint32_t)std::max(1, mx + 1);
  s->labels.alloc(std::max<uint64_t>(1, s->rows));
  s->d_train.alloc(std::max<uint64_t>(1, ntr));
  s->d_val.alloc(std::max<uint64_t>(1, nva));
  s->d_test.alloc(std::max<uint64_t>(1, nte));
  h2d(s->labels.p, s->h_labels.data(), s->h_labels.size(), st);
  h2d(s->d_train.p, s->h_train.data(), ntr, st);
  h2d(s->d_val.p, s->h_val.data(), nva, st);
  h2d(s->d_test.p, s->h_test.data(), nte, st);
  CG_CUDA(cudaStreamSynchronize(st));
}

std::unique_ptr<catgnn_shard_s> new_shard(catgnn_ctx ctx, uint64_t rows) {
  auto s = std::make_unique<catgnn_shard_s>();
  s->ctx = ctx;
  ctx_retain(ctx);
  s->rows = rows;
  return s;
}

// CSR from host local pairs.
void shard_csr_from_pairs(catgnn_shard_s* s, const uint32_t* pairs, uint64_t num_edges) {
  uint32_t* d = s->ctx->scratch_buf<uint32_t>("pairs", std::max<uint64_t>(1, 2 * num_edges));
  h2d(d, pairs, 2 * num_edges, s->ctx->stream);
  build_csr(s, d, num_edges);
}

// CSR from external-id edges mapped through the ascending node table.
void shard_csr_from_ext(catgnn_shard_s* s, const uint64_t* ext_ids, const uint64_t* edges,
                        uint64_t num_edges) {
  catgnn_ctx ctx = s->ctx;
  bool sorted = std::is_sorted(ext_ids, ext_ids + s->rows) &&
                std::adjacent_find(ext_ids, ext_ids + s->rows) == ext_ids + s->rows;
  uint32_t* d_pairs = ctx->scratch_buf<uint32_t>("pairs", std::max<uint64_t>(1, 2 * num_edges));
  if (sorted) {
    uint64_t* d_ext = ctx->scratch_buf<uint64_t>("ext_ids", std::max<uint64_t>(1, s->rows));
    uint64_t* d_edges = ctx->scratch_buf<uint64_t>("edges_ext", std::max<uint64_t>(1, 2 * num_edges));
    h2d(d_ext, ext_ids, s->rows, ctx->stream);
    h2d(d_edges, edges, 2 * num_edges, ctx->stream);
    map_ext_edges(ctx, d_ext, s->rows, d_edges, num_edges, d_pairs);
  } else {
    std::unordered_map<uint64_t, uint32_t> local;
    local.reserve(s->rows);
    for (uint64_t i = 0; i < s->rows; ++i) local[ext_ids[i]] = (uint32_t)i;
    std::vector<uint32_t> pairs(2 * num_edges);
    for (uint64_t k = 0; k < 2 * num_edges; ++k) {
      auto it = local.find(edges[k]);
      if (it == local.end())
        throw InternalError("partition edge endpoint missing from its node table (unordered_map::at)");
      pairs[k] = it->second;
    }
    h2d(d_pairs, pairs.data(), pairs.size(), ctx->stream);
  }
  build_csr(s, d_pairs, num_edges);
}

// train_epochs' shuffle (train.cpp:107-113): one `order` vector per call,
// shuffled in place once per epoch with mt19937_64(seed_for(seed, epoch)).
std::vector<uint32_t> epoch_orders(const std::vector<uint32_t>& train_rows, uint64_t epoch_begin,
                                   uint64_t epoch_end, uint64_t seed) {
  std::vector<uint32_t> order(train_rows), all;
  all.reserve(order.size() * (epoch_end - epoch_begin));
  for (uint64_t epoch = epoch_begin; epoch < epoch_end; ++epoch) {
    std::mt19937_64 rng(seed_for(seed, epoch));
    std::shuffle(order.begin(), order.end(), rng);
    all.insert(all.end(), order.begin(), order.end());
  }
  return all;
}

// Re-raise the error a nested ABI call recorded, with its category.
[[noreturn]] void throw_last_error_code(int rc) {
  if (rc == CATGNN_ECONFIG) throw ConfigError(g_last_error);
  if (rc == CATGNN_EDATA) throw DataError(g_last_error);
  throw InternalError(g_last_error);
}

void ensure_prop(catgnn_shard_s* s) {
  if (!s->xprop.p) throw ConfigError("features not propagated: call catgnn_sgc_propagate first");
}

std::vector<double> sync_weights_vec(const std::vector<uint64_t>& counts) {
  uint64_t total = 0;
  for (uint64_t c : counts) total += c;
  if (counts.empty() || total == 0)
    throw DataError("model averaging requires a nonzero training-node count");
  std::vector<double> alpha(counts.size());
  double partial = 0.0;
  for (size_t i = 0; i + 1 < counts.size(); ++i) {
    alpha[i] = static_cast<double>(counts[i]) / static_cast<double>(total);
    partial += alpha[i];
  }
  alpha.back() = 1.0 - partial;
  return alpha;
}

double micro_f1_from(uint64_t correct, uint64_t total) {
  // pooled TP/FP/FN (train.cpp:189-197): each miss is one FP and one FN
  uint64_t tp = correct, fp = total - correct, fn = total - correct;
  double denom = 2.0 * tp + fp + fn;
  return denom == 0 ? 0.0 : 2.0 * static_cast<double>(tp) / denom;
}

double eval_f1(catgnn_shard_s* s, const float* dW, const float* db, uint32_t C,
               const uint32_t* d_mask, uint64_t n_mask) {
  if (n_mask == 0) throw DataError("evaluation mask is empty");
  catgnn_ctx ctx = s->ctx;
  auto* cnt = ctx->scratch_buf<unsigned long long>("eval_cnt", 1);
  CG_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), ctx->stream));
  sgc_eval(ctx, s->xprop.p, s->ld, s->dim, dW, db, C, s->labels.p, d_mask, n_mask, cnt, nullptr);
  unsigned long long h = 0;
  CG_CUDA(cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  CG_CUDA(cudaStreamSynchronize(ctx->stream));
  return micro_f1_from(h, n_mask);
}

}  // namespace

extern "C" {

const char* catgnn_last_error(void) { return g_last_error.c_str(); }
int catgnn_version(void) { return 1; }

int catgnn_ctx_create(int device, void* stream, catgnn_ctx* out) {
  return guarded([&] {
    if (!out) throw ConfigError("null output");
    int n = 0;
    CG_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) throw ConfigError("device index out of range");
    CG_CUDA(cudaSetDevice(device));
    auto c = std::make_unique<catgnn_ctx_s>();
    c->device = device;
    if (stream) {
      c->stream = static_cast<cudaStream_t>(stream);
    } else {
      CG_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    CG_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    *out = c.release();
  });
}

int catgnn_ctx_destroy(catgnn_ctx ctx) {
  return guarded([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    ctx_release(ctx);
  });
}

int catgnn_ctx_wait(catgnn_ctx waiter, catgnn_ctx producer) {
  return guarded([&] {
    check_ctx(waiter);
    check_ctx(producer);
    if (waiter->device != producer->device) throw ConfigError("contexts are on different devices");
    waiter->wait_for(producer);
  });
}

int catgnn_ctx_set_sm_budget(catgnn_ctx ctx, int agg_sms, int gemm_sms) {
  return guarded([&] {
    check_ctx(ctx);
    if (agg_sms < 0 || gemm_sms < 0 || agg_sms > ctx->num_sms || gemm_sms > ctx->num_sms)
      throw ConfigError("SM budget out of range");
    ctx->agg_sms = agg_sms;
    ctx->gemm_sms = gemm_sms;
  });
}

int catgnn_ctx_synchronize(catgnn_ctx ctx) {
  return guarded([&] {
    check_ctx(ctx);
    CG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

uint64_t catgnn_ctx_launch_count(catgnn_ctx ctx) { return ctx ? ctx->launches : 0; }

int catgnn_ctx_set_kernel_timing(catgnn_ctx ctx, int enable) {
  return guarded([&] {
    check_ctx(ctx);
    ctx->drain_timing();
    ctx->timing = enable != 0;
    ctx->agg_ms = ctx->gemm_ms = 0;
    ctx->by_label.clear();
    ctx->agg_n = ctx->gemm_n = 0;
  });
}

// Per-label breakdown of the timed launches: record i (0 <= i < count) as
// "label\tms_total\tlaunches"; returns the record count in *count.
int catgnn_ctx_timing_record(catgnn_ctx ctx, uint32_t i, char* buf, uint32_t cap, uint32_t* count) {
  return guarded([&] {
    check_ctx(ctx);
    ctx->drain_timing();
    if (count) *count = (uint32_t)ctx->by_label.size();
    if (!buf || cap == 0) return;
    if (i >= ctx->by_label.size()) throw ConfigError("timing record index out of range");
    auto it = ctx->by_label.begin();
    std::advance(it, i);
    std::snprintf(buf, cap, "%s\t%.6f\t%llu", it->first.c_str(), it->second.first,
                  (unsigned long long)it->second.second);
  });
}

int catgnn_ctx_kernel_time(catgnn_ctx ctx, double* agg_ms, uint64_t* agg_launches, double* gemm_ms,
                           uint64_t* gemm_launches) {
  return guarded([&] {
    check_ctx(ctx);
    ctx->drain_timing();
    if (agg_ms) *agg_ms = ctx->agg_ms;
    if (agg_launches) *agg_launches = ctx->agg_n;
    if (gemm_ms) *gemm_ms = ctx->gemm_ms;
    if (gemm_launches) *gemm_launches = ctx->gemm_n;
  });
}

// -------------------------------------------------------------- artifact
int catgnn_artifact_open(const char* dir, catgnn_artifact* out) {
  return guarded([&] {
    if (!dir || !out) throw ConfigError("null argument");
    auto a = std::make_unique<catgnn_artifact_s>();
    open_artifact(a.get(), dir);
    *out = a.release();
  });
}

int catgnn_artifact_close(catgnn_artifact a) {
  return guarded([&] { delete a; });
}

int catgnn_artifact_get_info(catgnn_artifact a, catgnn_artifact_info* info) {
  return guarded([&] {
    if (!a || !info) throw ConfigError("null argument");
    info->num_partitions = a->num_partitions;
    info->num_nodes = a->num_nodes;
    info->num_edges = a->num_edges;
    info->feature_dim = a->feature_dim;
    info->has_features = a->has_features;
    info->has_meta = a->has_meta;
    info->add_reverse = a->add_reverse;
    info->replication_factor = a->replication_factor();
    info->manifest_replication_factor = a->manifest_rf;
  });
}

int catgnn_artifact_part_counts(catgnn_artifact a, uint32_t part, uint64_t* nodes, uint64_t* owned,
                                uint64_t* edges) {
  return guarded([&] {
    if (!a || part >= a->parts.size()) throw ConfigError("partition index out of range");
    const auto& t = a->parts[part];
    if (nodes) *nodes = t.ext.size();
    if (owned) *owned = t.m_owned;
    if (edges) *edges = t.edges.size() / 2;
  });
}

int catgnn_artifact_replica_map(catgnn_artifact a, uint32_t part, uint64_t* ext_ids, uint8_t* owner,
                                uint8_t* role, uint32_t* home) {
  return guarded([&] {
    if (!a || part >= a->parts.size()) throw ConfigError("partition index out of range");
    const auto& t = a->parts[part];
    const size_t n = t.ext.size();
    if (ext_ids) std::memcpy(ext_ids, t.ext.data(), n * 8);
    if (owner) std::memcpy(owner, t.owner.data(), n);
    if (role) std::memcpy(role, t.role.data(), n);
    if (home) {
      // owner partition of every external id: the unique partition whose node
      // table marks it owner (completion.cpp:46-50)
      std::vector<std::pair<uint64_t, uint32_t>> owners;
      for (uint32_t s = 0; s < a->parts.size(); ++s)
        for (size_t i = 0; i < a->parts[s].ext.size(); ++i)
          if (a->parts[s].owner[i]) owners.emplace_back(a->parts[s].ext[i], s);
      std::sort(owners.begin(), owners.end());
      for (size_t i = 0; i < n; ++i) {
        auto it = std::lower_bound(owners.begin(), owners.end(), std::make_pair(t.ext[i], 0u));
        if (it == owners.end() || it->first != t.ext[i])
          throw DataError("replica without an owner partition");
        home[i] = it->second;
      }
    }
  });
}

int catgnn_shard_train_views(catgnn_shard s, uint64_t* sub_rows, uint64_t* sub_nnz, uint64_t* nbr_nnz) {
  return guarded([&] {
    if (!s) throw ConfigError("null shard");
    CG_CUDA(cudaSetDevice(s->ctx->device));
    catgnn_shard_s* a = train_rows_view(s);
    catgnn_shard_s* b = train_nbr_view(s);
    if (sub_rows) *sub_rows = a ? a->rows : 0;
    if (sub_nnz) *sub_nnz = a ? a->nnz : 0;
    if (nbr_nnz) *nbr_nnz = b ? b->nnz : 0;
  });
}

int catgnn_shard_halo_map(catgnn_shard s, catgnn_artifact a, uint32_t* home, uint64_t* n_halo) {
  return guarded([&] {
    if (!s || !a) throw ConfigError("null argument");
    if (s->ext_ids.empty() && s->rows) throw ConfigError("shard was not loaded from a partition");
    CG_CUDA(cudaSetDevice(s->ctx->device));
    if (!s->d_ext.p && s->rows) {  // the device replica table (also the feature gathers' index)
      s->d_ext.alloc(s->rows);
      CG_CUDA(cudaMemcpyAsync(s->d_ext.p, s->ext_ids.data(), s->rows * 8, cudaMemcpyHostToDevice, s->ctx->stream));
    }
    std::vector<uint32_t> ids, parts;
    for (uint32_t q = 0; q < a->parts.size(); ++q)
      for (size_t i = 0; i < a->parts[q].ext.size(); ++i)
        if (a->parts[q].owner[i]) {
          if (a->parts[q].ext[i] > 0xffffffffull) throw ConfigError("halo map: ids beyond 2^32");
          ids.push_back((uint32_t)a->parts[q].ext[i]);
          parts.push_back(q);
        }
    const uint64_t h = halo_map(s, ids.data(), parts.data(), ids.size(), a->num_nodes, home);
    if (n_halo) *n_halo = h;
  });
}

// --------------------------------------------------------------- shards
int catgnn_shard_load(catgnn_ctx ctx, catgnn_artifact a, int32_t part, const char* input,
                      const char* features, catgnn_shard* out) {
  return guarded([&] {
    check_ctx(ctx);
    if (!a || !out) throw ConfigError("null argument");
    // train.cpp:220-221
    if (!a->has_meta) throw DataError("artifact has no labels; partition with --nodes to enable training");
    std::string feat_path = (features && *features) ? features : a->features;
    if (part < 0) {
      // global shard (train.cpp:224-252)
      std::string in_path = (input && *input) ? input : a->input;
      if (in_path.empty() || feat_path.empty())
        throw ConfigError("source edges/features not recorded in manifest; pass --input/--features");
      std::vector<float> feats;
      FeatureFile info;
      read_feature_matrix(feat_path, feats, &info);
      const uint64_t n = info.rows;
      if (n != a->num_nodes) throw DataError("feature file row count does not match the graph");
      std::vector<uint64_t> edges;
      read_edge_stream(in_path, a->add_reverse, edges);
      std::vector<uint32_t> pairs(edges.size());
      for (size_t k = 0; k < edges.size(); ++k) {
        if (edges[k] >= n) throw DataError("training requires dense external ids in [0,|V|)");
        pairs[k] = (uint32_t)edges[k];
      }
      std::vector<int32_t> labels(n, 0);
      std::vector<uint32_t> tr, va, te;
      for (const auto& m : a->meta) {
        if (m.node >= n) throw DataError("node meta refers to an id outside [0,|V|)");
        labels[m.node] = m.label;
        if (m.role == 1) tr.push_back((uint32_t)m.node);
        else if (m.role == 2) va.push_back((uint32_t)m.node);
        else if (m.role == 3) te.push_back((uint32_t)m.node);
      }
      auto s = new_shard(ctx, n);
      shard_csr_from_pairs(s.get(), pairs.data(), pairs.size() / 2);
      upload_features(s.get(), feats.data(), info.dim);
      set_labels(s.get(), labels.data(), tr.data(), tr.size(), va.data(), va.size(), te.data(), te.size());
      *out = s.release();
      return;
    }
    if ((uint32_t)part >= a->parts.size()) throw ConfigError("partition index out of range");
    const auto& t = a->parts[part];
    const uint64_t rows = t.ext.size();
    // train.cpp:258-267: local row = node-table position; train rows = owner && train
    std::vector<int32_t> labels(rows, 0);
    std::vector<uint32_t> tr;
    for (uint64_t i = 0; i < rows; ++i) {
      const MetaEntry* m = a->find_meta(t.ext[i]);
      labels[i] = m ? m->label : 0;
      if (t.owner[i] && t.role[i] == 1) tr.push_back((uint32_t)i);
    }
    auto s = new_shard(ctx, rows);
    s->ext_ids = t.ext;
    s->owner = t.owner;
    s->role = t.role;
    shard_csr_from_ext(s.get(), t.ext.data(), t.edges.data(), t.edges.size() / 2);
    std::vector<float> feats;
    uint32_t dim = 0;
    if (a->has_features) {
      FeatureFile info;
      read_feature_matrix((std::filesystem::path(a->dir) / t.dir / "features.bin").string(), feats, &info);
      dim = info.dim;
    } else {
      // gathered from the global matrix by external id (train.cpp:277-283)
      if (feat_path.empty()) throw ConfigError("source features not recorded in manifest; pass --features");
      std::vector<float> global;
      FeatureFile info;
      read_feature_matrix(feat_path, global, &info);
      dim = info.dim;
      feats.resize(rows * (size_t)dim);
      for (uint64_t i = 0; i < rows; ++i) {
        if (t.ext[i] >= info.rows)
          throw DataError("feature row " + std::to_string(t.ext[i]) + " out of range in " + feat_path);
        std::memcpy(feats.data() + i * dim, global.data() + t.ext[i] * dim, dim * 4);
      }
    }
    upload_features(s.get(), feats.data(), dim);
    set_labels(s.get(), labels.data(), tr.data(), tr.size(), nullptr, 0, nullptr, 0);
    *out = s.release();
  });
}

int catgnn_shard_create(catgnn_ctx ctx, uint32_t rows, const uint32_t* pairs, uint64_t num_edges,
                        const float* features, uint32_t dim, catgnn_shard* out) {
  return guarded([&] {
    check_ctx(ctx);
    if (!out || (num_edges && !pairs)) throw ConfigError("null argument");
    auto s = new_shard(ctx, rows);
    shard_csr_from_pairs(s.get(), pairs, num_edges);
    upload_features(s.get(), features, features ? dim : 0);
    set_labels(s.get(), nullptr, nullptr, 0, nullptr, 0, nullptr, 0);
    CG_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = s.release();
  });
}

int catgnn_shard_create_from_part(catgnn_ctx ctx, uint64_t rows, const uint64_t* ext_ids,
                                  const uint8_t* owner, const uint8_t* role, const int32_t* labels,
                                  const uint64_t* edges_ext, uint64_t num_edges,
                                  const float* features, uint32_t dim, catgnn_shard* out) {
  return guarded([&] {
    check_ctx(ctx);
    if (!out || !ext_ids || !owner || !role) throw ConfigError("null argument");
    auto s = new_shard(ctx, rows);
    s->ext_ids.assign(ext_ids, ext_ids + rows);
    s->owner.assign(owner, owner + rows);
    s->role.assign(role, role + rows);
    shard_csr_from_ext(s.get(), ext_ids, edges_ext, num_edges);
    upload_features(s.get(), features, features ? dim : 0);
    std::vector<uint32_t> tr;
    for (uint64_t i = 0; i < rows; ++i)
      if (owner[i] && role[i] == 1) tr.push_back((uint32_t)i);
    set_labels(s.get(), labels, tr.data(), tr.size(), nullptr, 0, nullptr, 0);
    *out = s.release();
  });
}

int catgnn_shard_destroy(catgnn_shard s) {
  return guarded([&] {
    if (!s) return;
    catgnn_ctx c = s->ctx;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    delete s;
    ctx_release(c);
  });
}

int catgnn_shard_set_labels(catgnn_shard s, const int32_t* labels, const uint32_t* train_rows,
                            uint64_t n_train, const uint32_t* val_rows, uint64_t n_val,
                            const uint32_t* test_rows, uint64_t n_test) {
  return guarded([&] {
    check_shard(s);
    set_labels(s, labels, train_rows, n_train, val_rows, n_val, test_rows, n_test);
  });
}

int catgnn_shard_upload_features(catgnn_shard s, const float* features, uint32_t dim) {
  return guarded([&] {
    check_shard(s);
    if (dim != s->dim || !s->x.p) {
      upload_features(s, features, dim);
      return;
    }
    if (s->rows && dim) copy_features_in(s, features, dim);
    });
}

int catgnn_shard_get_info(catgnn_shard s, catgnn_shard_info* info) {
  return guarded([&] {
    check_shard(s);
    if (!info) throw ConfigError("null argument");
    info->rows = s->rows;
    info->nnz = s->nnz;
    info->dim = s->dim;
    info->classes = s->classes;
    info->n_train = s->h_train.size();
    info->n_val = s->h_val.size();
    info->n_test = s->h_test.size();
    info->heavy_rows = s->n_heavy;
    info->tasks = s->n_units;
  });
}

int catgnn_csr_export(catgnn_shard s, uint64_t* offsets, uint32_t* neighbors) {
  return guarded([&] {
    check_shard(s);
    cudaStream_t st = s->ctx->stream;
    if (offsets)
      CG_CUDA(cudaMemcpyAsync(offsets, s->row_ptr.p, (s->rows + 1) * 8, cudaMemcpyDeviceToHost, st));
    if (neighbors && s->nnz)
      CG_CUDA(cudaMemcpyAsync(neighbors, s->col.p, s->nnz * 4, cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaStreamSynchronize(st));
  });
}

int catgnn_shard_role_rows(catgnn_shard s, int role, uint32_t* rows) {
  return guarded([&] {
    check_shard(s);
    const std::vector<uint32_t>* v = role == 1 ? &s->h_train : role == 2 ? &s->h_val
                                   : role == 3 ? &s->h_test : nullptr;
    if (!v) throw ConfigError("role must be 1 (train), 2 (val) or 3 (test)");
    if (rows) std::copy(v->begin(), v->end(), rows);
  });
}

int catgnn_shard_labels(catgnn_shard s, int32_t* labels) {
  return guarded([&] {
    check_shard(s);
    std::copy(s->h_labels.begin(), s->h_labels.end(), labels);
  });
}

int catgnn_shard_export_features(catgnn_shard s, int which, float* out) {
  return guarded([&] {
    check_shard(s);
    if (which == 0 && !s->x_fp32_valid)
      throw ConfigError("shard features are held as bf16x3 only (catgnn_shard_set_feature_layout)");
    const float* src = which == 0 ? s->x.p : s->xprop.p;
    if (!src) throw ConfigError("requested feature buffer is not materialised");
    if (s->rows && s->dim)
      CG_CUDA(cudaMemcpy2DAsync(out, s->dim * sizeof(float), src, s->ld * sizeof(float),
                                s->dim * sizeof(float), s->rows, cudaMemcpyDeviceToHost,
                                s->ctx->stream));
    CG_CUDA(cudaStreamSynchronize(s->ctx->stream));
  });
}

// ----------------------------------------------------------------- SGC
int catgnn_sgc_propagate(catgnn_shard s, uint32_t hops) {
  return guarded([&] {
    check_shard(s);
    catgnn_ctx ctx = s->ctx;
    const size_t n = std::max<uint64_t>(1, s->rows) * s->ld;
    s->xprop.reserve(n);
    if (!s->x_fp32_valid)
      throw ConfigError("shard features are held as bf16x3 only (catgnn_shard_set_feature_layout); upload them");
    if (hops == 0 || s->rows == 0) {  // k = 0 is the identity (train.hpp:29-32)
      if (s->rows) copy_rows(ctx, s->x.p, s->ld, s->xprop.p, s->ld, s->rows, s->ld);
      return;
    }
    float* tmp = ctx->scratch_buf<float>("sgc_pingpong", n);
    // ping-pong so that the final hop lands in xprop (train.cpp:53-63)
    const float* cur = s->x.p;
    for (uint32_t h = 0; h < hops; ++h) {
      float* dst = ((hops - 1 - h) % 2 == 0) ? s->xprop.p : tmp;
      AggArgs a;
      a.in = cur;
      a.in_ld = s->ld;
      a.out = dst;
      a.out_ld = s->ld;
      a.width = s->ld;
      a.self = 1;
      a.norm = kNormSgc;
      aggregate(s, a);
      cur = dst;
    }
    CG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int catgnn_softmax_loss(catgnn_shard s, const float* W, const float* b, uint32_t classes,
                        const uint32_t* rows, uint64_t n_rows, double* loss) {
  return guarded([&] {
    check_shard(s);
    ensure_prop(s);
    catgnn_ctx ctx = s->ctx;
    cudaStream_t st = ctx->stream;
    float* dW = ctx->scratch_buf<float>("p_W", (size_t)s->dim * classes);
    float* db = ctx->scratch_buf<float>("p_b", classes);
    uint32_t* dr = ctx->scratch_buf<uint32_t>("p_rows", std::max<uint64_t>(1, n_rows));
    double* rl = ctx->scratch_buf<double>("p_rowloss", std::max<uint64_t>(1, n_rows));
    h2d(dW, W, (size_t)s->dim * classes, st);
    h2d(db, b, classes, st);
    h2d(dr, rows, n_rows, st);
    if (n_rows) sgc_eval(ctx, s->xprop.p, s->ld, s->dim, dW, db, classes, s->labels.p, dr, n_rows, nullptr, rl);
    std::vector<double> h(n_rows);
    if (n_rows) CG_CUDA(cudaMemcpyAsync(h.data(), rl, n_rows * 8, cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaStreamSynchronize(st));
    double acc = 0.0;
    for (double v : h) acc += v;
    *loss = acc / static_cast<double>(n_rows);
  });
}

int catgnn_softmax_gradient(catgnn_shard s, const float* W, const float* b, uint32_t classes,
                            const uint32_t* rows, uint64_t n_rows, float* gW, float* gb) {
  return guarded([&] {
    check_shard(s);
    ensure_prop(s);
    catgnn_ctx ctx = s->ctx;
    cudaStream_t st = ctx->stream;
    const size_t wn = (size_t)s->dim * classes;
    float* dW = ctx->scratch_buf<float>("p_W", wn);
    float* db = ctx->scratch_buf<float>("p_b", classes);
    float* dgW = ctx->scratch_buf<float>("p_gW", wn);
    float* dgb = ctx->scratch_buf<float>("p_gb", classes);
    uint32_t* dr = ctx->scratch_buf<uint32_t>("p_rows", std::max<uint64_t>(1, n_rows));
    h2d(dW, W, wn, st);
    h2d(db, b, classes, st);
    h2d(dr, rows, n_rows, st);
    SgcReplicaHost r{s->xprop.p, s->ld, s->labels.p, dr, n_rows, dW, db, dgW, dgb};
    sgc_train(ctx, {r}, s->dim, classes, 0.f, (uint32_t)std::max<uint64_t>(1, n_rows), 1, true);
    CG_CUDA(cudaMemcpyAsync(gW, dgW, wn * 4, cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaMemcpyAsync(gb, dgb, classes * 4, cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaStreamSynchronize(st));
  });
}

int catgnn_train_epochs(uint32_t n, const catgnn_shard* shards, float* const* W, float* const* b,
                        uint32_t classes, double lr, uint32_t batch, uint64_t epoch_begin,
                        uint64_t epoch_end, const uint64_t* seeds) {
  return guarded([&] {
    if (n == 0) return;
    catgnn_ctx ctx = shards[0]->ctx;
    for (uint32_t i = 0; i < n; ++i) {
      check_shard(shards[i]);
      ensure_prop(shards[i]);
      if (shards[i]->ctx != ctx) throw ConfigError("replicas must share one context");
      if (shards[i]->dim != shards[0]->dim) throw DataError("model shapes differ across replicas");
    }
    const uint32_t dim = shards[0]->dim;
    const size_t wn = (size_t)dim * classes;
    cudaStream_t st = ctx->stream;
    std::vector<SgcReplicaHost> reps;
    std::vector<std::vector<uint32_t>> orders(n);
    bool any = false;
    for (uint32_t i = 0; i < n; ++i) {
      catgnn_shard s = shards[i];
      if (s->h_train.empty()) {
        // train.cpp:100-104
        std::fprintf(stderr, "warning: empty training set, parameters left unchanged\n");
        continue;
      }
      if (batch == 0) throw ConfigError("batch size must be >= 1");
      orders[i] = epoch_orders(s->h_train, epoch_begin, epoch_end, seeds[i]);
      any = true;
    }
    if (!any || epoch_end <= epoch_begin) return;
    float* dparams = ctx->scratch_buf<float>("te_params", (size_t)n * (wn + classes));
    size_t total_order = 0;
    for (auto& o : orders) total_order += o.size();
    uint32_t* dord = ctx->scratch_buf<uint32_t>("te_orders", std::max<size_t>(1, total_order));
    size_t off = 0;
    for (uint32_t i = 0; i < n; ++i) {
      if (orders[i].empty()) continue;
      float* pw = dparams + (size_t)i * (wn + classes);
      h2d(pw, W[i], wn, st);
      h2d(pw + wn, b[i], classes, st);
      h2d(dord + off, orders[i].data(), orders[i].size(), st);
      reps.push_back(SgcReplicaHost{shards[i]->xprop.p, shards[i]->ld, shards[i]->labels.p, dord + off,
                                    shards[i]->h_train.size(), pw, pw + wn});
      off += orders[i].size();
    }
    sgc_train(ctx, reps, dim, classes, (float)lr, batch, (uint32_t)(epoch_end - epoch_begin), false);
    for (uint32_t i = 0; i < n; ++i) {
      if (orders[i].empty()) continue;
      float* pw = dparams + (size_t)i * (wn + classes);
      CG_CUDA(cudaMemcpyAsync(W[i], pw, wn * 4, cudaMemcpyDeviceToHost, st));
      CG_CUDA(cudaMemcpyAsync(b[i], pw + wn, classes * 4, cudaMemcpyDeviceToHost, st));
    }
    CG_CUDA(cudaStreamSynchronize(st));
  });
}

// train_local (train.cpp:130-137): zero_params(dim, max label + 1) then
// train_epochs over [0, epochs) with cfg->seed, on the shard's features
// propagated prop_hops times (the caller, train-sim --compare-centralized,
// gnnpart.cpp:330-335, propagates the global shard first).  W == NULL queries
// the class count only.
int catgnn_train_local(catgnn_shard s, const catgnn_train_config* cfg, float* W, float* b, uint32_t* classes) {
  return guarded([&] {
    check_shard(s);
    if (!cfg) throw ConfigError("null argument");
    if (classes) *classes = s->classes;
    if (!W) return;
    if (!b) throw ConfigError("null argument");
    if (catgnn_sgc_propagate(s, cfg->prop_hops)) throw InternalError(g_last_error);
    std::fill(W, W + (size_t)s->dim * s->classes, 0.f);  // zero_params (train.cpp:67-72)
    std::fill(b, b + s->classes, 0.f);
    const uint64_t seed = cfg->seed;
    catgnn_shard_s* const sh = s;
    if (int rc = catgnn_train_epochs(1, &sh, &W, &b, s->classes, cfg->lr, cfg->batch, 0, cfg->epochs, &seed))
      throw_last_error_code(rc);
  });
}

int catgnn_sync_weights(const uint64_t* counts, uint32_t n, double* alpha) {
  return guarded([&] {
    std::vector<double> a = sync_weights_vec(std::vector<uint64_t>(counts, counts + n));
    std::copy(a.begin(), a.end(), alpha);
  });
}

int catgnn_model_average_host(catgnn_ctx ctx, uint32_t n, const float* const* params, uint64_t count,
                              const uint64_t* train_counts, float* out) {
  return guarded([&] {
    check_ctx(ctx);
    if (n == 0) throw DataError("model averaging needs one training count per replica");
    std::vector<double> alpha = sync_weights_vec(std::vector<uint64_t>(train_counts, train_counts + n));
    float* d = ctx->scratch_buf<float>("mah", (size_t)(n + 1) * count);
    std::vector<const float*> src(n);
    for (uint32_t i = 0; i < n; ++i) {
      h2d(d + (size_t)i * count, params[i], count, ctx->stream);
      src[i] = d + (size_t)i * count;
    }
    float* dout = d + (size_t)n * count;
    average_params(ctx, src, alpha, count, dout);
    CG_CUDA(cudaMemcpyAsync(out, dout, count * 4, cudaMemcpyDeviceToHost, ctx->stream));
    CG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int catgnn_evaluate_micro_f1(catgnn_shard s, const float* W, const float* b, uint32_t classes,
                             const uint32_t* mask_rows, uint64_t n_mask, double* f1) {
  return guarded([&] {
    check_shard(s);
    ensure_prop(s);
    if (n_mask == 0) throw DataError("evaluation mask is empty");
    catgnn_ctx ctx = s->ctx;
    cudaStream_t st = ctx->stream;
    float* dW = ctx->scratch_buf<float>("p_W", (size_t)s->dim * classes);
    float* db = ctx->scratch_buf<float>("p_b", classes);
    uint32_t* dm = ctx->scratch_buf<uint32_t>("p_rows", n_mask);
    h2d(dW, W, (size_t)s->dim * classes, st);
    h2d(db, b, classes, st);
    h2d(dm, mask_rows, n_mask, st);
    *f1 = eval_f1(s, dW, db, classes, dm, n_mask);
  });
}

int catgnn_distributed_train(uint32_t p, const catgnn_shard* shards, catgnn_shard global,
                             uint32_t workers, uint32_t sync_interval, const catgnn_train_config* cfg,
                             catgnn_dist_result* result) {
  return guarded([&] {
    // train.cpp:291-295
    if (workers == 0 || p == 0) throw ConfigError("need at least one worker and one partition");
    if (p % workers != 0) throw ConfigError("partition count must be a multiple of the worker count");
    if (sync_interval == 0) throw ConfigError("sync interval must be >= 1");
    check_shard(global);
    catgnn_ctx ctx = global->ctx;
    cudaStream_t st = ctx->stream;
    std::vector<uint64_t> counts;
    for (uint32_t i = 0; i < p; ++i) {
      check_shard(shards[i]);
      if (shards[i]->ctx != ctx) throw ConfigError("all shards must share one context");
      if (shards[i]->dim != global->dim) throw DataError("model shapes differ across replicas");
      if (catgnn_sgc_propagate(shards[i], cfg->prop_hops)) throw InternalError(g_last_error);
      counts.push_back(shards[i]->h_train.size());
    }
    if (catgnn_sgc_propagate(global, cfg->prop_hops)) throw InternalError(g_last_error);
    const uint32_t classes = global->classes;
    const uint32_t dim = global->dim;
    const size_t wn = (size_t)dim * classes, pn = wn + classes;
    // shared params + p replicas, all device-resident for the whole run
    float* shared = ctx->scratch_buf<float>("dt_shared", pn);
    float* reps = ctx->scratch_buf<float>("dt_reps", pn * p);
    CG_CUDA(cudaMemsetAsync(shared, 0, pn * 4, st));  // zero_params (train.cpp:67-72)
    std::vector<double> alpha = sync_weights_vec(counts);
    uint64_t done = 0, ops = 0;
    result->n_hist = 0;
    while (done < cfg->epochs) {
      const uint64_t chunk = std::min<uint64_t>(sync_interval, cfg->epochs - done);
      std::vector<SgcReplicaHost> rh;
      std::vector<std::vector<uint32_t>> orders(p);
      size_t total = 0;
      for (uint32_t i = 0; i < p; ++i) {
        CG_CUDA(cudaMemcpyAsync(reps + pn * i, shared, pn * 4, cudaMemcpyDeviceToDevice, st));
        if (shards[i]->h_train.empty()) {
          std::fprintf(stderr, "warning: empty training set, parameters left unchanged\n");
          continue;
        }
        if (cfg->batch == 0) throw ConfigError("batch size must be >= 1");
        orders[i] = epoch_orders(shards[i]->h_train, done, done + chunk, cfg->seed + i);
        total += orders[i].size();
      }
      uint32_t* dord = ctx->scratch_buf<uint32_t>("dt_orders", std::max<size_t>(1, total));
      size_t off = 0;
      for (uint32_t i = 0; i < p; ++i) {
        if (orders[i].empty()) continue;
        h2d(dord + off, orders[i].data(), orders[i].size(), st);
        rh.push_back(SgcReplicaHost{shards[i]->xprop.p, shards[i]->ld, shards[i]->labels.p, dord + off,
                                    shards[i]->h_train.size(), reps + pn * i, reps + pn * i + wn});
        off += orders[i].size();
      }
      if (!rh.empty()) sgc_train(ctx, rh, dim, classes, (float)cfg->lr, cfg->batch, (uint32_t)chunk, false);
      std::vector<const float*> src(p);
      for (uint32_t i = 0; i < p; ++i) src[i] = reps + pn * i;
      average_params(ctx, src, alpha, pn, shared);
      done += chunk;
      ops++;
      double vf = global->h_val.empty() ? 0.0 : eval_f1(global, shared, shared + wn, classes, global->d_val.p, global->h_val.size());
      double tf = global->h_test.empty() ? 0.0 : eval_f1(global, shared, shared + wn, classes, global->d_test.p, global->h_test.size());
      if (result->n_hist < result->hist_capacity) {
        uint64_t k = result->n_hist;
        if (result->hist_epoch) result->hist_epoch[k] = done;
        if (result->hist_syncs) result->hist_syncs[k] = ops;
        if (result->hist_val) result->hist_val[k] = vf;
        if (result->hist_test) result->hist_test[k] = tf;
      }
      result->n_hist++;
    }
    result->averaging_ops = ops;
    result->dim = dim;
    result->classes = classes;
    if (result->W) CG_CUDA(cudaMemcpyAsync(result->W, shared, wn * 4, cudaMemcpyDeviceToHost, st));
    if (result->b) CG_CUDA(cudaMemcpyAsync(result->b, shared + wn, classes * 4, cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaStreamSynchronize(st));
  });
}

}  // extern "C"
