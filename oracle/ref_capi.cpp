// TEST INFRASTRUCTURE ONLY — the CPU oracle.  Never linked into the product.
//
// extern "C" entry points over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile straight from
// the read-only tree with the Eigen-subset shim in oracle/eigen_shim).  Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs load this library (oracle/_ref/libgnnpart_ref.so).
//
// Each wrapper converts plain row-major arrays to the reference's types, calls
// the reference function, and converts back.  Error convention mirrors the
// reference CLI (proj/tools/gnnpart.cpp:387-399): ConfigError -> 2,
// DataError -> 3, anything else -> 4; message via ref_last_error().
#include <cstdint>
#include <cstring>
#include <exception>
#include <filesystem>
#include <iostream>
#include <memory>
#include <string>
#include <vector>

#include "gnnpart/baselines.hpp"
#include "gnnpart/completion.hpp"
#include "gnnpart/edge_stream.hpp"
#include "gnnpart/metrics.hpp"
#include "gnnpart/spring.hpp"
#include "gnnpart/store.hpp"
#include "gnnpart/synth.hpp"
#include "gnnpart/train.hpp"

using namespace gnnpart;
namespace fs = std::filesystem;

namespace {

thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    g_err.clear();
    return 0;
  } catch (const ConfigError& e) {
    g_err = std::string("bad-config: ") + e.what();
    return 2;
  } catch (const DataError& e) {
    g_err = std::string("bad-input: ") + e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = std::string("internal: ") + e.what();
    return 4;
  }
}

Eigen::MatrixXd from_rowmajor(const double* x, std::uint64_t rows, std::uint32_t cols) {
  Eigen::MatrixXd m(static_cast<Eigen::Index>(rows), cols);
  for (std::uint64_t i = 0; i < rows; ++i)
    for (std::uint32_t j = 0; j < cols; ++j)
      m(static_cast<Eigen::Index>(i), j) = x[i * cols + j];
  return m;
}

void to_rowmajor(const Eigen::MatrixXd& m, double* out) {
  const std::uint64_t cols = static_cast<std::uint64_t>(m.cols());
  for (Eigen::Index i = 0; i < m.rows(); ++i)
    for (Eigen::Index j = 0; j < m.cols(); ++j)
      out[static_cast<std::uint64_t>(i) * cols + static_cast<std::uint64_t>(j)] = m(i, j);
}

LocalAdjacency adjacency_from(std::uint32_t rows, const std::uint32_t* offsets,
                              const std::uint32_t* neighbors) {
  LocalAdjacency adj;
  adj.offsets.assign(offsets, offsets + rows + 1);
  adj.neighbors.assign(neighbors, neighbors + offsets[rows]);
  return adj;
}

ModelParams params_from(const double* W, const double* b, std::uint32_t dim, std::uint32_t C) {
  ModelParams p;
  p.weight = from_rowmajor(W, dim, C);
  p.bias = Eigen::VectorXd(C);
  for (std::uint32_t c = 0; c < C; ++c) p.bias(c) = b[c];
  return p;
}

void params_to(const ModelParams& p, double* W, double* b) {
  to_rowmajor(p.weight, W);
  for (Eigen::Index c = 0; c < p.bias.size(); ++c) b[c] = p.bias(c);
}

std::vector<std::int32_t> labels_from(const std::int32_t* y, std::uint64_t n) {
  return std::vector<std::int32_t>(y, y + n);
}

struct TDHandle {
  StoredArtifact artifact;
  TrainingData data;
};

const Shard& shard_of(const TDHandle* h, int s) {
  if (s < 0) return h->data.global;
  if (static_cast<std::size_t>(s) >= h->data.shards.size())
    throw ConfigError("shard index out of range");
  return h->data.shards[static_cast<std::size_t>(s)];
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- train.cpp:30-47 -----------------------------------------------------------
int ref_build_adjacency(std::uint32_t rows, const std::uint32_t* pairs, std::uint64_t num_edges,
                        std::uint32_t* offsets, std::uint32_t* neighbors,
                        std::uint64_t neighbor_capacity) {
  return guarded([&] {
    std::vector<std::pair<std::uint32_t, std::uint32_t>> edges(num_edges);
    for (std::uint64_t k = 0; k < num_edges; ++k) edges[k] = {pairs[2 * k], pairs[2 * k + 1]};
    LocalAdjacency adj = build_adjacency(rows, edges);
    if (adj.neighbors.size() > neighbor_capacity) throw ConfigError("neighbor buffer too small");
    std::memcpy(offsets, adj.offsets.data(), adj.offsets.size() * 4);
    std::memcpy(neighbors, adj.neighbors.data(), adj.neighbors.size() * 4);
  });
}

// ---- train.cpp:49-65 -----------------------------------------------------------
int ref_sgc_propagate(std::uint32_t rows, const std::uint32_t* offsets,
                      const std::uint32_t* neighbors, const double* x, std::uint32_t dim,
                      std::uint32_t hops, double* out) {
  return guarded([&] {
    LocalAdjacency adj = adjacency_from(rows, offsets, neighbors);
    Eigen::MatrixXd y = sgc_propagate(adj, from_rowmajor(x, rows, dim), hops);
    to_rowmajor(y, out);
  });
}

// Same as above but the input matrix is already column-major (no conversion
// inside the timed region of the CPU baseline).
int ref_sgc_propagate_colmajor(std::uint32_t rows, const std::uint32_t* offsets,
                               const std::uint32_t* neighbors, const double* x_colmajor,
                               std::uint32_t dim, std::uint32_t hops, double* out_colmajor) {
  return guarded([&] {
    LocalAdjacency adj = adjacency_from(rows, offsets, neighbors);
    Eigen::MatrixXd xm(rows, dim);
    std::memcpy(xm.data(), x_colmajor, sizeof(double) * rows * dim);
    Eigen::MatrixXd y = sgc_propagate(adj, xm, hops);
    std::memcpy(out_colmajor, y.data(), sizeof(double) * rows * dim);
  });
}

// ---- train.cpp:74-94 -----------------------------------------------------------
int ref_softmax_loss(const double* W, const double* b, std::uint32_t dim, std::uint32_t C,
                     const double* x, std::uint64_t rows, const std::int32_t* y,
                     double* loss) {
  return guarded([&] {
    ModelParams p = params_from(W, b, dim, C);
    *loss = softmax_loss(p.weight, p.bias, from_rowmajor(x, rows, dim), labels_from(y, rows));
  });
}

int ref_softmax_gradient(const double* W, const double* b, std::uint32_t dim, std::uint32_t C,
                         const double* x, std::uint64_t rows, const std::int32_t* y,
                         double* gW, double* gb) {
  return guarded([&] {
    ModelParams p = params_from(W, b, dim, C);
    Eigen::MatrixXd gw(dim, C);
    Eigen::VectorXd gbv(C);
    softmax_gradient(p.weight, p.bias, from_rowmajor(x, rows, dim), labels_from(y, rows), gw,
                     gbv);
    to_rowmajor(gw, gW);
    for (std::uint32_t c = 0; c < C; ++c) gb[c] = gbv(c);
  });
}

// ---- train.cpp:96-128 ----------------------------------------------------------
int ref_train_epochs(double* W, double* b, std::uint32_t dim, std::uint32_t C, const double* x,
                     std::uint64_t rows, const std::int32_t* labels,
                     const std::uint32_t* train_rows, std::uint64_t n_train, double lr,
                     std::uint32_t batch, std::uint64_t epoch_begin, std::uint64_t epoch_end,
                     std::uint64_t seed) {
  return guarded([&] {
    ModelParams p = params_from(W, b, dim, C);
    TrainConfig cfg;
    cfg.lr = lr;
    cfg.batch = batch;
    std::vector<std::uint32_t> tr(train_rows, train_rows + n_train);
    train_epochs(p, from_rowmajor(x, rows, dim), labels_from(labels, rows), tr, cfg,
                 epoch_begin, epoch_end, seed);
    params_to(p, W, b);
  });
}

// ---- train.cpp:139-172 ---------------------------------------------------------
int ref_sync_weights(const std::uint64_t* counts, std::uint32_t n, double* alpha) {
  return guarded([&] {
    std::vector<double> a = sync_weights(std::vector<std::uint64_t>(counts, counts + n));
    std::memcpy(alpha, a.data(), sizeof(double) * a.size());
  });
}

int ref_model_average(std::uint32_t n, std::uint32_t dim, std::uint32_t C, const double* Ws,
                      const double* bs, const std::uint64_t* counts, double* W_out,
                      double* b_out) {
  return guarded([&] {
    std::vector<ModelParams> reps;
    for (std::uint32_t i = 0; i < n; ++i)
      reps.push_back(params_from(Ws + std::uint64_t{i} * dim * C, bs + std::uint64_t{i} * C, dim, C));
    ModelParams avg = model_average(reps, std::vector<std::uint64_t>(counts, counts + n));
    params_to(avg, W_out, b_out);
  });
}

// ---- train.cpp:174-198 ---------------------------------------------------------
int ref_evaluate_micro_f1(const double* W, const double* b, std::uint32_t dim, std::uint32_t C,
                          const double* x, std::uint64_t rows, const std::int32_t* labels,
                          const std::uint32_t* mask, std::uint64_t n_mask, double* f1) {
  return guarded([&] {
    ModelParams p = params_from(W, b, dim, C);
    *f1 = evaluate_micro_f1(p, from_rowmajor(x, rows, dim), labels_from(labels, rows),
                            std::vector<std::uint32_t>(mask, mask + n_mask));
  });
}

// ---- partition pipeline: the `gnnpart partition` handler (tools/gnnpart.cpp:61-109,
// :254-268) restated over the same library calls -------------------------------------
int ref_partition(const char* input, const char* format, int add_reverse, const char* nodes,
                  const char* features, const char* algo, std::uint32_t partitions, double beta,
                  std::uint64_t tau_vol, double lambda, double balance_slack, std::uint32_t hops,
                  int no_completion, int shuffle_isolated, std::uint64_t seed,
                  const char* out_dir) {
  return guarded([&] {
    fs::path in(input);
    EdgeFormat fmt = (format && *format) ? parse_edge_format(format)
                                         : (in.extension() == ".bin" ? EdgeFormat::binary_u64
                                                                     : EdgeFormat::text_tsv);
    EdgeStream stream(in, fmt, add_reverse != 0);
    GraphIndex index = compute_degrees(stream);
    NodeMetaMap meta;
    std::string nodes_s = nodes ? nodes : "";
    std::string feat_s = features ? features : "";
    if (!nodes_s.empty()) meta = read_node_meta(nodes_s);
    std::string a = algo ? algo : "spring";
    std::uint64_t tau = tau_vol != 0 ? tau_vol : default_tau_vol(index.num_edges, partitions);
    HomeMap homes;
    if (a == "spring") {
      ClusterState state = cluster_stream(stream, index, tau);
      MergePlan plan = select_representatives(state, index);
      merge_clusters(state, plan, index, partitions, beta);
      homes = resolve_homes(assign_partitions(state, partitions, seed, shuffle_isolated != 0));
    } else if (a == "dbh") {
      homes = resolve_homes(dbh_partition(stream, index, partitions), index.num_nodes(), seed);
    } else if (a == "greedy") {
      homes = resolve_homes(greedy_partition(stream, index, partitions, balance_slack),
                            index.num_nodes(), seed);
    } else if (a == "hdrf") {
      homes = resolve_homes(hdrf_partition(stream, index, partitions, lambda), index.num_nodes(),
                            seed);
    } else if (a == "2ps") {
      homes = resolve_homes(two_phase_partition(stream, index, partitions, tau),
                            index.num_nodes(), seed);
    } else {
      throw ConfigError("unknown algorithm: " + a);
    }
    PartitionedGraph g = no_completion ? random_edge_assign(stream, index, homes, meta, seed)
                                       : complete_edges(stream, index, homes, meta, hops);
    nlohmann::json params{{"input", std::string(input)},
                          {"algorithm", a},
                          {"partitions", partitions},
                          {"beta", beta},
                          {"tau_vol", tau},
                          {"lambda", lambda},
                          {"balance_slack", balance_slack},
                          {"hops", hops},
                          {"completion", no_completion == 0},
                          {"add_reverse", add_reverse != 0},
                          {"seed", seed},
                          {"nodes", nodes_s},
                          {"features", feat_s}};
    fs::path fpath = feat_s;
    write_partitions(g, out_dir, a, params, nodes_s.empty() ? nullptr : &meta,
                     feat_s.empty() ? nullptr : &fpath);
  });
}

// SPRING home map only (dense first-seen order -> ext id, and partition per ext id);
// `home_by_ext` must hold max_ext+1 entries, filled with the home partition.
int ref_spring_homes(const char* input, int add_reverse, std::uint32_t partitions, double beta,
                     std::uint64_t tau_vol, std::uint64_t seed, std::uint32_t* home_by_ext,
                     std::uint64_t capacity) {
  return guarded([&] {
    fs::path in(input);
    EdgeFormat fmt = in.extension() == ".bin" ? EdgeFormat::binary_u64 : EdgeFormat::text_tsv;
    EdgeStream stream(in, fmt, add_reverse != 0);
    GraphIndex index = compute_degrees(stream);
    SpringParams sp;
    sp.partitions = partitions;
    sp.beta = beta;
    sp.tau_vol = tau_vol;
    sp.seed = seed;
    PartitionAssignment pa = spring_partition(stream, index, sp);
    for (NodeId v = 0; v < index.num_nodes(); ++v) {
      ExtNodeId e = index.dense_to_ext[v];
      if (e >= capacity) throw ConfigError("home buffer too small");
      home_by_ext[e] = pa.node_part[v];
    }
  });
}

// ---- edge_stream.cpp:192-215 compute_degrees -------------------------------------
// dense_to_ext / degree need `capacity` entries (2 x records is always enough).
int ref_compute_degrees(const char* input, int add_reverse, std::uint64_t* dense_to_ext, std::uint32_t* degree,
                        std::uint64_t capacity, std::uint64_t* num_nodes, std::uint64_t* num_edges,
                        std::uint64_t* num_self_loops) {
  return guarded([&] {
    fs::path in(input);
    EdgeFormat fmt = in.extension() == ".bin" ? EdgeFormat::binary_u64 : EdgeFormat::text_tsv;
    EdgeStream stream(in, fmt, add_reverse != 0);
    GraphIndex index = compute_degrees(stream);
    if (index.num_nodes() > capacity) throw ConfigError("index buffer too small");
    for (NodeId v = 0; v < index.num_nodes(); ++v) {
      dense_to_ext[v] = index.dense_to_ext[v];
      degree[v] = index.degree[v];
    }
    *num_nodes = index.num_nodes();
    *num_edges = index.num_edges;
    *num_self_loops = index.num_self_loops;
  });
}

// ---- metrics.cpp:9-12 over a stored artifact (store.cpp:269-333) ----------------
int ref_artifact_replication_factor(const char* dir, double* rf, double* manifest_rf) {
  return guarded([&] {
    StoredArtifact art = read_partitions(dir);
    *rf = replication_factor(art.graph);
    *manifest_rf = art.manifest.replication_factor;
  });
}

// ---- train.cpp:216-287 load_training_data -> handle ------------------------------
void* ref_td_load(const char* artifact_dir, const char* input_override,
                  const char* features_override) {
  TDHandle* h = nullptr;
  int rc = guarded([&] {
    auto owned = std::make_unique<TDHandle>();
    owned->artifact = read_partitions(artifact_dir);
    std::string input = (input_override && *input_override)
                            ? input_override
                            : owned->artifact.manifest.params.value("input", std::string{});
    std::string feats = (features_override && *features_override)
                            ? features_override
                            : owned->artifact.manifest.params.value("features", std::string{});
    if (input.empty() || feats.empty())
      throw ConfigError("source edges/features not recorded in manifest");
    fs::path in(input);
    EdgeStream stream(in, in.extension() == ".bin" ? EdgeFormat::binary_u64 : EdgeFormat::text_tsv,
                      owned->artifact.manifest.params.value("add_reverse", false));
    owned->data = load_training_data(owned->artifact, artifact_dir, stream, feats);
    h = owned.release();
  });
  return rc == 0 ? h : nullptr;
}

void ref_td_free(void* h) { delete static_cast<TDHandle*>(h); }

int ref_td_num_shards(void* h) { return static_cast<int>(static_cast<TDHandle*>(h)->data.shards.size()); }

int ref_td_shard_dims(void* hv, int s, std::uint64_t* rows, std::uint64_t* nnz, std::uint32_t* dim,
                      std::uint64_t* n_train, std::uint64_t* n_val, std::uint64_t* n_test) {
  return guarded([&] {
    const Shard& sh = shard_of(static_cast<TDHandle*>(hv), s);
    *rows = sh.adjacency.rows();
    *nnz = sh.adjacency.neighbors.size();
    *dim = static_cast<std::uint32_t>(sh.features.cols());
    *n_train = sh.train_rows.size();
    *n_val = sh.val_rows.size();
    *n_test = sh.test_rows.size();
  });
}

int ref_td_shard_export(void* hv, int s, std::uint32_t* offsets, std::uint32_t* neighbors,
                        double* features, std::int32_t* labels, std::uint32_t* train,
                        std::uint32_t* val, std::uint32_t* test) {
  return guarded([&] {
    const Shard& sh = shard_of(static_cast<TDHandle*>(hv), s);
    if (offsets) std::memcpy(offsets, sh.adjacency.offsets.data(), sh.adjacency.offsets.size() * 4);
    if (neighbors)
      std::memcpy(neighbors, sh.adjacency.neighbors.data(), sh.adjacency.neighbors.size() * 4);
    if (features) to_rowmajor(sh.features, features);
    if (labels) std::memcpy(labels, sh.labels.data(), sh.labels.size() * 4);
    if (train) std::memcpy(train, sh.train_rows.data(), sh.train_rows.size() * 4);
    if (val) std::memcpy(val, sh.val_rows.data(), sh.val_rows.size() * 4);
    if (test) std::memcpy(test, sh.test_rows.data(), sh.test_rows.size() * 4);
  });
}

// ---- train.cpp:289-340 distributed_train ----------------------------------------
int ref_td_distributed_train(void* hv, std::uint32_t workers, std::uint32_t sync_interval,
                             std::uint32_t epochs, double lr, std::uint32_t batch,
                             std::uint32_t prop_hops, std::uint64_t seed, double* W_out,
                             double* b_out, std::uint32_t* dim_out, std::uint32_t* classes_out,
                             std::uint64_t* hist_epoch, std::uint64_t* hist_syncs,
                             double* hist_val, double* hist_test, std::uint64_t hist_capacity,
                             std::uint64_t* n_hist, std::uint64_t* averaging_ops) {
  return guarded([&] {
    TrainConfig cfg;
    cfg.epochs = epochs;
    cfg.lr = lr;
    cfg.batch = batch;
    cfg.prop_hops = prop_hops;
    cfg.seed = seed;
    DistTrainResult r =
        distributed_train(static_cast<TDHandle*>(hv)->data, workers, sync_interval, cfg);
    *dim_out = static_cast<std::uint32_t>(r.params.weight.rows());
    *classes_out = static_cast<std::uint32_t>(r.params.weight.cols());
    if (W_out) params_to(r.params, W_out, b_out);
    *n_hist = r.history.size();
    *averaging_ops = r.averaging_ops;
    for (std::size_t k = 0; k < r.history.size() && k < hist_capacity; ++k) {
      hist_epoch[k] = r.history[k].epoch;
      hist_syncs[k] = r.history[k].syncs;
      hist_val[k] = r.history[k].val_f1;
      hist_test[k] = r.history[k].test_f1;
    }
  });
}

// ---- synth.cpp (DC-SBM alternate generator) -> dataset directory -----------------
int ref_write_synth(std::uint64_t nodes, std::uint64_t edges, std::uint32_t classes,
                    std::uint32_t dim, double mixing, std::uint64_t seed, const char* out_dir,
                    int binary) {
  return guarded([&] {
    SynthConfig cfg;
    cfg.nodes = nodes;
    cfg.edges = edges;
    cfg.classes = classes;
    cfg.feature_dim = dim;
    cfg.mixing = mixing;
    cfg.seed = seed;
    SynthDataset d = synth_graph(cfg);
    write_synth_dataset(d, cfg, out_dir, binary ? EdgeFormat::binary_u64 : EdgeFormat::text_tsv,
                        true);
  });
}

std::uint64_t ref_seed_for(std::uint64_t seed, std::uint64_t stream) { return seed_for(seed, stream); }

}  // extern "C"
