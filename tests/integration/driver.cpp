// TEST INFRASTRUCTURE ONLY — exercises INTEGRATION.md's binding
// (distributed_train_b200 / distributed_train_gnn_b200, compiled from the
// document) next to the reference's own distributed_train in one process, on
// one artifact: the train-sim path of proj/tools/gnnpart.cpp:310-321.
//
//   integration_driver ARTIFACT SYNC EPOCHS LR BATCH HOPS WORKERS
// prints one JSON line with the largest relative parameter differences and
// whether the sync histories agree (epoch / sync counts exactly, F1 per row).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <string>
#include <vector>

#include "catgnn.h"
#include "gnnpart/edge_stream.hpp"
#include "gnnpart/store.hpp"
#include "gnnpart/train.hpp"

namespace gnnpart {
DistTrainResult distributed_train_b200(const std::filesystem::path&, std::uint32_t, std::uint32_t,
                                       const TrainConfig&, int);
struct GnnTrainResult {
  std::vector<float> params;
  std::vector<double> losses;
  std::vector<SyncPoint> history;
  std::uint64_t averaging_ops = 0;
};
GnnTrainResult distributed_train_gnn_b200(const std::filesystem::path&, std::uint32_t, std::uint32_t,
                                          const TrainConfig&, int, std::uint32_t, std::uint32_t, int, int,
                                          catgnn_comm);
}  // namespace gnnpart

using namespace gnnpart;

static double rel(double num, double den) { return den > 0 ? std::sqrt(num / den) : std::sqrt(num); }

static double hist_f1_diff(const std::vector<SyncPoint>& a, const std::vector<SyncPoint>& b, bool* counts_ok) {
  *counts_ok = a.size() == b.size();
  double d = 0;
  for (size_t k = 0; k < a.size() && k < b.size(); ++k) {
    *counts_ok = *counts_ok && a[k].epoch == b[k].epoch && a[k].syncs == b[k].syncs;
    d = std::max({d, std::abs(a[k].val_f1 - b[k].val_f1), std::abs(a[k].test_f1 - b[k].test_f1)});
  }
  return d;
}

int main(int argc, char** argv) {
  if (argc != 8) {
    std::fprintf(stderr, "usage: integration_driver ARTIFACT SYNC EPOCHS LR BATCH HOPS WORKERS\n");
    return 2;
  }
  const std::filesystem::path dir = argv[1];
  const std::uint32_t sync = std::atoi(argv[2]), workers = std::atoi(argv[7]);
  TrainConfig cfg;
  cfg.epochs = std::atoi(argv[3]);
  cfg.lr = std::atof(argv[4]);
  cfg.batch = std::atoi(argv[5]);
  cfg.prop_hops = std::atoi(argv[6]);
  cfg.seed = 5;
  try {
    // the reference path (gnnpart.cpp:311-321)
    StoredArtifact art = read_partitions(dir);
    const std::string input = art.manifest.params.value("input", std::string{});
    const std::string feats = art.manifest.params.value("features", std::string{});
    EdgeStream stream(input,
                      std::filesystem::path(input).extension() == ".bin" ? EdgeFormat::binary_u64
                                                                        : EdgeFormat::text_tsv,
                      art.manifest.params.value("add_reverse", false));
    TrainingData data = load_training_data(art, dir, stream, feats);
    DistTrainResult ref = distributed_train(data, workers, sync, cfg);
    // the binding, SGC reference algorithm
    DistTrainResult b2 = distributed_train_b200(dir, workers, sync, cfg, 0);
    double dn = 0, dd = 0;
    for (Eigen::Index i = 0; i < ref.params.weight.rows(); ++i)
      for (Eigen::Index j = 0; j < ref.params.weight.cols(); ++j) {
        const double x = b2.params.weight(i, j) - ref.params.weight(i, j);
        dn += x * x;
        dd += ref.params.weight(i, j) * ref.params.weight(i, j);
      }
    const double w_rel = rel(dn, dd);
    bool counts_ok = false;
    const double f1d = hist_f1_diff(b2.history, ref.history, &counts_ok);
    // the binding, GNN loop with the SGC kind vs the reference at one hop, full batch
    TrainConfig fb = cfg;
    fb.batch = 0x7fffffffu;
    fb.prop_hops = 1;
    DistTrainResult ref1 = distributed_train(data, workers, sync, fb);
    GnnTrainResult g = distributed_train_gnn_b200(dir, workers, sync, fb, CATGNN_MODEL_SGC, 1, 0,
                                                  CATGNN_OPT_SGD, 0, nullptr);
    const Eigen::Index D = ref1.params.weight.rows(), C = ref1.params.weight.cols();
    dn = dd = 0;
    for (Eigen::Index i = 0; i < D; ++i)
      for (Eigen::Index j = 0; j < C; ++j) {  // library layout: W is classes x dim, then b
        const double x = g.params[(size_t)j * D + i] - ref1.params.weight(i, j);
        dn += x * x;
        dd += ref1.params.weight(i, j) * ref1.params.weight(i, j);
      }
    const double g_rel = rel(dn, dd);
    bool g_counts_ok = false;
    const double g_f1d = hist_f1_diff(g.history, ref1.history, &g_counts_ok);
    std::printf("{\"sgc_ref_w_rel\": %.3e, \"sgc_ref_hist_counts\": %s, \"sgc_ref_f1_diff\": %.6g, "
                "\"ops\": [%llu, %llu], \"gnn_sgc_w_rel\": %.3e, \"gnn_sgc_hist_counts\": %s, "
                "\"gnn_sgc_f1_diff\": %.6g, \"val_rows\": %zu, \"test_rows\": %zu}\n",
                w_rel, counts_ok ? "true" : "false", f1d, (unsigned long long)b2.averaging_ops,
                (unsigned long long)ref.averaging_ops, g_rel, g_counts_ok ? "true" : "false", g_f1d,
                data.global.val_rows.size(), data.global.test_rows.size());
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 4;
  }
  return 0;
}
