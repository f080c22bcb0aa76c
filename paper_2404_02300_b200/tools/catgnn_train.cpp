// catgnn_train — the C++ host of the B200 training path: `gnnpart train-sim`
// (/root/reference/proj/tools/gnnpart.cpp:203-217 options, :310-352 handler)
// over the C ABI, one process per GPU.
//
//   catgnn_train --artifact D [--input F] [--features F] [--workers q]
//                [--sync-interval s] [--epochs E] [--lr x] [--batch b]
//                [--prop-hops k] [--seed n] [--history csv] [--metrics json]
//                [--compare-centralized]
//                [--model sgc-ref|sgc|gcn|sage|gin] [--layers L] [--hidden H]
//                [--optimizer adam|sgd] [--device d] [--rendezvous FILE]
//
// --model sgc-ref (default) is the reference's own algorithm (sgc_propagate +
// mini-batch softmax regression, catgnn_distributed_train) and prints the
// reference's metrics JSON; the GNN models run catgnn_gnn_distributed_train
// (full-batch local iterations) and add the per-iteration
// losses.  Multi-GPU (GNN models): launch one process per GPU with RANK /
// WORLD_SIZE / LOCAL_RANK in the environment (torchrun, mpirun -x, a shell
// loop); rank 0 writes the NCCL unique id to the rendezvous file (default
// $CATGNN_RENDEZVOUS, else /tmp/catgnn_nccl_<MASTER_PORT or 29500>.id) and the
// other ranks read it, then partitions are trained cyclically per rank and the
// averages are NCCL all-reduces over NVLink.  Exit codes are the reference's:
// 2 bad config, 3 bad input, 4 internal (gnnpart.cpp:387-399).
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <nlohmann/json.hpp>

#include "catgnn.h"

using json = nlohmann::json;

namespace {

struct Fail : std::runtime_error {
  int code;
  Fail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void check(int rc) {
  if (rc != CATGNN_OK) throw Fail(rc == CATGNN_ECONFIG || rc == CATGNN_EDATA ? rc : 4, catgnn_last_error());
}

struct Args {
  std::string artifact, input, format, features, history, metrics, model = "sgc-ref", optimizer = "adam";
  std::string rendezvous;
  uint32_t workers = 1, sync = 1, epochs = 100, batch = 512, prop_hops = 2, layers = 2, hidden = 256;
  double lr = 0.01;
  uint64_t seed = 0;
  bool compare = false;
  int device = -1;
};

Args parse(int argc, char** argv) {
  Args a;
  auto need = [&](int& i) -> std::string {
    if (i + 1 >= argc) throw Fail(2, std::string(argv[i]) + " needs a value");
    return argv[++i];
  };
  auto u32 = [](const std::string& s) { return (uint32_t)std::stoul(s); };
  bool have_artifact = false;
  for (int i = 1; i < argc; ++i) {
    const std::string k = argv[i];
    try {
      if (k == "--artifact") { a.artifact = need(i); have_artifact = true; }
      else if (k == "--input") a.input = need(i);
      else if (k == "--format") a.format = need(i);
      else if (k == "--features") a.features = need(i);
      else if (k == "--workers") a.workers = u32(need(i));
      else if (k == "--sync-interval") a.sync = u32(need(i));
      else if (k == "--epochs") a.epochs = u32(need(i));
      else if (k == "--lr") a.lr = std::stod(need(i));
      else if (k == "--batch") a.batch = u32(need(i));
      else if (k == "--prop-hops") a.prop_hops = u32(need(i));
      else if (k == "--seed") a.seed = std::stoull(need(i));
      else if (k == "--history") a.history = need(i);
      else if (k == "--metrics") a.metrics = need(i);
      else if (k == "--compare-centralized") a.compare = true;
      else if (k == "--model") a.model = need(i);
      else if (k == "--layers") a.layers = u32(need(i));
      else if (k == "--hidden") a.hidden = u32(need(i));
      else if (k == "--optimizer") a.optimizer = need(i);
      else if (k == "--device") a.device = std::stoi(need(i));
      else if (k == "--rendezvous") a.rendezvous = need(i);
      else if (k == "-h" || k == "--help") {
        std::cout << "usage: catgnn_train --artifact DIR [train-sim options] [--model sgc-ref|sgc|gcn|sage|gin]\n";
        std::exit(0);
      } else {
        throw Fail(2, "unknown option " + k);
      }
    } catch (const std::invalid_argument&) {
      throw Fail(2, "bad value for " + k);
    } catch (const std::out_of_range&) {
      throw Fail(2, "value out of range for " + k);
    }
  }
  if (!have_artifact) throw Fail(2, "--artifact is required");
  return a;
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

// NCCL unique id exchange through a file on the node (rank 0 writes it
// atomically with a rename; the others wait for it).
void rendezvous(const std::string& path, int rank, char id[128]) {
  if (rank == 0) {
    check(catgnn_comm_unique_id(id));
    const std::string tmp = path + ".tmp";
    std::ofstream f(tmp, std::ios::binary | std::ios::trunc);
    f.write(id, 128);
    f.close();
    if (!f || std::rename(tmp.c_str(), path.c_str()) != 0) throw Fail(4, "cannot write rendezvous file " + path);
    return;
  }
  for (int t = 0; t < 6000; ++t) {
    std::ifstream f(path, std::ios::binary);
    if (f && f.read(id, 128) && f.gcount() == 128) return;
    std::this_thread::sleep_for(std::chrono::milliseconds(20));
  }
  throw Fail(4, "rendezvous file " + path + " did not appear");
}

void write_history(const std::string& path, const std::vector<uint64_t>& he, const std::vector<uint64_t>& hs,
                   const std::vector<double>& hv, const std::vector<double>& ht, uint64_t n) {
  if (path.empty()) return;
  std::ofstream csv(path, std::ios::trunc);  // gnnpart.cpp:340-345
  csv << "epoch,sync_count,val_f1,test_f1\n";
  for (uint64_t k = 0; k < n; ++k) csv << he[k] << ',' << hs[k] << ',' << hv[k] << ',' << ht[k] << '\n';
}

int run(int argc, char** argv) {
  Args a = parse(argc, argv);
  const int world = env_int("WORLD_SIZE", 1), rank = env_int("RANK", 0);
  const int device = a.device >= 0 ? a.device : env_int("LOCAL_RANK", 0);
  catgnn_ctx ctx = nullptr;
  check(catgnn_ctx_create(device, nullptr, &ctx));
  json metrics;
  const uint64_t cap = a.epochs / std::max(a.sync, 1u) + 2;
  std::vector<uint64_t> he(cap), hs(cap);
  std::vector<double> hv(cap), ht(cap);

  if (a.model == "sgc-ref") {
    // the reference algorithm (train-sim, gnnpart.cpp:310-339)
    if (world > 1) throw Fail(2, "--model sgc-ref runs in one process; use a GNN model for multi-GPU");
    catgnn_artifact art;
    check(catgnn_artifact_open(a.artifact.c_str(), &art));
    catgnn_artifact_info info;
    check(catgnn_artifact_get_info(art, &info));
    catgnn_shard global = nullptr;
    check(catgnn_shard_load(ctx, art, -1, a.input.c_str(), a.features.c_str(), &global));
    std::vector<catgnn_shard> shards(info.num_partitions);
    for (uint32_t s = 0; s < info.num_partitions; ++s)
      check(catgnn_shard_load(ctx, art, (int32_t)s, a.input.c_str(), a.features.c_str(), &shards[s]));
    catgnn_shard_info gi;
    check(catgnn_shard_get_info(global, &gi));
    std::vector<float> W((size_t)gi.dim * gi.classes), b(gi.classes);
    catgnn_train_config tc{a.epochs, a.lr, a.batch, a.prop_hops, a.seed};
    catgnn_dist_result r{W.data(), b.data(), 0, 0, he.data(), hs.data(), hv.data(), ht.data(), cap, 0, 0};
    check(catgnn_distributed_train(info.num_partitions, shards.data(), global, a.workers, a.sync, &tc, &r));
    const uint64_t n = std::min<uint64_t>(r.n_hist, cap);
    metrics = json{{"epochs", a.epochs},
                   {"sync_interval", a.sync},
                   {"workers", a.workers},
                   {"averaging_ops", r.averaging_ops},
                   {"final_val_f1", n ? hv[n - 1] : 0.0},
                   {"final_test_f1", n ? ht[n - 1] : 0.0}};
    if (a.compare) {  // gnnpart.cpp:330-339
      uint32_t classes = 0;
      check(catgnn_train_local(global, &tc, nullptr, nullptr, &classes));
      std::vector<float> cW((size_t)gi.dim * classes), cb(classes);
      check(catgnn_train_local(global, &tc, cW.data(), cb.data(), &classes));
      std::vector<uint32_t> test(gi.n_test);
      check(catgnn_shard_role_rows(global, 3, test.data()));
      double central = 0.0;
      check(catgnn_evaluate_micro_f1(global, cW.data(), cb.data(), classes, test.data(), test.size(), &central));
      metrics["centralized_test_f1"] = central;
      metrics["gap"] = std::abs(central - metrics["final_test_f1"].get<double>());
    }
    write_history(a.history, he, hs, hv, ht, n);
    for (auto s : shards) catgnn_shard_destroy(s);
    catgnn_shard_destroy(global);
    catgnn_artifact_close(art);
  } else {
    int kind = a.model == "gcn" ? CATGNN_MODEL_GCN : a.model == "sage" ? CATGNN_MODEL_SAGE
             : a.model == "gin" ? CATGNN_MODEL_GIN : a.model == "sgc" ? CATGNN_MODEL_SGC : 0;
    if (!kind) throw Fail(2, "unknown model " + a.model);
    if (a.optimizer != "adam" && a.optimizer != "sgd") throw Fail(2, "unknown optimizer " + a.optimizer);
    catgnn_comm comm = nullptr;
    if (world > 1) {
      std::string path = a.rendezvous;
      if (path.empty()) {
        const char* e = std::getenv("CATGNN_RENDEZVOUS");
        const char* port = std::getenv("MASTER_PORT");
        path = e && *e ? e : std::string("/tmp/catgnn_nccl_") + (port ? port : "29500") + ".id";
      }
      char id[128];
      rendezvous(path, rank, id);
      check(catgnn_comm_create(ctx, world, rank, id, &comm));
    }
    catgnn_gnn_train_config gc{};
    gc.model.kind = kind;
    gc.model.layers = kind == CATGNN_MODEL_SGC && a.layers == 2 ? 1 : a.layers;
    gc.model.hidden = a.hidden;
    gc.model.optimizer = a.optimizer == "adam" ? CATGNN_OPT_ADAM : CATGNN_OPT_SGD;
    gc.model.lr = a.lr;
    gc.model.beta1 = 0.9;
    gc.model.beta2 = 0.999;
    gc.model.eps = 1e-8;
    gc.model.seed = a.seed;
    gc.epochs = a.epochs;
    gc.sync_interval = a.sync;
    gc.workers = a.workers;
    gc.eval_global = 1;
    std::vector<double> losses(std::max(a.epochs, 1u));
    catgnn_gnn_result r{};
    r.losses = losses.data();
    r.loss_capacity = losses.size();
    r.hist_epoch = he.data(); r.hist_syncs = hs.data(); r.hist_val = hv.data(); r.hist_test = ht.data();
    r.hist_capacity = cap;
    check(catgnn_gnn_distributed_train(ctx, a.artifact.c_str(), a.input.c_str(), a.features.c_str(), &gc, comm, &r));
    const uint64_t n = std::min<uint64_t>(r.n_hist, cap);
    metrics = json{{"epochs", a.epochs},
                   {"sync_interval", a.sync},
                   {"workers", a.workers},
                   {"averaging_ops", r.averaging_ops},
                   {"final_val_f1", n ? hv[n - 1] : 0.0},
                   {"final_test_f1", n ? ht[n - 1] : 0.0},
                   {"model", a.model},
                   {"ranks", world},
                   {"losses", std::vector<double>(losses.begin(), losses.begin() + r.n_losses)}};
    if (rank == 0) write_history(a.history, he, hs, hv, ht, n);
    if (comm) catgnn_comm_destroy(comm);
  }
  if (rank == 0) {
    if (!a.metrics.empty()) {
      std::ofstream mj(a.metrics, std::ios::trunc);
      mj << metrics.dump(2) << '\n';
    }
    std::cout << metrics.dump(2) << '\n';
  }
  catgnn_ctx_destroy(ctx);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    return run(argc, argv);
  } catch (const Fail& e) {  // gnnpart.cpp:387-399
    const char* what = e.code == 2 ? "bad-config" : e.code == 3 ? "bad-input" : "internal";
    std::cerr << "error: " << what << ": " << e.what() << '\n';
    return e.code;
  } catch (const std::exception& e) {
    std::cerr << "error: internal: " << e.what() << '\n';
    return 4;
  }
}
