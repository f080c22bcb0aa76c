// Device neighbour completion: the B200 restatement of gnnpart::complete_edges
// (/root/reference/proj/src/completion.cpp:130-171) with PartitionBuilder
// (:13-58) — the step between SPRING's node->home assignment and the
// per-partition shards, SURVEY.md §8(f) row 1 (papers100M-scale streams do not
// fit the reference's per-partition unordered_set in host RAM).
//
// For dense external ids (ext < num_nodes, the form load_training_data
// requires, train.cpp:234-240) and hops in {1,2,3}:
//   reach[v]  = 1 << home[v], grown hops-1 times over the stream (:150-160)
//   edge k goes to every partition s in reach[u] | reach[v] (:161-166; for
//   hops = 1 that is {home[u], home[v]}, :140-144)
//   per partition, one record per unordered pair: the FIRST occurrence in
//   stream order, original orientation (add_edge, :18-23)
//   node table: endpoints of kept edges + every node homed at s, ascending
//   ext id, owner = home == s, role only on owners (finish, :25-57).
// Per partition: select the stream positions routed to s (stream order), sort
// (pair key, position) with a stable radix sort, keep the first of each key,
// scatter the keep flags back and compact — the kept edges stay in stream
// order.  Node presence is a byte map over the node ids.  All integer work:
// HBM-bound sorts and compactions, no tensor cores.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <string>
#include <vector>

#include "artifact.hpp"
#include "index.hpp"
#include "shard.hpp"

struct catgnn_completion_s {
  uint32_t p = 0;
  uint64_t num_nodes = 0;
  struct Part {
    std::vector<uint64_t> edges;  // 2 x E, ext ids, stream order
    std::vector<uint64_t> ext;    // ascending
    std::vector<uint8_t> owner, role;
  };
  std::vector<Part> parts;
};

namespace catgnn {
namespace {

inline unsigned grid_of(uint64_t n) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148ull * 32));
}

__global__ void check_edges_kernel(const uint64_t* __restrict__ e, uint64_t m, uint64_t n, int* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
    if (e[i] >= n) *bad = 1;
}

__global__ void init_reach_kernel(const uint32_t* __restrict__ home, uint64_t n, unsigned long long* reach) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x)
    reach[v] = 1ull << home[v];
}

// next[u] |= reach[v], next[v] |= reach[u]  (completion.cpp:153-158)
__global__ void grow_reach_kernel(const uint64_t* __restrict__ e, uint64_t m, const unsigned long long* __restrict__ reach,
                                  unsigned long long* next) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = e[2 * k], v = e[2 * k + 1];
    const unsigned long long ru = reach[u], rv = reach[v];
    if ((next[u] | rv) != next[u]) atomicOr(next + u, rv);
    if ((next[v] | ru) != next[v]) atomicOr(next + v, ru);
  }
}

__global__ void route_flags_kernel(const uint64_t* __restrict__ e, uint64_t m, const unsigned long long* __restrict__ reach,
                                   uint32_t s, uint8_t* __restrict__ flag) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m; k += (uint64_t)gridDim.x * blockDim.x)
    flag[k] = (uint8_t)(((reach[e[2 * k]] | reach[e[2 * k + 1]]) >> s) & 1ull);
}

// unordered pair key (completion.cpp:20-21) of the selected stream positions
__global__ void pair_keys_kernel(const uint64_t* __restrict__ e, const uint64_t* __restrict__ sel, uint64_t ns,
                                 uint64_t* __restrict__ key, uint64_t* __restrict__ idx) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ns; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = sel[i];
    const uint64_t u = e[2 * k], v = e[2 * k + 1];
    key[i] = (min(u, v) << 32) | max(u, v);
    idx[i] = i;
  }
}

// keep[idx_sorted[j]] = first of its key run (stable sort: smallest position)
__global__ void first_of_key_kernel(const uint64_t* __restrict__ skey, const uint64_t* __restrict__ sidx, uint64_t ns,
                                    uint8_t* __restrict__ keep) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < ns; j += (uint64_t)gridDim.x * blockDim.x)
    keep[sidx[j]] = (uint8_t)(j == 0 || skey[j] != skey[j - 1]);
}

__global__ void gather_edges_mark_kernel(const uint64_t* __restrict__ e, const uint64_t* __restrict__ ext,
                                         const uint64_t* __restrict__ kept, uint64_t nk, uint64_t* __restrict__ out,
                                         uint8_t* __restrict__ present) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nk; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = kept[i];
    out[2 * i] = ext[2 * k];  // original record, original orientation
    out[2 * i + 1] = ext[2 * k + 1];
    present[e[2 * k]] = 1;
    present[e[2 * k + 1]] = 1;
  }
}

__global__ void ids_to_ext_kernel(uint64_t* __restrict__ ids, uint64_t n, const uint64_t* __restrict__ id_to_ext) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    ids[i] = id_to_ext[ids[i]];
}

__global__ void runs_to_u64_kernel(const uint32_t* __restrict__ runs, uint64_t n, uint64_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = runs[i];
}

// per run: home / role of its dense id (HomeMap and NodeMetaMap are by dense id)
__global__ void by_run_kernel(const uint32_t* __restrict__ dense_of_run, uint64_t n, const uint32_t* __restrict__ home,
                              const uint8_t* __restrict__ roles, uint32_t* __restrict__ home_run,
                              uint8_t* __restrict__ roles_run) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n; r += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t d = dense_of_run[r];
    home_run[r] = home[d];
    if (roles) roles_run[r] = roles[d];
  }
}

__global__ void mark_owned_kernel(const uint32_t* __restrict__ home, uint64_t n, uint32_t s, uint8_t* __restrict__ present) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x)
    if (home[v] == s) present[v] = 1;
}

__global__ void node_records_kernel(const uint64_t* __restrict__ ids, uint64_t nn, const uint32_t* __restrict__ home,
                                    const uint8_t* __restrict__ roles, uint32_t s, uint8_t* __restrict__ owner,
                                    uint8_t* __restrict__ role) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nn; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = ids[i];
    const bool own = home[v] == s;
    owner[i] = own ? 1 : 0;
    role[i] = (own && roles) ? roles[v] : 0;
  }
}

// cub temp storage helper
struct Temp {
  catgnn_ctx ctx;
  void* get(size_t bytes) { return ctx->scratch_buf<unsigned char>("cmp_cub", std::max<size_t>(bytes, 1)); }
};

template <typename T>
T* dev(catgnn_ctx ctx, const char* name, size_t n) {
  return ctx->scratch_buf<T>(name, std::max<size_t>(n, 1));
}

// add_reverse expansion of one streamed chunk (EdgeReader::next,
// edge_stream.cpp:138-148): record k -> (u, v) and, when u != v, (v, u), at
// the output position given by the exclusive scan of the per-record counts.
__global__ void expand_count_kernel(const uint64_t* __restrict__ rec, uint64_t n, uint32_t* cnt) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x)
    cnt[k] = rec[2 * k] != rec[2 * k + 1] ? 2u : 1u;
}
__global__ void expand_scatter_kernel(const uint64_t* __restrict__ rec, uint64_t n, const uint64_t* __restrict__ off,
                                      uint64_t* __restrict__ out) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = rec[2 * k], v = rec[2 * k + 1], o = off[k];
    out[2 * o] = u;
    out[2 * o + 1] = v;
    if (u != v) {
      out[2 * o + 2] = v;
      out[2 * o + 3] = u;
    }
  }
}
struct Count32To64 {
  __host__ __device__ uint64_t operator()(uint32_t x) const { return x; }
};

// The per-partition work on node ids 0..n-1 (dense ids, or the ascending-ext
// "runs" of a graph index): d_e routes and keys, d_ext is the original record
// for the output, id_to_ext (ascending in id) maps node-table ids back.
void complete_core(catgnn_ctx ctx, const uint64_t* d_e, const uint64_t* d_ext, uint64_t m, const uint32_t* d_home,
                   const uint8_t* d_roles, uint64_t n, const uint64_t* id_to_ext, uint32_t p, uint32_t hops,
                   catgnn_completion_s* res) {
  cudaStream_t st = ctx->stream;
  // reach masks
  unsigned long long* reach = dev<unsigned long long>(ctx, "cmp_reach", n);
  if (n) init_reach_kernel<<<grid_of(n), 256, 0, st>>>(d_home, n, reach);
  for (uint32_t r = 1; r < hops; ++r) {
    unsigned long long* next = dev<unsigned long long>(ctx, "cmp_reach_next", n);
    CG_CUDA(cudaMemcpyAsync(next, reach, n * 8, cudaMemcpyDeviceToDevice, st));
    if (m) grow_reach_kernel<<<grid_of(m), 256, 0, st>>>(d_e, m, reach, next);
    CG_CUDA(cudaMemcpyAsync(reach, next, n * 8, cudaMemcpyDeviceToDevice, st));
  }
  CG_CHECK_LAUNCH();

  res->p = p;
  res->num_nodes = n;
  res->parts.resize(p);
  uint8_t* flag = dev<uint8_t>(ctx, "cmp_flag", m);
  uint64_t* sel = dev<uint64_t>(ctx, "cmp_sel", m);
  // per-partition buffers are sized by the routed count (grow-only scratch)
  uint64_t *key = nullptr, *key2 = nullptr, *idx = nullptr, *idx2 = nullptr, *kept = nullptr, *oute = nullptr;
  uint8_t* keep = nullptr;
  uint8_t* present = dev<uint8_t>(ctx, "cmp_present", n);
  uint64_t* ids = dev<uint64_t>(ctx, "cmp_ids", n);
  uint8_t* own = dev<uint8_t>(ctx, "cmp_own", n);
  uint8_t* rol = dev<uint8_t>(ctx, "cmp_rol", n);
  uint64_t* count = dev<uint64_t>(ctx, "cmp_count", 1);
  Temp tmp{ctx};
  auto counted = [&]() {
    uint64_t c = 0;
    CG_CUDA(cudaMemcpyAsync(&c, count, 8, cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaStreamSynchronize(st));
    return c;
  };
  thrust::counting_iterator<uint64_t> pos(0);
  const int key_bits = 64;
  for (uint32_t s = 0; s < p; ++s) {
    auto& P = res->parts[s];
    uint64_t nk = 0;
    if (m) {
      route_flags_kernel<<<grid_of(m), 256, 0, st>>>(d_e, m, reach, s, flag);
      size_t tb = 0;
      CG_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, pos, flag, sel, count, m, st));
      CG_CUDA(cub::DeviceSelect::Flagged(tmp.get(tb), tb, pos, flag, sel, count, m, st));
      const uint64_t ns = counted();
      key = dev<uint64_t>(ctx, "cmp_key", ns);
      key2 = dev<uint64_t>(ctx, "cmp_key2", ns);
      idx = dev<uint64_t>(ctx, "cmp_idx", ns);
      idx2 = dev<uint64_t>(ctx, "cmp_idx2", ns);
      keep = dev<uint8_t>(ctx, "cmp_keep", ns);
      kept = dev<uint64_t>(ctx, "cmp_kept", ns);
      oute = dev<uint64_t>(ctx, "cmp_oute", 2 * ns);
      if (ns) {
        pair_keys_kernel<<<grid_of(ns), 256, 0, st>>>(d_e, sel, ns, key, idx);
        CG_CHECK_LAUNCH();
        tb = 0;
        CG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key2, idx, idx2, ns, 0, key_bits, st));
        CG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(tb), tb, key, key2, idx, idx2, ns, 0, key_bits, st));
        first_of_key_kernel<<<grid_of(ns), 256, 0, st>>>(key2, idx2, ns, keep);
        CG_CHECK_LAUNCH();
        tb = 0;
        CG_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, sel, keep, kept, count, ns, st));
        CG_CUDA(cub::DeviceSelect::Flagged(tmp.get(tb), tb, sel, keep, kept, count, ns, st));
        nk = counted();
      }
    }
    if (n) CG_CUDA(cudaMemsetAsync(present, 0, n, st));
    if (nk) gather_edges_mark_kernel<<<grid_of(nk), 256, 0, st>>>(d_e, d_ext, kept, nk, oute, present);
    if (n) mark_owned_kernel<<<grid_of(n), 256, 0, st>>>(d_home, n, s, present);
    CG_CHECK_LAUNCH();
    uint64_t nn = 0;
    if (n) {
      size_t tb = 0;
      CG_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, pos, present, ids, count, n, st));
      CG_CUDA(cub::DeviceSelect::Flagged(tmp.get(tb), tb, pos, present, ids, count, n, st));
      nn = counted();
    }
    if (nn) node_records_kernel<<<grid_of(nn), 256, 0, st>>>(ids, nn, d_home, d_roles, s, own, rol);
    if (nn && id_to_ext) ids_to_ext_kernel<<<grid_of(nn), 256, 0, st>>>(ids, nn, id_to_ext);
    CG_CHECK_LAUNCH();
    P.edges.resize(2 * nk);
    P.ext.resize(nn);
    P.owner.resize(nn);
    P.role.resize(nn);
    if (nk) CG_CUDA(cudaMemcpyAsync(P.edges.data(), oute, 2 * nk * 8, cudaMemcpyDeviceToHost, st));
    if (nn) {
      CG_CUDA(cudaMemcpyAsync(P.ext.data(), ids, nn * 8, cudaMemcpyDeviceToHost, st));
      CG_CUDA(cudaMemcpyAsync(P.owner.data(), own, nn, cudaMemcpyDeviceToHost, st));
      CG_CUDA(cudaMemcpyAsync(P.role.data(), rol, nn, cudaMemcpyDeviceToHost, st));
    }
    CG_CUDA(cudaStreamSynchronize(st));
    ctx->launches += 6;
  }
}

}  // namespace
}  // namespace catgnn

using namespace catgnn;

namespace {

void check_completion_args(const uint32_t* home, uint64_t num_nodes, uint32_t p, uint32_t hops) {
  if (hops < 1 || hops > 3) throw ConfigError("hop count must be in {1,2,3}");                 // :133
  if (p == 0) throw DataError("home map does not cover the node set");                         // :65-66
  if (p > 64) throw ConfigError("device completion supports at most 64 partitions");           // :147-148
  if (num_nodes >= (1ull << 32)) throw ConfigError("node ids must fit 32 bits");
  for (uint64_t v = 0; v < num_nodes; ++v)
    if (home[v] >= p) throw DataError("home partition out of range");                         // :67-68
}

// d_e (m records, dense ids) is on the device: upload the home map and roles,
// check the endpoints, run the per-partition completion, release the scratch.
catgnn_completion_s* complete_dense(catgnn_ctx ctx, uint64_t* d_e, uint64_t m, const uint32_t* home,
                                    const uint8_t* roles, uint64_t n, uint32_t p, uint32_t hops) {
  cudaStream_t st = ctx->stream;
  uint32_t* d_home = dev<uint32_t>(ctx, "cmp_home", n);
  uint8_t* d_roles = roles ? dev<uint8_t>(ctx, "cmp_roles", n) : nullptr;
  if (n) CG_CUDA(cudaMemcpyAsync(d_home, home, n * 4, cudaMemcpyHostToDevice, st));
  if (roles && n) CG_CUDA(cudaMemcpyAsync(d_roles, roles, n, cudaMemcpyHostToDevice, st));
  int* bad = dev<int>(ctx, "cmp_bad", 1);
  CG_CUDA(cudaMemsetAsync(bad, 0, 4, st));
  if (m) check_edges_kernel<<<grid_of(2 * m), 256, 0, st>>>(d_e, 2 * m, n, bad);
  int h_bad = 0;
  CG_CUDA(cudaMemcpyAsync(&h_bad, bad, 4, cudaMemcpyDeviceToHost, st));
  CG_CUDA(cudaStreamSynchronize(st));
  if (h_bad) throw DataError("edge endpoint outside the node set (external ids must be dense)");
  auto res = std::make_unique<catgnn_completion_s>();
  complete_core(ctx, d_e, d_e, m, d_home, d_roles, n, nullptr, p, hops, res.get());
  // the completion scratch is sized by the stream: give it back
  for (auto it = ctx->scratch.begin(); it != ctx->scratch.end();)
    it = it->first.rfind("cmp_", 0) == 0 ? ctx->scratch.erase(it) : std::next(it);
  return res.release();
}

}  // namespace

int catgnn_complete_edges(catgnn_ctx ctx, const uint64_t* edges, uint64_t num_edges, const uint32_t* home,
                          const uint8_t* roles, uint64_t num_nodes, uint32_t p, uint32_t hops,
                          catgnn_completion* out) {
  return guarded([&] {
    if (!ctx || !out || (num_edges && !edges) || (num_nodes && !home)) throw ConfigError("null argument");
    check_completion_args(home, num_nodes, p, hops);
    CG_CUDA(cudaSetDevice(ctx->device));
    const uint64_t m = num_edges;
    uint64_t* d_e = dev<uint64_t>(ctx, "cmp_edges", 2 * m);
    if (m) CG_CUDA(cudaMemcpyAsync(d_e, edges, 2 * m * 8, cudaMemcpyHostToDevice, ctx->stream));
    *out = complete_dense(ctx, d_e, m, home, roles, num_nodes, p, hops);
  });
}

// complete_edges over an EDG1 edge file streamed in chunks (SURVEY §8(f) row 1:
// the papers100M-scale stream, 1.6 B records / 26 GB, never sits in host RAM —
// only a pinned chunk does — and the reference's per-partition unordered_set is
// replaced by the device sort).  add_reverse expands each record on the device.
// Chunk size: CATGNN_STREAM_CHUNK records (default 4 M = 64 MB).
int catgnn_complete_edges_file(catgnn_ctx ctx, const char* path, int add_reverse, const uint32_t* home,
                               const uint8_t* roles, uint64_t num_nodes, uint32_t p, uint32_t hops,
                               catgnn_completion* out) {
  return guarded([&] {
    if (!ctx || !out || !path || (num_nodes && !home)) throw ConfigError("null argument");
    check_completion_args(home, num_nodes, p, hops);
    CG_CUDA(cudaSetDevice(ctx->device));
    namespace fs = std::filesystem;
    if (fs::path(path).extension() != ".bin") {  // text streams: host read, then the same path
      std::vector<uint64_t> e;
      read_edge_stream(path, add_reverse != 0, e);
      const uint64_t m = e.size() / 2;
      uint64_t* d_e = dev<uint64_t>(ctx, "cmp_edges", 2 * m);
      if (m) CG_CUDA(cudaMemcpyAsync(d_e, e.data(), 2 * m * 8, cudaMemcpyHostToDevice, ctx->stream));
      *out = complete_dense(ctx, d_e, m, home, roles, num_nodes, p, hops);
      return;
    }
    std::error_code ec;
    if (!fs::is_regular_file(path, ec)) throw DataError(std::string("edge file not readable: ") + path);
    FILE* f = std::fopen(path, "rb");
    if (!f) throw DataError(std::string("cannot open edge file: ") + path);
    struct Closer {
      FILE* f;
      ~Closer() { std::fclose(f); }
    } closer{f};
    const uint64_t size = fs::file_size(path);
    char magic[4] = {0, 0, 0, 0};
    uint64_t off = 0;
    if (size >= 4 && std::fread(magic, 1, 4, f) == 4 && std::memcmp(magic, "EDG1", 4) == 0) off = 4;
    std::fseek(f, (long)off, SEEK_SET);
    if ((size - off) % 16 != 0) throw DataError(std::string("binary edge file has truncated record: ") + path);
    const uint64_t records = (size - off) / 16;
    const uint64_t cap = add_reverse ? 2 * records : records;  // expanded records, upper bound
    uint64_t* d_e = dev<uint64_t>(ctx, "cmp_edges", 2 * cap);
    static const uint64_t chunk = [] {
      const char* v = std::getenv("CATGNN_STREAM_CHUNK");
      return (uint64_t)(v && *v ? std::max(1LL, std::atoll(v)) : (4LL << 20));
    }();
    cudaStream_t st = ctx->stream;
    uint64_t* pinned = nullptr;
    CG_CUDA(cudaMallocHost(&pinned, std::max<uint64_t>(1, std::min(chunk, records)) * 16));
    struct Pinned {
      uint64_t* p;
      ~Pinned() { cudaFreeHost(p); }
    } pin{pinned};
    uint64_t* d_raw = add_reverse ? dev<uint64_t>(ctx, "cmp_raw", 2 * std::min(chunk, records)) : nullptr;
    uint32_t* d_cnt = add_reverse ? dev<uint32_t>(ctx, "cmp_cnt", std::min(chunk, records)) : nullptr;
    uint64_t* d_off = add_reverse ? dev<uint64_t>(ctx, "cmp_off", std::min(chunk, records) + 1) : nullptr;
    Temp tmp{ctx};
    uint64_t m = 0;  // expanded records so far
    for (uint64_t done = 0; done < records;) {
      const uint64_t n = std::min(chunk, records - done);
      if (std::fread(pinned, 16, n, f) != n) throw DataError(std::string("short edge read: ") + path);
      if (!add_reverse) {
        CG_CUDA(cudaMemcpyAsync(d_e + 2 * m, pinned, n * 16, cudaMemcpyHostToDevice, st));
        m += n;
      } else {
        CG_CUDA(cudaMemcpyAsync(d_raw, pinned, n * 16, cudaMemcpyHostToDevice, st));
        expand_count_kernel<<<grid_of(n), 256, 0, st>>>(d_raw, n, d_cnt);
        auto cnt64 = thrust::make_transform_iterator(d_cnt, Count32To64{});
        size_t tb = 0;
        CG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt64, d_off, n + 0, st));
        CG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(tb), tb, cnt64, d_off, n, st));
        expand_scatter_kernel<<<grid_of(n), 256, 0, st>>>(d_raw, n, d_off, d_e + 2 * m);
        CG_CHECK_LAUNCH();
        ctx->launches += 2;
        uint64_t last_off = 0;
        uint32_t last_cnt = 0;
        CG_CUDA(cudaMemcpyAsync(&last_off, d_off + n - 1, 8, cudaMemcpyDeviceToHost, st));
        CG_CUDA(cudaMemcpyAsync(&last_cnt, d_cnt + n - 1, 4, cudaMemcpyDeviceToHost, st));
        CG_CUDA(cudaStreamSynchronize(st));
        m += last_off + last_cnt;
      }
      CG_CUDA(cudaStreamSynchronize(st));  // the pinned chunk is refilled next
      done += n;
    }
    *out = complete_dense(ctx, d_e, m, home, roles, num_nodes, p, hops);
  });
}

int catgnn_complete_edges_indexed(catgnn_ctx ctx, catgnn_index index, const uint64_t* edges, uint64_t num_edges,
                                  const uint32_t* home, const uint8_t* roles, uint32_t p, uint32_t hops,
                                  catgnn_completion* out) {
  return guarded([&] {
    if (!ctx || !index || !out || (num_edges && !edges) || (index->n && !home)) throw ConfigError("null argument");
    if (index->ctx->device != ctx->device) throw ConfigError("index and context must share one device");
    if (hops < 1 || hops > 3) throw ConfigError("hop count must be in {1,2,3}");                 // :133
    if (p == 0) throw DataError("home map does not cover the node set");                         // :65-66
    if (p > 64) throw ConfigError("device completion supports at most 64 partitions");           // :147-148
    const uint64_t m = num_edges, n = index->n;
    for (uint64_t v = 0; v < n; ++v)
      if (home[v] >= p) throw DataError("home partition out of range");                         // :67-68
    CG_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    uint64_t* d_ext = dev<uint64_t>(ctx, "cmp_ext", 2 * m);
    uint64_t* d_e = dev<uint64_t>(ctx, "cmp_edges", 2 * m);
    uint32_t* runs = dev<uint32_t>(ctx, "cmp_runs", 2 * m);
    uint32_t* home_d = dev<uint32_t>(ctx, "cmp_home_dense", n);
    uint8_t* roles_d = roles ? dev<uint8_t>(ctx, "cmp_roles_dense", n) : nullptr;
    uint32_t* home_run = dev<uint32_t>(ctx, "cmp_home", n);
    uint8_t* roles_run = roles ? dev<uint8_t>(ctx, "cmp_roles", n) : nullptr;
    if (m) CG_CUDA(cudaMemcpyAsync(d_ext, edges, 2 * m * 8, cudaMemcpyHostToDevice, st));
    if (n) CG_CUDA(cudaMemcpyAsync(home_d, home, n * 4, cudaMemcpyHostToDevice, st));
    if (roles && n) CG_CUDA(cudaMemcpyAsync(roles_d, roles, n, cudaMemcpyHostToDevice, st));
    int* missing = dev<int>(ctx, "cmp_bad", 1);
    CG_CUDA(cudaMemsetAsync(missing, 0, 4, st));
    // GraphIndex::dense (edge_stream.hpp:113-118) for every endpoint, as runs
    if (m) map_to_runs_kernel<<<grid_of(2 * m), 256, 0, st>>>(index->sorted_ext.p, n, d_ext, 2 * m, runs, missing);
    if (m) runs_to_u64_kernel<<<grid_of(2 * m), 256, 0, st>>>(runs, 2 * m, d_e);
    if (n) by_run_kernel<<<grid_of(n), 256, 0, st>>>(index->dense_of_run.p, n, home_d, roles_d, home_run, roles_run);
    CG_CHECK_LAUNCH();
    int h_missing = 0;
    CG_CUDA(cudaMemcpyAsync(&h_missing, missing, 4, cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaStreamSynchronize(st));
    if (h_missing) throw DataError("node missing from degree table");                           // :115-116
    auto res = std::make_unique<catgnn_completion_s>();
    complete_core(ctx, d_e, d_ext, m, home_run, roles_run, n, index->sorted_ext.p, p, hops, res.get());
    for (auto it = ctx->scratch.begin(); it != ctx->scratch.end();)
      it = it->first.rfind("cmp_", 0) == 0 ? ctx->scratch.erase(it) : std::next(it);
    *out = res.release();
  });
}

int catgnn_completion_part_counts(catgnn_completion c, uint32_t part, uint64_t* edges, uint64_t* nodes,
                                  uint64_t* owned) {
  return guarded([&] {
    if (!c) throw ConfigError("null completion");
    if (part >= c->p) throw ConfigError("partition index out of range");
    const auto& P = c->parts[part];
    if (edges) *edges = P.edges.size() / 2;
    if (nodes) *nodes = P.ext.size();
    if (owned) {
      uint64_t o = 0;
      for (uint8_t x : P.owner) o += x;
      *owned = o;
    }
  });
}

int catgnn_completion_part(catgnn_completion c, uint32_t part, uint64_t* edges, uint64_t* ext, uint8_t* owner,
                           uint8_t* role) {
  return guarded([&] {
    if (!c) throw ConfigError("null completion");
    if (part >= c->p) throw ConfigError("partition index out of range");
    const auto& P = c->parts[part];
    if (edges) std::copy(P.edges.begin(), P.edges.end(), edges);
    if (ext) std::copy(P.ext.begin(), P.ext.end(), ext);
    if (owner) std::copy(P.owner.begin(), P.owner.end(), owner);
    if (role) std::copy(P.role.begin(), P.role.end(), role);
  });
}

int catgnn_completion_destroy(catgnn_completion c) {
  return guarded([&] { delete c; });
}
