// Device graph index: the B200 restatement of gnnpart::compute_degrees
// (/root/reference/proj/src/edge_stream.cpp:192-215, GraphIndex
// edge_stream.hpp:104-128), SURVEY.md §8(f) row 3.
//
// The reference interns external ids through an unordered_map in first-seen
// order (record k = (u, v): u before v) and counts degrees (a self-loop counts
// 2).  Here the 2E endpoint occurrences (key = ext id, value = stream position
// 2k / 2k+1) are radix-sorted; each run of equal ids is one node, its length
// is the degree (a self-loop contributes two occurrences) and its first value
// the first-seen position, so sorting the runs by that position yields
// dense_to_ext exactly.  The sorted run keys double as the ext -> dense lookup
// table (binary search) that catgnn_complete_edges_indexed uses to route
// arbitrary 64-bit ids.  Integer, HBM/sort-bound work.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <memory>
#include <vector>

#include "index.hpp"

namespace catgnn {
namespace {

inline unsigned grid_of(uint64_t n) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148ull * 32));
}

__global__ void iota_kernel(uint64_t* __restrict__ v, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    v[i] = i;
}

__global__ void run_starts_kernel(const uint64_t* __restrict__ sk, uint64_t n, uint8_t* __restrict__ flag) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x)
    flag[j] = (uint8_t)(j == 0 || sk[j] != sk[j - 1]);
}

__global__ void self_loops_kernel(const uint64_t* __restrict__ e, uint64_t m, unsigned long long* count) {
  unsigned long long c = 0;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m; k += (uint64_t)gridDim.x * blockDim.x)
    c += e[2 * k] == e[2 * k + 1];
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

__global__ void run_lengths_kernel(const uint64_t* __restrict__ starts, uint64_t n, uint32_t* __restrict__ len) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n; r += (uint64_t)gridDim.x * blockDim.x)
    len[r] = (uint32_t)(starts[r + 1] - starts[r]);
}

// inverse permutation: dense_of_run[order[i]] = i
__global__ void invert_kernel(const uint64_t* __restrict__ order, uint64_t n, uint32_t* __restrict__ dense_of_run) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    dense_of_run[order[i]] = (uint32_t)i;
}

__global__ void gather_u64_kernel(const uint64_t* __restrict__ src, const uint64_t* __restrict__ idx, uint64_t n,
                                  uint64_t* __restrict__ dst) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}
__global__ void gather_u32_kernel(const uint32_t* __restrict__ src, const uint64_t* __restrict__ idx, uint64_t n,
                                  uint32_t* __restrict__ dst) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

}  // namespace

// ext id -> run (position in the ascending unique-id table) by binary search;
// run = n when absent (sets *missing).
__global__ void map_to_runs_kernel(const uint64_t* __restrict__ sorted_ext, uint64_t n, const uint64_t* __restrict__ ids,
                                   uint64_t m, uint32_t* __restrict__ runs, int* missing) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = ids[i];
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (sorted_ext[mid] < x) lo = mid + 1;
      else hi = mid;
    }
    if (lo < n && sorted_ext[lo] == x) {
      runs[i] = (uint32_t)lo;
    } else {
      runs[i] = (uint32_t)n;
      *missing = 1;
    }
  }
}

void build_index(catgnn_ctx ctx, const uint64_t* d_edges, uint64_t m, catgnn_index_s* idx) {
  cudaStream_t st = ctx->stream;
  const uint64_t n2 = 2 * m;
  auto buf = [&](const char* name, size_t bytes) { return ctx->scratch_buf<unsigned char>(name, std::max<size_t>(bytes, 8)); };
  uint64_t* pos = reinterpret_cast<uint64_t*>(buf("idx_pos", n2 * 8));
  uint64_t* sk = reinterpret_cast<uint64_t*>(buf("idx_sk", n2 * 8));
  uint64_t* sv = reinterpret_cast<uint64_t*>(buf("idx_sv", n2 * 8));
  uint8_t* flag = buf("idx_flag", n2);
  uint64_t* runs_first = reinterpret_cast<uint64_t*>(buf("idx_first", n2 * 8));
  uint64_t* count = reinterpret_cast<uint64_t*>(buf("idx_count", 8));
  idx->m = m;
  if (m == 0) {
    idx->n = 0;
    idx->self_loops = 0;
    return;
  }
  iota_kernel<<<grid_of(n2), 256, 0, st>>>(pos, n2);
  size_t tb = 0;
  CG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, d_edges, sk, pos, sv, n2, 0, 64, st));
  CG_CUDA(cub::DeviceRadixSort::SortPairs(buf("idx_cub", tb), tb, d_edges, sk, pos, sv, n2, 0, 64, st));
  run_starts_kernel<<<grid_of(n2), 256, 0, st>>>(sk, n2, flag);
  // unique ids (ascending) and the first stream position of each
  idx->sorted_ext.alloc(n2);
  tb = 0;
  CG_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, sk, flag, idx->sorted_ext.p, count, n2, st));
  CG_CUDA(cub::DeviceSelect::Flagged(buf("idx_cub", tb), tb, sk, flag, idx->sorted_ext.p, count, n2, st));
  uint64_t n = 0;
  CG_CUDA(cudaMemcpyAsync(&n, count, 8, cudaMemcpyDeviceToHost, st));
  CG_CUDA(cudaStreamSynchronize(st));
  tb = 0;
  CG_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, sv, flag, runs_first, count, n2, st));
  CG_CUDA(cub::DeviceSelect::Flagged(buf("idx_cub", tb), tb, sv, flag, runs_first, count, n2, st));
  // degree = run length: positions of the run starts, differenced
  uint64_t* starts = reinterpret_cast<uint64_t*>(buf("idx_starts", (n2 + 1) * 8));
  thrust::counting_iterator<uint64_t> it(0);
  tb = 0;
  CG_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, it, flag, starts, count, n2, st));
  CG_CUDA(cub::DeviceSelect::Flagged(buf("idx_cub", tb), tb, it, flag, starts, count, n2, st));
  CG_CUDA(cudaMemcpyAsync(starts + n, &n2, 8, cudaMemcpyHostToDevice, st));
  CG_CUDA(cudaStreamSynchronize(st));
  uint32_t* deg_run = reinterpret_cast<uint32_t*>(buf("idx_degrun", n * 4));
  run_lengths_kernel<<<grid_of(n), 256, 0, st>>>(starts, n, deg_run);
  // first-seen order: sort runs by their first position
  uint64_t* run_ids = reinterpret_cast<uint64_t*>(buf("idx_runids", n * 8));
  uint64_t* first_sorted = reinterpret_cast<uint64_t*>(buf("idx_firstsorted", n * 8));
  uint64_t* order = reinterpret_cast<uint64_t*>(buf("idx_order", n * 8));
  iota_kernel<<<grid_of(n), 256, 0, st>>>(run_ids, n);
  tb = 0;
  CG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, runs_first, first_sorted, run_ids, order, n, 0, 64, st));
  CG_CUDA(cub::DeviceRadixSort::SortPairs(buf("idx_cub", tb), tb, runs_first, first_sorted, run_ids, order, n, 0,
                                          64, st));
  idx->dense_of_run.alloc(std::max<uint64_t>(n, 1));
  invert_kernel<<<grid_of(n), 256, 0, st>>>(order, n, idx->dense_of_run.p);
  uint64_t* d2e = reinterpret_cast<uint64_t*>(buf("idx_d2e", n * 8));
  uint32_t* degd = reinterpret_cast<uint32_t*>(buf("idx_degd", n * 4));
  gather_u64_kernel<<<grid_of(n), 256, 0, st>>>(idx->sorted_ext.p, order, n, d2e);
  gather_u32_kernel<<<grid_of(n), 256, 0, st>>>(deg_run, order, n, degd);
  unsigned long long* slc = reinterpret_cast<unsigned long long*>(buf("idx_slc", 8));
  CG_CUDA(cudaMemsetAsync(slc, 0, 8, st));
  self_loops_kernel<<<grid_of(m), 256, 0, st>>>(d_edges, m, slc);
  CG_CHECK_LAUNCH();
  idx->n = n;
  idx->dense_to_ext.resize(n);
  idx->degree.resize(n);
  unsigned long long h_sl = 0;
  CG_CUDA(cudaMemcpyAsync(idx->dense_to_ext.data(), d2e, n * 8, cudaMemcpyDeviceToHost, st));
  CG_CUDA(cudaMemcpyAsync(idx->degree.data(), degd, n * 4, cudaMemcpyDeviceToHost, st));
  CG_CUDA(cudaMemcpyAsync(&h_sl, slc, 8, cudaMemcpyDeviceToHost, st));
  CG_CUDA(cudaStreamSynchronize(st));
  idx->self_loops = h_sl;
  ctx->launches += 8;
  for (auto itr = ctx->scratch.begin(); itr != ctx->scratch.end();)
    itr = itr->first.rfind("idx_", 0) == 0 ? ctx->scratch.erase(itr) : std::next(itr);
}

}  // namespace catgnn

using namespace catgnn;

int catgnn_index_build(catgnn_ctx ctx, const uint64_t* edges, uint64_t num_edges, catgnn_index* out) {
  return guarded([&] {
    if (!ctx || !out || (num_edges && !edges)) throw ConfigError("null argument");
    CG_CUDA(cudaSetDevice(ctx->device));
    auto idx = std::make_unique<catgnn_index_s>();
    idx->ctx = ctx;
    DevBuf<uint64_t> d_e;
    d_e.alloc(std::max<uint64_t>(2 * num_edges, 1));
    if (num_edges)
      CG_CUDA(cudaMemcpyAsync(d_e.p, edges, 2 * num_edges * 8, cudaMemcpyHostToDevice, ctx->stream));
    build_index(ctx, d_e.p, num_edges, idx.get());
    if (idx->n >= (1ull << 32)) throw ConfigError("more than 2^32 nodes");
    ctx_retain(ctx);
    *out = idx.release();
  });
}

int catgnn_index_info(catgnn_index idx, uint64_t* num_nodes, uint64_t* num_edges, uint64_t* num_self_loops) {
  return guarded([&] {
    if (!idx) throw ConfigError("null index");
    if (num_nodes) *num_nodes = idx->n;
    if (num_edges) *num_edges = idx->m;
    if (num_self_loops) *num_self_loops = idx->self_loops;
  });
}

int catgnn_index_export(catgnn_index idx, uint64_t* dense_to_ext, uint32_t* degree) {
  return guarded([&] {
    if (!idx) throw ConfigError("null index");
    if (dense_to_ext) std::copy(idx->dense_to_ext.begin(), idx->dense_to_ext.end(), dense_to_ext);
    if (degree) std::copy(idx->degree.begin(), idx->degree.end(), degree);
  });
}

int catgnn_index_destroy(catgnn_index idx) {
  return guarded([&] {
    if (!idx) return;
    catgnn_ctx c = idx->ctx;
    delete idx;
    ctx_release(c);
  });
}
