// K1 — device CSR builder, the B200 restatement of gnnpart::build_adjacency
// (/root/reference/proj/src/train.cpp:30-47) and of the local-id mapping in
// load_training_data (train.cpp:255-273).
//
// build_adjacency fills each row with a cursor walked in edge order: edge k =
// (u,v) appends v to row u and, when u != v, u to row v.  Expanding edge k into
// the two entries (u->v) at position 2k and (v->u) at 2k+1 (dropped for
// self-loops) and STABLY sorting by source row reproduces that order exactly:
// inside a row the entries stay in ascending (k, side) order.  The sort is an
// LSD radix sort over only ceil(log2(rows+1)) key bits (CUB onesweep), the
// offsets are a degree histogram + scan.  Everything is int32 column indices
// and int64 offsets (train.hpp:19's u32 offsets overflow at papers scale).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <cstdlib>

#include "shard.hpp"

namespace catgnn {

namespace {

__global__ void count_degrees_kernel(const uint32_t* __restrict__ pairs, uint64_t num_edges,
                                     uint32_t rows, int32_t* __restrict__ deg,
                                     int* __restrict__ bad) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < num_edges;
       k += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t u = pairs[2 * k], v = pairs[2 * k + 1];
    if (u >= rows || v >= rows) {
      *bad = 1;
      continue;
    }
    atomicAdd(&deg[u], 1);
    if (u != v) atomicAdd(&deg[v], 1);
  }
}

__global__ void expand_entries_kernel(const uint32_t* __restrict__ pairs, uint64_t num_edges,
                                      uint32_t sentinel, uint32_t* __restrict__ keys,
                                      uint32_t* __restrict__ vals) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < num_edges;
       k += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t u = pairs[2 * k], v = pairs[2 * k + 1];
    keys[2 * k] = u;
    vals[2 * k] = v;
    keys[2 * k + 1] = (u != v) ? v : sentinel;  // a self-loop is stored once
    vals[2 * k + 1] = u;
  }
}

struct ToI64 {
  __host__ __device__ int64_t operator()(int32_t x) const { return x; }
};

__global__ void degree_scales_kernel(const int64_t* __restrict__ row_ptr, uint64_t rows,
                                     float* __restrict__ dinv, float* __restrict__ inv_deg,
                                     float* __restrict__ inv_deg1) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x) {
    float d = (float)(row_ptr[r + 1] - row_ptr[r]);
    dinv[r] = 1.0f / sqrtf(1.0f + d);
    inv_deg[r] = d > 0.f ? 1.0f / d : 0.0f;
    inv_deg1[r] = 1.0f / (1.0f + d);  // sgc_propagate's scale (train.cpp:60), as K2's kNormSgc
  }
}

__global__ void map_ext_kernel(const uint64_t* __restrict__ ext, uint64_t rows,
                               const uint64_t* __restrict__ edges, uint64_t n_ids,
                               uint32_t* __restrict__ out, int* __restrict__ missing) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_ids;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t key = edges[i];
    uint64_t lo = 0, hi = rows;
    while (lo < hi) {
      uint64_t mid = (lo + hi) >> 1;
      if (ext[mid] < key) lo = mid + 1; else hi = mid;
    }
    if (lo >= rows || ext[lo] != key) {
      *missing = 1;
      out[i] = 0;
    } else {
      out[i] = (uint32_t)lo;
    }
  }
}

__global__ void copy_rows_kernel(const float4* __restrict__ in, uint32_t in_ld4,
                                 float4* __restrict__ out, uint32_t out_ld4, uint64_t rows,
                                 uint32_t w4) {
  uint64_t total = rows * w4;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t r = i / w4;
    uint32_t c = (uint32_t)(i % w4);
    out[r * out_ld4 + c] = in[r * in_ld4 + c];
  }
}


inline unsigned grid_for(uint64_t n, unsigned block = 256) {
  uint64_t g = (n + block - 1) / block;
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(g, 148ull * 64));
}

uint32_t env_unit_cost() {
  const char* s = std::getenv("CATGNN_UNIT");
  if (s && *s) {
    long v = std::strtol(s, nullptr, 10);
    if (v >= 32) return (uint32_t)v;
  }
  return 512;
}

// Aggregation work plan.  Light units pack consecutive rows until their cost
// (deg + 2 per row) reaches U; a row with deg > U is split into ceil(deg/U)
// chunk units whose partial sums a fix-up pass combines in chunk order, so the
// result is deterministic run to run.
void build_plan(catgnn_shard_s* s, const std::vector<int64_t>& rp) {
  const uint32_t U = env_unit_cost();
  static const uint64_t row_cost = [] {  // per-row overhead in edge units (A/B knob)
    const char* v = std::getenv("CATGNN_ROW_COST");
    return (uint64_t)(v && *v ? std::max(1L, std::strtol(v, nullptr, 10)) : 32L);  // 32: measured best on the reddit shards (scripts/plan_sweep.sh)
  }();
  std::vector<int4> units, heavy;
  uint64_t chunks = 0, cost = 0, begin = 0;
  for (uint64_t r = 0; r < s->rows; ++r) {
    uint64_t deg = (uint64_t)(rp[r + 1] - rp[r]);
    if (deg > U) {
      if (r > begin) units.push_back(make_int4((int)begin, (int)r, -1, 0));
      uint64_t nch = (deg + U - 1) / U;
      heavy.push_back(make_int4((int)r, (int)chunks, (int)nch, 0));
      for (uint64_t c = 0; c < nch; ++c)
        units.push_back(make_int4((int)r, (int)c, (int)(chunks + c), 0));
      chunks += nch;
      begin = r + 1;
      cost = 0;
    } else {
      cost += deg + row_cost;
      if (cost >= U) {
        units.push_back(make_int4((int)begin, (int)(r + 1), -1, 0));
        begin = r + 1;
        cost = 0;
      }
    }
  }
  if (begin < s->rows) units.push_back(make_int4((int)begin, (int)s->rows, -1, 0));
  s->unit_cost = U;
  s->n_units = units.size();
  s->n_heavy = heavy.size();
  s->n_chunks = chunks;
  s->units.alloc(std::max<size_t>(1, units.size()));
  s->heavy.alloc(std::max<size_t>(1, heavy.size()));
  if (!units.empty())
    CG_CUDA(cudaMemcpyAsync(s->units.p, units.data(), units.size() * sizeof(int4),
                            cudaMemcpyHostToDevice, s->ctx->stream));
  if (!heavy.empty())
    CG_CUDA(cudaMemcpyAsync(s->heavy.p, heavy.data(), heavy.size() * sizeof(int4),
                            cudaMemcpyHostToDevice, s->ctx->stream));
  CG_CUDA(cudaStreamSynchronize(s->ctx->stream));
}

}  // namespace

void build_csr(catgnn_shard_s* s, const uint32_t* d_pairs, uint64_t num_edges) {
  catgnn_ctx ctx = s->ctx;
  cudaStream_t st = ctx->stream;
  if (s->rows >= 0x7fffffffull) throw ConfigError("shard rows exceed the int32 column index range");
  const uint32_t rows = (uint32_t)s->rows;
  s->num_edges = num_edges;
  s->row_ptr.alloc(rows + 1);
  int32_t* deg = ctx->scratch_buf<int32_t>("k1_deg", rows + 1);
  int* bad = ctx->scratch_buf<int>("k1_flag", 1);
  CG_CUDA(cudaMemsetAsync(deg, 0, sizeof(int32_t) * (rows + 1), st));
  CG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
  if (num_edges) {
    count_degrees_kernel<<<grid_for(num_edges), 256, 0, st>>>(d_pairs, num_edges, rows, deg, bad);
    CG_CHECK_LAUNCH();
    ctx->launches++;
  }
  int h_bad = 0;
  CG_CUDA(cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  CG_CUDA(cudaStreamSynchronize(st));
  if (h_bad) throw DataError("edge endpoint outside the row space");

  // offsets: row_ptr[0] = 0, row_ptr[1..] = inclusive scan of deg
  CG_CUDA(cudaMemsetAsync(s->row_ptr.p, 0, sizeof(int64_t), st));
  {
    auto it = thrust::make_transform_iterator(deg, ToI64());
    size_t tmp_bytes = 0;
    CG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, it, s->row_ptr.p + 1, (int)rows, st));
    void* tmp = ctx->scratch_buf<unsigned char>("k1_cub", tmp_bytes);
    CG_CUDA(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, it, s->row_ptr.p + 1, (int)rows, st));
    ctx->launches += 2;
  }
  std::vector<int64_t> rp(rows + 1);
  CG_CUDA(cudaMemcpyAsync(rp.data(), s->row_ptr.p, sizeof(int64_t) * (rows + 1),
                          cudaMemcpyDeviceToHost, st));
  CG_CUDA(cudaStreamSynchronize(st));
  s->nnz = (uint64_t)rp[rows];
  if (s->nnz >= 0x7fffffffull * 2) throw ConfigError("shard nnz exceeds the sort index range");

  s->col.alloc(std::max<uint64_t>(1, s->nnz));
  if (num_edges) {
    const uint64_t n2 = 2 * num_edges;
    uint32_t* k_in = ctx->scratch_buf<uint32_t>("k1_kin", n2);
    uint32_t* v_in = ctx->scratch_buf<uint32_t>("k1_vin", n2);
    uint32_t* k_out = ctx->scratch_buf<uint32_t>("k1_kout", n2);
    uint32_t* v_out = ctx->scratch_buf<uint32_t>("k1_vout", n2);
    expand_entries_kernel<<<grid_for(num_edges), 256, 0, st>>>(d_pairs, num_edges, rows, k_in, v_in);
    CG_CHECK_LAUNCH();
    ctx->launches++;
    int end_bit = 1;
    while (end_bit < 32 && (1ull << end_bit) <= rows) ++end_bit;  // sentinel = rows must fit
    size_t tmp_bytes = 0;
    CG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k_in, k_out, v_in, v_out,
                                            (int64_t)n2, 0, end_bit, st));
    void* tmp = ctx->scratch_buf<unsigned char>("k1_cub", tmp_bytes);
    CG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k_in, k_out, v_in, v_out,
                                            (int64_t)n2, 0, end_bit, st));
    ctx->launches += 4;
    // entries with a real source come first (sentinel = rows sorts last)
    CG_CUDA(cudaMemcpyAsync(s->col.p, v_out, s->nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  }
  s->dinv.alloc(std::max<uint32_t>(1, rows));
  s->inv_deg.alloc(std::max<uint32_t>(1, rows));
  s->inv_deg1.alloc(std::max<uint32_t>(1, rows));
  if (rows) {
    degree_scales_kernel<<<grid_for(rows), 256, 0, st>>>(s->row_ptr.p, rows, s->dinv.p, s->inv_deg.p,
                                                         s->inv_deg1.p);
    CG_CHECK_LAUNCH();
    ctx->launches++;
  }
  build_plan(s, rp);
}

void map_ext_edges(catgnn_ctx ctx, const uint64_t* d_ext_ids, uint64_t rows,
                   const uint64_t* d_edges_ext, uint64_t num_edges, uint32_t* d_pairs) {
  int* missing = ctx->scratch_buf<int>("k1_missing", 1);
  CG_CUDA(cudaMemsetAsync(missing, 0, sizeof(int), ctx->stream));
  if (num_edges) {
    map_ext_kernel<<<grid_for(2 * num_edges), 256, 0, ctx->stream>>>(d_ext_ids, rows, d_edges_ext,
                                                                   2 * num_edges, d_pairs, missing);
    CG_CHECK_LAUNCH();
    ctx->launches++;
  }
  int h = 0;
  CG_CUDA(cudaMemcpyAsync(&h, missing, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CG_CUDA(cudaStreamSynchronize(ctx->stream));
  // load_training_data uses unordered_map::at (train.cpp:271): a missing
  // endpoint escapes as std::out_of_range, i.e. the CLI's "internal" category.
  if (h) throw InternalError("partition edge endpoint missing from its node table (unordered_map::at)");
}

void copy_rows(catgnn_ctx ctx, const float* in, uint32_t in_ld, float* out, uint32_t out_ld,
               uint64_t rows, uint32_t width) {
  if (!rows || !width) return;
  uint32_t w4 = width / 4;
  copy_rows_kernel<<<grid_for(rows * w4), 256, 0, ctx->stream>>>(
      reinterpret_cast<const float4*>(in), in_ld / 4, reinterpret_cast<float4*>(out), out_ld / 4,
      rows, w4);
  CG_CHECK_LAUNCH();
  ctx->launches++;
}


}  // namespace catgnn
