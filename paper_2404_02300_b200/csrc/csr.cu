// K1 — device CSR builder, the B200 restatement of gnnpart::build_adjacency
// (/root/reference/proj/src/train.cpp:30-47) and of the local-id mapping in
// load_training_data (train.cpp:255-273).
//
// build_adjacency fills each row with a cursor walked in edge order: edge k =
// (u,v) appends v to row u and, when u != v, u to row v.  Expanding edge k into
// the two entries (u->v) at position 2k and (v->u) at 2k+1 (dropped for
// self-loops) and STABLY sorting by source row reproduces that order exactly:
// inside a row the entries stay in ascending (k, side) order.  The sort is our
// own stable LSD radix sort (radix.cu) over only ceil(log2(rows+1)) key bits,
// the offsets are a degree histogram + scan.  Everything is int32 column indices
// and int64 offsets (train.hpp:19's u32 offsets overflow at papers scale).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "radix.hpp"
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

// Aggregation work plan, built on the device.  A row with deg > U is split
// into ceil(deg/U) chunk units whose partial sums a fix-up pass combines in
// chunk order; the other (light) rows are packed into units of consecutive
// rows by their cost deg + row_cost: with P_r the exclusive prefix of those
// costs, a light row starts a unit when floor(P_r / U) differs from its light
// predecessor's or a heavy row lies in between, so units carry ~U cost each.
// Units are listed in row order (the persistent K2 grid pulls them in that
// order).  A light row's sum never depends on where its unit starts or ends
// (each row is one warp's edge walk from its own first edge), and chunking is
// fixed by U, so the plan changes no result bit.
//
// plan_rows_kernel: per row, the units it emits (1 for a unit start, nch for a
// heavy row, else 0), its heavy flag and its chunk count.
__global__ void plan_rows_kernel(const int64_t* __restrict__ row_ptr, uint64_t rows, uint32_t U,
                                 uint64_t row_cost, uint64_t* __restrict__ cost, uint32_t* __restrict__ nch,
                                 unsigned long long* __restrict__ big) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t deg = (uint64_t)(row_ptr[r + 1] - row_ptr[r]);
    const bool heavy = deg > U;
    cost[r] = heavy ? 0 : deg + row_cost;
    nch[r] = heavy ? (uint32_t)((deg + U - 1) / U) : 0;
    if (heavy && nch[r] > 16) atomicAdd(big, 1ull);  // aggregate.cu kWarpFixChunks
  }
}
// emit[r]: units row r opens (needs the exclusive cost prefix P)
__global__ void plan_emit_kernel(const uint64_t* __restrict__ P, const uint32_t* __restrict__ nch, uint64_t rows,
                                 uint32_t U, uint32_t* __restrict__ emit, uint32_t* __restrict__ is_heavy) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t h = nch[r];
    is_heavy[r] = h ? 1u : 0u;
    uint32_t e = h;
    if (!h) {  // light: a unit start after a heavy row, at row 0, or at a new cost bucket
      const bool start = r == 0 || nch[r - 1] != 0 || (P[r] / U) != (P[r - 1] / U);
      e = start ? 1u : 0u;
    }
    emit[r] = e;
  }
}
// scatter: light unit starts (end filled by plan_ends_kernel), chunk units and
// the heavy table
__global__ void plan_scatter_kernel(const uint32_t* __restrict__ nch, const uint32_t* __restrict__ emit,
                                    const uint64_t* __restrict__ upos, const uint64_t* __restrict__ hpos,
                                    const uint64_t* __restrict__ cpos, uint64_t rows, int4* __restrict__ units,
                                    int4* __restrict__ heavy) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t h = nch[r];
    if (h) {
      const uint64_t c0 = cpos[r];
      heavy[hpos[r]] = make_int4((int)r, (int)c0, (int)h, 0);
      for (uint32_t c = 0; c < h; ++c) units[upos[r] + c] = make_int4((int)r, (int)c, (int)(c0 + c), 0);
    } else if (emit[r]) {
      units[upos[r]] = make_int4((int)r, -1, -1, 0);
    }
  }
}
// a light unit ends where the next unit (light start or heavy row) begins
__global__ void plan_ends_kernel(int4* __restrict__ units, uint64_t n_units, uint64_t rows) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_units;
       i += (uint64_t)gridDim.x * blockDim.x) {
    int4 u = units[i];
    if (u.z >= 0) continue;
    u.y = i + 1 < n_units ? units[i + 1].x : (int)rows;
    units[i] = u;
  }
}

template <typename InIt, typename Out>
void exclusive_scan(catgnn_ctx ctx, InIt in, Out* out, uint64_t n) {
  size_t tmp_bytes = 0;
  CG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, in, out, (int64_t)n, ctx->stream));
  void* tmp = ctx->scratch_buf<unsigned char>("k1_cub", tmp_bytes);
  CG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, in, out, (int64_t)n, ctx->stream));
  ctx->launches += 2;
}

struct U32ToU64 {
  __host__ __device__ uint64_t operator()(uint32_t x) const { return x; }
};

void build_plan(catgnn_shard_s* s) {
  catgnn_ctx ctx = s->ctx;
  cudaStream_t st = ctx->stream;
  const uint32_t U = env_unit_cost();
  static const uint64_t row_cost = [] {  // per-row overhead in edge units (A/B knob)
    const char* v = std::getenv("CATGNN_ROW_COST");
    return (uint64_t)(v && *v ? std::max(1L, std::strtol(v, nullptr, 10)) : 32L);  // 32: measured best on the reddit shards (scripts/plan_sweep.sh)
  }();
  const uint64_t rows = s->rows;
  s->unit_cost = U;
  if (rows == 0) {
    s->n_units = s->n_heavy = s->n_chunks = s->n_big_heavy = 0;
    s->units.alloc(1);
    s->heavy.alloc(1);
    return;
  }
  const uint64_t n1 = rows + 1;  // one extra slot: the scans' totals
  uint64_t* cost = ctx->scratch_buf<uint64_t>("k1_plan_cost", n1);
  uint64_t* P = ctx->scratch_buf<uint64_t>("k1_plan_P", n1);
  uint32_t* nch = ctx->scratch_buf<uint32_t>("k1_plan_nch", n1);
  uint32_t* emit = ctx->scratch_buf<uint32_t>("k1_plan_emit", n1);
  uint32_t* ish = ctx->scratch_buf<uint32_t>("k1_plan_heavy", n1);
  uint64_t* upos = ctx->scratch_buf<uint64_t>("k1_plan_upos", n1);
  uint64_t* hpos = ctx->scratch_buf<uint64_t>("k1_plan_hpos", n1);
  uint64_t* cpos = ctx->scratch_buf<uint64_t>("k1_plan_cpos", n1);
  CG_CUDA(cudaMemsetAsync(cost + rows, 0, 8, st));
  CG_CUDA(cudaMemsetAsync(nch + rows, 0, 4, st));
  CG_CUDA(cudaMemsetAsync(emit + rows, 0, 4, st));
  CG_CUDA(cudaMemsetAsync(ish + rows, 0, 4, st));
  unsigned long long* big = ctx->scratch_buf<unsigned long long>("k1_plan_big", 1);
  CG_CUDA(cudaMemsetAsync(big, 0, 8, st));
  plan_rows_kernel<<<grid_for(rows), 256, 0, st>>>(s->row_ptr.p, rows, U, row_cost, cost, nch, big);
  CG_CHECK_LAUNCH();
  exclusive_scan(ctx, cost, P, n1);
  plan_emit_kernel<<<grid_for(rows), 256, 0, st>>>(P, nch, rows, U, emit, ish);
  CG_CHECK_LAUNCH();
  auto e64 = thrust::make_transform_iterator(emit, U32ToU64());
  auto h64 = thrust::make_transform_iterator(ish, U32ToU64());
  auto c64 = thrust::make_transform_iterator(nch, U32ToU64());
  exclusive_scan(ctx, e64, upos, n1);
  exclusive_scan(ctx, h64, hpos, n1);
  exclusive_scan(ctx, c64, cpos, n1);
  uint64_t tot[4];
  CG_CUDA(cudaMemcpyAsync(&tot[0], upos + rows, 8, cudaMemcpyDeviceToHost, st));
  CG_CUDA(cudaMemcpyAsync(&tot[1], hpos + rows, 8, cudaMemcpyDeviceToHost, st));
  CG_CUDA(cudaMemcpyAsync(&tot[2], cpos + rows, 8, cudaMemcpyDeviceToHost, st));
  CG_CUDA(cudaMemcpyAsync(&tot[3], big, 8, cudaMemcpyDeviceToHost, st));
  CG_CUDA(cudaStreamSynchronize(st));
  s->n_units = tot[0];
  s->n_heavy = tot[1];
  s->n_chunks = tot[2];
  s->n_big_heavy = tot[3];
  if (s->n_units >= 0x7fffffffull || s->n_chunks >= 0x7fffffffull)
    throw ConfigError("aggregation plan exceeds the int32 unit range");
  s->units.alloc(std::max<uint64_t>(1, s->n_units));
  s->heavy.alloc(std::max<uint64_t>(1, s->n_heavy));
  plan_scatter_kernel<<<grid_for(rows), 256, 0, st>>>(nch, emit, upos, hpos, cpos, rows, s->units.p, s->heavy.p);
  CG_CHECK_LAUNCH();
  plan_ends_kernel<<<grid_for(s->n_units), 256, 0, st>>>(s->units.p, s->n_units, rows);
  CG_CHECK_LAUNCH();
  ctx->launches += 4;
}

// train-row views (train_rows_view / train_nbr_view)
__global__ void view_deg_kernel(const int64_t* __restrict__ row_ptr, const uint32_t* __restrict__ rows_sel,
                                uint64_t n, uint64_t* __restrict__ deg) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t r = rows_sel[i];
    deg[i] = (uint64_t)(row_ptr[r + 1] - row_ptr[r]);
  }
}
// warp per selected row: its neighbour list copied in order
__global__ void view_copy_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                                 const uint32_t* __restrict__ rows_sel, uint64_t n,
                                 const int64_t* __restrict__ vptr, int32_t* __restrict__ vcol) {
  const int lane = threadIdx.x & 31;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
    const uint32_t r = rows_sel[i];
    const int64_t b = row_ptr[r], e = row_ptr[r + 1], o = vptr[i];
    for (int64_t k = b + lane; k < e; k += 32) vcol[o + (k - b)] = col[k];
  }
}
__global__ void mark_rows_kernel(const uint32_t* __restrict__ rows_sel, uint64_t n, uint8_t* __restrict__ flag) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    flag[rows_sel[i]] = 1;
}
// warp per row: neighbours that are flagged (counted, then compacted in order)
__global__ void filter_count_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                                    uint64_t rows, const uint8_t* __restrict__ flag, uint64_t* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < rows;
       r += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
    uint32_t c = 0;
    for (int64_t k = row_ptr[r] + lane; k < row_ptr[r + 1]; k += 32) c += flag[col[k]];
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) c += __shfl_xor_sync(0xffffffffu, c, m);
    if (lane == 0) cnt[r] = c;
  }
}
__global__ void filter_copy_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                                   uint64_t rows, const uint8_t* __restrict__ flag, const int64_t* __restrict__ fptr,
                                   int32_t* __restrict__ fcol) {
  const int lane = threadIdx.x & 31;
  for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < rows;
       r += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
    int64_t o = fptr[r];
    const int64_t e1 = row_ptr[r + 1];
    for (int64_t k0 = row_ptr[r]; k0 < e1; k0 += 32) {
      const int64_t k = k0 + lane;
      const int32_t j = k < e1 ? col[k] : 0;
      const bool keep = k < e1 && flag[j];
      const uint32_t m = __ballot_sync(0xffffffffu, keep);
      if (keep) fcol[o + __popc(m & ((1u << lane) - 1u))] = j;
      o += __popc(m);
    }
  }
}

unsigned warps_grid(uint64_t n) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 7) / 8, 148ull * 16));
}

// A view shard sharing the parent's context: CSR (row_ptr from per-row counts)
// + its own K2 work plan.
std::unique_ptr<catgnn_shard_s> make_view(catgnn_shard_s* s, uint64_t rows, const uint64_t* d_cnt) {
  auto v = std::make_unique<catgnn_shard_s>();
  v->ctx = s->ctx;
  v->rows = rows;
  v->row_ptr.alloc(rows + 1);
  uint64_t* tmp = s->ctx->scratch_buf<uint64_t>("sub_scan", rows + 1);
  CG_CUDA(cudaMemcpyAsync(tmp, d_cnt, rows * 8, cudaMemcpyDeviceToDevice, s->ctx->stream));
  CG_CUDA(cudaMemsetAsync(tmp + rows, 0, 8, s->ctx->stream));
  exclusive_scan(s->ctx, tmp, reinterpret_cast<uint64_t*>(v->row_ptr.p), rows + 1);
  int64_t nnz = 0;
  CG_CUDA(cudaMemcpyAsync(&nnz, v->row_ptr.p + rows, 8, cudaMemcpyDeviceToHost, s->ctx->stream));
  CG_CUDA(cudaStreamSynchronize(s->ctx->stream));
  v->nnz = (uint64_t)nnz;
  v->col.alloc(std::max<uint64_t>(1, v->nnz));
  return v;
}

}  // namespace

catgnn_shard_s* train_rows_view(catgnn_shard_s* s) {
  const uint64_t n = s->h_train.size();
  if (!n) return nullptr;
  if (!s->train_sub) {
    cudaStream_t st = s->ctx->stream;
    uint64_t* deg = s->ctx->scratch_buf<uint64_t>("sub_cnt", n);
    view_deg_kernel<<<grid_for(n), 256, 0, st>>>(s->row_ptr.p, s->d_train.p, n, deg);
    CG_CHECK_LAUNCH();
    auto v = make_view(s, n, deg);
    view_copy_kernel<<<warps_grid(n), 256, 0, st>>>(s->row_ptr.p, s->col.p, s->d_train.p, n, v->row_ptr.p, v->col.p);
    CG_CHECK_LAUNCH();
    v->row_map.alloc(n);
    CG_CUDA(cudaMemcpyAsync(v->row_map.p, s->d_train.p, n * 4, cudaMemcpyDeviceToDevice, st));
    build_plan(v.get());
    s->ctx->launches += 3;
    s->ctx->release_scratch({"k1_", "sub_"});
    s->train_sub = std::move(v);
  }
  return s->train_sub.get();
}

catgnn_shard_s* train_nbr_view(catgnn_shard_s* s) {
  const uint64_t n = s->h_train.size();
  if (!n || !s->rows) return nullptr;
  if (!s->train_nbr) {
    cudaStream_t st = s->ctx->stream;
    uint8_t* flag = s->ctx->scratch_buf<uint8_t>("sub_flag", s->rows);
    CG_CUDA(cudaMemsetAsync(flag, 0, s->rows, st));
    mark_rows_kernel<<<grid_for(n), 256, 0, st>>>(s->d_train.p, n, flag);
    CG_CHECK_LAUNCH();
    uint64_t* cnt = s->ctx->scratch_buf<uint64_t>("sub_cnt", s->rows);
    filter_count_kernel<<<warps_grid(s->rows), 256, 0, st>>>(s->row_ptr.p, s->col.p, s->rows, flag, cnt);
    CG_CHECK_LAUNCH();
    auto v = make_view(s, s->rows, cnt);
    filter_copy_kernel<<<warps_grid(s->rows), 256, 0, st>>>(s->row_ptr.p, s->col.p, s->rows, flag, v->row_ptr.p,
                                                           v->col.p);
    CG_CHECK_LAUNCH();
    build_plan(v.get());
    s->ctx->launches += 4;
    s->ctx->release_scratch({"k1_", "sub_"});
    s->train_nbr = std::move(v);
  }
  return s->train_nbr.get();
}

void build_csr(catgnn_shard_s* s, const uint32_t* d_pairs, uint64_t num_edges) {
  catgnn_ctx ctx = s->ctx;
  cudaStream_t st = ctx->stream;
  if (s->rows >= 0x7fffffffull) throw ConfigError("shard rows exceed the int32 column index range");
  const uint32_t rows = (uint32_t)s->rows;
  s->num_edges = num_edges;
  s->train_sub.reset();  // views of the previous CSR
  s->train_nbr.reset();
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
  int64_t nnz = 0;
  CG_CUDA(cudaMemcpyAsync(&nnz, s->row_ptr.p + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CG_CUDA(cudaStreamSynchronize(st));
  s->nnz = (uint64_t)nnz;
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
    uint32_t *k_res = nullptr, *v_res = nullptr;
    radix_sort_pairs(ctx, k_in, v_in, k_out, v_out, n2, end_bit, &k_res, &v_res);  // stable (radix.cu)
    // entries with a real source come first (sentinel = rows sorts last)
    CG_CUDA(cudaMemcpyAsync(s->col.p, v_res, s->nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
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
  build_plan(s);
  // K1's temporaries (expanded entries, radix buffers, plan scans: ~70 B per nnz)
  ctx->release_scratch({"k1_", "radix_", "pairs", "edges_ext", "ext_ids"});
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

namespace {
__global__ void halo_lookup_kernel(const uint64_t* __restrict__ ext, uint64_t rows, const uint32_t* __restrict__ ids,
                                   const uint32_t* __restrict__ parts, uint64_t n, uint32_t* __restrict__ home,
                                   unsigned int* __restrict__ missing) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t key = ext[r];
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if ((uint64_t)ids[mid] < key) lo = mid + 1; else hi = mid;
    }
    if (lo < n && ids[lo] == key) home[r] = parts[lo];
    else { home[r] = 0xFFFFFFFFu; atomicAdd(missing, 1u); }
  }
}
}  // namespace

uint64_t halo_map(catgnn_shard_s* s, const uint32_t* owner_ids, const uint32_t* owner_parts, uint64_t n_owned,
                  uint64_t num_ids, uint32_t* home_host) {
  catgnn_ctx ctx = s->ctx;
  cudaStream_t st = ctx->stream;
  if (num_ids > 0xffffffffull) throw ConfigError("halo map: ids beyond 2^32");
  const uint64_t n = std::max<uint64_t>(1, n_owned);
  uint32_t* k = ctx->scratch_buf<uint32_t>("halo_k", n);
  uint32_t* v = ctx->scratch_buf<uint32_t>("halo_v", n);
  uint32_t* k2 = ctx->scratch_buf<uint32_t>("halo_k2", n);
  uint32_t* v2 = ctx->scratch_buf<uint32_t>("halo_v2", n);
  uint32_t* home = ctx->scratch_buf<uint32_t>("halo_home", std::max<uint64_t>(1, s->rows));
  unsigned int* missing = ctx->scratch_buf<unsigned int>("halo_missing", 1);
  CG_CUDA(cudaMemcpyAsync(k, owner_ids, n_owned * 4, cudaMemcpyHostToDevice, st));
  CG_CUDA(cudaMemcpyAsync(v, owner_parts, n_owned * 4, cudaMemcpyHostToDevice, st));
  CG_CUDA(cudaMemsetAsync(missing, 0, sizeof(unsigned int), st));
  int bits = 1;
  while (bits < 32 && (1ull << bits) < num_ids) ++bits;
  uint32_t *ks = nullptr, *vs = nullptr;
  radix_sort_pairs(ctx, k, v, k2, v2, n_owned, bits, &ks, &vs);
  if (s->rows) {
    halo_lookup_kernel<<<grid_for(s->rows), 256, 0, st>>>(s->d_ext.p, s->rows, ks, vs, n_owned, home, missing);
    CG_CHECK_LAUNCH();
    ctx->launches++;
  }
  unsigned int h_missing = 0;
  CG_CUDA(cudaMemcpyAsync(&h_missing, missing, sizeof(h_missing), cudaMemcpyDeviceToHost, st));
  std::vector<uint32_t> hh(s->rows);
  if (s->rows) CG_CUDA(cudaMemcpyAsync(hh.data(), home, s->rows * 4, cudaMemcpyDeviceToHost, st));
  CG_CUDA(cudaStreamSynchronize(st));
  if (h_missing) throw DataError("replica without an owner partition");
  uint64_t halo = 0;
  for (uint64_t r = 0; r < s->rows; ++r) halo += s->owner.empty() ? 0 : (s->owner[r] == 0);
  if (home_host && s->rows) std::memcpy(home_host, hh.data(), s->rows * 4);
  return halo;
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
