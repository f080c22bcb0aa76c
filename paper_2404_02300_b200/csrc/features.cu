// Global feature store + per-shard row gather: the device form of
// load_training_data's "features gathered from the global matrix" branch
// (/root/reference/proj/src/train.cpp:277-283: X_i.row(r) = global.row(ext_r)).
//
// The global matrix lives on the device exactly as it lies in host memory
// (rows x dim f32, dense, FEA1 row order) so a host->device refresh is one
// contiguous pinned copy of |V|*dim*4 bytes instead of the RF-times larger
// per-shard copies (reddit-shaped p=8: 0.6 GB vs 3.9 GB).  The gather writes
// the shard's padded layout x[r][0..ld) with ld = round_up(dim, 4); padding
// columns stay zero.  HBM-bound: rows*dim*4 read + rows*ld*4 written.
#include <algorithm>
#include <cstdio>
#include <filesystem>
#include <map>

#include <cuda_bf16.h>

#include "artifact.hpp"
#include "comm.hpp"
#include "shard.hpp"

// Uploads run on the store's context stream (a dedicated copy stream when the
// store is created on its own context); gathers on the shard's stream.  Two
// events order them without host syncs: a gather waits for the last upload,
// an upload waits until every stream that gathered from the previous contents
// is done — so a caller can double-buffer stores and copy step t+1's features
// while step t computes.
struct catgnn_features_s {
  catgnn_ctx ctx = nullptr;
  uint64_t rows = 0;
  uint32_t dim = 0;
  catgnn::DevBuf<float> x;  // rows x dim, dense
  cudaEvent_t uploaded = nullptr;
  bool has_upload = false;  // `uploaded` marks an upload consumers must wait for
  std::map<cudaStream_t, cudaEvent_t> consumed;  // per consumer stream: last gather
  ~catgnn_features_s() {
    if (uploaded) cudaEventDestroy(uploaded);
    for (auto& kv : consumed) cudaEventDestroy(kv.second);
  }
};

namespace catgnn {
namespace {

// One warp per destination row.  Source rows are dim*4 bytes apart, so their
// alignment is 16 B only when dim % 4 == 0 (float4 path); otherwise 8 B
// (dim even: float2) or 4 B.
template <int V>
__global__ void __launch_bounds__(256) gather_rows_kernel(const float* __restrict__ src, uint32_t dim,
                                                          const uint64_t* __restrict__ ext, uint64_t rows,
                                                          float* __restrict__ dst, uint32_t ld,
                                                          __nv_bfloat16* __restrict__ hi,
                                                          __nv_bfloat16* __restrict__ lo, uint32_t sld) {
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (uint64_t r = warp; r < rows; r += nwarps) {
    const float* s = src + __ldg(ext + r) * dim;
    float* d = dst ? dst + r * ld : nullptr;
    // bf16x3 copy for the GNN's tensor-core GEMMs (hi = bf16(x), lo = bf16(x - hi)),
    // written from the same registers instead of a separate split pass
    __nv_bfloat16* dh = hi ? hi + r * sld : nullptr;
    __nv_bfloat16* dl = lo ? lo + r * sld : nullptr;
    // U vector loads in flight per lane before their stores (a 602-wide row is
    // 10 float2 per lane: one round trip instead of ten)
    constexpr int U = 8;
    constexpr uint32_t step = 32 * V;
    for (uint32_t c0 = lane * V; c0 < dim; c0 += step * U) {
      if (V == 4) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (c0 + u * step < dim) v[u] = __ldg(reinterpret_cast<const float4*>(s + c0 + u * step));
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (c0 + u * step < dim) {
            if (d) *reinterpret_cast<float4*>(d + c0 + u * step) = v[u];
            if (dh) {
              const __nv_bfloat162 h0 = __floats2bfloat162_rn(v[u].x, v[u].y), h1 = __floats2bfloat162_rn(v[u].z, v[u].w);
              const __nv_bfloat162 l0 = __floats2bfloat162_rn(v[u].x - __low2float(h0), v[u].y - __high2float(h0));
              const __nv_bfloat162 l1 = __floats2bfloat162_rn(v[u].z - __low2float(h1), v[u].w - __high2float(h1));
              reinterpret_cast<__nv_bfloat162*>(dh + c0 + u * step)[0] = h0;
              reinterpret_cast<__nv_bfloat162*>(dh + c0 + u * step)[1] = h1;
              reinterpret_cast<__nv_bfloat162*>(dl + c0 + u * step)[0] = l0;
              reinterpret_cast<__nv_bfloat162*>(dl + c0 + u * step)[1] = l1;
            }
          }
      } else if (V == 2) {
        float2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (c0 + u * step < dim) v[u] = __ldg(reinterpret_cast<const float2*>(s + c0 + u * step));
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (c0 + u * step < dim) {
            if (d) *reinterpret_cast<float2*>(d + c0 + u * step) = v[u];
            if (dh) {
              const __nv_bfloat162 h = __floats2bfloat162_rn(v[u].x, v[u].y);
              *reinterpret_cast<__nv_bfloat162*>(dh + c0 + u * step) = h;
              *reinterpret_cast<__nv_bfloat162*>(dl + c0 + u * step) =
                  __floats2bfloat162_rn(v[u].x - __low2float(h), v[u].y - __high2float(h));
            }
          }
      } else {
        float v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (c0 + u * step < dim) v[u] = __ldg(s + c0 + u * step);
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (c0 + u * step < dim) {
            if (d) d[c0 + u * step] = v[u];
            if (dh) {
              const __nv_bfloat16 h = __float2bfloat16_rn(v[u]);
              dh[c0 + u * step] = h;
              dl[c0 + u * step] = __float2bfloat16_rn(v[u] - __bfloat162float(h));
            }
          }
      }
    }
  }
}

void check_features(catgnn_features f) {
  if (!f || !f->ctx) throw ConfigError("null feature store");
}

}  // namespace
}  // namespace catgnn

using namespace catgnn;

int catgnn_features_create(catgnn_ctx ctx, uint64_t rows, uint32_t dim, catgnn_features* out) {
  return guarded([&] {
    if (!ctx || !out) throw ConfigError("null argument");
    if (dim == 0) throw ConfigError("feature width must be positive");
    auto f = new catgnn_features_s();
    f->ctx = ctx;
    f->rows = rows;
    f->dim = dim;
    try {
      CG_CUDA(cudaSetDevice(ctx->device));
      f->x.alloc(std::max<uint64_t>(1, rows) * dim);
      CG_CUDA(cudaEventCreateWithFlags(&f->uploaded, cudaEventDisableTiming));
    } catch (...) {
      delete f;
      throw;
    }
    ctx_retain(ctx);
    *out = f;
  });
}

int catgnn_features_destroy(catgnn_features f) {
  return guarded([&] {
    if (!f) return;
    catgnn_ctx c = f->ctx;
    delete f;
    ctx_release(c);
  });
}

int catgnn_features_upload(catgnn_features f, const float* host, uint64_t row_begin, uint64_t nrows) {
  return guarded([&] {
    check_features(f);
    if (row_begin > f->rows || nrows > f->rows - row_begin) throw ConfigError("feature rows out of range");
    if (nrows && !host) throw ConfigError("null argument");
    if (!nrows) return;
    cudaStream_t st = f->ctx->stream;
    for (auto& kv : f->consumed)
      if (kv.first != st) CG_CUDA(cudaStreamWaitEvent(st, kv.second, 0));
    CG_CUDA(cudaMemcpyAsync(f->x.p + row_begin * f->dim, host, nrows * f->dim * sizeof(float),
                            cudaMemcpyHostToDevice, st));
    CG_CUDA(cudaEventRecord(f->uploaded, st));
    f->has_upload = true;
  });
}

int catgnn_features_allgather(catgnn_features f, catgnn_comm c, uint64_t rows_per_rank) {
  return guarded([&] {
    check_features(f);
    if (!c || !c->comm) throw ConfigError("null communicator");
    if (rows_per_rank * (uint64_t)c->nranks > std::max<uint64_t>(f->rows, 1) || !rows_per_rank)
      throw ConfigError("feature store too small for rows_per_rank x ranks");
    cudaStream_t st = f->ctx->stream;
    for (auto& kv : f->consumed)
      if (kv.first != st) CG_CUDA(cudaStreamWaitEvent(st, kv.second, 0));
    const size_t count = rows_per_rank * f->dim;
    float* mine = f->x.p + (size_t)c->rank * count;
    const ncclResult_t r = ncclAllGather(mine, f->x.p, count, ncclFloat32, c->comm, st);  // in place
    if (r != ncclSuccess) throw InternalError(std::string("ncclAllGather: ") + ncclGetErrorString(r));
    CG_CUDA(cudaEventRecord(f->uploaded, st));
    f->has_upload = true;
  });
}

// Forget the recorded upload / gather events: the caller orders the store's
// producers and consumers by stream order from here on (e.g. before capturing
// a CUDA graph whose replays must not wait on events of uncaptured work).
int catgnn_features_reset_deps(catgnn_features f) {
  return guarded([&] {
    check_features(f);
    for (auto& kv : f->consumed) CG_CUDA(cudaEventDestroy(kv.second));
    f->consumed.clear();
    f->has_upload = false;
  });
}

int catgnn_shard_gather_features(catgnn_shard s, catgnn_features f) {
  return guarded([&] {
    if (!s || !s->ctx) throw ConfigError("null shard");
    check_features(f);
    if (f->ctx->device != s->ctx->device) throw ConfigError("shard and feature store must share one device");
    if (s->ext_ids.size() != s->rows)
      throw ConfigError("shard has no replica map (create it from a partition)");
    cudaStream_t st = s->ctx->stream;
    if (s->rows && !s->d_ext.p) {
      // the node table is ascending (completion.cpp:54-55), but do not rely on it here
      s->ext_max = *std::max_element(s->ext_ids.begin(), s->ext_ids.end());
      s->d_ext.alloc(s->rows);
      CG_CUDA(cudaMemcpyAsync(s->d_ext.p, s->ext_ids.data(), s->rows * 8, cudaMemcpyHostToDevice, st));
    }
    if (s->rows && s->ext_max >= f->rows)  // train.cpp:279-281
      throw DataError("feature row " + std::to_string(s->ext_max) + " out of range of the feature store");
    const uint32_t ld = round_up(f->dim, 4);
    s->x_version++;  // the bf16x3 copy (gnn.cu) is re-split on next use
    if (s->dim != f->dim || !s->x.p) {
      s->dim = f->dim;
      s->ld = ld;
      s->x.alloc(std::max<uint64_t>(1, s->rows) * ld);
      if (ld != f->dim) CG_CUDA(cudaMemsetAsync(s->x.p, 0, s->x.bytes(), st));
    }
    s->xprop.release();
    if (!s->rows) return;
    if (f->ctx->stream != st && f->has_upload) CG_CUDA(cudaStreamWaitEvent(st, f->uploaded, 0));
    const unsigned grid = (unsigned)std::min<uint64_t>((s->rows + 7) / 8, (uint64_t)s->ctx->num_sms * 8);
    const int t = s->ctx->begin_timed(2, s->ctx->timing ? "K6 feature gather d" + std::to_string(f->dim) : std::string());
    // a shard a bf16x3 model has read keeps its split copy current from here;
    // with the split-only layout it is the only copy written
    const uint32_t sld = round_up(f->dim, 8);
    if (s->x_split_only && (!s->xs_hi.p || s->xs_ld != sld)) {
      const size_t n = std::max<uint64_t>(1, s->rows) * sld;
      s->xs_hi.alloc(n);
      s->xs_lo.alloc(n);
      s->xs_ld = sld;
      CG_CUDA(cudaMemsetAsync(s->xs_hi.p, 0, n * 2, st));  // zero padding columns
      CG_CUDA(cudaMemsetAsync(s->xs_lo.p, 0, n * 2, st));
    }
    const bool split = s->xs_hi.p && s->xs_ld == sld;
    float* xdst = (s->x_split_only && split) ? nullptr : s->x.p;
    auto* hi = split ? reinterpret_cast<__nv_bfloat16*>(s->xs_hi.p) : nullptr;
    auto* lo = split ? reinterpret_cast<__nv_bfloat16*>(s->xs_lo.p) : nullptr;
    if (f->dim % 4 == 0)
      gather_rows_kernel<4><<<grid, 256, 0, st>>>(f->x.p, f->dim, s->d_ext.p, s->rows, xdst, ld, hi, lo, s->xs_ld);
    else if (f->dim % 2 == 0)
      gather_rows_kernel<2><<<grid, 256, 0, st>>>(f->x.p, f->dim, s->d_ext.p, s->rows, xdst, ld, hi, lo, s->xs_ld);
    else
      gather_rows_kernel<1><<<grid, 256, 0, st>>>(f->x.p, f->dim, s->d_ext.p, s->rows, xdst, ld, hi, lo, s->xs_ld);
    if (split) s->xs_version = s->x_version;
    s->x_fp32_valid = xdst != nullptr;
    CG_CHECK_LAUNCH();
    s->ctx->end_timed(t);
    s->ctx->launches++;
    if (f->ctx->stream != st) {
      cudaEvent_t& ev = f->consumed[st];
      if (!ev) CG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      CG_CUDA(cudaEventRecord(ev, st));
    }
  });
}

// split_features (store.cpp:97-116): part-<s>/features.bin = the rows of the
// global FEA1 matrix named by partition s's node table, in node-table order.
// The reference seeks and reads one row per node record; here the matrix is
// read once (bulk, pinned), uploaded, and every partition's rows are gathered
// on the device and written back as FEA1 files.
int catgnn_split_features(catgnn_ctx ctx, catgnn_artifact a, const char* features, const char* out_dir,
                          uint32_t* files_written) {
  return guarded([&] {
    if (!ctx || !a || !features || !out_dir) throw ConfigError("null argument");
    CG_CUDA(cudaSetDevice(ctx->device));
    namespace fs = std::filesystem;
    const FeatureFile h = read_feature_header(features);
    const size_t total = h.rows * (size_t)h.dim;
    cudaStream_t st = ctx->stream;
    // the pinned buffer is also the D2H target of every partition's rows: size
    // it for the largest node table too (a table may repeat ids; the reference
    // writes one row per record, store.cpp:104-112)
    size_t max_part = 0;
    for (const auto& t : a->parts) max_part = std::max(max_part, t.ext.size() * (size_t)h.dim);
    float* pinned = nullptr;
    CG_CUDA(cudaMallocHost(&pinned, std::max<size_t>({1, total, max_part}) * 4));
    struct Pinned {
      float* p;
      ~Pinned() { cudaFreeHost(p); }
    } guard{pinned};
    {
      FILE* f = std::fopen(features, "rb");
      if (!f) throw DataError(std::string("cannot open feature file: ") + features);
      std::fseek(f, 20, SEEK_SET);
      const size_t got = total ? std::fread(pinned, 4, total, f) : 0;
      std::fclose(f);
      if (got != total) throw DataError(std::string("short feature read: ") + features);
    }
    DevBuf<float> src;
    src.alloc(std::max<size_t>(1, total));
    if (total) CG_CUDA(cudaMemcpyAsync(src.p, pinned, total * 4, cudaMemcpyHostToDevice, st));
    uint32_t written = 0;
    for (uint32_t s = 0; s < a->num_partitions; ++s) {
      const auto& ext = a->parts[s].ext;
      for (uint64_t id : ext)  // FeatureFileReader::read_row (store.cpp:55-58)
        if (id >= h.rows)
          throw DataError("feature row " + std::to_string(id) + " out of range in " + std::string(features));
      const uint64_t rows = ext.size();
      DevBuf<uint64_t> ids;
      DevBuf<float> dst;
      ids.alloc(std::max<uint64_t>(1, rows));
      dst.alloc(std::max<size_t>(1, rows * (size_t)h.dim));
      if (rows) {
        CG_CUDA(cudaMemcpyAsync(ids.p, ext.data(), rows * 8, cudaMemcpyHostToDevice, st));
        const unsigned grid = (unsigned)std::min<uint64_t>((rows + 7) / 8, (uint64_t)ctx->num_sms * 8);
        if (h.dim % 4 == 0)
          gather_rows_kernel<4><<<grid, 256, 0, st>>>(src.p, h.dim, ids.p, rows, dst.p, h.dim, nullptr, nullptr, 0);
        else if (h.dim % 2 == 0)
          gather_rows_kernel<2><<<grid, 256, 0, st>>>(src.p, h.dim, ids.p, rows, dst.p, h.dim, nullptr, nullptr, 0);
        else
          gather_rows_kernel<1><<<grid, 256, 0, st>>>(src.p, h.dim, ids.p, rows, dst.p, h.dim, nullptr, nullptr, 0);
        CG_CHECK_LAUNCH();
        ctx->launches++;
        CG_CUDA(cudaMemcpyAsync(pinned, dst.p, rows * (size_t)h.dim * 4, cudaMemcpyDeviceToHost, st));
      }
      CG_CUDA(cudaStreamSynchronize(st));
      const fs::path part_dir = fs::path(out_dir) / ("part-" + std::to_string(s));
      fs::create_directories(part_dir);
      const std::string out_path = (part_dir / "features.bin").string();
      FILE* f = std::fopen(out_path.c_str(), "wb");
      if (!f) throw DataError("cannot write feature file: " + out_path);
      const uint32_t dtype = 1;
      bool ok = std::fwrite("FEA1", 1, 4, f) == 4 && std::fwrite(&rows, 8, 1, f) == 1 &&
                std::fwrite(&h.dim, 4, 1, f) == 1 && std::fwrite(&dtype, 4, 1, f) == 1;
      const size_t n = rows * (size_t)h.dim;
      if (ok && n) ok = std::fwrite(pinned, 4, n, f) == n;
      ok = (std::fclose(f) == 0) && ok;
      if (!ok) throw DataError("short write: " + out_path);
      ++written;
    }
    if (files_written) *files_written = written;
  });
}

// Feature layout of a shard (no reference counterpart: a device-memory layout
// choice).  split_only = 1: catgnn_shard_gather_features writes only the
// bf16x3 (hi, lo) copy the GNN layers' tensor-core GEMMs read, not the fp32
// rows; calls that need fp32 features (SGC propagation, feature export, a
// model whose first layer is not on the bf16x3 path) fail with ConfigError
// until the next catgnn_shard_upload_features.
int catgnn_shard_set_feature_layout(catgnn_shard s, int split_only) {
  return guarded([&] {
    if (!s) throw ConfigError("null shard");
    CG_CUDA(cudaSetDevice(s->ctx->device));
    s->x_split_only = split_only != 0;
  });
}
