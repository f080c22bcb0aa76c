// Read-bandwidth probe for the roofline denominators bench.py reports beside
// MEASURED_PEAKS.json: streams a device buffer with 128-bit ld.global.cg
// loads (cached in L2 only), grid = 8 CTAs x 148 SMs.  A buffer well under the
// 126 MB L2 measures the L2 read rate that bounds K2's gathers on the
// reddit-shaped graph (69% L2 hit rate); a multi-GB buffer measures HBM read.
#include <algorithm>

#include "common.hpp"

namespace catgnn {
namespace {

__global__ void __launch_bounds__(512) read_probe_kernel(const float4* __restrict__ buf, uint64_t n4, int passes,
                                                         float* __restrict__ sink) {
  float acc = 0.f;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (int p = 0; p < passes; ++p) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += 4 * stride) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint64_t k = i + u * stride;
        v[u] = k < n4 ? __ldcg(buf + k) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
  }
  if (acc == 1.2345e-30f) sink[0] = acc;  // keeps the loads live, never taken
}

}  // namespace
}  // namespace catgnn

using namespace catgnn;

extern "C" int catgnn_probe_read_bandwidth(catgnn_ctx ctx, uint64_t bytes, int passes, double* gbs) {
  return guarded([&] {
    if (!ctx || !gbs || bytes < 16 || passes < 1) throw ConfigError("bad probe arguments");
    CG_CUDA(cudaSetDevice(ctx->device));
    const uint64_t n4 = bytes / 16;
    DevBuf<float4> buf;
    buf.alloc(n4);
    float* sink = ctx->scratch_buf<float>("probe_sink", 1);
    CG_CUDA(cudaMemsetAsync(buf.p, 0, n4 * 16, ctx->stream));
    const unsigned grid = (unsigned)ctx->num_sms * 4;
    read_probe_kernel<<<grid, 512, 0, ctx->stream>>>(buf.p, n4, 1, sink);  // warm (fills L2 when it fits)
    CG_CHECK_LAUNCH();
    cudaEvent_t a, b;
    CG_CUDA(cudaEventCreate(&a));
    CG_CUDA(cudaEventCreate(&b));
    CG_CUDA(cudaEventRecord(a, ctx->stream));
    read_probe_kernel<<<grid, 512, 0, ctx->stream>>>(buf.p, n4, passes, sink);
    CG_CUDA(cudaEventRecord(b, ctx->stream));
    CG_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    CG_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    ctx->launches += 2;
    *gbs = (double)n4 * 16.0 * passes / (ms * 1e-3) / 1e9;
  });
}
