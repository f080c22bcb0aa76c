// Stable LSD radix sort of (uint32 key, uint32 value) pairs over the low
// `bits` key bits — K1's sort (csr.cu: the expanded (row, neighbour) entries
// by row, which must keep edge order inside a row, train.cpp:41-45).
//
// One pass per 8-bit digit, three kernels per pass, all HBM-streaming:
//   histogram  per 4096-item tile, the count of every digit (shared-memory
//              atomics), stored digit-major: counts[d * tiles + t];
//   scan       exclusive prefix of the digit-major counts = each (digit, tile)
//              bucket's first output position (a reduce / scan / add chain);
//   scatter    each tile reloads its items, ranks them stably inside the tile
//              (8 warps own consecutive 512-item runs; per 32-item round a
//              warp groups equal digits with match.any, its rank is the number
//              of equal-digit lanes below it plus the warp's running count,
//              warps offset by the per-warp digit histograms of the warps
//              before them) and writes key and value to bucket base + rank.
// Stability: inside a tile the order is (warp, round, lane) = input order;
// across tiles the digit-major scan orders tiles.  Passes ping-pong between
// the caller's two buffer pairs; the result lands in (keys_out, vals_out).
#include <algorithm>

#include "radix.hpp"

namespace catgnn {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 16;                    // per thread
constexpr int kTile = kThreads * kItems;      // 4096
constexpr int kRadix = 256;
constexpr int kRunPerWarp = kTile / kWarps;   // 512 consecutive items per warp

__global__ void __launch_bounds__(kThreads) radix_hist_kernel(const uint32_t* __restrict__ keys, uint64_t n,
                                                             int shift, uint32_t tiles, uint32_t* __restrict__ counts) {
  __shared__ uint32_t h[kRadix];
  for (uint32_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    h[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t base = (uint64_t)t * kTile;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const uint64_t k = base + (uint64_t)i * kThreads + threadIdx.x;
      if (k < n) atomicAdd(&h[(__ldg(keys + k) >> shift) & (kRadix - 1)], 1u);
    }
    __syncthreads();
    counts[(uint64_t)threadIdx.x * tiles + t] = h[threadIdx.x];
    __syncthreads();
  }
}

// --- exclusive scan of a uint32 array (length L) -------------------------
// block b sums items [b*kTile, (b+1)*kTile)
__global__ void __launch_bounds__(kThreads) scan_reduce_kernel(const uint32_t* __restrict__ in, uint64_t L,
                                                              uint32_t* __restrict__ sums) {
  __shared__ uint32_t w[kWarps];
  const uint64_t base = (uint64_t)blockIdx.x * kTile;
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t k = base + (uint64_t)i * kThreads + threadIdx.x;
    if (k < L) s += in[k];
  }
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int i = 0; i < kWarps; ++i) t += w[i];
    sums[blockIdx.x] = t;
  }
}
// single block: exclusive scan of the block sums in place (sequential chunks per thread)
__global__ void __launch_bounds__(1024) scan_sums_kernel(uint32_t* __restrict__ sums, uint32_t nb) {
  __shared__ uint32_t part[1024];
  const uint32_t per = (nb + 1023) / 1024;
  const uint32_t b0 = threadIdx.x * per, b1 = min(nb, b0 + per);
  uint32_t s = 0;
  for (uint32_t i = b0; i < b1; ++i) s += sums[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {  // inclusive Hillis-Steele over the 1024 chunk sums
    const uint32_t v = threadIdx.x >= (uint32_t)off ? part[threadIdx.x - off] : 0u;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  uint32_t run = threadIdx.x ? part[threadIdx.x - 1] : 0u;
  for (uint32_t i = b0; i < b1; ++i) {
    const uint32_t v = sums[i];
    sums[i] = run;
    run += v;
  }
}
// block b: exclusive scan of its tile, offset by the scanned block sum
__global__ void __launch_bounds__(kThreads) scan_apply_kernel(const uint32_t* __restrict__ in, uint64_t L,
                                                             const uint32_t* __restrict__ sums,
                                                             uint32_t* __restrict__ out) {
  __shared__ uint32_t w[kWarps];
  // thread t owns the consecutive items [t*kItems, (t+1)*kItems) of the tile
  const uint64_t base = (uint64_t)blockIdx.x * kTile + (uint64_t)threadIdx.x * kItems;
  uint32_t v[kItems];
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    v[i] = base + i < L ? in[base + i] : 0u;
    s += v[i];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = s;
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, m);
    if (lane >= m) incl += y;
  }
  if (lane == 31) w[warp] = incl;
  __syncthreads();
  uint32_t wb = 0;
  for (int i = 0; i < warp; ++i) wb += w[i];
  uint32_t run = sums[blockIdx.x] + wb + incl - s;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    if (base + i < L) out[base + i] = run;
    run += v[i];
  }
}

__global__ void __launch_bounds__(kThreads) radix_scatter_kernel(const uint32_t* __restrict__ keys,
                                                                const uint32_t* __restrict__ vals, uint64_t n,
                                                                int shift, uint32_t tiles,
                                                                const uint32_t* __restrict__ offs,
                                                                uint32_t* __restrict__ keys_out,
                                                                uint32_t* __restrict__ vals_out) {
  __shared__ uint32_t whist[kWarps][kRadix];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  for (uint32_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    for (int i = threadIdx.x; i < kWarps * kRadix; i += kThreads) (&whist[0][0])[i] = 0;
    __syncthreads();
    const uint64_t base = (uint64_t)t * kTile + (uint64_t)warp * kRunPerWarp;
    uint32_t k[kItems], v[kItems];
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
      const uint64_t idx = base + (uint64_t)r * 32 + lane;
      const bool ok = idx < n;
      k[r] = ok ? __ldg(keys + idx) : 0u;
      v[r] = ok ? __ldg(vals + idx) : 0u;
      const uint32_t d = (k[r] >> shift) & (kRadix - 1);
      const uint32_t act = __ballot_sync(0xffffffffu, ok);
      const uint32_t peers = __match_any_sync(0xffffffffu, ok ? d : 0x1000u) & act;
      if (ok && (peers & lt) == 0) whist[warp][d] += __popc(peers);  // lowest equal-digit lane
      __syncwarp();
    }
    __syncthreads();
    {  // per digit: bucket base of this tile + the counts of the warps before
      const int d = threadIdx.x;
      uint32_t run = offs[(uint64_t)d * tiles + t];
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        const uint32_t c = whist[w][d];
        whist[w][d] = run;
        run += c;
      }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
      const uint64_t idx = base + (uint64_t)r * 32 + lane;
      const bool ok = idx < n;
      const uint32_t d = (k[r] >> shift) & (kRadix - 1);
      const uint32_t act = __ballot_sync(0xffffffffu, ok);
      const uint32_t peers = __match_any_sync(0xffffffffu, ok ? d : 0x1000u) & act;
      const uint32_t pos = ok ? whist[warp][d] + __popc(peers & lt) : 0u;
      __syncwarp();
      if (ok) {
        keys_out[pos] = k[r];
        vals_out[pos] = v[r];
        if ((peers & lt) == 0) whist[warp][d] += __popc(peers);
      }
      __syncwarp();
    }
    __syncthreads();
  }
}

unsigned grid_tiles(uint64_t tiles, int sms) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(tiles, (uint64_t)sms * 8));
}

void exclusive_scan_u32(catgnn_ctx ctx, const uint32_t* in, uint64_t L, uint32_t* out) {
  const uint64_t nb = (L + kTile - 1) / kTile;
  if (nb > 0xffffffffull) throw ConfigError("radix sort: scan too long");
  uint32_t* sums = ctx->scratch_buf<uint32_t>("radix_scan_sums", std::max<uint64_t>(1, nb));
  scan_reduce_kernel<<<(unsigned)nb, kThreads, 0, ctx->stream>>>(in, L, sums);
  CG_CHECK_LAUNCH();
  scan_sums_kernel<<<1, 1024, 0, ctx->stream>>>(sums, (uint32_t)nb);
  CG_CHECK_LAUNCH();
  scan_apply_kernel<<<(unsigned)nb, kThreads, 0, ctx->stream>>>(in, L, sums, out);
  CG_CHECK_LAUNCH();
  ctx->launches += 3;
}

}  // namespace

void radix_sort_pairs(catgnn_ctx ctx, uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt,
                      uint64_t n, int bits, uint32_t** keys_result, uint32_t** vals_result) {
  *keys_result = keys;
  *vals_result = vals;
  if (n == 0 || bits <= 0) return;
  if (n > 0xffffffffull) throw ConfigError("radix sort: more than 2^32 items");
  const uint64_t tiles64 = (n + kTile - 1) / kTile;
  const uint32_t tiles = (uint32_t)tiles64;
  const uint64_t L = (uint64_t)kRadix * tiles;
  uint32_t* counts = ctx->scratch_buf<uint32_t>("radix_counts", L);
  uint32_t* offs = ctx->scratch_buf<uint32_t>("radix_offs", L);
  const unsigned g = grid_tiles(tiles, ctx->num_sms);
  uint32_t *ki = keys, *vi = vals, *ko = keys_alt, *vo = vals_alt;
  for (int shift = 0; shift < bits; shift += 8) {
    radix_hist_kernel<<<g, kThreads, 0, ctx->stream>>>(ki, n, shift, tiles, counts);
    CG_CHECK_LAUNCH();
    exclusive_scan_u32(ctx, counts, L, offs);
    radix_scatter_kernel<<<g, kThreads, 0, ctx->stream>>>(ki, vi, n, shift, tiles, offs, ko, vo);
    CG_CHECK_LAUNCH();
    ctx->launches += 2;
    std::swap(ki, ko);
    std::swap(vi, vo);
  }
  *keys_result = ki;
  *vals_result = vi;
}

}  // namespace catgnn
