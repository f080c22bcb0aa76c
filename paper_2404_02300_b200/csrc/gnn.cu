// GNN models of the north star (GCN-norm / SAGE-mean / GIN-sum), full-batch
// per partition: forward, loss, backward, optimizer, model averaging and the
// NCCL all-reduce of the averaged parameters.
//
// The reference trains SGC (propagation once, then a linear softmax model;
// proj/src/train.cpp) and has no GCN/SAGE/GIN; these layers follow its
// conventions: local CSR degrees, local rows in
// node-table order, loss = mean cross-entropy over owned train rows, alpha-
// weighted averaging of every parameter tensor (train.cpp:154-172), one "local
// iteration" = one full-batch step.  Parity is against the NumPy restatement in
// oracle/gnn_oracle.py (unpinned by the reference: it has no such models).
//
// Per layer, the aggregation runs at min(d_in, d_out):
//   GCN  transform-first: T = dinv*(H W^T)  [K3 epi: row scale]
//                         Z = dinv*(T_self + sum T_nbr) + b, H = relu(Z)   [K2]
//   GCN  aggregate-first: A = dinv*(dinv*H_self + sum dinv*H_nbr)          [K2 pre+post]
//                         Z = A W^T + b, H = relu(Z)                       [K3 epi]
//   SAGE aggregate-first: cat = [H | mean_N(H)] ; Z = cat [W_s|W_n]^T + b
//   SAGE transform-first: P = H [W_s;W_n]^T ; Z = P_s + mean_N(P_n) + b
//   GIN  (eps = 0): as GCN with plain sums (no normalisation)
// Backward uses the same CSR (A is symmetric, train.cpp:41-45 inserts both
// directions) with the source-row scale applied as K2's `pre`, and the
// weight gradients as split-K K3 GEMMs that read the row-major activations as
// MN-major tensor-core operands, and the input gradients read W itself as an
// MN-major operand (no transposes anywhere).
#include <nccl.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "artifact.hpp"
#include "comm.hpp"
#include "gemm.hpp"
#include "model.hpp"
#include "sgc.hpp"
#include "shard.hpp"

using namespace catgnn;

namespace catgnn {

namespace {



__device__ __forceinline__ float wsum(float v) {
#pragma unroll
  for (int m = 16; m; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}
__device__ __forceinline__ float wmax(float v) {
#pragma unroll
  for (int m = 16; m; m >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, m));
  return v;
}

// K4: softmax cross-entropy over the train rows.  dZ[r] = (softmax(z_r) - onehot)
// / n_train (rows not listed keep the caller's zeros); per-row loss for a
// deterministic reduction.  Warp per row, lanes over classes.  With rs, also
// writes dZs[r] = rs[r] * dZ[r] (the GCN source scale D^-1/2 of the next
// backward aggregation, so K2 needs no per-edge scale loads).  With dZh, that
// row (rs = 1 when null) is written instead as fp16, times hscale (2^k ~ n:
// |hscale * dZ| <= 1 stays in the fp16 normal range), the fp16 K2 pass's input.
__global__ void softmax_ce_kernel(const float* __restrict__ Z, uint32_t ldz, uint32_t C,
                                  const int32_t* __restrict__ labels, const uint32_t* __restrict__ rows,
                                  uint64_t n, float* __restrict__ dZ, uint32_t lddz,
                                  double* __restrict__ row_loss, const float* __restrict__ rs,
                                  float* __restrict__ dZs, __half* __restrict__ dZh, uint32_t ldh,
                                  float hscale) {
  const int lane = threadIdx.x & 31;
  const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const float inv_n = 1.0f / (float)n;
  for (uint64_t i = wid; i < n; i += nw) {
    const uint32_t r = rows[i];
    const float* z = Z + (size_t)r * ldz;
    const int y = labels[r];
    float m = -INFINITY;
    for (uint32_t c = lane; c < C; c += 32) m = fmaxf(m, z[c]);
    m = wmax(m);
    float s = 0.f, zy = 0.f;
    for (uint32_t c = lane; c < C; c += 32) {
      s += expf(z[c] - m);
      if ((int)c == y) zy = z[c];
    }
    s = wsum(s);
    zy = wsum(zy);
    const float sc = rs ? rs[r] : 0.f;
    for (uint32_t c = lane; c < C; c += 32) {
      float p = expf(z[c] - m) / s;
      if ((int)c == y) p -= 1.0f;
      if (dZ) dZ[(size_t)r * lddz + c] = p * inv_n;
      if (dZh) dZh[(size_t)r * ldh + c] = __float2half_rn((rs ? sc : 1.f) * (p * inv_n) * hscale);
      else if (rs) dZs[(size_t)r * lddz + c] = sc * (p * inv_n);
    }
    if (lane == 0) row_loss[i] = (double)m + log((double)s) - (double)zy;
  }
}

// Deterministic sum of n doubles (single block of 1024, 4 loads in flight per
// thread, fixed order per thread, tree).
__global__ void __launch_bounds__(1024) sum_doubles_kernel(const double* __restrict__ v, uint64_t n, double* out) {
  __shared__ double sh[1024];
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  const uint64_t T = blockDim.x;
  uint64_t i = threadIdx.x;
  for (; i + 3 * T < n; i += 4 * T) {
    a0 += v[i]; a1 += v[i + T]; a2 += v[i + 2 * T]; a3 += v[i + 3 * T];
  }
  for (; i < n; i += T) a0 += v[i];
  sh[threadIdx.x] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// Per-row argmax (first maximum) over role rows -> correct count.
__global__ void argmax_correct_kernel(const float* __restrict__ Z, uint32_t ldz, uint32_t C,
                                      const int32_t* __restrict__ labels, const uint32_t* __restrict__ rows,
                                      uint64_t n, unsigned long long* correct) {
  const int lane = threadIdx.x & 31;
  const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = wid; i < n; i += nw) {
    const uint32_t r = rows[i];
    const float* z = Z + (size_t)r * ldz;
    float best = -INFINITY;
    int bi = 0x7fffffff;
    for (uint32_t c = lane; c < C; c += 32)
      if (z[c] > best) { best = z[c]; bi = (int)c; }
#pragma unroll
    for (int m = 16; m; m >>= 1) {
      float ob = __shfl_xor_sync(0xffffffffu, best, m);
      int oi = __shfl_xor_sync(0xffffffffu, bi, m);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (lane == 0 && bi == labels[r]) atomicAdd(correct, 1ull);
  }
}

// Column sums of rows x width (ld % 4 == 0): each block reduces a slab of rows
// with float4 loads (tpr threads per row, 256/tpr rows in flight), partials
// per block, then a fixed-order reduce — deterministic.
// H16: X is fp16 rows holding rs[r] * x / scale (the fp16 K2 inputs); the sum
// is of x (the division by rs happens per row here, by scale in the reduce).
template <bool H16>
__device__ __forceinline__ float4 colsum_ld(const void* X, uint64_t r, uint32_t ld, uint32_t c,
                                            const float* __restrict__ rs) {
  if constexpr (H16) {
    const uint2 u = __ldg(reinterpret_cast<const uint2*>(static_cast<const __half*>(X) + r * ld) + c);
    const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
    const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
    const float f = rs ? 1.0f / __ldg(rs + r) : 1.0f;
    return make_float4(a.x * f, a.y * f, b.x * f, b.y * f);
  } else {
    return __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(X) + r * ld) + c);
  }
}
template <bool H16>
__global__ void colsum_partial_kernel(const void* __restrict__ X, uint32_t ld, uint64_t rows,
                                      uint32_t width, float* __restrict__ partial, const float* __restrict__ rsc) {
  __shared__ float4 red[256];
  const uint32_t w4 = (width + 3) / 4;
  const uint64_t per = (rows + gridDim.x - 1) / gridDim.x;
  const uint64_t r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
  const uint32_t tpr = min(w4, 256u), rpi = 256 / tpr;
  const uint32_t c4 = threadIdx.x % tpr, rs = threadIdx.x / tpr;
  for (uint32_t cb = 0; cb < w4; cb += tpr) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const uint32_t c = cb + c4;
    if (rs < rpi && c < w4) {
      // 4 independent row loads in flight per thread, combined in a fixed order
      float4 a1 = acc, a2 = acc, a3 = acc;
      uint64_t r = r0 + rs;
      for (; r + 3 * rpi < r1; r += 4 * rpi) {
        const float4 v0 = colsum_ld<H16>(X, r, ld, c, rsc), v1 = colsum_ld<H16>(X, r + rpi, ld, c, rsc);
        const float4 v2 = colsum_ld<H16>(X, r + 2 * rpi, ld, c, rsc), v3 = colsum_ld<H16>(X, r + 3 * rpi, ld, c, rsc);
        acc.x += v0.x; acc.y += v0.y; acc.z += v0.z; acc.w += v0.w;
        a1.x += v1.x; a1.y += v1.y; a1.z += v1.z; a1.w += v1.w;
        a2.x += v2.x; a2.y += v2.y; a2.z += v2.z; a2.w += v2.w;
        a3.x += v3.x; a3.y += v3.y; a3.z += v3.z; a3.w += v3.w;
      }
      for (; r < r1; r += rpi) {
        const float4 v = colsum_ld<H16>(X, r, ld, c, rsc);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      acc.x += a1.x + (a2.x + a3.x); acc.y += a1.y + (a2.y + a3.y);
      acc.z += a1.z + (a2.z + a3.z); acc.w += a1.w + (a2.w + a3.w);
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    if (rs == 0 && c < w4) {
      float4 s = red[c4];
      for (uint32_t k = 1; k < rpi; ++k) {
        const float4 v = red[k * tpr + c4];
        s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
      }
      float* dst = partial + (size_t)blockIdx.x * w4 * 4 + c * 4;
      dst[0] = s.x; dst[1] = s.y; dst[2] = s.z; dst[3] = s.w;
    }
    __syncthreads();
  }
}
// fp16 rows (rs[r] * x / scale, the fp16 K2 inputs): 16-byte loads of 8
// columns, tpr threads per row, 256/tpr rows in flight, 4 loads in flight per
// thread, fixed-order partials per block (deterministic); the per-row division
// by rs is one reciprocal per loaded vector.
__global__ void colsum_h16_kernel(const __half* __restrict__ X, uint32_t ld, uint64_t rows, uint32_t width,
                                  float* __restrict__ partial, const float* __restrict__ rsc) {
  __shared__ float4 red[256][2];
  const uint32_t w8 = (width + 7) / 8;
  const uint64_t per = (rows + gridDim.x - 1) / gridDim.x;
  const uint64_t r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
  const uint32_t tpr = min(w8, 256u), rpi = 256 / tpr;
  const uint32_t c8 = threadIdx.x % tpr, rs = threadIdx.x / tpr;
  auto ld8 = [&](uint64_t r, float4& a, float4& b) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(X + r * ld) + c8);
    const float f = rsc ? 1.0f / __ldg(rsc + r) : 1.0f;
    const float2 x0 = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
    const float2 x1 = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
    const float2 x2 = __half22float2(*reinterpret_cast<const __half2*>(&u.z));
    const float2 x3 = __half22float2(*reinterpret_cast<const __half2*>(&u.w));
    a = make_float4(x0.x * f, x0.y * f, x1.x * f, x1.y * f);
    b = make_float4(x2.x * f, x2.y * f, x3.x * f, x3.y * f);
  };
  float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), b0 = a0, a1 = a0, b1 = a0;
  if (rs < rpi && c8 < w8) {
    uint64_t r = r0 + rs;
    for (; r + rpi < r1; r += 2 * rpi) {
      float4 x, y, z, w;
      ld8(r, x, y);
      ld8(r + rpi, z, w);
      a0.x += x.x; a0.y += x.y; a0.z += x.z; a0.w += x.w; b0.x += y.x; b0.y += y.y; b0.z += y.z; b0.w += y.w;
      a1.x += z.x; a1.y += z.y; a1.z += z.z; a1.w += z.w; b1.x += w.x; b1.y += w.y; b1.z += w.z; b1.w += w.w;
    }
    if (r < r1) {
      float4 x, y;
      ld8(r, x, y);
      a0.x += x.x; a0.y += x.y; a0.z += x.z; a0.w += x.w; b0.x += y.x; b0.y += y.y; b0.z += y.z; b0.w += y.w;
    }
    a0.x += a1.x; a0.y += a1.y; a0.z += a1.z; a0.w += a1.w; b0.x += b1.x; b0.y += b1.y; b0.z += b1.z; b0.w += b1.w;
  }
  red[threadIdx.x][0] = a0;
  red[threadIdx.x][1] = b0;
  __syncthreads();
  if (rs == 0 && c8 < w8) {
    float4 sa = red[c8][0], sb = red[c8][1];
    for (uint32_t k = 1; k < rpi; ++k) {
      const float4 va = red[k * tpr + c8][0], vb = red[k * tpr + c8][1];
      sa.x += va.x; sa.y += va.y; sa.z += va.z; sa.w += va.w; sb.x += vb.x; sb.y += vb.y; sb.z += vb.z; sb.w += vb.w;
    }
    float* dst = partial + (size_t)blockIdx.x * w8 * 8 + c8 * 8;
    dst[0] = sa.x; dst[1] = sa.y; dst[2] = sa.z; dst[3] = sa.w; dst[4] = sb.x; dst[5] = sb.y; dst[6] = sb.z; dst[7] = sb.w;
  }
}

// One warp per column: lanes stride the block partials, then a fixed xor tree.
__global__ void colsum_reduce_kernel(const float* __restrict__ partial, uint32_t blocks, uint32_t width,
                                     uint32_t pstride, float* __restrict__ out, float scale) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= width) return;
  float acc = 0.f;
  for (uint32_t b = lane; b < blocks; b += 32) acc += partial[(size_t)b * pstride + c];
  acc = wsum(acc);
  if (lane == 0) out[c] = acc * scale;
}

// K5: fused optimizer over the flat parameter vector.
// The step count lives on the device (step[0] = completed updates, step[1] =
// block ticket), so a CUDA graph replaying train steps applies the right bias
// correction every replay: each block reads t = step[0] + 1, and the last
// block to finish advances step[0].
__global__ void adam_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                            float* __restrict__ v, uint64_t n, float lr, float b1, float b2, float eps,
                            double b1d, double b2d, unsigned long long* step) {
  __shared__ float bc[2];
  if (threadIdx.x == 0) {
    const double t = (double)(*(volatile unsigned long long*)step + 1);
    bc[0] = (float)(1.0 - pow(b1d, t));
    bc[1] = (float)(1.0 - pow(b2d, t));
  }
  __syncthreads();
  const float bc1 = bc[0], bc2 = bc[1];
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const float gi = g[i];
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    p[i] -= lr * (mi / bc1) / (sqrtf(vi / bc2) + eps);
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(step + 1, 1ull) == gridDim.x - 1) {  // every block has read step[0]
      step[0] += 1;
      step[1] = 0;
    }
  }
}
__global__ void sgd_kernel(float* __restrict__ p, const float* __restrict__ g, uint64_t n, float lr) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    p[i] -= lr * g[i];
}
__global__ void scale_kernel(float* __restrict__ p, uint64_t n, double a) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = (float)((double)p[i] * a);
}

// GEMM precision: 3xTF32 in both directions.  With plain TF32 operands the
// forward's ~1e-3 relative error flips a few ReLU masks, which moves the
// first-layer weight gradient by ~1% (scripts/diag_gnn.py); 3xTF32 keeps every
// intermediate within ~1e-6 of the f64 oracle.  Override with
// CATGNN_{FWD,BWD}_PRECISION=1 for plain TF32.
int env_precision(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return (v && (v[0] == '1' || v[0] == '3')) ? v[0] - '0' : dflt;
}
const int kBwdPrecision = env_precision("CATGNN_BWD_PRECISION", 3);
const int kFwdPrecision = env_precision("CATGNN_FWD_PRECISION", 3);

unsigned grid1d(uint64_t n) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148 * 16));
}

double unit_uniform(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }

}  // namespace
}  // namespace catgnn



namespace catgnn {
namespace {

void check_model(catgnn_model m) {
  if (!m) throw ConfigError("null model");
  CG_CUDA(cudaSetDevice(m->ctx->device));
}

// Named activation buffer; zero-filled whenever its shape changes so padding
// columns (never written by narrower producers) are exactly zero.
float* act(catgnn_ctx ctx, const std::string& name, uint64_t rows, uint32_t ld, bool zero) {
  float* p = ctx->scratch_buf<float>(name, std::max<uint64_t>(1, rows) * ld);
  auto sig = std::make_pair(rows, ld);
  auto it = ctx->act_shape.find(name);
  if (zero || it == ctx->act_shape.end() || it->second != sig) {
    CG_CUDA(cudaMemsetAsync(p, 0, std::max<uint64_t>(1, rows) * ld * 4, ctx->stream));
    ctx->act_shape[name] = sig;
  }
  return p;
}

// Row stride of a layer activation.  Narrow rows are padded to 16 floats
// (64 B) so every gathered row starts on a sector pair and the 44-wide class
// rows of the reddit shape become 48 (agg_kernel<2,8>).
constexpr uint32_t kPadNarrow = 16;
uint32_t act_width(uint32_t d) { return d < 128 ? round_up(d, kPadNarrow) : round_up(d, 4); }
const bool kSageInPlace = [] {  // A/B knob (CATGNN_SAGE_INPLACE=0: copy h into [h | mean])
  const char* v = std::getenv("CATGNN_SAGE_INPLACE");
  return v ? v[0] != '0' : true;
}();

void plan_layers(catgnn_model_s* M) {
  const auto& c = M->cfg;
  M->layers.clear();
  uint64_t off = 0;
  for (uint32_t l = 0; l < c.layers; ++l) {
    Layer L;
    L.d_in = l == 0 ? c.in_dim : c.hidden;
    L.d_out = l + 1 == c.layers ? c.classes : c.hidden;
    L.K_in = l == 0 ? round_up(L.d_in, 4) : act_width(L.d_in);  // layer 0 reads the shard's x
    L.D_out = act_width(L.d_out);
    L.ld_act = L.D_out;  // (64-float strides for 33-64-wide rows measured no faster: not wavefront bound)
    if (c.kind == CATGNN_MODEL_SAGE) {
      L.agg_first = L.d_in <= L.d_out;
      if (L.agg_first) {
        L.w_rows = L.d_out; L.w_cols = 2 * L.K_in;
        L.lw_rows = L.d_out; L.lw_cols = 2 * L.d_in;
        L.gemm_n = L.d_out;
      } else {
        L.w_rows = L.D_out + L.d_out; L.w_cols = L.K_in;
        L.lw_rows = 2 * L.d_out; L.lw_cols = L.d_in;
        L.gemm_n = L.D_out + L.d_out;
      }
    } else {
      L.agg_first = L.d_in < L.d_out;
      L.w_rows = L.d_out; L.w_cols = L.K_in;
      L.lw_rows = L.d_out; L.lw_cols = L.d_in;
      L.gemm_n = L.d_out;
    }
    L.off_w = off;
    off += (uint64_t)L.w_rows * L.w_cols;
    L.off_b = off;
    off += L.D_out;
    M->layers.push_back(L);
  }
  M->n_params = off;
  // A hidden layer followed by a SAGE aggregate-first layer writes its output
  // straight into that layer's [h | mean] buffer (left half): no row copy.
  for (size_t l = 0; l + 1 < M->layers.size(); ++l) {
    const Layer& N = M->layers[l + 1];
    M->layers[l].out_in_next_mid = c.kind == CATGNN_MODEL_SAGE && N.agg_first && N.K_in == M->layers[l].D_out &&
                                   kSageInPlace;
  }
}

// logical (row, col) of layer L -> internal index
uint64_t internal_w_index(const catgnn_model_s* M, const Layer& L, uint32_t r, uint32_t c) {
  uint32_t ir = r, ic = c;
  if (M->cfg.kind == CATGNN_MODEL_SAGE) {
    if (L.agg_first) ic = c < L.d_in ? c : L.K_in + (c - L.d_in);
    else ir = r < L.d_out ? r : L.D_out + (r - L.d_out);
  }
  return L.off_w + (uint64_t)ir * L.w_cols + ic;
}

uint64_t logical_count(const catgnn_model_s* M) {
  uint64_t n = 0;
  for (const auto& L : M->layers) n += (uint64_t)L.lw_rows * L.lw_cols + L.d_out;
  return n;
}

// logical flat <-> internal flat (host)
void logical_to_internal(const catgnn_model_s* M, const float* in, std::vector<float>& out) {
  out.assign(M->n_params, 0.f);
  uint64_t k = 0;
  for (const auto& L : M->layers) {
    for (uint32_t r = 0; r < L.lw_rows; ++r)
      for (uint32_t c = 0; c < L.lw_cols; ++c) out[internal_w_index(M, L, r, c)] = in[k++];
    for (uint32_t j = 0; j < L.d_out; ++j) out[L.off_b + j] = in[k++];
  }
}
void internal_to_logical(const catgnn_model_s* M, const std::vector<float>& in, float* out) {
  uint64_t k = 0;
  for (const auto& L : M->layers) {
    for (uint32_t r = 0; r < L.lw_rows; ++r)
      for (uint32_t c = 0; c < L.lw_cols; ++c) out[k++] = in[internal_w_index(M, L, r, c)];
    for (uint32_t j = 0; j < L.d_out; ++j) out[k++] = in[L.off_b + j];
  }
}


// Column sums of fp32 rows, or (Xh) of fp16 rows stored as rs[r] * x / scale.
void colsum(catgnn_ctx ctx, const float* X, uint32_t ld, uint64_t rows, uint32_t width, float* out,
            const __half* Xh = nullptr, const float* rs = nullptr, float scale = 1.0f) {
  if (ld % 4) throw ConfigError("column sum needs a row stride multiple of 4");
  const uint32_t blocks = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(1, (rows + 255) / 256), 592);
  const uint32_t pstride = round_up(width, 4);
  float* part = ctx->scratch_buf<float>("colsum_part", (size_t)blocks * pstride);
  if (Xh) {
    if (ld % 8) throw ConfigError("fp16 column sum needs a row stride multiple of 8");
    const uint32_t hb = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(1, (rows + 63) / 64), 1184);
    const uint32_t hs = round_up(width, 8);
    float* hpart = ctx->scratch_buf<float>("colsum_part_h", (size_t)hb * hs);
    colsum_h16_kernel<<<hb, 256, 0, ctx->stream>>>(Xh, ld, rows, width, hpart, rs);
    CG_CHECK_LAUNCH();
    colsum_reduce_kernel<<<(width + 7) / 8, 256, 0, ctx->stream>>>(hpart, hb, width, hs, out, scale);
  } else {
    colsum_partial_kernel<false><<<blocks, 256, 0, ctx->stream>>>(X, ld, rows, width, part, nullptr);
    CG_CHECK_LAUNCH();
    colsum_reduce_kernel<<<(width + 7) / 8, 256, 0, ctx->stream>>>(part, blocks, width, pstride, out, scale);
  }
  CG_CHECK_LAUNCH();
  ctx->launches += 2;
}

// Forward aggregation of a layer: post ⊙ (A + I)(pre ⊙ h) with
//   GCN  pre = post = (1+deg)^-1/2,  SGC  pre = 1, post = 1/(1+deg)  (train.cpp:60),
//   GIN  pre = post = 1.
// A is symmetric, so the backward is pre ⊙ (A + I)(post ⊙ g): bwd_pre / bwd_norm.
int agg_norm(const catgnn_model_s* M) {
  return M->cfg.kind == CATGNN_MODEL_GCN ? kNormGcn : M->cfg.kind == CATGNN_MODEL_SGC ? kNormSgc : kNormNone;
}
const float* bwd_pre(const catgnn_model_s* M, const catgnn_shard_s* S) {
  return M->cfg.kind == CATGNN_MODEL_GCN ? S->dinv.p : M->cfg.kind == CATGNN_MODEL_SGC ? S->inv_deg1.p : nullptr;
}
int bwd_norm(const catgnn_model_s* M) { return M->cfg.kind == CATGNN_MODEL_GCN ? kNormGcn : kNormNone; }

// bf16x3 activation: hi / lo bf16 rows (row stride ld, a multiple of 8)
struct Split {
  uint16_t* hi = nullptr;
  uint16_t* lo = nullptr;
  uint32_t ld = 0;
  explicit operator bool() const { return hi != nullptr; }
};
SplitOperand op16(const Split& s, bool mn) {
  return SplitOperand{reinterpret_cast<const __nv_bfloat16*>(s.hi), reinterpret_cast<const __nv_bfloat16*>(s.lo),
                      s.ld, mn};
}

struct Bufs {
  const float* in;  // H_{l-1}
  uint32_t in_ld;
  float* mid;       // T / A / cat / P
  uint32_t mid_ld;
  float* out;       // H_l (nullptr when H_l exists only as `split`)
  uint32_t out_ld;
  uint32_t* bits = nullptr;  // H_l > 0, one bit per column (ReLU layers): the backward's mask
  uint32_t bits_words = 0;
  Split in_split;  // bf16x3 layers: H_{l-1} (or x) as the GEMMs' pre-split operand
  Split split;     // H_l written by K2 as the next bf16x3 layer's operand
};

// bf16x3 GEMM path (default; CATGNN_GEMM_BF16X3=0: 3xTF32 everywhere): the
// transform-first GCN / GIN / SGC layers, whose GEMM operands are produced by
// K2 epilogues (H_l, dT_l), the features (split once per upload) or the
// weights (split per forward) — written straight as bf16 (hi, lo) pairs, so
// the GEMM has no conversion pass and runs kind::f16 MMAs (2x the tf32 rate,
// half the shared-memory bytes per MMA); ~2^-16 relative per product.
const bool kBf16x3 = [] {
  const char* v = std::getenv("CATGNN_GEMM_BF16X3");
  return v ? v[0] != '0' : true;
}();
bool bf_layer(const catgnn_model_s* M, size_t l) {
  const int k = M->cfg.kind;
  return kBf16x3 && l < M->layers.size() && !M->layers[l].agg_first &&
         (k == CATGNN_MODEL_GCN || k == CATGNN_MODEL_GIN || k == CATGNN_MODEL_SGC);
}

// Named bf16x3 activation pair, zero-filled whenever its shape changes; hi and
// lo are one allocation (lo follows hi), so a dead pair can host a rows x ld
// fp32 array (backward lean).
Split act16(catgnn_ctx ctx, const std::string& name, uint64_t rows, uint32_t ld) {
  Split s;
  s.ld = ld;
  const size_t n = std::max<uint64_t>(1, rows) * ld;
  s.hi = ctx->scratch_buf<uint16_t>(name + "_hl", 2 * n);
  s.lo = s.hi + n;
  auto sig = std::make_pair(rows, ld);
  auto it = ctx->act_shape.find(name + "_s");
  if (it == ctx->act_shape.end() || it->second != sig) {
    CG_CUDA(cudaMemsetAsync(s.hi, 0, n * 2, ctx->stream));
    CG_CUDA(cudaMemsetAsync(s.lo, 0, n * 2, ctx->stream));
    ctx->act_shape[name + "_s"] = sig;
  }
  return s;
}

// fp16 K2 inputs (default; CATGNN_ACT_F16=0: fp32).  The transform-first GCN
// layers gather the producer-scaled gradient s * dZ backward, and the last
// layer its GEMM output T = s (H W) forward, as fp16 rows: the K2 passes are
// bound by the L2 -> SM bytes of the gathered rows, which this halves.  The
// source scale s = D^-1/2 is applied by the producer before rounding, and the
// backward rows carry a power-of-two factor 2^k <= n_train (|dZ| <= 1/n_train)
// so gradients stay in the fp16 normal range; each element is rounded once
// (2^-11 relative) and summed in fp32: gradients move by ~2e-4 relative
// (north-star gate 2e-3).  Not for:
//  * a hidden layer's forward — its output feeds a ReLU, and rounding T flips
//    the masks of near-zero pre-activations (5 of 98 k on the small test graph
//    moved dW0 by 4e-3); the logits have no ReLU;
//  * GIN — sum aggregation grows with the degree (RMAT hubs: 54 k neighbours),
//    so neither activations nor gradients have a bounded range;
//  * SGC — pinned to the reference's f64 sgc_propagate at 1e-4.
const bool kActF16 = [] {
  const char* v = std::getenv("CATGNN_ACT_F16");
  return v ? v[0] != '0' : true;
}();
bool f16_bwd(const catgnn_model_s* M, size_t l) {
  return M->act_f16 && bf_layer(M, l) && M->cfg.kind == CATGNN_MODEL_GCN;
}
bool f16_fwd(const catgnn_model_s* M, size_t l) { return f16_bwd(M, l) && l + 1 == M->layers.size(); }
// A hidden GCN layer's forward as a guarded fp16 pass (aggregate.cu epilogue_row
// GUARD): K2 gathers fp16 T and flags every element whose pre-activation lies
// within 8 standard deviations of the rounding error of zero; those (~0.5%)
// are recomputed in fp32 from an fp32 copy of T, so every ReLU mask bit is the
// fp32 path's.  256-wide layers (CATGNN_ACT_F16_GUARD=0: fp32 forward).
const bool kGuardEnv = [] {
  const char* v = std::getenv("CATGNN_ACT_F16_GUARD");
  return v ? v[0] != '0' : true;
}();
bool f16_guard(const catgnn_model_s* M, size_t l) {
  return kGuardEnv && f16_bwd(M, l) && l + 1 < M->layers.size() && M->layers[l].D_out == 256;
}
// fp16 row stride: 32 / 64 halves (one 64- / 128-byte line) for narrow rows
uint32_t ld_h16(uint32_t w) { return w <= 32 ? 32 : w <= 64 ? 64 : round_up(w, 8); }
// (rows + 1) x ld: row `rows` stays zero (K2's idle-slot target)
__half* act_h(catgnn_ctx ctx, const std::string& name, uint64_t rows, uint32_t ld) {
  const size_t n = (rows + 1) * ld;
  __half* p = reinterpret_cast<__half*>(ctx->scratch_buf<uint16_t>(name, n));
  auto sig = std::make_pair(rows, ld);
  auto it = ctx->act_shape.find(name);
  if (it == ctx->act_shape.end() || it->second != sig) {  // padding columns are read (as zeros)
    CG_CUDA(cudaMemsetAsync(p, 0, n * 2, ctx->stream));
    ctx->act_shape[name] = sig;
  }
  return p;
}

// The shard's features as a bf16x3 pair, re-split when they changed.
Split shard_x_split(catgnn_shard_s* S) {
  const uint32_t ld = round_up(std::max<uint32_t>(S->dim, 1), 8);
  if (S->xs_version != S->x_version || S->xs_ld != ld || !S->xs_hi.p) {
    if (!S->x_fp32_valid) throw InternalError("bf16x3 feature copy is stale and the fp32 rows are not held");
    const size_t n = std::max<uint64_t>(1, S->rows) * ld;
    if (S->xs_ld != ld || !S->xs_hi.p) {
      S->xs_hi.alloc(n);
      S->xs_lo.alloc(n);
      S->xs_ld = ld;
    }
    split_bf16(S->ctx, S->x.p, S->ld, S->rows, S->dim, reinterpret_cast<__nv_bfloat16*>(S->xs_hi.p),
               reinterpret_cast<__nv_bfloat16*>(S->xs_lo.p), ld);
    S->xs_version = S->x_version;
  }
  return Split{S->xs_hi.p, S->xs_lo.p, ld};
}

// Weights of layer l as a bf16x3 pair (split from the fp32 master copy).
Split weight_split(catgnn_model_s* M, size_t l) {
  const Layer& L = M->layers[l];
  return Split{M->ws_hi.p + M->ws_off[l], M->ws_lo.p + M->ws_off[l], round_up(L.w_cols, 8)};
}
void split_weights(catgnn_model_s* M) {
  for (size_t l = 0; l < M->layers.size(); ++l) {
    if (!bf_layer(M, l)) continue;
    const Layer& L = M->layers[l];
    const Split w = weight_split(M, l);
    split_bf16(M->ctx, M->params.p + L.off_w, L.w_cols, L.w_rows, L.w_cols, reinterpret_cast<__nv_bfloat16*>(w.hi),
               reinterpret_cast<__nv_bfloat16*>(w.lo), w.ld);
  }
}

uint32_t* act_bits(catgnn_ctx ctx, const std::string& name, uint64_t rows, uint32_t words) {
  return ctx->scratch_buf<uint32_t>(name, std::max<uint64_t>(1, rows) * words);
}

std::string nm(const char* base, size_t l) { return std::string(base) + std::to_string(l); }

// Forward over the shard; returns the logits buffer (rows x D_out of the last layer).
// lean (train steps): the last layer's logits are computed for the train rows
// only (the loss reads nothing else; K2 over the shard's train-row view) —
// forward_backward and evaluation compute every row.
std::vector<Bufs> forward(catgnn_model_s* M, catgnn_shard_s* S, bool lean = false) {
  catgnn_ctx ctx = M->ctx;
  const uint64_t rows = S->rows;
  const bool gcn = M->cfg.kind == CATGNN_MODEL_GCN;
  const bool sage = M->cfg.kind == CATGNN_MODEL_SAGE;
  std::vector<Bufs> B(M->layers.size());
  const float* in = S->x.p;
  uint32_t in_ld = S->ld;
  const bool fresh = M->last_rows != rows;
  split_weights(M);
  M->h_split_only.assign(M->layers.size(), false);
  if (!S->x_fp32_valid && !bf_layer(M, 0))
    throw ConfigError("shard features are held as bf16x3 only; this model's first layer reads fp32 features");
  for (size_t l = 0; l < M->layers.size(); ++l) {
    const Layer& L = M->layers[l];
    const bool last = l + 1 == M->layers.size();
    Bufs& b = B[l];
    b.in = in;
    b.in_ld = in_ld;
    // output consumed only by the next (bf16x3) layer's GEMMs: written as a
    // bf16x3 pair, no fp32 copy (by K2 for a transform-first layer, by the
    // GEMM epilogue for an aggregate-first GCN / GIN layer)
    const bool h_split = !last && bf_layer(M, l + 1) && !L.out_in_next_mid &&
                         (!L.agg_first || M->cfg.kind != CATGNN_MODEL_SAGE);
    if (L.out_in_next_mid) {  // the next layer's [h | mean], left half
      b.out_ld = 2 * M->layers[l + 1].K_in;
      b.out = act(ctx, nm("mid", l + 1), rows, b.out_ld, fresh);
    } else if (!h_split) {
      b.out_ld = L.ld_act;
      b.out = act(ctx, nm("H", l), rows, b.out_ld, fresh);
    } else {
      b.out_ld = L.ld_act;
      b.out = nullptr;
    }
    if (!last) {
      b.bits_words = (L.D_out + 31) / 32;
      b.bits = act_bits(ctx, nm("Hbits", l), rows, b.bits_words);
    }
    const float* bias = M->params.p + L.off_b;
    if (sage && L.agg_first) {
      b.mid_ld = 2 * L.K_in;
      const bool inplace = l > 0 && M->layers[l - 1].out_in_next_mid;  // h already in the left half
      b.mid = act(ctx, nm("mid", l), rows, b.mid_ld, fresh && !inplace);
      if (!inplace) copy_rows(ctx, in, in_ld, b.mid, b.mid_ld, rows, L.K_in);
      AggArgs a;
      a.in = in; a.in_ld = in_ld; a.out = b.mid; a.out_ld = b.mid_ld; a.out_col = L.K_in;
      a.width = L.K_in; a.norm = kNormMean;
      aggregate(S, a);
      GemmEpi e; e.out = b.out; e.ld_out = b.out_ld; e.bias = bias; e.relu = !last;
      e.bits_out = b.bits; e.bits_words = b.bits_words;
      gemm_tn(ctx, b.mid, b.mid_ld, M->params.p + L.off_w, L.w_cols, (uint32_t)rows, L.d_out, L.w_cols, e, 1, kFwdPrecision);
    } else if (sage) {
      b.mid_ld = 2 * L.D_out;  // [P_s (D_out, padded) | P_n (d_out) | zero padding]
      b.mid = act(ctx, nm("mid", l), rows, b.mid_ld, fresh);
      GemmEpi e; e.out = b.mid; e.ld_out = b.mid_ld;
      gemm_tn(ctx, in, in_ld, M->params.p + L.off_w, L.w_cols, (uint32_t)rows, L.gemm_n, L.K_in, e, 1, kFwdPrecision);
      AggArgs a;
      a.in = b.mid; a.in_ld = b.mid_ld; a.in_col = L.D_out;
      a.out = b.out; a.out_ld = b.out_ld; a.width = L.D_out; a.norm = kNormMean;
      a.residual = b.mid; a.res_ld = b.mid_ld; a.res_col = 0;
      a.bias = bias; a.relu = !last;
      a.bits_out = b.bits; a.bits_words = b.bits_words;
      aggregate(S, a);
    } else if (L.agg_first) {  // GCN / GIN aggregate-first
      b.mid_ld = L.K_in;
      b.mid = act(ctx, nm("mid", l), rows, b.mid_ld, fresh);
      AggArgs a;
      a.in = in; a.in_ld = in_ld; a.out = b.mid; a.out_ld = b.mid_ld; a.width = L.K_in;
      a.self = 1; a.norm = agg_norm(M); a.pre = gcn ? S->dinv.p : nullptr;
      aggregate(S, a);
      GemmEpi e; e.out = b.out; e.ld_out = b.out_ld; e.bias = bias; e.relu = !last;
      e.bits_out = b.bits; e.bits_words = b.bits_words;
      if (!L.out_in_next_mid) e.store_cols = b.out_ld;  // zero padding (bias is zero-padded)
      if (h_split) {  // H_l straight into the next bf16x3 layer's operand pair
        b.split = act16(ctx, nm("Hs", l), rows, round_up(L.D_out, 8));
        e.out = nullptr;
        e.out_bhi = reinterpret_cast<__nv_bfloat16*>(b.split.hi);
        e.out_blo = reinterpret_cast<__nv_bfloat16*>(b.split.lo);
        e.ld_out = b.split.ld;
        e.store_cols = b.split.ld;
        M->h_split_only[l] = true;
      }
      gemm_tn(ctx, b.mid, b.mid_ld, M->params.p + L.off_w, L.w_cols, (uint32_t)rows, L.d_out, L.K_in, e, 1, kFwdPrecision);
    } else {  // GCN / GIN / SGC transform-first
      const bool h16 = f16_fwd(M, l);
      const bool guard = f16_guard(M, l);
      __half* mid_h = nullptr;
      float* smax = nullptr;
      __half* mid_lo = nullptr;
      GemmEpi e; e.rowscale = gcn ? S->dinv.p : nullptr;
      if (h16) {  // T as fp16 rows: the K2 pass's only input
        b.mid_ld = ld_h16(L.D_out);
        mid_h = act_h(ctx, nm("midh", l), rows, b.mid_ld);
        e.out_h = mid_h; e.ld_out = b.mid_ld;
        e.store_cols = round_up(L.D_out, 8);  // the vectors K2 reads, zero padding included
      } else if (guard) {  // fp16 T gathered, its rounding residual for the flagged elements, per-row max |T|
        b.mid_ld = ld_h16(L.D_out);
        mid_h = act_h(ctx, nm("midh", l), rows, b.mid_ld);
        mid_lo = act_h(ctx, nm("midl", l), rows, b.mid_ld);
        smax = ctx->scratch_buf<float>(nm("smax", l), rows + 1);
        CG_CUDA(cudaMemsetAsync(smax, 0, (rows + 1) * sizeof(float), ctx->stream));
        e.out_h = mid_h; e.out_hl = mid_lo; e.ld_out = b.mid_ld;
        e.rowmax = smax;
        e.store_cols = round_up(L.D_out, 8);
      } else {
        b.mid_ld = L.ld_act;
        b.mid = act(ctx, nm("mid", l), rows + 1, b.mid_ld, fresh);  // + zero row (K2's idle-slot target)
        e.out = b.mid; e.ld_out = b.mid_ld;
        e.store_cols = b.mid_ld;  // the padding of T is zero either way: staged stores for the ragged tail
      }
      if (bf_layer(M, l)) {
        // the layer input as a pre-split pair: the features, the previous K2's
        // bf16x3 output, or (previous layer on another path) a split of its fp32 rows
        if (l == 0) b.in_split = shard_x_split(S);
        else if (B[l - 1].split) b.in_split = B[l - 1].split;
        else {
          b.in_split = act16(ctx, nm("Hin", l), rows, round_up(L.K_in, 8));
          split_bf16(ctx, in, in_ld, rows, L.K_in, reinterpret_cast<__nv_bfloat16*>(b.in_split.hi),
                     reinterpret_cast<__nv_bfloat16*>(b.in_split.lo), b.in_split.ld);
        }
        gemm_bf16x3(ctx, op16(b.in_split, false), op16(weight_split(M, l), false), (uint32_t)rows, L.d_out, L.K_in,
                    e, 1);
      } else {
        gemm_tn(ctx, in, in_ld, M->params.p + L.off_w, L.w_cols, (uint32_t)rows, L.d_out, L.K_in, e, 1,
                kFwdPrecision);
      }
      AggArgs a;
      a.in = b.mid; a.in_ld = b.mid_ld; a.out = b.out; a.out_ld = b.out_ld; a.width = L.D_out;
      if (h16) { a.in = nullptr; a.in_h = mid_h; }
      else if (guard) {
        a.in = nullptr; a.in_h = mid_h;
        a.guard_smax = smax; a.guard_lo = mid_lo;
        a.guard_flags = act_bits(ctx, nm("Hflags", l), rows, b.bits_words);
      }
      else a.in_zero_row = true;
      a.self = 1; a.norm = agg_norm(M); a.bias = bias; a.relu = !last;
      a.bits_out = b.bits; a.bits_words = b.bits_words;
      if (h_split) {  // H_l is only the next bf16x3 layer's GEMM operand
        b.split = act16(ctx, nm("Hs", l), rows, round_up(L.D_out, 8));
        a.out = nullptr;
        a.out_hi = b.split.hi; a.out_lo = b.split.lo; a.out_s_ld = b.split.ld;
        M->h_split_only[l] = true;
      }
      catgnn_shard_s* V = (lean && last && bf_layer(M, l)) ? train_rows_view(S) : nullptr;
      if (V) {  // train rows only: the view's rows map back to the shard's
        a.row_map = V->row_map.p;
        a.zero_row = (int64_t)rows;
      }
      aggregate(V ? V : S, a);
    }
    in = b.out;
    in_ld = b.out_ld;
  }
  M->last_rows = rows;
  return B;
}

// Loss + backward; fills M->grads.  Returns the loss when want_loss.
// lean (train steps): a hidden layer's output kept only as a bf16x3 pair is
// dead once the next layer's weight gradient has read it, so that layer's
// fp32 dZ (written by the next layer's dX GEMM) takes its place — one rows x
// width activation less (a papers-scale GIN partition of 31 M rows then fits
// one B200); forward_backward keeps every activation for export.
double backward(catgnn_model_s* M, catgnn_shard_s* S, const std::vector<Bufs>& B, bool want_loss,
                bool lean = false) {
  catgnn_ctx ctx = M->ctx;
  cudaStream_t st = ctx->stream;
  const uint64_t rows = S->rows;
  const uint32_t R4 = round_up((uint32_t)std::max<uint64_t>(rows, 1), 4);
  const bool sage = M->cfg.kind == CATGNN_MODEL_SAGE;
  const size_t nl = M->layers.size();
  // K4: dZ of the last layer
  const Layer& LL = M->layers[nl - 1];
  // A transform-first GCN / GIN / SGC last layer's fp32 T (its K2 input) is dead
  // once the logits exist: K4 writes dZ over it (one rows x ld activation less —
  // 22 GB on a 31 M-row papers-scale partition)
  const bool reuse_t = !LL.agg_first && M->cfg.kind != CATGNN_MODEL_SAGE && B[nl - 1].mid &&
                       B[nl - 1].mid_ld == LL.ld_act;
  // with fp16 backward inputs the last layer's dZ exists only as the fp16 K2
  // input (its bias gradient sums those rows): no fp32 copy is written
  const bool last_h = f16_bwd(M, nl - 1);
  float* dZ = last_h ? nullptr : reuse_t ? B[nl - 1].mid : act(ctx, nm("dZ", nl - 1), rows, LL.ld_act, false);
  M->dz_last = dZ;
  M->dz_ptr.assign(nl, nullptr);
  M->dz_ptr[nl - 1] = dZ;
  if (dZ) CG_CUDA(cudaMemsetAsync(dZ, 0, std::max<uint64_t>(1, rows) * LL.ld_act * 4, st));
  const uint64_t ntr = S->h_train.size();
  // fp16 gradient rows carry 2^k <= n_train (|dZ| <= 1 / n_train)
  const float gscale = std::ldexp(1.0f, (int)std::floor(std::log2((double)std::max<uint64_t>(ntr, 1))));
  M->dz_f16.assign(nl, {});
  double loss = 0.0;
  double* row_loss = ctx->scratch_buf<double>("row_loss", std::max<uint64_t>(1, ntr));
  if (!M->loss_dev.p) M->loss_dev.alloc(1);
  double* loss_dev = M->loss_dev.p;
  CG_CUDA(cudaMemsetAsync(loss_dev, 0, 8, st));
  M->loss_rows = ntr;
  // GCN / SGC transform-first: the last layer's backward aggregation gathers
  // bwd_pre * dZ, produced here by K4 instead of per edge in K2
  float* dZs = nullptr;
  __half* dZh = nullptr;  // fp16 K2 input of the last layer's backward pass
  if (f16_bwd(M, nl - 1)) {
    const uint32_t ldh = ld_h16(LL.D_out);
    dZh = act_h(ctx, nm("dZh", nl - 1), rows, ldh);
    CG_CUDA(cudaMemsetAsync(dZh, 0, std::max<uint64_t>(1, rows) * ldh * 2, st));
  } else if (bwd_pre(M, S) && !LL.agg_first) {
    dZs = act(ctx, "dZs", rows, LL.ld_act, false);
    CG_CUDA(cudaMemsetAsync(dZs, 0, std::max<uint64_t>(1, rows) * LL.ld_act * 4, st));
  }
  if (ntr) {
    softmax_ce_kernel<<<grid1d(ntr * 32), 256, 0, st>>>(B[nl - 1].out, B[nl - 1].out_ld, LL.d_out,
                                                      S->labels.p, S->d_train.p, ntr, dZ, LL.ld_act, row_loss,
                                                      (dZs || dZh) ? bwd_pre(M, S) : nullptr, dZs, dZh,
                                                      ld_h16(LL.D_out), gscale);
    CG_CHECK_LAUNCH();
    sum_doubles_kernel<<<1, 1024, 0, st>>>(row_loss, ntr, loss_dev);
    CG_CHECK_LAUNCH();
    ctx->launches += 2;
  }
  uint32_t dZ_ld = LL.ld_act;
  // dZ of the current layer as fp16 rows (rs * dZ * scale): the K2 input
  __half* dzh = dZh;
  if (dZh) M->dz_f16[nl - 1] = {true, bwd_pre(M, S), gscale, ld_h16(LL.D_out)};
  for (size_t li = nl; li-- > 0;) {
    const Layer& L = M->layers[li];
    const Bufs& b = B[li];
    float* gW = M->grads.p + L.off_w;
    if (dzh) {
      const auto& z = M->dz_f16[li];
      colsum(ctx, nullptr, z.ld, rows, L.d_out, M->grads.p + L.off_b, dzh, z.rs, 1.0f / z.scale);
    } else {
      colsum(ctx, dZ, dZ_ld, rows, L.d_out, M->grads.p + L.off_b);
    }
    const bool need_dx = li > 0;
    // ReLU mask of the previous layer's output: its bits
    const uint32_t* hbits = li > 0 ? B[li - 1].bits : nullptr;
    const uint32_t hwords = li > 0 ? B[li - 1].bits_words : 0;
    // layer li-1's backward K2 gathers dZ_{li-1} as fp16 when it is an fp16
    // layer and this layer's dX GEMM produces it (bf16x3 transform-first)
    const bool prev_h = need_dx && f16_bwd(M, li - 1) && bf_layer(M, li);
    const bool onto_h = lean && need_dx && !prev_h && bf_layer(M, li) && M->h_split_only[li - 1] &&
                        B[li - 1].split && B[li - 1].split.ld == L.K_in;
    float* dZprev = need_dx && !prev_h
                        ? (onto_h ? reinterpret_cast<float*>(B[li - 1].split.hi) : act(ctx, nm("dZ", li - 1), rows, L.K_in, false))
                        : nullptr;
    if (need_dx) M->dz_ptr[li - 1] = dZprev;
    __half* dzh_prev = prev_h ? act_h(ctx, nm("dZh", li - 1), rows, ld_h16(L.K_in)) : nullptr;
    if (sage && L.agg_first) {
      // dW = dZ^T cat (both operands read MN-major in place)
      GemmEpi e; e.out = gW; e.ld_out = L.w_cols;
      gemm(ctx, GemmOperand{dZ, dZ_ld, true}, GemmOperand{b.mid, b.mid_ld, true}, L.d_out, L.w_cols,
           (uint32_t)rows, e, 0, kBwdPrecision);
      if (need_dx) {
        float* dcat = act(ctx, "dmid", rows, b.mid_ld, false);
        GemmEpi e2; e2.out = dcat; e2.ld_out = b.mid_ld;
        gemm(ctx, GemmOperand{dZ, dZ_ld, false}, GemmOperand{M->params.p + L.off_w, L.w_cols, true}, (uint32_t)rows,
             L.w_cols, L.d_out, e2, 1, kBwdPrecision);
        AggArgs a;
        a.in = dcat; a.in_ld = b.mid_ld; a.in_col = L.K_in; a.pre = S->inv_deg.p;
        a.out = dZprev; a.out_ld = L.K_in; a.width = L.K_in; a.norm = kNormNone;
        a.residual = dcat; a.res_ld = b.mid_ld; a.res_col = 0;
        a.mask_bits = hbits; a.mask_words = hwords;
        aggregate(S, a);
      }
    } else if (sage) {
      // dP = [dZ | sum_{i in N(j)} dZ_i / deg_i]
      float* dP = act(ctx, "dmid", rows, b.mid_ld, false);
      copy_rows(ctx, dZ, dZ_ld, dP, b.mid_ld, rows, L.D_out);
      AggArgs a;
      a.in = dZ; a.in_ld = dZ_ld; a.pre = S->inv_deg.p;
      a.out = dP; a.out_ld = b.mid_ld; a.out_col = L.D_out; a.width = L.D_out; a.norm = kNormNone;
      aggregate(S, a);
      // dW = dP^T H_prev (MN-major operands, no transposes)
      GemmEpi e; e.out = gW; e.ld_out = L.w_cols;
      gemm(ctx, GemmOperand{dP, b.mid_ld, true}, GemmOperand{b.in, b.in_ld, true}, L.gemm_n, L.w_cols,
           (uint32_t)rows, e, 0, kBwdPrecision);
      if (need_dx) {
        GemmEpi e2; e2.out = dZprev; e2.ld_out = L.K_in; e2.mask_bits = hbits; e2.mask_words = hwords;
        gemm(ctx, GemmOperand{dP, b.mid_ld, false}, GemmOperand{M->params.p + L.off_w, L.w_cols, true},
             (uint32_t)rows, L.w_cols, L.gemm_n, e2, 1, kBwdPrecision);
      }
    } else if (L.agg_first) {  // GCN / GIN
      GemmEpi e; e.out = gW; e.ld_out = L.w_cols;
      gemm(ctx, GemmOperand{dZ, dZ_ld, true}, GemmOperand{b.mid, b.mid_ld, true}, L.d_out, L.w_cols,
           (uint32_t)rows, e, 0, kBwdPrecision);
      if (need_dx) {
        float* dA = act(ctx, "dmid", rows, L.K_in, false);
        GemmEpi e2; e2.out = dA; e2.ld_out = L.K_in;
        gemm(ctx, GemmOperand{dZ, dZ_ld, false}, GemmOperand{M->params.p + L.off_w, L.w_cols, true}, (uint32_t)rows,
             L.w_cols, L.d_out, e2, 1, kBwdPrecision);
        AggArgs a;
        a.in = dA; a.in_ld = L.K_in; a.pre = bwd_pre(M, S); a.self = 1; a.norm = bwd_norm(M);
        a.out = dZprev; a.out_ld = L.K_in; a.width = L.K_in;
        a.mask_bits = hbits; a.mask_words = hwords;
        aggregate(S, a);
      }
    } else if (bf_layer(M, li)) {  // GCN / GIN / SGC transform-first, bf16x3 GEMMs
      // dT = pre (A+I)(post dZ) straight into a bf16x3 pair: both GEMMs' operand
      const Split dT = act16(ctx, "dTs", rows, round_up(L.ld_act, 8));
      AggArgs a;
      a.in = dZ; a.in_ld = dZ_ld; a.pre = bwd_pre(M, S); a.self = 1; a.norm = bwd_norm(M);
      if (li == nl - 1 && dZs) { a.in = dZs; a.pre = nullptr; }  // pre-scaled by K4
      if (dzh) {  // fp16 rows pre-scaled by their producer (K4 or the next layer's dX GEMM)
        const auto& z = M->dz_f16[li];
        a.in = nullptr; a.in_h = dzh; a.in_ld = z.ld; a.pre = nullptr; a.in_scale = 1.0f / z.scale;
      }
      a.out = nullptr; a.out_hi = dT.hi; a.out_lo = dT.lo; a.out_s_ld = dT.ld; a.width = L.D_out;
      // the last layer's gradient is non-zero on the train rows only: gather from
      // those neighbours (the shard's train-neighbour view; every row keeps its
      // full degree's post scale)
      catgnn_shard_s* V = (lean && li == nl - 1 && ntr) ? train_nbr_view(S) : nullptr;
      if (V) {
        a.zero_row = (int64_t)rows;
        if (a.norm == kNormGcn) a.post_arr = S->dinv.p;
        else if (a.norm != kNormNone) V = nullptr;  // (no per-row table for other norms)
      }
      aggregate(V ? V : S, a);
      GemmEpi e; e.out = gW; e.ld_out = L.w_cols;  // dW = dT^T H_{l-1} (both MN-major, in place)
      gemm_bf16x3(ctx, op16(dT, true), op16(b.in_split, true), L.d_out, L.w_cols, (uint32_t)rows, e, 0);
      if (need_dx) {  // dZ_{l-1} = mask (dT W)
        GemmEpi e2; e2.out = dZprev; e2.ld_out = L.K_in; e2.mask_bits = hbits; e2.mask_words = hwords;
        if (prev_h) {  // fp16 rows bwd_pre * dZ * 2^k: the input of layer li-1's K2 pass
          e2.out = nullptr; e2.out_h = dzh_prev; e2.ld_out = ld_h16(L.K_in);
          e2.store_cols = round_up(L.K_in, 8);
          e2.rowscale = bwd_pre(M, S); e2.out_scale = gscale;
          M->dz_f16[li - 1] = {true, bwd_pre(M, S), gscale, e2.ld_out};
        }
        gemm_bf16x3(ctx, op16(dT, false), op16(weight_split(M, li), true), (uint32_t)rows, L.w_cols, L.d_out, e2, 1);
      }
    } else {  // GCN / GIN transform-first
      float* dT = act(ctx, "dmid", rows, L.ld_act, false);
      AggArgs a;
      a.in = dZ; a.in_ld = dZ_ld; a.pre = bwd_pre(M, S); a.self = 1; a.norm = bwd_norm(M);
      if (li == nl - 1 && dZs) { a.in = dZs; a.pre = nullptr; }  // pre-scaled by K4
      a.out = dT; a.out_ld = L.ld_act; a.width = L.D_out;
      aggregate(S, a);
      GemmEpi e; e.out = gW; e.ld_out = L.w_cols;
      gemm(ctx, GemmOperand{dT, L.ld_act, true}, GemmOperand{b.in, b.in_ld, true}, L.d_out, L.w_cols,
           (uint32_t)rows, e, 0, kBwdPrecision);
      if (need_dx) {
        GemmEpi e2; e2.out = dZprev; e2.ld_out = L.K_in; e2.mask_bits = hbits; e2.mask_words = hwords;
        gemm(ctx, GemmOperand{dT, L.ld_act, false}, GemmOperand{M->params.p + L.off_w, L.w_cols, true},
             (uint32_t)rows, L.w_cols, L.d_out, e2, 1, kBwdPrecision);
      }
    }
    dZ = dZprev;
    dZ_ld = L.K_in;
    dzh = dzh_prev;
  }
  if (want_loss && ntr) {
    CG_CUDA(cudaMemcpyAsync(&loss, loss_dev, 8, cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaStreamSynchronize(st));
    loss /= (double)ntr;
    bool any_h = false;
    for (size_t l = 0; l < nl; ++l) any_h = any_h || f16_bwd(M, l);
    if (any_h && !std::isfinite(loss))
      throw DataError("non-finite loss with fp16 aggregation inputs (range +-65504 exceeded?); "
                      "CATGNN_ACT_F16=0 keeps them fp32");
  }
  return loss;
}

void optimizer_step(catgnn_model_s* M) {
  catgnn_ctx ctx = M->ctx;
  M->step++;
  const auto& c = M->cfg;
  if (c.optimizer == CATGNN_OPT_ADAM) {
    adam_kernel<<<grid1d(M->n_params), 256, 0, ctx->stream>>>(M->params.p, M->grads.p, M->m.p, M->v.p,
                                                             M->n_params, (float)c.lr, (float)c.beta1,
                                                             (float)c.beta2, (float)c.eps, c.beta1, c.beta2,
                                                             M->step_dev.p);
  } else {
    sgd_kernel<<<grid1d(M->n_params), 256, 0, ctx->stream>>>(M->params.p, M->grads.p, M->n_params, (float)c.lr);
  }
  CG_CHECK_LAUNCH();
  ctx->launches++;
}

void check_pair(catgnn_model m, catgnn_shard s) {
  check_model(m);
  if (!s) throw ConfigError("null shard");
  if (s->ctx != m->ctx) throw ConfigError("model and shard must share one context");
  if (s->dim != m->cfg.in_dim) throw DataError("shard feature width differs from the model input width");
  // a train label outside [0, classes) would silently drop its one-hot term in K4
  if (!s->h_train.empty() && (s->train_label_min < 0 || (uint32_t)s->train_label_max >= m->cfg.classes))
    throw DataError("train-row label outside [0, classes) of the model");
}

__global__ void loss_accum_kernel(const double* __restrict__ loss_sum, double weight, double* acc) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *acc += weight * *loss_sum;
}

}  // namespace

void model_train_step(catgnn_model m, catgnn_shard s) {
  check_pair(m, s);
  auto B = forward(m, s, true);
  backward(m, s, B, false, true);
  optimizer_step(m);
  m->last_shard = s;
}

void model_weighted_sum(const std::vector<catgnn_model>& src, const std::vector<double>& alpha,
                        catgnn_model dst) {
  check_model(dst);
  if (src.empty() || src.size() != alpha.size()) throw DataError("model averaging needs one weight per replica");
  std::vector<const float*> ptrs(src.size());
  for (size_t i = 0; i < src.size(); ++i) {
    check_model(src[i]);
    if (src[i]->n_params != dst->n_params) throw DataError("model shapes differ across replicas");
    if (src[i]->ctx->device != dst->ctx->device) throw ConfigError("models are on different devices");
    dst->ctx->wait_for(src[i]->ctx);  // replicas trained on other contexts' streams finish first
    ptrs[i] = src[i]->params.p;
  }
  float* tmp = dst->ctx->scratch_buf<float>("avg_tmp", dst->n_params);
  average_params(dst->ctx, ptrs, alpha, dst->n_params, tmp);
  CG_CUDA(cudaMemcpyAsync(dst->params.p, tmp, dst->n_params * 4, cudaMemcpyDeviceToDevice, dst->ctx->stream));
}

void model_accumulate_loss(catgnn_model m, double weight, double* acc) {
  check_model(m);
  if (!m->loss_dev.p || m->loss_rows == 0) return;
  loss_accum_kernel<<<1, 32, 0, m->ctx->stream>>>(m->loss_dev.p, weight / (double)m->loss_rows, acc);
  CG_CHECK_LAUNCH();
  m->ctx->launches++;
}

}  // namespace catgnn


extern "C" {

int catgnn_model_create(catgnn_ctx ctx, const catgnn_model_config* cfg, catgnn_model* out) {
  return guarded([&] {
    if (!ctx || !cfg || !out) throw ConfigError("null argument");
    CG_CUDA(cudaSetDevice(ctx->device));
    if (cfg->kind != CATGNN_MODEL_GCN && cfg->kind != CATGNN_MODEL_SAGE && cfg->kind != CATGNN_MODEL_GIN &&
        cfg->kind != CATGNN_MODEL_SGC)
      throw ConfigError("unknown model kind");
    if (cfg->layers < 1 || cfg->in_dim < 1 || cfg->classes < 1 || (cfg->layers > 1 && cfg->hidden < 1))
      throw ConfigError("model needs >= 1 layer and positive widths");
    if (cfg->optimizer != CATGNN_OPT_SGD && cfg->optimizer != CATGNN_OPT_ADAM)
      throw ConfigError("unknown optimizer");
    auto M = std::make_unique<catgnn_model_s>();
    M->ctx = ctx;
    M->cfg = *cfg;
    M->act_f16 = kActF16;
    ctx_retain(ctx);
    plan_layers(M.get());
    M->params.alloc(M->n_params);
    M->grads.alloc(M->n_params);
    {  // bf16x3 weight copies (layers on the bf16x3 path only)
      uint64_t ws = 0;
      M->ws_off.assign(M->layers.size(), 0);
      for (size_t l = 0; l < M->layers.size(); ++l) {
        M->ws_off[l] = ws;
        if (bf_layer(M.get(), l)) ws += (uint64_t)M->layers[l].w_rows * round_up(M->layers[l].w_cols, 8);
      }
      M->ws_hi.alloc(std::max<uint64_t>(1, ws));
      M->ws_lo.alloc(std::max<uint64_t>(1, ws));
    }
    M->m.alloc(M->n_params);
    M->v.alloc(M->n_params);
    CG_CUDA(cudaMemsetAsync(M->grads.p, 0, M->n_params * 4, ctx->stream));
    CG_CUDA(cudaMemsetAsync(M->m.p, 0, M->n_params * 4, ctx->stream));
    CG_CUDA(cudaMemsetAsync(M->v.p, 0, M->n_params * 4, ctx->stream));
    M->step_dev.alloc(2);
    CG_CUDA(cudaMemsetAsync(M->step_dev.p, 0, 2 * sizeof(unsigned long long), ctx->stream));
    // Glorot-uniform init: W[i] = (2u-1)*sqrt(6/(d_in+d_out)), u from
    // splitmix64(seed_for(seed, layer) + i) over the logical row-major index;
    // biases zero.  The SGC kind is the reference's model and is
    // zero-initialised like it (zero_params, train.cpp:67-72).
    std::vector<float> logical(logical_count(M.get()), 0.f);
    uint64_t k = 0;
    for (size_t l = 0; l < M->layers.size() && cfg->kind != CATGNN_MODEL_SGC; ++l) {
      const Layer& L = M->layers[l];
      const double a = std::sqrt(6.0 / (double)(L.d_in + L.d_out));
      const uint64_t base = seed_for(cfg->seed, l);
      const uint64_t nw = (uint64_t)L.lw_rows * L.lw_cols;
      for (uint64_t i = 0; i < nw; ++i)
        logical[k++] = (float)((2.0 * unit_uniform(mix64(base + i)) - 1.0) * a);
      k += L.d_out;
    }
    std::vector<float> internal;
    logical_to_internal(M.get(), logical.data(), internal);
    CG_CUDA(cudaMemcpyAsync(M->params.p, internal.data(), M->n_params * 4, cudaMemcpyHostToDevice, ctx->stream));
    CG_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = M.release();
  });
}

int catgnn_model_set_act_f16(catgnn_model m, int on) {
  return guarded([&] {
    check_model(m);
    m->act_f16 = on != 0;
  });
}

int catgnn_model_destroy(catgnn_model m) {
  return guarded([&] {
    if (!m) return;
    catgnn_ctx c = m->ctx;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    delete m;
    ctx_release(c);
  });
}

uint64_t catgnn_model_num_params(catgnn_model m) { return m ? logical_count(m) : 0; }

int catgnn_model_layer_shape(catgnn_model m, uint32_t layer, uint32_t* w_rows, uint32_t* w_cols,
                             uint64_t* offset_w, uint64_t* offset_b) {
  return guarded([&] {
    check_model(m);
    if (layer >= m->layers.size()) throw ConfigError("layer index out of range");
    uint64_t off = 0;
    for (uint32_t l = 0; l < layer; ++l)
      off += (uint64_t)m->layers[l].lw_rows * m->layers[l].lw_cols + m->layers[l].d_out;
    const Layer& L = m->layers[layer];
    if (w_rows) *w_rows = L.lw_rows;
    if (w_cols) *w_cols = L.lw_cols;
    if (offset_w) *offset_w = off;
    if (offset_b) *offset_b = off + (uint64_t)L.lw_rows * L.lw_cols;
  });
}

static void export_flat(catgnn_model m, const float* dev, float* out) {
  std::vector<float> h(m->n_params);
  CG_CUDA(cudaMemcpyAsync(h.data(), dev, m->n_params * 4, cudaMemcpyDeviceToHost, m->ctx->stream));
  CG_CUDA(cudaStreamSynchronize(m->ctx->stream));
  internal_to_logical(m, h, out);
}

int catgnn_model_get_params(catgnn_model m, float* out) {
  return guarded([&] {
    check_model(m);
    export_flat(m, m->params.p, out);
  });
}

int catgnn_model_get_grads(catgnn_model m, float* out) {
  return guarded([&] {
    check_model(m);
    export_flat(m, m->grads.p, out);
  });
}

int catgnn_model_set_params(catgnn_model m, const float* in) {
  return guarded([&] {
    check_model(m);
    std::vector<float> internal;
    logical_to_internal(m, in, internal);
    CG_CUDA(cudaMemcpyAsync(m->params.p, internal.data(), m->n_params * 4, cudaMemcpyHostToDevice, m->ctx->stream));
    CG_CUDA(cudaStreamSynchronize(m->ctx->stream));
  });
}

int catgnn_model_copy_params(catgnn_model dst, catgnn_model src) {
  return guarded([&] {
    check_model(dst);
    check_model(src);
    if (dst->n_params != src->n_params) throw DataError("model shapes differ across replicas");
    if (dst->ctx->device != src->ctx->device) throw ConfigError("models are on different devices");
    dst->ctx->wait_for(src->ctx);  // src's pending updates first (contexts on other streams)
    CG_CUDA(cudaMemcpyAsync(dst->params.p, src->params.p, dst->n_params * 4, cudaMemcpyDeviceToDevice,
                            dst->ctx->stream));
  });
}

int catgnn_model_forward_backward(catgnn_model m, catgnn_shard s, double* loss) {
  return guarded([&] {
    check_pair(m, s);
    auto B = forward(m, s);
    double l = backward(m, s, B, loss != nullptr);
    if (loss) *loss = l;
    m->last_shard = s;
  });
}

int catgnn_model_train_step(catgnn_model m, catgnn_shard s, double* loss) {
  return guarded([&] {
    check_pair(m, s);
    auto B = forward(m, s, true);
    double l = backward(m, s, B, loss != nullptr, true);
    optimizer_step(m);
    if (loss) *loss = l;
    m->last_shard = s;
  });
}

// Loss of the model's last train step (mean CE over its train rows), read
// back now: a caller training several replicas per step issues every
// train_step without a host sync and reads the losses once at the end.
int catgnn_model_last_loss(catgnn_model m, double* loss) {
  return guarded([&] {
    check_model(m);
    if (!loss) throw ConfigError("null argument");
    *loss = 0.0;
    if (!m->loss_dev.p || m->loss_rows == 0) return;
    double sum = 0.0;
    CG_CUDA(cudaMemcpyAsync(&sum, m->loss_dev.p, 8, cudaMemcpyDeviceToHost, m->ctx->stream));
    CG_CUDA(cudaStreamSynchronize(m->ctx->stream));
    *loss = sum / (double)m->loss_rows;
  });
}

// Asynchronous form: enqueues the D2H copy of the last step's loss sum into
// host_sum (pinned memory; capturable) and returns its train-row count, so
// the mean is *host_sum / *rows once the context's stream has synchronised.
int catgnn_model_last_loss_async(catgnn_model m, double* host_sum, uint64_t* rows) {
  return guarded([&] {
    check_model(m);
    if (!host_sum || !rows) throw ConfigError("null argument");
    *rows = m->loss_rows;
    if (!m->loss_dev.p || m->loss_rows == 0) {
      *host_sum = 0.0;
      return;
    }
    CG_CUDA(cudaMemcpyAsync(host_sum, m->loss_dev.p, 8, cudaMemcpyDeviceToHost, m->ctx->stream));
  });
}

int catgnn_model_forward(catgnn_model m, catgnn_shard s, float* logits, int role, double* f1) {
  return guarded([&] {
    check_pair(m, s);
    auto B = forward(m, s);
    m->last_shard = s;
    catgnn_ctx ctx = m->ctx;
    const Layer& LL = m->layers.back();
    if (logits && s->rows)
      CG_CUDA(cudaMemcpy2DAsync(logits, LL.d_out * 4, B.back().out, B.back().out_ld * 4, LL.d_out * 4, s->rows,
                                cudaMemcpyDeviceToHost, ctx->stream));
    if (f1) {
      const uint32_t* rows = role == 1 ? s->d_train.p : role == 2 ? s->d_val.p : s->d_test.p;
      const uint64_t n = role == 1 ? s->h_train.size() : role == 2 ? s->h_val.size() : s->h_test.size();
      if (role < 1 || role > 3) throw ConfigError("role must be 1, 2 or 3");
      if (n == 0) throw DataError("evaluation mask is empty");
      auto* cnt = ctx->scratch_buf<unsigned long long>("eval_cnt", 1);
      CG_CUDA(cudaMemsetAsync(cnt, 0, 8, ctx->stream));
      argmax_correct_kernel<<<grid1d(n * 32), 256, 0, ctx->stream>>>(B.back().out, B.back().out_ld, LL.d_out,
                                                                     s->labels.p, rows, n, cnt);
      CG_CHECK_LAUNCH();
      ctx->launches++;
      unsigned long long h = 0;
      CG_CUDA(cudaMemcpyAsync(&h, cnt, 8, cudaMemcpyDeviceToHost, ctx->stream));
      CG_CUDA(cudaStreamSynchronize(ctx->stream));
      // micro-F1 from pooled counts (train.cpp:189-197) == accuracy
      const double tp = (double)h, miss = (double)(n - h);
      *f1 = (2 * tp + 2 * miss) == 0 ? 0.0 : 2 * tp / (2 * tp + 2 * miss);
    }
    CG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int catgnn_model_export(catgnn_model m, uint32_t layer, int what, float* out, uint32_t* width) {
  return guarded([&] {
    check_model(m);
    if (layer >= m->layers.size()) throw ConfigError("layer index out of range");
    catgnn_shard s = m->last_shard;
    if (!s) throw ConfigError("no forward pass has run");
    const Layer& L = m->layers[layer];
    const float* src = nullptr;
    uint32_t ld = 0, w = L.d_out;
    if (what == 0 && layer < m->h_split_only.size() && m->h_split_only[layer]) {
      // H_l kept only as the bf16x3 pair: export hi + lo
      const uint32_t sld = round_up(L.D_out, 8);
      const uint16_t* hi = m->ctx->scratch_buf<uint16_t>(nm("Hs", layer) + "_hl", 1);
      const uint16_t* lo = hi + std::max<uint64_t>(1, s->rows) * sld;  // act16: lo follows hi
      if (width) *width = w;
      if (out && s->rows) {
        std::vector<uint16_t> h(s->rows * (size_t)sld), lw(s->rows * (size_t)sld);
        CG_CUDA(cudaMemcpyAsync(h.data(), hi, h.size() * 2, cudaMemcpyDeviceToHost, m->ctx->stream));
        CG_CUDA(cudaMemcpyAsync(lw.data(), lo, lw.size() * 2, cudaMemcpyDeviceToHost, m->ctx->stream));
        CG_CUDA(cudaStreamSynchronize(m->ctx->stream));
        auto f = [](uint16_t v) { uint32_t u = (uint32_t)v << 16; float x; std::memcpy(&x, &u, 4); return x; };
        for (uint64_t r = 0; r < s->rows; ++r)
          for (uint32_t c = 0; c < w; ++c) out[r * w + c] = f(h[r * sld + c]) + f(lw[r * sld + c]);
      }
      return;
    }
    if (what == 0 && L.out_in_next_mid) {
      src = m->ctx->scratch_buf<float>(nm("mid", layer + 1), 1);
      ld = 2 * m->layers[layer + 1].K_in;
    } else if (what == 0) {
      src = m->ctx->scratch_buf<float>(nm("H", layer), 1);
      ld = L.ld_act;
    }
    else if (what == 2 && layer < m->dz_f16.size() && m->dz_f16[layer].on) {
      // dZ_l held only as fp16 rows rs[r] * dZ * scale
      const auto& z = m->dz_f16[layer];
      const uint16_t* h = m->ctx->scratch_buf<uint16_t>(nm("dZh", layer), 1);
      if (width) *width = w;
      if (out && s->rows) {
        std::vector<__half> hv(s->rows * (size_t)z.ld);
        std::vector<float> rs(z.rs ? s->rows : 0);
        CG_CUDA(cudaMemcpyAsync(hv.data(), h, hv.size() * 2, cudaMemcpyDeviceToHost, m->ctx->stream));
        if (z.rs) CG_CUDA(cudaMemcpyAsync(rs.data(), z.rs, rs.size() * 4, cudaMemcpyDeviceToHost, m->ctx->stream));
        CG_CUDA(cudaStreamSynchronize(m->ctx->stream));
        for (uint64_t r = 0; r < s->rows; ++r)
          for (uint32_t c = 0; c < w; ++c)
            out[r * w + c] = __half2float(hv[r * z.ld + c]) / ((z.rs ? rs[r] : 1.0f) * z.scale);
      }
      return;
    }
    else if (what == 2) {
      src = (layer < m->dz_ptr.size() && m->dz_ptr[layer]) ? m->dz_ptr[layer]
                                                           : m->ctx->scratch_buf<float>(nm("dZ", layer), 1);
      ld = L.ld_act;
    }
    else throw ConfigError("export: what must be 0 (H) or 2 (dZ)");
    if (width) *width = w;
    if (out && s->rows)
      CG_CUDA(cudaMemcpy2DAsync(out, w * 4, src, ld * 4, w * 4, s->rows, cudaMemcpyDeviceToHost, m->ctx->stream));
    CG_CUDA(cudaStreamSynchronize(m->ctx->stream));
  });
}

int catgnn_model_average(uint32_t n, const catgnn_model* src, const uint64_t* train_counts, catgnn_model dst) {
  return guarded([&] {
    check_model(dst);
    if (n == 0) throw DataError("model averaging needs one training count per replica");
    std::vector<double> alpha(n);
    {
      uint64_t total = 0;
      for (uint32_t i = 0; i < n; ++i) total += train_counts[i];
      if (total == 0) throw DataError("model averaging requires a nonzero training-node count");
      double partial = 0;
      for (uint32_t i = 0; i + 1 < n; ++i) {
        alpha[i] = (double)train_counts[i] / (double)total;
        partial += alpha[i];
      }
      alpha[n - 1] = 1.0 - partial;
    }
    model_weighted_sum(std::vector<catgnn_model>(src, src + n), alpha, dst);
  });
}

// A rank's share of the model average across ranks: dst = sum_i alpha_i src_i
// with the GLOBAL sync_weights of its partitions (a rank whose partitions hold
// no train rows contributes zeros, as the reference weights them by 0).
int catgnn_model_weighted_sum(uint32_t n, const catgnn_model* src, const double* alpha, catgnn_model dst) {
  return guarded([&] {
    if (n == 0 || !src || !alpha) throw DataError("model averaging needs one weight per replica");
    model_weighted_sum(std::vector<catgnn_model>(src, src + n), std::vector<double>(alpha, alpha + n), dst);
  });
}

int catgnn_model_scale(catgnn_model m, double alpha) {
  return guarded([&] {
    check_model(m);
    scale_kernel<<<grid1d(m->n_params), 256, 0, m->ctx->stream>>>(m->params.p, m->n_params, alpha);
    CG_CHECK_LAUNCH();
    m->ctx->launches++;
  });
}

int catgnn_comm_unique_id(char id[128]) {
  return guarded([&] {
    ncclUniqueId u;
    if (ncclGetUniqueId(&u) != ncclSuccess) throw InternalError("ncclGetUniqueId failed");
    static_assert(sizeof(u) == 128, "NCCL unique id size");
    std::memcpy(id, &u, 128);
  });
}

int catgnn_comm_create(catgnn_ctx ctx, int nranks, int rank, const char id[128], catgnn_comm* out) {
  return guarded([&] {
    if (!ctx || !out) throw ConfigError("null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) throw ConfigError("bad rank / world size");
    CG_CUDA(cudaSetDevice(ctx->device));
    auto c = std::make_unique<catgnn_comm_s>();
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    ncclResult_t r = ncclCommInitRank(&c->comm, nranks, u, rank);
    if (r != ncclSuccess) throw InternalError(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    c->ctx = ctx;
    c->nranks = nranks;
    c->rank = rank;
    *out = c.release();
  });
}

int catgnn_comm_destroy(catgnn_comm c) {
  return guarded([&] {
    if (!c) return;
    if (c->comm) ncclCommDestroy(c->comm);
    delete c;
  });
}

// C1: sum over ranks of the (alpha-prescaled) parameters, in place, on the
// context stream (NCCL over NVLink / NVSwitch).
int catgnn_model_allreduce(catgnn_model m, catgnn_comm c) {
  return guarded([&] {
    check_model(m);
    if (!c) throw ConfigError("null communicator");
    ncclResult_t r = ncclAllReduce(m->params.p, m->params.p, m->n_params, ncclFloat32, ncclSum, c->comm,
                                   m->ctx->stream);
    if (r != ncclSuccess) throw InternalError(std::string("ncclAllReduce: ") + ncclGetErrorString(r));
  });
}

}  // extern "C"
