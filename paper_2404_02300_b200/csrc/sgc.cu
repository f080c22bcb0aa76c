// SGC path of the reference (/root/reference/proj/src/train.cpp:13-26, :74-198):
// softmax regression trained by mini-batch SGD over pre-propagated features,
// proportional model averaging and micro-F1 evaluation.
//
// sgc_train_kernel runs whole epochs for one replica per CTA: the parameters
// (W dim x C, b) stay in shared memory for the entire call, batches follow
// the host-generated libstdc++ shuffle order (seed_for(seed, epoch) +
// std::shuffle, train.cpp:111-113), and each batch does
//   phase A (warp per row): z = x W + b, P = softmax(z), P[y] -= 1, P /= count
//   phase B (thread per feature k): W[k,:] -= lr * sum_b x_b[k] P_b  (train.cpp:92,123)
//                                   b      -= lr * colsum(P)         (train.cpp:93,124)
// exactly the reference's update order (gradient with the pre-batch weights).
#include <algorithm>
#include <cstdio>

#include "sgc.hpp"

namespace catgnn {

namespace {

constexpr int kSgcThreads = 512;

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int m = 16; m; m >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, m));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int m = 16; m; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}

// Reduce-scatter of 32 per-lane partial vectors: afterwards lane L holds
// sum over lanes of z[L] in z[0].  31 shuffles for 32 values.
__device__ __forceinline__ float reduce_scatter32(float (&z)[32], int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool upper = lane & s;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      float send = upper ? z[i] : z[i + s];
      float keep = upper ? z[i + s] : z[i];
      z[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return z[0];
}

// Logits of one row for class chunk [c0, c0+32): returns z for class c0+lane.
__device__ __forceinline__ float row_logit_chunk(const float* __restrict__ x, uint32_t dim,
                                                 const float* W, uint32_t C, uint32_t c0,
                                                 int lane) {
  float z[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) z[i] = 0.f;
  const uint32_t cn = min(32u, C - c0);
  for (uint32_t k = lane; k < dim; k += 32) {
    const float xv = x[k];
    const float* wr = W + (size_t)k * C + c0;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < (int)cn) z[i] = fmaf(xv, wr[i], z[i]);
  }
  return reduce_scatter32(z, lane);
}

struct Replica {
  const float* x;
  uint32_t ld;
  const int32_t* labels;
  const uint32_t* order;  // n_epochs x n_train row ids (or the batch rows in gradient mode)
  uint64_t n_train;
  float* W;  // dim x C
  float* b;  // C
  float* gW; // gradient-only mode outputs
  float* gb;
};

template <int CT>
__global__ void __launch_bounds__(kSgcThreads) sgc_train_kernel(const Replica* __restrict__ reps,
                                                                uint32_t dim, uint32_t C, float lr,
                                                                uint32_t batch, uint32_t n_epochs,
                                                                int grad_only) {
  extern __shared__ float sm[];
  const Replica rep = reps[blockIdx.x];
  float* Ws = sm;                                  // dim*C
  float* bs = Ws + (size_t)dim * C;                // C (padded to 4)
  float* P = bs + ((C + 3) & ~3u);                 // batch*C
  uint32_t* rows = reinterpret_cast<uint32_t*>(P + (size_t)batch * C);  // batch
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  if (rep.n_train == 0) return;
  for (size_t i = tid; i < (size_t)dim * C; i += blockDim.x) Ws[i] = rep.W[i];
  for (uint32_t c = tid; c < C; c += blockDim.x) bs[c] = rep.b[c];
  __syncthreads();
  for (uint32_t ep = 0; ep < n_epochs; ++ep) {
    const uint32_t* ord = rep.order + (size_t)ep * rep.n_train;
    for (uint64_t start = 0; start < rep.n_train; start += batch) {
      const uint32_t cnt = (uint32_t)(batch < rep.n_train - start ? (uint64_t)batch : rep.n_train - start);
      for (uint32_t i = tid; i < cnt; i += blockDim.x) rows[i] = ord[start + i];
      __syncthreads();
      // phase A: probabilities minus one-hot, scaled by 1/count
      const float inv_cnt = 1.0f / (float)cnt;
      for (uint32_t bi = warp; bi < cnt; bi += nwarps) {
        const uint32_t row = rows[bi];
        const float* x = rep.x + (size_t)row * rep.ld;
        float z[CT];
        float m = -INFINITY;
#pragma unroll
        for (int t = 0; t < CT; ++t) {
          const uint32_t c0 = 32u * t;
          z[t] = -INFINITY;
          if (c0 < C) {
            float v = row_logit_chunk(x, dim, Ws, C, c0, lane);
            if (c0 + lane < C) z[t] = v + bs[c0 + lane];
          }
          m = fmaxf(m, z[t]);
        }
        m = warp_max(m);
        float s = 0.f;
#pragma unroll
        for (int t = 0; t < CT; ++t) {
          z[t] = (32u * t + lane < C) ? expf(z[t] - m) : 0.f;
          s += z[t];
        }
        s = warp_sum(s);
        const int y = rep.labels[row];
#pragma unroll
        for (int t = 0; t < CT; ++t) {
          const uint32_t c = 32u * t + lane;
          if (c < C) {
            float p = z[t] / s;
            if ((int)c == y) p -= 1.0f;
            P[(size_t)bi * C + c] = p * inv_cnt;
          }
        }
      }
      __syncthreads();
      // phase B: gradient and update; thread owns feature k
      for (uint32_t k = tid; k < dim; k += blockDim.x) {
        for (uint32_t c0 = 0; c0 < C; c0 += 32) {
          const uint32_t cn = min(32u, C - c0);
          float g[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) g[i] = 0.f;
          for (uint32_t bi = 0; bi < cnt; ++bi) {
            const float xv = rep.x[(size_t)rows[bi] * rep.ld + k];
            const float* pr = P + (size_t)bi * C + c0;
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (i < (int)cn) g[i] = fmaf(xv, pr[i], g[i]);
          }
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (i < (int)cn) {
              if (grad_only) rep.gW[(size_t)k * C + c0 + i] = g[i];
              else Ws[(size_t)k * C + c0 + i] -= lr * g[i];
            }
        }
      }
      for (uint32_t c = tid; c < C; c += blockDim.x) {
        float gbv = 0.f;
        for (uint32_t bi = 0; bi < cnt; ++bi) gbv += P[(size_t)bi * C + c];
        if (grad_only) rep.gb[c] = gbv;
        else bs[c] -= lr * gbv;
      }
      __syncthreads();
    }
  }
  if (!grad_only) {
    for (size_t i = tid; i < (size_t)dim * C; i += blockDim.x) rep.W[i] = Ws[i];
    for (uint32_t c = tid; c < C; c += blockDim.x) rep.b[c] = bs[c];
  }
}

// Shapes that do not fit one CTA's shared memory (dim*C + batch*C floats over
// 227 KB, e.g. the reference's default batch 512 with 128-d features and 172
// classes, or softmax_gradient over a whole train set) or with more than 256
// classes: the same algorithm and update order as sgc_train_kernel, with W/b
// updated in place in global memory and the batch's P and row ids in a
// per-replica global scratch slab.  __syncthreads orders the block's global
// writes exactly as it orders the shared-memory ones above.
__global__ void __launch_bounds__(kSgcThreads) sgc_train_global_kernel(const Replica* __restrict__ reps,
                                                                       float* scratch, size_t slab,
                                                                       uint32_t dim, uint32_t C, float lr,
                                                                       uint32_t batch, uint32_t n_epochs,
                                                                       int grad_only) {
  const Replica rep = reps[blockIdx.x];
  float* P = scratch + (size_t)blockIdx.x * slab;                      // batch*C
  uint32_t* rows = reinterpret_cast<uint32_t*>(P + (size_t)batch * C);  // batch
  float* W = rep.W;
  float* bv = rep.b;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  if (rep.n_train == 0) return;
  for (uint32_t ep = 0; ep < n_epochs; ++ep) {
    const uint32_t* ord = rep.order + (size_t)ep * rep.n_train;
    for (uint64_t start = 0; start < rep.n_train; start += batch) {
      const uint32_t cnt = (uint32_t)(batch < rep.n_train - start ? (uint64_t)batch : rep.n_train - start);
      for (uint32_t i = tid; i < cnt; i += blockDim.x) rows[i] = ord[start + i];
      __syncthreads();
      const float inv_cnt = 1.0f / (float)cnt;
      for (uint32_t bi = warp; bi < cnt; bi += nwarps) {
        const uint32_t row = rows[bi];
        const float* x = rep.x + (size_t)row * rep.ld;
        float* pr = P + (size_t)bi * C;
        float m = -INFINITY;
        for (uint32_t c0 = 0; c0 < C; c0 += 32) {  // logits, chunk by chunk
          const float v = row_logit_chunk(x, dim, W, C, c0, lane);
          if (c0 + lane < C) {
            pr[c0 + lane] = v + bv[c0 + lane];
            m = fmaxf(m, pr[c0 + lane]);
          }
        }
        m = warp_max(m);
        float s = 0.f;
        for (uint32_t c = lane; c < C; c += 32) {
          const float e = expf(pr[c] - m);
          pr[c] = e;
          s += e;
        }
        s = warp_sum(s);
        const int y = rep.labels[row];
        for (uint32_t c = lane; c < C; c += 32) {
          float p = pr[c] / s;
          if ((int)c == y) p -= 1.0f;
          pr[c] = p * inv_cnt;
        }
      }
      __syncthreads();
      for (uint32_t k = tid; k < dim; k += blockDim.x) {
        for (uint32_t c0 = 0; c0 < C; c0 += 32) {
          const uint32_t cn = min(32u, C - c0);
          float g[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) g[i] = 0.f;
          for (uint32_t bi = 0; bi < cnt; ++bi) {
            const float xv = rep.x[(size_t)rows[bi] * rep.ld + k];
            const float* pr = P + (size_t)bi * C + c0;
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (i < (int)cn) g[i] = fmaf(xv, pr[i], g[i]);
          }
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (i < (int)cn) {
              if (grad_only) rep.gW[(size_t)k * C + c0 + i] = g[i];
              else W[(size_t)k * C + c0 + i] -= lr * g[i];
            }
        }
      }
      for (uint32_t c = tid; c < C; c += blockDim.x) {
        float gbv = 0.f;
        for (uint32_t bi = 0; bi < cnt; ++bi) gbv += P[(size_t)bi * C + c];
        if (grad_only) rep.gb[c] = gbv;
        else bv[c] -= lr * gbv;
      }
      __syncthreads();
    }
  }
}

// Any class count (> 256): logits chunk by chunk with an online max / sum of
// exponentials, so nothing per row is stored; first-maximum argmax because the
// chunks are visited in increasing class order and only a strictly larger
// logit replaces the best.
__global__ void sgc_eval_any_kernel(const float* __restrict__ x, uint32_t ld, uint32_t dim,
                                    const float* __restrict__ W, const float* __restrict__ b, uint32_t C,
                                    const int32_t* __restrict__ labels, const uint32_t* __restrict__ mask,
                                    uint64_t n_mask, unsigned long long* correct, double* row_loss) {
  const int lane = threadIdx.x & 31;
  const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = wid; i < n_mask; i += nw) {
    const uint32_t row = mask[i];
    const float* xr = x + (size_t)row * ld;
    const int y = labels[row];
    float best = -INFINITY, s = 0.f, zy = 0.f;
    int bidx = 0x7fffffff;
    for (uint32_t c0 = 0; c0 < C; c0 += 32) {
      const float v = row_logit_chunk(xr, dim, W, C, c0, lane);
      if (c0 + lane < C) {
        const float z = v + b[c0 + lane];
        if (z > best) {
          s = s * expf(best - z) + 1.0f;  // rescale the running sum to the new maximum
          best = z;
          bidx = (int)(c0 + lane);
        } else {
          s += expf(z - best);
        }
        if ((int)(c0 + lane) == y) zy = z;
      }
    }
    float gbest = best;
    int gidx = bidx;
#pragma unroll
    for (int m = 16; m; m >>= 1) {
      float ob = __shfl_xor_sync(0xffffffffu, gbest, m);
      int oi = __shfl_xor_sync(0xffffffffu, gidx, m);
      if (ob > gbest || (ob == gbest && oi < gidx)) { gbest = ob; gidx = oi; }
    }
    if (row_loss) {
      const float ls = best == -INFINITY ? 0.f : s * expf(best - gbest);
      const float tot = warp_sum(ls);
      zy = warp_sum(zy);
      if (lane == 0) row_loss[i] = (double)gbest + log((double)tot) - (double)zy;
    }
    if (lane == 0 && correct && gidx == y) atomicAdd(correct, 1ull);
  }
}

// Per mask row: argmax (first maximum, like Eigen's maxCoeff) vs label, plus
// the row's cross-entropy for the loss hook.
template <int CT>
__global__ void sgc_eval_kernel(const float* __restrict__ x, uint32_t ld, uint32_t dim,
                                const float* __restrict__ W, const float* __restrict__ b, uint32_t C,
                                const int32_t* __restrict__ labels, const uint32_t* __restrict__ mask,
                                uint64_t n_mask, unsigned long long* correct, double* row_loss) {
  const int lane = threadIdx.x & 31;
  const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = wid; i < n_mask; i += nw) {
    const uint32_t row = mask[i];
    const float* xr = x + (size_t)row * ld;
    float z[CT];
    float best = -INFINITY;
    int bidx = 0x7fffffff;
#pragma unroll
    for (int t = 0; t < CT; ++t) {
      const uint32_t c0 = 32u * t;
      z[t] = -INFINITY;
      if (c0 < C) {
        float v = row_logit_chunk(xr, dim, W, C, c0, lane);
        if (c0 + lane < C) {
          z[t] = v + b[c0 + lane];
          if (z[t] > best) { best = z[t]; bidx = (int)(c0 + lane); }
        }
      }
    }
#pragma unroll
    for (int m = 16; m; m >>= 1) {
      float ob = __shfl_xor_sync(0xffffffffu, best, m);
      int oi = __shfl_xor_sync(0xffffffffu, bidx, m);
      if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
    }
    const int y = labels[row];
    if (row_loss) {
      float s = 0.f, zy = 0.f;
#pragma unroll
      for (int t = 0; t < CT; ++t) {
        const uint32_t c = 32u * t + lane;
        if (c < C) {
          s += expf(z[t] - best);
          if ((int)c == y) zy = z[t];
        }
      }
      s = warp_sum(s);
      zy = warp_sum(zy);
      if (lane == 0) row_loss[i] = (double)best + log((double)s) - (double)zy;
    }
    if (lane == 0 && correct && bidx == y) atomicAdd(correct, 1ull);
  }
}

__global__ void average_kernel(const float* const* __restrict__ src, const double* __restrict__ alpha,
                               uint32_t n, uint64_t count, float* __restrict__ out) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < count;
       j += (uint64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;  // model_average starts from zero params (train.cpp:164-169)
    for (uint32_t i = 0; i < n; ++i) acc += alpha[i] * (double)src[i][j];
    out[j] = (float)acc;
  }
}

// Replica pointers and weights passed by value (kernel parameters): no
// host-to-device staging, so averaging needs no host synchronisation and a
// step that ends with it can be enqueued (or graph-captured) back to back.
constexpr uint32_t kAvgByValue = 32;
struct AvgArgs {
  const float* src[kAvgByValue];
  double alpha[kAvgByValue];
};
__global__ void average_kernel_v(const AvgArgs a, uint32_t n, uint64_t count, float* __restrict__ out) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < count;
       j += (uint64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;  // same order and arithmetic as average_kernel
    for (uint32_t i = 0; i < n; ++i) acc += a.alpha[i] * (double)__ldg(a.src[i] + j);
    out[j] = (float)acc;
  }
}

size_t sgc_smem_bytes(uint32_t dim, uint32_t C, uint32_t batch) {
  return sizeof(float) * ((size_t)dim * C + ((C + 3) & ~3u) + (size_t)batch * C) +
         sizeof(uint32_t) * batch;
}

template <int CT>
void launch_train(const Replica* d_reps, uint32_t n, uint32_t dim, uint32_t C, float lr,
                  uint32_t batch, uint32_t n_epochs, int grad_only, size_t smem, cudaStream_t st) {
  auto fn = sgc_train_kernel<CT>;
  CG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  fn<<<n, kSgcThreads, smem, st>>>(d_reps, dim, C, lr, batch, n_epochs, grad_only);
  CG_CHECK_LAUNCH();
}

template <int CT>
void launch_eval(const float* x, uint32_t ld, uint32_t dim, const float* W, const float* b,
                 uint32_t C, const int32_t* labels, const uint32_t* mask, uint64_t n_mask,
                 unsigned long long* correct, double* row_loss, cudaStream_t st) {
  unsigned grid = (unsigned)std::min<uint64_t>((n_mask + 7) / 8, 148 * 16);
  sgc_eval_kernel<CT><<<std::max(1u, grid), 256, 0, st>>>(x, ld, dim, W, b, C, labels, mask, n_mask,
                                                         correct, row_loss);
  CG_CHECK_LAUNCH();
}

}  // namespace

void sgc_train(catgnn_ctx ctx, const std::vector<SgcReplicaHost>& reps, uint32_t dim, uint32_t C,
               float lr, uint32_t batch, uint32_t n_epochs, bool grad_only) {
  if (C == 0) throw ConfigError("class count must be >= 1");
  if (batch == 0) throw ConfigError("batch size must be >= 1");
  std::vector<Replica> h(reps.size());
  for (size_t i = 0; i < reps.size(); ++i)
    h[i] = Replica{reps[i].x, reps[i].ld, reps[i].labels, reps[i].order, reps[i].n_train,
                   reps[i].W, reps[i].b, reps[i].gW, reps[i].gb};
  Replica* d = ctx->scratch_buf<Replica>("sgc_reps", h.size());
  CG_CUDA(cudaMemcpyAsync(d, h.data(), h.size() * sizeof(Replica), cudaMemcpyHostToDevice, ctx->stream));
  const uint32_t n = (uint32_t)h.size();
  // a batch never holds more rows than the largest train set
  uint64_t max_rows = 1;
  for (const auto& r : reps) max_rows = std::max<uint64_t>(max_rows, r.n_train);
  const uint32_t eff_batch = (uint32_t)std::min<uint64_t>(batch, max_rows);
  const size_t smem = sgc_smem_bytes(dim, C, eff_batch);
  if (C <= 256 && smem <= 227 * 1024) {
    const int ct = (int)((C + 31) / 32);
    switch (ct) {
      case 1: launch_train<1>(d, n, dim, C, lr, eff_batch, n_epochs, grad_only, smem, ctx->stream); break;
      case 2: launch_train<2>(d, n, dim, C, lr, eff_batch, n_epochs, grad_only, smem, ctx->stream); break;
      case 3: case 4: launch_train<4>(d, n, dim, C, lr, eff_batch, n_epochs, grad_only, smem, ctx->stream); break;
      default: launch_train<8>(d, n, dim, C, lr, eff_batch, n_epochs, grad_only, smem, ctx->stream); break;
    }
  } else {
    // W/b stay where the caller put them (global); P + rows per replica in scratch
    const size_t slab = round_up64((uint64_t)eff_batch * C + eff_batch, 4);
    float* scratch = ctx->scratch_buf<float>("sgc_global_slab", slab * n);
    sgc_train_global_kernel<<<n, kSgcThreads, 0, ctx->stream>>>(d, scratch, slab, dim, C, lr, eff_batch,
                                                                 n_epochs, grad_only);
    CG_CHECK_LAUNCH();
  }
  ctx->launches++;
  CG_CUDA(cudaStreamSynchronize(ctx->stream));
}

void sgc_eval(catgnn_ctx ctx, const float* x, uint32_t ld, uint32_t dim, const float* W,
              const float* b, uint32_t C, const int32_t* labels, const uint32_t* mask,
              uint64_t n_mask, unsigned long long* correct, double* row_loss) {
  if (C == 0) throw ConfigError("class count must be >= 1");
  const int ct = (int)((C + 31) / 32);
  switch (ct) {
    case 1: launch_eval<1>(x, ld, dim, W, b, C, labels, mask, n_mask, correct, row_loss, ctx->stream); break;
    case 2: launch_eval<2>(x, ld, dim, W, b, C, labels, mask, n_mask, correct, row_loss, ctx->stream); break;
    case 3: case 4: launch_eval<4>(x, ld, dim, W, b, C, labels, mask, n_mask, correct, row_loss, ctx->stream); break;
    case 5: case 6: case 7: case 8:
      launch_eval<8>(x, ld, dim, W, b, C, labels, mask, n_mask, correct, row_loss, ctx->stream); break;
    default: {
      unsigned grid = (unsigned)std::min<uint64_t>((n_mask + 7) / 8, 148 * 16);
      sgc_eval_any_kernel<<<std::max(1u, grid), 256, 0, ctx->stream>>>(x, ld, dim, W, b, C, labels, mask,
                                                                       n_mask, correct, row_loss);
      CG_CHECK_LAUNCH();
    }
  }
  ctx->launches++;
}

void average_params(catgnn_ctx ctx, const std::vector<const float*>& d_src,
                    const std::vector<double>& alpha, uint64_t count, float* d_out) {
  const uint32_t n = (uint32_t)d_src.size();
  unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((count + 255) / 256, 148 * 8));
  if (n <= kAvgByValue) {
    AvgArgs a{};
    for (uint32_t i = 0; i < n; ++i) { a.src[i] = d_src[i]; a.alpha[i] = alpha[i]; }
    average_kernel_v<<<grid, 256, 0, ctx->stream>>>(a, n, count, d_out);
    CG_CHECK_LAUNCH();
    ctx->launches++;
    return;
  }
  const float** dp = ctx->scratch_buf<const float*>("avg_src", n);
  double* da = ctx->scratch_buf<double>("avg_alpha", n);
  CG_CUDA(cudaMemcpyAsync(dp, d_src.data(), n * sizeof(float*), cudaMemcpyHostToDevice, ctx->stream));
  CG_CUDA(cudaMemcpyAsync(da, alpha.data(), n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  average_kernel<<<grid, 256, 0, ctx->stream>>>(dp, da, n, count, d_out);
  CG_CHECK_LAUNCH();
  ctx->launches++;
  // the host vectors above must outlive the async copies
  CG_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace catgnn
