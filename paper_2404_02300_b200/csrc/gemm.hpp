#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.hpp"

namespace catgnn {

// Fused epilogue of K3, applied per output element (row, col):
//   v = acc; v *= rowscale[row] (cols >= scale_col_begin); v += bias[col];
//   v = relu(v); v = bit(mask_bits, row, col) ? v : 0;  v *= out_scale;
//   out[row][out_col+col] = v   (or out_h[...] = fp16(v))
//   bits_out: bit (row, col) = v > 0 (the ReLU mask of this output's backward)
struct GemmEpi {
  float* out = nullptr;
  uint32_t ld_out = 0, out_col = 0;
  const float* rowscale = nullptr;
  uint32_t scale_col_begin = 0;
  const float* bias = nullptr;
  int relu = 0;
  const uint32_t* mask_bits = nullptr;  // 32-bit words per row: mask_words
  uint32_t mask_words = 0;
  uint32_t* bits_out = nullptr;
  uint32_t bits_words = 0;
  // columns [N, store_cols) of the output rows are padding the caller wants
  // written with the epilogue of a zero accumulator (zero when bias is
  // zero-padded): lets a ragged last 32-column chunk (N = 41 classes) use the
  // staged, line-coalesced stores; 0 = write only [0, N)
  uint32_t store_cols = 0;
  // fp16 output rows instead of `out` (ld_out / out_col in halves, multiples
  // of 8): the input of an fp16 K2 pass; out_scale (a power of two) keeps
  // small values (gradients) in the fp16 normal range
  // (out and out_h may both be set: the staged path writes both copies)
  __half* out_h = nullptr;
  uint32_t ld_h = 0;  // out_h row stride in halves when both outputs are set (0: ld_out)
  __half* out_hl = nullptr;  // with out_h: fp16 (v - fp16(v)) * 2^11, same layout (hi + lo * 2^-11 ~ v to 2^-22)
  // bf16x3 pair output (hi = bf16(v), lo = bf16(v - hi); row stride ld_h or
  // ld_out): the next bf16x3 GEMM's pre-split operand, written directly
  __nv_bfloat16* out_bhi = nullptr;
  __nv_bfloat16* out_blo = nullptr;
  float out_scale = 1.0f;
  // per output row: max |v| over its columns, merged with atomicMax on the
  // float bits (caller zero-fills; order-independent, so deterministic)
  float* rowmax = nullptr;
  float* partial = nullptr;  // internal (split-K workspace)
};

// C[M x N] = A[M x K] . B[N x K]^T with A (row stride lda) and B (row stride
// ldb) K-major fp32 device matrices.  split_k = 0 picks a split automatically
// (deterministic reduction in split order).  precision 1 = TF32 (inputs
// truncated to 10 mantissa bits), 3 = 3xTF32 (hi*hi + hi*lo + lo*hi, ~fp32).
// Operand of K3: row-major fp32 with row stride ld.  K-major: [M or N rows][K];
// MN-major: [K rows][M or N] (read in place by the tensor core, no transpose).
struct GemmOperand {
  const float* ptr = nullptr;
  uint32_t ld = 0;
  bool mn_major = false;
};

void gemm(catgnn_ctx ctx, GemmOperand a, GemmOperand b, uint32_t M, uint32_t N, uint32_t K, const GemmEpi& epi,
          uint32_t split_k = 1, int precision = 1);

// bf16x3 operand: x = hi + lo with hi = bf16(x), lo = bf16(x - hi) (~16
// significant bits, relative error ~2^-17), row-major with row stride ld
// (multiple of 8 elements).  K-major / MN-major as GemmOperand.
struct SplitOperand {
  const __nv_bfloat16* hi = nullptr;
  const __nv_bfloat16* lo = nullptr;
  uint32_t ld = 0;
  bool mn_major = false;
};

// C = A . B^T on pre-split operands: lo*hi + hi*lo + hi*hi on the tcgen05
// kind::f16 tensor cores (fp32 accumulation in TMEM), no conversion pass in
// the GEMM; same epilogue / split-K as gemm().
void gemm_bf16x3(catgnn_ctx ctx, SplitOperand a, SplitOperand b, uint32_t M, uint32_t N, uint32_t K,
                 const GemmEpi& epi, uint32_t split_k = 1);

// fp32 rows x cols (row stride ld_in) -> (hi, lo) rows x ld_out; columns
// [cols, ld_out) are written as zeros.
void split_bf16(catgnn_ctx ctx, const float* in, uint32_t ld_in, uint64_t rows, uint32_t cols, __nv_bfloat16* hi,
                __nv_bfloat16* lo, uint32_t ld_out);

void gemm_tn(catgnn_ctx ctx, const float* A, uint32_t lda, const float* B, uint32_t ldb, uint32_t M,
             uint32_t N, uint32_t K, const GemmEpi& epi, uint32_t split_k = 1, int precision = 1);

}  // namespace catgnn
