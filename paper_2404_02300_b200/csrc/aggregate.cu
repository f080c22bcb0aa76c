// K2 — neighbourhood aggregation, the B200 restatement of the gather loop of
// gnnpart::sgc_propagate (/root/reference/proj/src/train.cpp:55-62) generalised
// to the north-star layers (SGC mean-with-self, GCN-norm, SAGE-mean, GIN-sum).
//
//   out[r] = epi( post(deg_r) * ( self * pre[r]*in[r] + sum_{j in N(r)} pre[j]*in[j] ) )
//   epi    = (+ residual[r]) (+ bias) (ReLU) (* mask bit (r, c)); optionally
//            also writes the bits (out > 0) for the backward's ReLU mask
//
// Roofline: HBM-bound gather.  Algorithmic bytes per pass =
//   nnz*(4 + 4*width) + rows*(4*width*(1+self) + 8)
// (int32 column index + one fp32 row per edge; own row read when self, output
// row written, int64 offset read).  The kernel is persistent: warps pull work
// units (see csr.cu build_plan) from an atomic counter, prefetching the next
// unit index while the current one streams.  Inside a unit a warp walks whole
// rows: 32 column indices per coalesced load, then neighbour rows gathered with
// 128-bit read-only loads, UNROLL neighbours in flight per lane group.  Rows
// narrower than 128 floats are processed by sub-warp groups (LPN lanes per
// neighbour, 32/LPN neighbours at once) reduced with xor-shuffles.  Rows with
// more than U neighbours are chunked; chunk partials are combined in chunk
// order by agg_fixup_kernel, so results are deterministic.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "shard.hpp"

namespace catgnn {

namespace {

struct AggKernelArgs {
  const int64_t* __restrict__ row_ptr;
  const int32_t* __restrict__ col;
  const int4* __restrict__ units;
  const int4* __restrict__ heavy;
  unsigned long long n_units;
  unsigned long long n_heavy;
  unsigned int* counter;
  float* __restrict__ partials;  // [n_chunks][w4*4]
  uint32_t U;
  const float* __restrict__ in;
  const __half* __restrict__ in_h;  // fp16 input rows instead of `in` (in_ld / in_col in halves)
  uint32_t in_ld, in_col;
  float in_scale;                   // folded into the post scale (fp16 inputs stored scaled by 1/in_scale)
  int zero_row;                     // fp16 inputs: index of an all-zero row (= rows), the target of idle loads
  const int32_t* __restrict__ row_map;  // row views: a view row's row in the buffers
  const float* __restrict__ post_arr;   // per-row post scale (filtered views), else from the degree
  // guarded fp16 forward (GUARD): per-row max |T_j| of the fp16-rounded rows,
  // flagged-column bits, the rows with flags and their count, the threshold
  // factor (see epilogue_row)
  const float* __restrict__ gsmax;
  uint32_t* __restrict__ flag_bits;
  uint32_t* __restrict__ fix_rows;     // flagged light rows (warp-per-row fix)
  unsigned int* fix_count;
  uint32_t* __restrict__ fix_heavy;    // flagged split rows (block-per-row fix)
  unsigned int* fix_hcount;
  float* __restrict__ guard_part;      // per chunk: its neighbours' sum of squared row maxima
  float* __restrict__ guard_pre;       // rows x 256: the fp16-path pre-activation of each flagged element
  float guard_k;
  float* __restrict__ out;
  uint32_t out_ld, out_col;
  uint32_t w4;
  const float* __restrict__ pre;
  int self;
  int norm;
  const float* __restrict__ bias;
  const float* __restrict__ residual;
  uint32_t res_ld, res_col;
  int relu;
  int stream_hint;  // column indices and output rows with evict-first hints
  const uint32_t* __restrict__ mask_bits;  // ReLU-backward mask, 1 bit per column
  uint32_t mask_words;                     // 32-bit words per row
  uint32_t* __restrict__ bits_out;         // output > 0 bits (forward ReLU layers)
  uint32_t bits_words;
  uint2* __restrict__ out_hi;  // bf16x3 output pair (4 bf16 per float4 column group)
  uint2* __restrict__ out_lo;
  uint32_t out_s_ld;           // in bf16 elements
};

__device__ __forceinline__ float4 ldg4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}
// Packed fp32 pairs (sm_100 FADD2 / FFMA2): same IEEE round-to-nearest
// arithmetic per element as two scalar ops, half the issue slots.
__device__ __forceinline__ void add2(float& x, float& y, float u, float w) {
  asm("{\n\t.reg .b64 a, b;\n\tmov.b64 a, {%0, %1};\n\tmov.b64 b, {%2, %3};\n\t"
      "add.rn.f32x2 a, a, b;\n\tmov.b64 {%0, %1}, a;\n\t}"
      : "+f"(x), "+f"(y) : "f"(u), "f"(w));
}
__device__ __forceinline__ void fma2(float& x, float& y, float s, float u, float w) {
  asm("{\n\t.reg .b64 a, b, c;\n\tmov.b64 a, {%0, %1};\n\tmov.b64 b, {%2, %3};\n\t"
      "mov.b64 c, {%4, %4};\n\tfma.rn.f32x2 a, c, b, a;\n\tmov.b64 {%0, %1}, a;\n\t}"
      : "+f"(x), "+f"(y) : "f"(u), "f"(w), "f"(s));
}
__device__ __forceinline__ void fma4(float4& a, float s, const float4& v) {  // a += s * v
  fma2(a.x, a.y, s, v.x, v.y);
  fma2(a.z, a.w, s, v.z, v.w);
}
__device__ __forceinline__ void add4(float4& a, const float4& v) {
  add2(a.x, a.y, v.x, v.y);
  add2(a.z, a.w, v.z, v.w);
}
// 8 fp16 columns -> two float4 (exact)
__device__ __forceinline__ void h8_to_f4(const uint4& r, float4& a, float4& b) {
  const float2 x0 = __half22float2(*reinterpret_cast<const __half2*>(&r.x));
  const float2 x1 = __half22float2(*reinterpret_cast<const __half2*>(&r.y));
  const float2 x2 = __half22float2(*reinterpret_cast<const __half2*>(&r.z));
  const float2 x3 = __half22float2(*reinterpret_cast<const __half2*>(&r.w));
  a = make_float4(x0.x, x0.y, x1.x, x1.y);
  b = make_float4(x2.x, x2.y, x3.x, x3.y);
}
// One gathered 16-byte vector (CPV = 1: 4 fp32 columns, 2: 8 fp16 columns)
// into the accumulators a[0, CPV).
// f32 += f16, one instruction (sm_100 FHADD): exact conversion, IEEE RN add
__device__ __forceinline__ void fhadd(float& a, uint32_t h2, bool hi) {
  unsigned short h0, h1;
  asm("mov.b32 {%0, %1}, %2;" : "=h"(h0), "=h"(h1) : "r"(h2));
  asm("add.rn.f32.f16 %0, %1, %0;" : "+f"(a) : "h"(hi ? h1 : h0));
}
template <int CPV, bool PRE>
__device__ __forceinline__ void acc_raw(float4* a, const uint4& r, float s) {
  if constexpr (CPV == 2 && !PRE) {
    fhadd(a[0].x, r.x, false); fhadd(a[0].y, r.x, true); fhadd(a[0].z, r.y, false); fhadd(a[0].w, r.y, true);
    fhadd(a[1].x, r.z, false); fhadd(a[1].y, r.z, true); fhadd(a[1].z, r.w, false); fhadd(a[1].w, r.w, true);
  } else if constexpr (CPV == 1) {
    const float4 v = make_float4(__uint_as_float(r.x), __uint_as_float(r.y), __uint_as_float(r.z), __uint_as_float(r.w));
    if (PRE) fma4(a[0], s, v);
    else add4(a[0], v);
  } else {
    float4 v0, v1;
    h8_to_f4(r, v0, v1);
    if (PRE) { fma4(a[0], s, v0); fma4(a[1], s, v1); }
    else { add4(a[0], v0); add4(a[1], v1); }
  }
}
template <int CPV>
__device__ __forceinline__ void raw_to_f4(float4* a, const uint4& r) {
  if constexpr (CPV == 1) a[0] = make_float4(__uint_as_float(r.x), __uint_as_float(r.y), __uint_as_float(r.z), __uint_as_float(r.w));
  else h8_to_f4(r, a[0], a[1]);
}
// The row's own input columns [4 c4, 4 c4 + 4) (fp32 or fp16 rows)
__device__ __forceinline__ float4 self4(const AggKernelArgs& p, int64_t r, uint32_t c4) {
  if (p.in_h) {
    const uint2 u = __ldg(reinterpret_cast<const uint2*>(p.in_h + (size_t)r * p.in_ld + p.in_col + c4 * 4));
    const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
    const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
    return make_float4(a.x, a.y, b.x, b.y);
  }
  return __ldg(reinterpret_cast<const float4*>(p.in + (size_t)r * p.in_ld + p.in_col + c4 * 4));
}

__device__ __forceinline__ float4 shfl_xor4(const float4& v, int m) {
  return make_float4(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m),
                     __shfl_xor_sync(0xffffffffu, v.z, m), __shfl_xor_sync(0xffffffffu, v.w, m));
}

// Column index e: read once per pass, so with stream_hint it is loaded
// evict-first and leaves L2 to the gathered feature rows.
__device__ __forceinline__ int ld_col(const AggKernelArgs& p, int64_t e) {
  return p.stream_hint ? __ldcs(p.col + e) : __ldg(p.col + e);
}
__device__ __forceinline__ int ld_col(const AggKernelArgs& p, const int* __restrict__ base, int e) {
  return p.stream_hint ? __ldcs(base + e) : __ldg(base + e);
}

__device__ __forceinline__ float post_scale(int norm, float deg) {
  switch (norm) {
    case kNormSgc: return 1.0f / (1.0f + deg);
    case kNormGcn: return 1.0f / sqrtf(1.0f + deg);
    case kNormMean: return deg > 0.f ? 1.0f / deg : 0.0f;
    default: return 1.0f;
  }
}

// Final epilogue for one output row.  `acc` holds the neighbour sum for the
// float4 columns c4 = (li + LPN*q)*CPV + h at acc[q*CPV + h] (CPV = 2 for fp16
// input rows: a 16-byte vector then carries 8 columns).
// selfv: the row's own input columns when already loaded (light units).
// GUARD (fp16 forward of a ReLU layer): s2 = sum over the row's gathered rows
// (self included) of max_c |T_j[c]|^2.  Rounding T_j[c] to fp16 moves it by at
// most 2^-11 |T_j[c]| (RN, uniform in +-half an ulp: variance <= 2^-22 T^2 / 3),
// so the pre-activation a = post * sum + b carries an error of standard
// deviation <= post * 2^-11 * sqrt(s2 / 3) (max_c |T_j[c]| over-estimates each
// element's scale, so this bounds the true deviation).  Elements with |a| <
// guard_k * post * sqrt(s2) (guard_k = 6 * 2^-11 / sqrt(3): 6 bounding standard
// deviations, a tail probability < 2e-9; for rows with <= 12 terms also the
// worst case n * 2^-11 * max) could have the other sign in exact arithmetic:
// they are flagged (flag_bits), their fp16-path pre-activation kept
// (guard_pre) and their row listed (fix_rows / fix_heavy) for the exact fix.
template <int VPL, int LPN, bool BITS, int CPV, bool GUARD = false>
__device__ __forceinline__ void epilogue_row(const AggKernelArgs& p, int64_t rv, float deg,
                                             const float4 (&acc)[VPL * CPV], int li,
                                             const float4 (*selfv)[VPL * CPV] = nullptr, float s2 = 0.f) {
  const int64_t r = p.row_map ? (int64_t)__ldg(p.row_map + rv) : rv;  // the row in the output / input buffers
  // lanes [0, LPN) run this together (bit words are assembled across them)
  constexpr unsigned kLanes = LPN == 32 ? 0xffffffffu : ((1u << LPN) - 1u);
  constexpr int kGroup = LPN < 8 / CPV ? LPN : 8 / CPV;  // lanes whose nibbles form one 32-bit word
  const float post = (p.post_arr ? __ldg(p.post_arr + r) : post_scale(p.norm, deg)) * p.in_scale;
  const float selfs = p.pre ? __ldg(p.pre + r) : 1.0f;
  uint32_t nib[VPL * CPV];  // (out > 0) per column of each float4, for bits_out
  uint32_t fnib[VPL * CPV];  // GUARD: flagged columns
  float tau = 0.f;
  if (GUARD) {  // + (deg + 1) * 2^-28: fp16 subnormals round to an absolute 2^-25
    const float sm = __ldg(p.gsmax + r);
    tau = p.guard_k * post * sqrtf(s2 + sm * sm + (deg + 1.f) * 0x1p-28f);
  }
#pragma unroll
  for (int q = 0; q < VPL; ++q)
#pragma unroll
    for (int h = 0; h < CPV; ++h) {
      const int k = q * CPV + h;
      const uint32_t c4 = (li + LPN * q) * CPV + h;
      nib[k] = 0;
      fnib[k] = 0;
      if (c4 >= p.w4) continue;
      float4 a = acc[k];
      if (p.self) fma4(a, selfs, selfv ? (*selfv)[k] : self4(p, r, c4));
      a.x *= post; a.y *= post; a.z *= post; a.w *= post;
      if (p.residual) add4(a, ldg4(p.residual + (size_t)r * p.res_ld + p.res_col + c4 * 4));
      if (p.bias) add4(a, ldg4(p.bias + c4 * 4));
      if (GUARD) {
        fnib[k] = (fabsf(a.x) < tau) | ((fabsf(a.y) < tau) << 1) | ((fabsf(a.z) < tau) << 2) | ((fabsf(a.w) < tau) << 3);
        if (fnib[k])  // kept for the exact fix: it only adds the rounding residuals' contribution
          *reinterpret_cast<float4*>(p.guard_pre + (size_t)r * 256 + c4 * 4) = a;
      }
      if (p.relu) {
        a.x = fmaxf(a.x, 0.f); a.y = fmaxf(a.y, 0.f); a.z = fmaxf(a.z, 0.f); a.w = fmaxf(a.w, 0.f);
      }
      if (BITS && p.mask_bits) {  // ReLU backward: bit (r, col) of the forward activation
        const uint32_t m = __ldg(p.mask_bits + (size_t)r * p.mask_words + c4 / 8) >> ((c4 % 8) * 4);
        a.x = (m & 1u) ? a.x : 0.f; a.y = (m & 2u) ? a.y : 0.f;
        a.z = (m & 4u) ? a.z : 0.f; a.w = (m & 8u) ? a.w : 0.f;
      }
      if (BITS) nib[k] = (a.x > 0.f) | ((a.y > 0.f) << 1) | ((a.z > 0.f) << 2) | ((a.w > 0.f) << 3);
      if (p.out) {
        float4* dst = reinterpret_cast<float4*>(p.out + (size_t)r * p.out_ld + p.out_col + c4 * 4);
        if (p.stream_hint) __stcs(dst, a);  // evict-first: keep L2 for the gathered rows
        else *dst = a;
      }
      if (p.out_hi) {  // hi = bf16(v), lo = bf16(v - hi): the next GEMM's pre-split operand
        const __nv_bfloat162 h0 = __floats2bfloat162_rn(a.x, a.y), h1 = __floats2bfloat162_rn(a.z, a.w);
        const __nv_bfloat162 l0 = __floats2bfloat162_rn(a.x - __low2float(h0), a.y - __high2float(h0));
        const __nv_bfloat162 l1 = __floats2bfloat162_rn(a.z - __low2float(h1), a.w - __high2float(h1));
        const size_t o = ((size_t)r * p.out_s_ld + c4 * 4) / 4;
        p.out_hi[o] = make_uint2(*reinterpret_cast<const uint32_t*>(&h0), *reinterpret_cast<const uint32_t*>(&h1));
        p.out_lo[o] = make_uint2(*reinterpret_cast<const uint32_t*>(&l0), *reinterpret_cast<const uint32_t*>(&l1));
      }
    }
  if (BITS && p.bits_out) {  // 1 bit per output element (> 0): the next backward's ReLU mask
    bool anyf = false;
#pragma unroll
    for (int q = 0; q < VPL; ++q) {
      const uint32_t c40 = (li + LPN * q) * CPV;
      uint32_t w = 0, fw = 0;
#pragma unroll
      for (int h = 0; h < CPV; ++h) {
        w |= nib[q * CPV + h] << (((c40 + h) % 8) * 4);
        if (GUARD) fw |= fnib[q * CPV + h] << (((c40 + h) % 8) * 4);
      }
#pragma unroll
      for (int m = 1; m < kGroup; m <<= 1) {
        w |= __shfl_xor_sync(kLanes, w, m);
        if (GUARD) fw |= __shfl_xor_sync(kLanes, fw, m);
      }
      if (c40 < p.w4 && c40 % 8 == 0) {
        p.bits_out[(size_t)r * p.bits_words + c40 / 8] = w;
        if (GUARD) p.flag_bits[(size_t)r * p.bits_words + c40 / 8] = fw;
      }
      anyf |= fw != 0;
    }
    if (GUARD && __any_sync(kLanes, anyf) && li == 0) {
      if (deg > (float)p.U) p.fix_heavy[atomicAdd(p.fix_hcount, 1u)] = (uint32_t)r;
      else p.fix_rows[atomicAdd(p.fix_count, 1u)] = (uint32_t)r;
    }
  }
}

// Lane base address of the gathered rows: row j's 16-byte vector li + LPN*q
// sits at base + j*ldb + q*LPN*16 (one IMAD.WIDE per neighbour, the q offset
// an immediate).  fp16 rows (CPV = 2) hold 8 columns per vector.
template <int CPV>
__device__ __forceinline__ const char* lane_base(const AggKernelArgs& p, int li) {
  const char* b = CPV == 2 ? reinterpret_cast<const char*>(p.in_h + p.in_col) + li * 16
                           : reinterpret_cast<const char*>(p.in + p.in_col) + li * 16;
  // opaque: each neighbour address is then one IMAD.WIDE (j * row bytes + base)
  asm volatile("" : "+l"(b));
  return b;
}
template <int CPV>
__device__ __forceinline__ uint32_t row_bytes(const AggKernelArgs& p) { return p.in_ld * (CPV == 2 ? 2u : 4u); }
template <int CPV>
__device__ __forceinline__ uint32_t n_vec(const AggKernelArgs& p) { return CPV == 2 ? (p.w4 + 1) / 2 : p.w4; }
template <int VPL, int LPN>
__device__ __forceinline__ uint4 ld_nbr(const char* base, uint32_t ldb, int j, int q) {
  return __ldg(reinterpret_cast<const uint4*>(base + (uint64_t)(uint32_t)j * ldb + q * LPN * 16));
}

// Sum of pre[j]*in[j] over edges [e0, e1) into acc (reduced across groups).
// Loads past the end of the range, and by lanes whose columns lie past the
// row width, are skipped and contribute zeros.
template <int VPL, int LPN, bool PRE, int CPV, bool FULLW, bool ZR, bool GUARD>
__device__ __forceinline__ void gather(const AggKernelArgs& p, int64_t e0, int64_t e1,
                                       float4 (&acc)[VPL * CPV], int lane, float* ss_out = nullptr) {
  float ss = 0.f;  // GUARD: this chunk's sum of squared row maxima
  constexpr int G = 32 / LPN;  // neighbours processed side by side
  constexpr int UNROLL = VPL * CPV >= 4 ? 2 : (VPL * CPV >= 2 ? 4 : 8);
  const int g = lane / LPN, li = lane % LPN;
  const char* base = lane_base<CPV>(p, li);
  const uint32_t ldb = row_bytes<CPV>(p);
  bool colok[VPL];
#pragma unroll
  for (int q = 0; q < VPL; ++q) colok[q] = FULLW || li + LPN * q < (int)n_vec<CPV>(p);
#pragma unroll
  for (int k = 0; k < VPL * CPV; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t e = e0; e < e1; e += 32) {
    const int n = (int)((e1 - e) < 32 ? (e1 - e) : 32);
    const int myj = lane < n ? ld_col(p, e + lane) : 0;
    float mys = 1.0f;
    if (PRE) mys = lane < n ? __ldg(p.pre + myj) : 0.0f;
    if (GUARD) {
      const float sj = lane < n ? __ldg(p.gsmax + myj) : 0.0f;
      ss = fmaf(sj, sj, ss);
    }
    for (int kb = 0; kb < n; kb += G * UNROLL) {
      uint4 v[UNROLL][VPL];
      float s[UNROLL];
      bool ok[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const int kk = kb + u * G + g;
        const int j = __shfl_sync(0xffffffffu, myj, kk & 31);
        s[u] = PRE ? __shfl_sync(0xffffffffu, mys, kk & 31) : 1.0f;
        ok[u] = kk < n;
#pragma unroll
        for (int q = 0; q < VPL; ++q) {
          if constexpr (ZR)  // idle slots load the zero row
            v[u][q] = colok[q] ? ld_nbr<VPL, LPN>(base, ldb, ok[u] ? j : p.zero_row, q) : make_uint4(0u, 0u, 0u, 0u);
          else
            v[u][q] = (ok[u] && colok[q]) ? ld_nbr<VPL, LPN>(base, ldb, j, q) : make_uint4(0u, 0u, 0u, 0u);
        }
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u)
#pragma unroll
        for (int q = 0; q < VPL; ++q) acc_raw<CPV, PRE>(acc + q * CPV, v[u][q], s[u]);
    }
  }
#pragma unroll
  for (int m = LPN; m < 32; m <<= 1)
#pragma unroll
    for (int k = 0; k < VPL * CPV; ++k) add4(acc[k], shfl_xor4(acc[k], m));
  if (GUARD) {
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, m);
    *ss_out = ss;
  }
}

// A light unit (whole rows [r0, r1), edges contiguous in col[]) walked as one
// edge stream: the column indices (and source scales) of the unit are held in
// two 32-edge register chunks, the next chunk loaded while the current one is
// consumed, so a row costs no dependent index load; row offsets are fetched
// 32 rows per coalesced load and each row's own input row (self term) is
// requested together with its first neighbour batch.  Per row the G lane
// groups split the neighbours, UNROLL batches in flight, xor-shuffle reduce.
template <int VPL, int LPN, bool PRE, bool BITS, int CPV, bool FULLW, bool ZR, bool GUARD>
__device__ __forceinline__ void light_unit(const AggKernelArgs& p, int64_t r0, int64_t r1, int lane) {
  constexpr int G = 32 / LPN;
  static_assert(!GUARD || (G == 1 && !PRE && BITS), "guarded passes: whole-warp rows, no source scale, ReLU bits");
  // per-neighbour scalar streamed with the column indices: the source scale
  // (PRE) or the guard's row max (GUARD)
  constexpr bool SC = PRE || GUARD;
  const float* __restrict__ sarr = PRE ? p.pre : p.gsmax;
#ifndef AGG_NARROW_UNROLL
#define AGG_NARROW_UNROLL 4
#endif
#ifndef AGG_WIDE_UNROLL
#define AGG_WIDE_UNROLL 6
#endif
#ifndef AGG_H16_WIDE_UNROLL
#define AGG_H16_WIDE_UNROLL 8
#endif
  constexpr int UNROLL0 = CPV == 2 ? (LPN < 32 ? AGG_NARROW_UNROLL : (VPL == 1 ? AGG_H16_WIDE_UNROLL : (VPL == 2 ? AGG_WIDE_UNROLL : 2)))
                          : (LPN < 32 && VPL == 2) ? AGG_NARROW_UNROLL
                          : (LPN == 32 && VPL == 2) ? AGG_WIDE_UNROLL
                                                    : (VPL >= 4 ? 2 : (VPL >= 2 ? 4 : 8));
  constexpr int UNROLL = G * UNROLL0 > 32 ? 32 / G : UNROLL0;
  constexpr int B = G * UNROLL;  // neighbours per batch (<= 32)
  static_assert(B <= 32, "batch must fit one index chunk");
  const int g = lane / LPN, li = lane % LPN;
  const bool writer = lane < LPN;
  // edge offsets are 32-bit, relative to the unit's first edge (a light unit
  // holds < 2^31 edges); only the unit base is 64-bit
  const int64_t E0 = __ldg(p.row_ptr + r0);
  const int NE = (int)(__ldg(p.row_ptr + r1) - E0);
  const int* __restrict__ colu = p.col + E0;
  int cb = 0;  // first edge of the current chunk
  int cur = (lane < NE) ? ld_col(p, colu, lane) : 0;
  int nxt = (32 + lane < NE) ? ld_col(p, colu, 32 + lane) : 0;
  float curs = 1.f, nxts = 1.f;
  if (SC) {
    curs = (lane < NE) ? __ldg(sarr + cur) : 0.f;
    nxts = (32 + lane < NE) ? __ldg(sarr + nxt) : 0.f;
  }
  const char* base = lane_base<CPV>(p, li);
  const uint32_t ldb = row_bytes<CPV>(p);
  const int zrow = p.zero_row;
  bool colok[VPL];
#pragma unroll
  for (int q = 0; q < VPL; ++q) colok[q] = FULLW || li + LPN * q < (int)n_vec<CPV>(p);
  for (int64_t rb = r0; rb < r1; rb += 32) {
    const int64_t rr = rb + lane;
    const int rpa = rr < r1 ? (int)(__ldg(p.row_ptr + rr) - E0) : 0;
    const int rpb = rr < r1 ? (int)(__ldg(p.row_ptr + rr + 1) - E0) : 0;
    const int nr = (int)((r1 - rb) < 32 ? (r1 - rb) : 32);
    for (int i = 0; i < nr; ++i) {
      const int64_t r = rb + i;
      const int e0 = __shfl_sync(0xffffffffu, rpa, i), e1 = __shfl_sync(0xffffffffu, rpb, i);
#ifdef AGG_SKIP_SHORT  // diagnostics build: the cost of short rows (wrong results)
      if (e1 - e0 < AGG_SKIP_SHORT) continue;
#endif
      float4 selfv[VPL * CPV];
      const int64_t rsrc = p.row_map ? (int64_t)__ldg(p.row_map + r) : r;  // own input row (row views)
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        const uint4 sv = (p.self && writer && colok[q]) ? ld_nbr<VPL, LPN>(base, ldb, (int)rsrc, q) : make_uint4(0u, 0u, 0u, 0u);
        raw_to_f4<CPV>(selfv + q * CPV, sv);
      }
      float4 acc[VPL * CPV];
#pragma unroll
      for (int k = 0; k < VPL * CPV; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      float ss = 0.f;  // GUARD: per lane, the squared maxima of the window slots it held (summed at the row end)
      for (int e = e0; e < e1; e += B) {
        while (e >= cb + 32) {  // warp-uniform: advance the index window by one chunk
          cb += 32;
          cur = nxt;
          curs = nxts;
          const bool ok = cb + 32 + lane < NE;
          nxt = ok ? ld_col(p, colu, cb + 32 + lane) : 0;
          if (SC) nxts = ok ? __ldg(sarr + nxt) : 0.f;
        }
        uint4 v[UNROLL][VPL];
        float s[UNROLL];
        bool ok[UNROLL];
        if constexpr (G == 1) {
          // whole-warp rows: realign the window to this batch once (lane l <-
          // edge e + l), then each neighbour is one shuffle of a constant lane
          const int off = e - cb + lane;  // < 64
          const int wa = __shfl_sync(0xffffffffu, cur, off & 31);
          const int wb = __shfl_sync(0xffffffffu, nxt, off & 31);
          const int win = off < 32 ? wa : wb;
          float wins = 1.f;
          if (SC) {
            const float sa = __shfl_sync(0xffffffffu, curs, off & 31);
            const float sb = __shfl_sync(0xffffffffu, nxts, off & 31);
            wins = off < 32 ? sa : sb;
          }
          const int rem = min(e1 - e, B);  // valid neighbours of the batch
          if (GUARD && lane < rem) ss = fmaf(wins, wins, ss);  // lane l holds edge e + l's row max
#pragma unroll
          for (int uu = 0; uu < UNROLL; ++uu) {
            const int j = __shfl_sync(0xffffffffu, win, uu);
            s[uu] = PRE ? __shfl_sync(0xffffffffu, wins, uu) : 1.f;
            ok[uu] = uu < rem;
#pragma unroll
            for (int q = 0; q < VPL; ++q) {
              if constexpr (ZR)  // idle slots load the zero row
                v[uu][q] = colok[q] ? ld_nbr<VPL, LPN>(base, ldb, ok[uu] ? j : zrow, q) : make_uint4(0u, 0u, 0u, 0u);
              else
                v[uu][q] = (ok[uu] && colok[q]) ? ld_nbr<VPL, LPN>(base, ldb, j, q) : make_uint4(0u, 0u, 0u, 0u);
            }
          }
        } else {
          // lane groups: the window is realigned once per batch (lane l <-
          // edge e + l), then group g's neighbour of slot uu is one shuffle
          // of lane uu*G + g
          const int off = e - cb + lane;  // < 64
          const int wa = __shfl_sync(0xffffffffu, cur, off & 31);
          const int wb = __shfl_sync(0xffffffffu, nxt, off & 31);
          const int win = off < 32 ? wa : wb;
          float wins = 1.f;
          if (PRE) {
            const float sa = __shfl_sync(0xffffffffu, curs, off & 31);
            const float sb = __shfl_sync(0xffffffffu, nxts, off & 31);
            wins = off < 32 ? sa : sb;
          }
          const int rem = min(e1 - e, B);  // valid neighbours of the batch
#pragma unroll
          for (int uu = 0; uu < UNROLL; ++uu) {
            const int k = uu * G + g;
            const int j = __shfl_sync(0xffffffffu, win, k);
            s[uu] = PRE ? __shfl_sync(0xffffffffu, wins, k) : 1.f;
            ok[uu] = k < rem;
#pragma unroll
            for (int q = 0; q < VPL; ++q) {
              if constexpr (ZR)  // idle slots and lanes past the row width load the zero row
                v[uu][q] = ld_nbr<VPL, LPN>(base, ldb, (ok[uu] && colok[q]) ? j : zrow, q);
              else
                v[uu][q] = (ok[uu] && colok[q]) ? ld_nbr<VPL, LPN>(base, ldb, j, q) : make_uint4(0u, 0u, 0u, 0u);
            }
          }
        }
#pragma unroll
        for (int uu = 0; uu < UNROLL; ++uu)
#pragma unroll
          for (int q = 0; q < VPL; ++q) acc_raw<CPV, PRE>(acc + q * CPV, v[uu][q], s[uu]);
      }
#pragma unroll
      for (int m = LPN; m < 32; m <<= 1)
#pragma unroll
        for (int k = 0; k < VPL * CPV; ++k) add4(acc[k], shfl_xor4(acc[k], m));
      if (GUARD) {
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, m);
      }
      if (writer) epilogue_row<VPL, LPN, BITS, CPV, GUARD>(p, r, (float)(e1 - e0), acc, li, &selfv, ss);
    }
  }
}

// Persistent unit loop shared by both aggregation kernels: warps pull work
// units from the atomic counter (the next one prefetched by lane 0).
template <int VPL, int LPN, bool PRE, bool BITS, int CPV, bool FULLW, bool ZR, bool GUARD>
__device__ __forceinline__ void unit_loop(const AggKernelArgs& p) {
  const int lane = threadIdx.x & 31;
  const int li = lane % LPN;
  const bool writer = lane < LPN;
  unsigned int u = 0;
  if (lane == 0) u = atomicAdd(p.counter, 1u);
  u = __shfl_sync(0xffffffffu, u, 0);
  while (u < p.n_units) {
    unsigned int next = 0;
    if (lane == 0) next = atomicAdd(p.counter, 1u);  // prefetch the next unit
    const int4 w = __ldg(p.units + u);
    if (w.z < 0) {
      light_unit<VPL, LPN, PRE, BITS, CPV, FULLW, ZR, GUARD>(p, w.x, w.y, lane);
    } else {
      float4 acc[VPL * CPV];
      const int64_t r = w.x;
      const int64_t rb = __ldg(p.row_ptr + r), re = __ldg(p.row_ptr + r + 1);
      const int64_t e0 = rb + (int64_t)w.y * p.U;
      const int64_t e1 = (re < e0 + (int64_t)p.U) ? re : e0 + (int64_t)p.U;
      float ss = 0.f;
      gather<VPL, LPN, PRE, CPV, FULLW, ZR, GUARD>(p, e0, e1, acc, lane, &ss);
      if (GUARD && lane == 0) p.guard_part[w.z] = ss;
      if (writer) {
        float* dst = p.partials + (size_t)w.z * p.w4 * 4;
#pragma unroll
        for (int q = 0; q < VPL; ++q)
#pragma unroll
          for (int h = 0; h < CPV; ++h) {
            const uint32_t c4 = (li + LPN * q) * CPV + h;
            if (c4 < p.w4) *reinterpret_cast<float4*>(dst + c4 * 4) = acc[q * CPV + h];
          }
      }
    }
    u = __shfl_sync(0xffffffffu, next, 0);
  }
}

// BITS: the epilogue reads / writes ReLU bit masks (a separate instantiation
// keeps the plain passes' register budget: the narrow kernel runs at 64).
// CPV = 2: fp16 input rows.
// FULLW: the row width fills every lane's vectors (no column predicate).
// ZR: the input has a zero row at index rows (fp16 inputs always): idle
// neighbour slots load it instead of being predicated off and zeroed.
// GUARD: guarded fp16 forward of a ReLU layer (epilogue_row).
template <int VPL, int LPN, bool PRE, int MINB, bool BITS, int CPV, bool FULLW = false, bool ZR = (CPV == 2),
          bool GUARD = false>
__global__ void __launch_bounds__(256, MINB) agg_kernel(const AggKernelArgs p) {
  unit_loop<VPL, LPN, PRE, BITS, CPV, FULLW, ZR, GUARD>(p);
}

// One CTA per split row.  Warp w sums the row's chunk partials c = w, w+8,
// w+16, ... (two independent load chains per warp), the eight warp sums are
// combined in warp order through shared memory, and warp 0 applies the same
// epilogue as a light row.  The summation order is fixed by the plan, so the
// result is deterministic run to run.  Hub rows with ~100 chunks finish in
// ~7 dependent loads instead of ~25 with one warp per row.
constexpr int kFixWarps = 8;
// split rows with at most this many chunks are combined by one warp each
// (agg_fixup_warp_kernel); hubs with more keep a whole block
constexpr int kWarpFixChunks = 16;
// warps [w0, w0 + nw) of the grid, one split row each
template <int VPL, bool GUARD>
__device__ __forceinline__ void fixup_warp_rows(const AggKernelArgs& p, uint64_t w0, uint64_t nw) {
  const int lane = threadIdx.x & 31;
  for (uint64_t h = w0; h < p.n_heavy; h += nw) {
    const int4 hv = __ldg(p.heavy + h);
    if (hv.z > kWarpFixChunks) continue;  // a block-per-row hub (agg_fixup_kernel)
    const int64_t r = hv.x;
    float ss = 0.f;
    if (GUARD) {
      for (int c = lane; c < hv.z; c += 32) ss += __ldcg(p.guard_part + hv.y + c);
#pragma unroll
      for (int m = 16; m > 0; m >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, m);
    }
    float4 a0[VPL], a1[VPL];
#pragma unroll
    for (int q = 0; q < VPL; ++q) a0[q] = a1[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    const float* base = p.partials + (size_t)hv.y * p.w4 * 4;
    const size_t cs = (size_t)p.w4 * 4;
    int c = 0;
    for (; c + 1 < hv.z; c += 2) {  // chunk pairs in flight, fixed combination order
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        const uint32_t c4 = lane + 32 * q;
        if (c4 < p.w4) {
          add4(a0[q], __ldcg(reinterpret_cast<const float4*>(base + (size_t)c * cs + c4 * 4)));
          add4(a1[q], __ldcg(reinterpret_cast<const float4*>(base + (size_t)(c + 1) * cs + c4 * 4)));
        }
      }
    }
    if (c < hv.z) {
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        const uint32_t c4 = lane + 32 * q;
        if (c4 < p.w4) add4(a0[q], __ldcg(reinterpret_cast<const float4*>(base + (size_t)c * cs + c4 * 4)));
      }
    }
#pragma unroll
    for (int q = 0; q < VPL; ++q) add4(a0[q], a1[q]);
    const float deg = (float)(__ldg(p.row_ptr + r + 1) - __ldg(p.row_ptr + r));
    epilogue_row<VPL, 32, true, 1, GUARD>(p, r, deg, a0, lane, nullptr, ss);
  }
}
// blocks [b0, b0 + nb), one hub row each
template <int VPL, bool GUARD>
__device__ __forceinline__ void fixup_hub_rows(const AggKernelArgs& p, float4 (&part)[kFixWarps][32 * VPL],
                                               uint64_t b0, uint64_t nb) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint64_t h = b0; h < p.n_heavy; h += nb) {
    const int4 hv = __ldg(p.heavy + h);
    if (hv.z <= kWarpFixChunks) continue;  // combined by agg_fixup_warp_kernel
    const int64_t r = hv.x;
    float ss = 0.f;
    if (GUARD) {  // the guard's sum over the row's chunks (fixed order)
      for (int c = lane; c < hv.z; c += 32) ss += __ldcg(p.guard_part + hv.y + c);
#pragma unroll
      for (int m = 16; m > 0; m >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, m);
    }
    float4 acc[VPL], acc2[VPL];
#pragma unroll
    for (int q = 0; q < VPL; ++q) acc[q] = acc2[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    const float* base = p.partials + (size_t)hv.y * p.w4 * 4;
    const size_t cs = (size_t)p.w4 * 4;
    int c = warp;
    for (; c + kFixWarps < hv.z; c += 2 * kFixWarps) {
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        const uint32_t c4 = lane + 32 * q;
        if (c4 < p.w4) {
          const float* src = base + (size_t)c * cs + c4 * 4;
          add4(acc[q], __ldcg(reinterpret_cast<const float4*>(src)));
          add4(acc2[q], __ldcg(reinterpret_cast<const float4*>(src + kFixWarps * cs)));
        }
      }
    }
    if (c < hv.z) {
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        const uint32_t c4 = lane + 32 * q;
        if (c4 < p.w4) add4(acc[q], __ldcg(reinterpret_cast<const float4*>(base + (size_t)c * cs + c4 * 4)));
      }
    }
#pragma unroll
    for (int q = 0; q < VPL; ++q) {
      add4(acc[q], acc2[q]);
      part[warp][lane + 32 * q] = acc[q];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        float4 t = part[0][lane + 32 * q];
#pragma unroll
        for (int w = 1; w < kFixWarps; ++w) add4(t, part[w][lane + 32 * q]);
        acc[q] = t;
      }
      const float deg = (float)(__ldg(p.row_ptr + r + 1) - __ldg(p.row_ptr + r));
      epilogue_row<VPL, 32, true, 1, GUARD>(p, r, deg, acc, lane, nullptr, ss);
    }
    __syncthreads();
  }
}
template <int VPL, bool GUARD = false>
__global__ void __launch_bounds__(256) agg_fixup_warp_kernel(const AggKernelArgs p) {
  fixup_warp_rows<VPL, GUARD>(p, (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5,
                              ((uint64_t)gridDim.x * blockDim.x) >> 5);
}
template <int VPL, bool GUARD = false>
__global__ void __launch_bounds__(256) agg_fixup_kernel(const AggKernelArgs p) {
  __shared__ float4 part[kFixWarps][32 * VPL];
  fixup_hub_rows<VPL, GUARD>(p, part, blockIdx.x, gridDim.x);
}
// both in one launch: the first hb blocks look for hub rows (dispatched first,
// so a hub's long combine overlaps the warp-per-row combines)
template <int VPL, bool GUARD = false>
__global__ void __launch_bounds__(256) agg_fixup_merged_kernel(const AggKernelArgs p, unsigned hb) {
  __shared__ float4 part[kFixWarps][32 * VPL];
  if (blockIdx.x < hb) fixup_hub_rows<VPL, GUARD>(p, part, blockIdx.x, hb);
  else
    fixup_warp_rows<VPL, GUARD>(p, ((blockIdx.x - hb) * (uint64_t)blockDim.x + threadIdx.x) >> 5,
                                ((uint64_t)(gridDim.x - hb) * blockDim.x) >> 5);
}

// Exact recomputation of the guard's flagged elements (epilogue_row GUARD).
// The producing GEMM wrote lo = (T - fp16(T)) * 2^11 next to the fp16 T K2
// gathered, so the exact pre-activation is the fp16 path's (kept in
// guard_pre by the epilogue) plus post * 2^-11 * (sum of lo over the row's
// neighbours and itself): per flagged row, its flagged columns in groups of
// four, each group one walk over the row's edges (one column-index load and up
// to four residual loads per edge), lanes strided over the edges and a fixed
// xor / warp-order reduction — deterministic.  Then bias is already in, ReLU;
// the value replaces the fp16-path result in the bf16x3 output pair (and fp32
// output) and its ReLU bit is set or cleared.  Light rows: a warp each; split
// (heavy) rows: a 256-thread block each.
__device__ __forceinline__ void fix_store(const AggKernelArgs& p, uint32_t r, uint32_t c, float lo_sum,
                                          const __half* __restrict__ lo, float post) {
  const float selfs = p.pre ? __ldg(p.pre + r) : 1.0f;
  float s = lo_sum;
  if (p.self) s = fmaf(selfs, __half2float(__ldg(lo + (size_t)r * p.in_ld + p.in_col + c)), s);
  float v = fmaf(post * 0x1p-11f, s, p.guard_pre[(size_t)r * 256 + c]);
  if (p.relu) v = fmaxf(v, 0.f);
  if (p.out) p.out[(size_t)r * p.out_ld + p.out_col + c] = v;
  if (p.out_hi) {
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    const __nv_bfloat16 l = __float2bfloat16_rn(v - __bfloat162float(h));
    reinterpret_cast<__nv_bfloat16*>(p.out_hi)[(size_t)r * p.out_s_ld + c] = h;
    reinterpret_cast<__nv_bfloat16*>(p.out_lo)[(size_t)r * p.out_s_ld + c] = l;
  }
  uint32_t* bw = p.bits_out + (size_t)r * p.bits_words + c / 32;
  if (v > 0.f) atomicOr(bw, 1u << (c % 32));
  else atomicAnd(bw, ~(1u << (c % 32)));
}
// the next up-to-4 flagged columns of a row at or after word w / remaining
// bits fw; the row's 8 flag words sit in lanes 0-7 of `words` (one load)
__device__ __forceinline__ int next_cols(uint32_t words, uint32_t& w, uint32_t& fw, uint32_t (&cols)[4]) {
  int nc = 0;
  while (nc < 4) {
    while (!fw) {
      if (++w >= 8) return nc;
      fw = __shfl_sync(0xffffffffu, words, w);
    }
    cols[nc++] = w * 32 + (__ffs(fw) - 1);
    fw &= fw - 1;
  }
  return nc;
}
__device__ __forceinline__ float lo_at(const __half* __restrict__ lo, size_t i) { return __half2float(__ldg(lo + i)); }
// light rows: warp per row, warps [w0, w0 + nw) of the grid
__device__ __forceinline__ void exact_fix_light(const AggKernelArgs& p, const __half* __restrict__ lo, unsigned w0,
                                                unsigned nw) {
  const int lane = threadIdx.x & 31;
  const unsigned n = *p.fix_count;
  for (unsigned i = w0; i < n; i += nw) {
    const uint32_t r = p.fix_rows[i];
    const int64_t e0 = __ldg(p.row_ptr + r), e1 = __ldg(p.row_ptr + r + 1);
    const float post = post_scale(p.norm, (float)(e1 - e0));
    const uint32_t words = lane < 8 ? p.flag_bits[(size_t)r * 8 + lane] : 0u;
    uint32_t w = 0, fw = __shfl_sync(0xffffffffu, words, 0);
    uint32_t cols[4];
    for (int nc; (nc = next_cols(words, w, fw, cols)) > 0;) {
      float a[4] = {0.f, 0.f, 0.f, 0.f};
      for (int64_t e = e0 + lane; e < e1; e += 32) {
        const size_t jb = (size_t)__ldg(p.col + e) * p.in_ld + p.in_col;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (k < nc) a[k] += lo_at(lo, jb + cols[k]);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) a[k] += __shfl_xor_sync(0xffffffffu, a[k], m);
      if (lane < nc) {
        float mine = a[0];
#pragma unroll
        for (int k = 1; k < 4; ++k) mine = lane == k ? a[k] : mine;
        fix_store(p, r, cols[lane], mine, lo, post);
      }
    }
  }
}
// split (hub) rows: block per row, blocks [b0, b0 + nb)
__device__ __forceinline__ void exact_fix_heavy(const AggKernelArgs& p, const __half* __restrict__ lo,
                                                float (&red)[8][4], unsigned b0, unsigned nb) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned n = *p.fix_hcount;
  for (unsigned i = b0; i < n; i += nb) {
    const uint32_t r = p.fix_heavy[i];
    const int64_t e0 = __ldg(p.row_ptr + r), e1 = __ldg(p.row_ptr + r + 1);
    const float post = post_scale(p.norm, (float)(e1 - e0));
    const uint32_t words = lane < 8 ? p.flag_bits[(size_t)r * 8 + lane] : 0u;
    uint32_t w = 0, fw = __shfl_sync(0xffffffffu, words, 0);
    uint32_t cols[4];
    for (int nc; (nc = next_cols(words, w, fw, cols)) > 0;) {
      float a[4] = {0.f, 0.f, 0.f, 0.f}, b[4] = {0.f, 0.f, 0.f, 0.f};
      int64_t e = e0 + threadIdx.x;
      for (; e + 256 < e1; e += 512) {  // two edges in flight per thread
        const size_t ja = (size_t)__ldg(p.col + e) * p.in_ld + p.in_col;
        const size_t jb = (size_t)__ldg(p.col + e + 256) * p.in_ld + p.in_col;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (k < nc) { a[k] += lo_at(lo, ja + cols[k]); b[k] += lo_at(lo, jb + cols[k]); }
      }
      if (e < e1) {
        const size_t ja = (size_t)__ldg(p.col + e) * p.in_ld + p.in_col;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (k < nc) a[k] += lo_at(lo, ja + cols[k]);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        a[k] += b[k];
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) a[k] += __shfl_xor_sync(0xffffffffu, a[k], m);
      }
      if (lane == 0)
#pragma unroll
        for (int k = 0; k < 4; ++k) red[warp][k] = a[k];
      __syncthreads();
      if (warp == 0 && lane < nc) {
        float s = 0.f;
#pragma unroll
        for (int ww = 0; ww < 8; ++ww) s += red[ww][lane];
        fix_store(p, r, cols[lane], s, lo, post);
      }
      __syncthreads();
    }
  }
}
__global__ void __launch_bounds__(256, 8) agg_exact_fix_kernel(const AggKernelArgs p, const __half* __restrict__ lo) {
  exact_fix_light(p, lo, (blockIdx.x * blockDim.x + threadIdx.x) >> 5, (gridDim.x * blockDim.x) >> 5);
}
__global__ void __launch_bounds__(256) agg_exact_fix_heavy_kernel(const AggKernelArgs p,
                                                                  const __half* __restrict__ lo) {
  __shared__ float red[8][4];
  exact_fix_heavy(p, lo, red, blockIdx.x, gridDim.x);
}
// one launch for both: the first hb blocks take the hub rows (dispatched first,
// so their long edge walks overlap the light rows instead of following them)
__global__ void __launch_bounds__(256, 8) agg_exact_fix_merged_kernel(const AggKernelArgs p,
                                                                      const __half* __restrict__ lo, unsigned hb) {
  __shared__ float red[8][4];
  if (blockIdx.x < hb) exact_fix_heavy(p, lo, red, blockIdx.x, hb);
  else exact_fix_light(p, lo, ((blockIdx.x - hb) * blockDim.x + threadIdx.x) >> 5, ((gridDim.x - hb) * blockDim.x) >> 5);
}

using AggFn = void (*)(const AggKernelArgs);

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

template <int VPL, int LPN>
AggFn pick_pre(bool pre, bool bits) {
  // 3 CTAs/SM for rows >= 128 floats, 4 for plain narrow rows (<= 80 / 64 registers)
#ifndef AGG_NARROW_MINB
#define AGG_NARROW_MINB 4
#endif
#ifndef AGG_WIDE_MINB
#define AGG_WIDE_MINB 3
#endif
  constexpr int MINB = LPN < 32 ? AGG_NARROW_MINB : AGG_WIDE_MINB;
  if (bits) return pre ? agg_kernel<VPL, LPN, true, 3, true, 1> : agg_kernel<VPL, LPN, false, 3, true, 1>;
  return pre ? agg_kernel<VPL, LPN, true, MINB, false, 1> : agg_kernel<VPL, LPN, false, MINB, false, 1>;
}
// fp16 input rows (the source scale is folded into the producer: no PRE)
template <int VPL, int LPN, bool FULLW = false>
AggFn pick_h16(bool bits) {
  constexpr int MINB = LPN < 32 ? AGG_NARROW_MINB : AGG_WIDE_MINB;
  return bits ? agg_kernel<VPL, LPN, false, 3, true, 2, FULLW> : agg_kernel<VPL, LPN, false, MINB, false, 2, FULLW>;
}

// 6 standard deviations of the fp16 rounding error (epilogue_row GUARD)
constexpr float kGuardK = 6.0f * 0x1p-11f / 1.7320508f;

// Width slab handled by one launch: at most 32 lanes x 8 float4 = 1024 floats.
constexpr uint32_t kMaxSlab4 = 256;


AggFn pick_kernel(uint32_t w4, bool pre, bool bits, bool h16, bool zr, bool guard, int* lpn_out) {
  if (guard) {  // guarded fp16 forward: 256 columns, ReLU bits (checked by aggregate())
    *lpn_out = 32;
    return agg_kernel<1, 32, false, 3, true, 2, true, true, true>;
  }
  if (!h16 && zr && w4 == 64) {  // 256 fp32 columns, zero row: no predicates in the gather
    *lpn_out = 32;
    if (bits) return pre ? agg_kernel<2, 32, true, 3, true, 1, true, true> : agg_kernel<2, 32, false, 3, true, 1, true, true>;
    return pre ? agg_kernel<2, 32, true, AGG_WIDE_MINB, false, 1, true, true>
               : agg_kernel<2, 32, false, AGG_WIDE_MINB, false, 1, true, true>;
  }
  if (h16) {  // 16-byte vectors of 8 halves: 48-wide class rows = 6 of 8 lanes (4 neighbours per load)
    const uint32_t w8 = (w4 + 1) / 2;
    if (w8 <= 4) { *lpn_out = 4; return pick_h16<1, 4>(bits); }
    if (w8 <= 8) { *lpn_out = 8; return pick_h16<1, 8>(bits); }
    if (w8 <= 16) { *lpn_out = 16; return pick_h16<1, 16>(bits); }
    *lpn_out = 32;
    if (w8 == 32) return pick_h16<1, 32, true>(bits);  // 256 columns
    switch ((w8 + 31) / 32) {
      case 1: return pick_h16<1, 32>(bits);
      case 2: return pick_h16<2, 32>(bits);
      case 3: return pick_h16<3, 32>(bits);
      default: return pick_h16<4, 32>(bits);
    }
  }
  // lanes per neighbour x float4 per lane; the narrow class rows (41-48 floats)
  // use 8 lanes x 2 float4 (4 neighbours per load instruction)
  if (w4 <= 4) { *lpn_out = 4; return pick_pre<1, 4>(pre, bits); }
  if (w4 <= 8) { *lpn_out = 8; return pick_pre<1, 8>(pre, bits); }
  if (w4 <= 16) { *lpn_out = 8; return pick_pre<2, 8>(pre, bits); }
  // 129-192 floats (e.g. 172 classes): 16 lanes x 3 float4, two neighbours per
  // load instruction (48 float4 slots instead of 64)
  static const int mid16 = env_int("CATGNN_AGG_MID16", 1);
  if (mid16 && w4 > 32 && w4 <= 48) { *lpn_out = 16; return pick_pre<3, 16>(pre, bits); }
  *lpn_out = 32;
  switch ((w4 + 31) / 32) {
    case 1: return pick_pre<1, 32>(pre, bits);
    case 2: return pick_pre<2, 32>(pre, bits);
    case 3: return pick_pre<3, 32>(pre, bits);
    case 4: return pick_pre<4, 32>(pre, bits);
    case 5: return pick_pre<5, 32>(pre, bits);
    case 6: return pick_pre<6, 32>(pre, bits);
    case 7: return pick_pre<7, 32>(pre, bits);
    default: return pick_pre<8, 32>(pre, bits);
  }
}

AggFn pick_fixup(uint32_t w4, bool warp) {
  switch ((w4 + 31) / 32) {
    case 1: return warp ? agg_fixup_warp_kernel<1> : agg_fixup_kernel<1>;
    case 2: return warp ? agg_fixup_warp_kernel<2> : agg_fixup_kernel<2>;
    case 3: return warp ? agg_fixup_warp_kernel<3> : agg_fixup_kernel<3>;
    case 4: return warp ? agg_fixup_warp_kernel<4> : agg_fixup_kernel<4>;
    case 5: return warp ? agg_fixup_warp_kernel<5> : agg_fixup_kernel<5>;
    case 6: return warp ? agg_fixup_warp_kernel<6> : agg_fixup_kernel<6>;
    case 7: return warp ? agg_fixup_warp_kernel<7> : agg_fixup_kernel<7>;
    default: return warp ? agg_fixup_warp_kernel<8> : agg_fixup_kernel<8>;
  }
}

int blocks_per_sm(int device, AggFn fn) {
  // keyed by device ordinal (the occupancy query is per device); callers on
  // several host threads share the cache
  static std::mutex mu;
  static std::map<std::pair<int, AggFn>, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({device, fn});
  if (it != cache.end()) return it->second;
  int b = 0;
  CG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, 256, 0));
  b = std::max(1, b);
  cache[{device, fn}] = b;
  return b;
}

}  // namespace

void aggregate(catgnn_shard_s* s, const AggArgs& a) {
  catgnn_ctx ctx = s->ctx;
  if (a.width % 4 || a.in_ld % 4 || a.out_ld % 4 || a.in_col % 4 || a.out_col % 4 ||
      (a.residual && (a.res_ld % 4 || a.res_col % 4)))
    throw ConfigError("aggregation widths/strides must be multiples of 4 floats");
  // one buffer may be both input and output when the column ranges are disjoint
  // (SAGE: mean(h) into the right half of [h | mean])
  if (a.in == a.out && a.in && a.in_ld == a.out_ld && a.in_col < a.out_col + a.width && a.out_col < a.in_col + a.width)
    throw ConfigError("aggregation cannot run in place");
  if (a.in == a.out && a.in && a.in_ld != a.out_ld) throw ConfigError("aggregation cannot run in place");
  if (s->rows == 0 || a.width == 0) return;
  if (!a.out && !a.out_hi) throw ConfigError("aggregation needs an output");
  if (a.guard_smax && a.row_map) throw ConfigError("guarded aggregation over a row view");
  if (a.guard_smax && (!a.in_h || a.width != 256 || !a.bits_out || !a.relu || a.pre || a.mask_bits || a.residual ||
                       !a.guard_flags || !a.guard_lo || a.bits_words != 8))
    throw ConfigError("guarded fp16 aggregation: fp16 input, 256 columns, ReLU with bit output, fp16 residual");
  if (a.in_h && (a.in || a.pre || a.in_ld % 8 || a.in_col % 8 || a.in_ld < a.in_col + round_up(a.width, 8)))
    throw ConfigError("fp16 aggregation input: no fp32 input / source scale, row stride and column a multiple of 8");
  if (a.out_hi && (!a.out_lo || a.out_s_ld % 8 || a.out_s_ld < a.width))
    throw ConfigError("bf16 aggregation output needs hi and lo rows of >= width elements, a multiple of 8");
  const uint32_t W4 = a.width / 4;
  for (uint32_t c4 = 0; c4 < W4; c4 += kMaxSlab4) {
    const uint32_t w4 = std::min(kMaxSlab4, W4 - c4);
    AggKernelArgs p{};
    p.row_ptr = s->row_ptr.p;
    p.col = s->col.p;
    p.units = s->units.p;
    p.heavy = s->heavy.p;
    p.n_units = s->n_units;
    p.n_heavy = s->n_heavy;
    p.counter = ctx->scratch_buf<unsigned int>("k2_counter", 1);
    p.partials = s->n_chunks ? ctx->scratch_buf<float>("k2_partials", s->n_chunks * (size_t)w4 * 4)
                             : nullptr;
    p.U = s->unit_cost;
    p.in = a.in;
    p.in_h = static_cast<const __half*>(a.in_h);
    p.in_scale = a.in_scale;
    p.zero_row = (int)(a.zero_row >= 0 ? a.zero_row : (int64_t)s->rows);
    p.row_map = a.row_map;
    p.post_arr = a.post_arr;
    p.in_ld = a.in_ld;
    p.in_col = a.in_col + c4 * 4;
    p.out = a.out;
    p.out_ld = a.out_ld;
    p.out_col = a.out_col + c4 * 4;
    p.w4 = w4;
    p.pre = a.pre;
    p.self = a.self;
    p.norm = a.norm;
    p.bias = a.bias ? a.bias + c4 * 4 : nullptr;
    p.residual = a.residual;
    p.res_ld = a.res_ld;
    p.res_col = a.res_col + c4 * 4;
    p.relu = a.relu;
    if ((a.mask_bits || a.bits_out) && c4 % 8)
      throw ConfigError("bit masks need 32-column aligned aggregation slabs");
    p.mask_bits = a.mask_bits ? a.mask_bits + c4 / 8 : nullptr;
    p.mask_words = a.mask_words;
    p.bits_out = a.bits_out ? a.bits_out + c4 / 8 : nullptr;
    p.bits_words = a.bits_words;
    p.out_hi = a.out_hi ? reinterpret_cast<uint2*>(static_cast<uint16_t*>(a.out_hi) + c4 * 4) : nullptr;
    p.out_lo = a.out_lo ? reinterpret_cast<uint2*>(static_cast<uint16_t*>(a.out_lo) + c4 * 4) : nullptr;
    p.out_s_ld = a.out_s_ld;
    static const int hint = env_int("CATGNN_AGG_HINT", 1);
    p.stream_hint = hint;
    int lpn = 32;
    const bool guard = a.guard_smax != nullptr;
    if (guard) {
      p.gsmax = a.guard_smax;
      p.flag_bits = a.guard_flags;
      p.fix_rows = ctx->scratch_buf<uint32_t>("k2_fix_rows", std::max<uint64_t>(1, s->rows));
      p.fix_heavy = ctx->scratch_buf<uint32_t>("k2_fix_heavy", std::max<uint64_t>(1, s->n_heavy));
      p.fix_count = ctx->scratch_buf<unsigned int>("k2_fix_count", 2);
      p.fix_hcount = p.fix_count + 1;
      p.guard_part = ctx->scratch_buf<float>("k2_guard_part", std::max<uint64_t>(1, s->n_chunks));
      p.guard_pre = ctx->scratch_buf<float>("k2_guard_pre", std::max<uint64_t>(1, s->rows) * 256);
      p.guard_k = kGuardK;
      CG_CUDA(cudaMemsetAsync(p.fix_count, 0, 2 * sizeof(unsigned int), ctx->stream));
    }
    AggFn fn = pick_kernel(w4, a.pre != nullptr, a.mask_bits || a.bits_out, a.in_h != nullptr,
                           a.in_zero_row && W4 == w4, guard, &lpn);
    CG_CUDA(cudaMemsetAsync(p.counter, 0, sizeof(unsigned int), ctx->stream));
    static const int detail = env_int("CATGNN_TIMING_DETAIL", 0);  // label per shard (rows)
    int t = ctx->begin_timed(0, ctx->timing ? "K2 agg w" + std::to_string(w4 * 4) + (a.in_h ? " f16" : "") +
                                                   (a.pre ? " pre" : "") +
                                                   (a.mask_bits || a.bits_out ? " bits" : "") +
                                                   (detail ? " rows=" + std::to_string(s->rows) : std::string())
                                             : std::string());
    const int bps = blocks_per_sm(ctx->device, fn);
    static const int sms_env = env_int("CATGNN_AGG_SMS", 0);  // A/B knob: SMs the persistent grid covers
    const uint64_t warps_needed = std::max<uint64_t>(1, s->n_units);
    const unsigned grid = (unsigned)std::max<uint64_t>(
        1, std::min<uint64_t>((uint64_t)(sms_env > 0 ? sms_env : (ctx->agg_sms ? ctx->agg_sms : ctx->num_sms)) * bps,
                              (warps_needed + 7) / 8));
    fn<<<grid, 256, 0, ctx->stream>>>(p);
    CG_CHECK_LAUNCH();
    ctx->launches++;
    if (s->n_heavy) {  // split rows: warp per row up to kWarpFixChunks chunks, block per hub row
      AggFn fw = guard ? agg_fixup_warp_kernel<2, true> : pick_fixup(w4, true);
      const unsigned gw = (unsigned)std::min<uint64_t>((s->n_heavy + 7) / 8, (uint64_t)ctx->num_sms * 8);
      static const int fix_merged = env_int("CATGNN_FIX_MERGED", 1);
      const unsigned vpl = (w4 + 31) / 32;
      if (s->n_big_heavy && fix_merged && vpl <= 2) {
        const unsigned hb = (unsigned)std::min<uint64_t>(s->n_heavy, (uint64_t)ctx->num_sms * 16);
        auto fm = guard ? agg_fixup_merged_kernel<2, true>
                        : (vpl == 1 ? agg_fixup_merged_kernel<1> : agg_fixup_merged_kernel<2>);
        fm<<<hb + gw, 256, 0, ctx->stream>>>(p, hb);
        CG_CHECK_LAUNCH();
      } else {
        fw<<<gw, 256, 0, ctx->stream>>>(p);
        CG_CHECK_LAUNCH();
      }
      if (s->n_big_heavy && !(fix_merged && vpl <= 2)) {
        AggFn fx = guard ? agg_fixup_kernel<2, true> : pick_fixup(w4, false);
        const unsigned g2 = (unsigned)std::min<uint64_t>(s->n_heavy, (uint64_t)ctx->num_sms * 16);
        fx<<<g2, 256, 0, ctx->stream>>>(p);
        CG_CHECK_LAUNCH();
        ctx->launches++;
      }
      ctx->launches++;
    }
    if (guard) {  // exact fp32 recomputation of the flagged elements
      int tf = ctx->begin_timed(3, ctx->timing ? std::string("(within K2 w256) guard exact fix") : std::string());
      static const int merged = env_int("CATGNN_FIX_MERGED", 1);
      const unsigned hb = (unsigned)std::min<uint64_t>(s->n_heavy, (uint64_t)ctx->num_sms * 2);
      if (merged) {
        agg_exact_fix_merged_kernel<<<ctx->num_sms * 8 + hb, 256, 0, ctx->stream>>>(
            p, static_cast<const __half*>(a.guard_lo), hb);
      } else {
        agg_exact_fix_kernel<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(p, static_cast<const __half*>(a.guard_lo));
      }
      CG_CHECK_LAUNCH();
      if (s->n_heavy && !merged) {
        agg_exact_fix_heavy_kernel<<<(unsigned)std::min<uint64_t>(s->n_heavy, ctx->num_sms * 4), 256, 0,
                                     ctx->stream>>>(p, static_cast<const __half*>(a.guard_lo));
        CG_CHECK_LAUNCH();
        ctx->launches++;
      }
      ctx->end_timed(tf);
      ctx->launches++;
      static const int stats = env_int("CATGNN_GUARD_STATS", 0);  // diagnostics: flagged rows per pass
      if (stats) {
        unsigned n = 0;
        CG_CUDA(cudaMemcpyAsync(&n, p.fix_count, sizeof(n), cudaMemcpyDeviceToHost, ctx->stream));
        CG_CUDA(cudaStreamSynchronize(ctx->stream));
        unsigned nh = 0;
        CG_CUDA(cudaMemcpy(&nh, p.fix_hcount, sizeof(nh), cudaMemcpyDeviceToHost));
        std::vector<uint32_t> fl(s->rows * 8);
        CG_CUDA(cudaMemcpy(fl.data(), p.flag_bits, fl.size() * 4, cudaMemcpyDeviceToHost));
        std::vector<int64_t> rp(s->rows + 1);
        CG_CUDA(cudaMemcpy(rp.data(), s->row_ptr.p, rp.size() * 8, cudaMemcpyDeviceToHost));
        uint64_t el = 0, work = 0;
        for (uint64_t r = 0; r < s->rows; ++r) {
          int c = 0;
          for (int w = 0; w < 8; ++w) c += __builtin_popcount(fl[r * 8 + w]);
          el += c;
          work += (uint64_t)c * (uint64_t)(rp[r + 1] - rp[r] + 1);
        }
        fprintf(stderr, "[guard] rows %llu flagged rows %u + split rows %u of %llu; elements %llu (%.3f%%), "
                "residual loads %llu (%.2f per edge)\n", (unsigned long long)s->rows, n, nh,
                (unsigned long long)s->n_heavy, (unsigned long long)el, 100.0 * el / (s->rows * 256.0),
                (unsigned long long)work, (double)work / (double)s->nnz);
      }
    }
    ctx->end_timed(t);
  }
}

}  // namespace catgnn
