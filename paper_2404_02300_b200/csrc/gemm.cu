// K3 — dense layer transform on the 5th-generation tensor cores.
//
//   C[M x N] = A[M x K] . B[N x K]^T        (A, B K-major fp32 in HBM, TF32 MMA,
//                                            fp32 accumulation in TMEM)
//
// Persistent CTAs (one per SM) walk 128 x BN output tiles (x split-K ranges):
//   warp 0      TMA producer: operand tiles into an S-stage shared-memory ring
//               (cp.async.bulk.tensor ... mbarrier::complete_tx).  K-major
//               operands: one {32 x rows} SWIZZLE_128B box; MN-major operands
//               (row-major activations read in place for weight gradients):
//               {32 x 32} boxes in the SWIZZLE_128B_BASE32B layout
//   warp 1      TMEM allocation + one elected thread issuing tcgen05.mma
//               .cta_group::1.kind::tf32 (M=128, N=BN, K=8 per instruction)
//               into one of two TMEM accumulators, so the epilogue of tile i
//               overlaps the MMAs of tile i+1; tcgen05.commit frees stages
//   warps 2..5  3xTF32 converters: lo = x - tf32(x) tiles into a ring of L
//               residual slots (slot it % L, freed by the MMAs of stage it - L),
//               MMA issues lo*hi + hi*lo + hi*hi (~fp32 accuracy)
//   warps 6..   epilogue (4 warps, or 8 for short K loops — two per TMEM lane
//               quarter splitting the 32-column chunks): tcgen05.ld 32x32b.x32 (warp w reads TMEM lanes
//               32*(w%4)..+31 = tile rows), fused row-scale / bias / ReLU /
//               ReLU-backward bit mask, staged line-coalesced stores — or raw split-K partials
//               that gemm_reduce_kernel sums in split order (deterministic).
// Tail rows/columns and K past the tensor extent are zero-filled by TMA.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <array>
#include <map>
#include <mutex>

#include "gemm.hpp"

namespace catgnn {

namespace {

constexpr int BM = 128;
constexpr int BK = 32;              // fp32 elements per k-block row = 128 bytes
constexpr int A_STAGE = BM * BK * 4;  // 16 KB
#ifndef GEMM_CONV_WARPS
#define GEMM_CONV_WARPS 4
#endif
constexpr int kConvWarps = GEMM_CONV_WARPS;  // 3xTF32 converter warps (8 measured no faster)
constexpr int kEpiWarp0 = 2 + kConvWarps;    // first epilogue warp
// Epilogue warps per CTA (template EPIW): 4, one per TMEM lane quarter, or 8,
// two per quarter splitting the 32-column chunks — for GEMMs with a short K
// loop, which are bound by draining and storing the accumulator.
template <int EPIW>
constexpr int threads_for() { return 32 * (kEpiWarp0 + EPIW); }  // TMA, MMA, converters, epilogue
constexpr uint32_t kTileLd4 = 9;
constexpr uint32_t kMaxLo = 8;     // residual-slot barriers reserved (>= stages for CATGNN_GEMM_LO_SLOTS=0)
constexpr uint32_t kMaxStages = 8;
// barrier block: full/empty/conv per stage, tfull/tempty x2, lo_empty x kMaxLo, TMEM holder
__host__ __device__ constexpr uint32_t kBarBytes(uint32_t S) { return ((3 * S + 4 + kMaxLo) * 8 + 8 + 15) / 16 * 16; }  // epilogue staging tile row stride in float4 (144 B)
constexpr size_t epi_smem(int epiw) { return (size_t)epiw * 32 * kTileLd4 * 16; }

struct GemmArgs {
  uint32_t M, N, K;
  uint32_t BN;
  uint32_t bk;        // K elements per k-block (stage): 32 fp32 / 64 bf16 = 128-byte rows
  uint32_t stages;
  uint32_t lo_slots;  // 3xTF32: ring of lo (residual) tile slots, decoupled from the TMA stages
  uint32_t kb_per_split;
  uint32_t tmem_cols;
  uint32_t idesc;
  uint32_t split3;  // 1: 3xTF32 (hi*hi + hi*lo + lo*hi), 0: plain TF32
  uint32_t mt, nt, splits, tiles;
  uint32_t a_mn, b_mn;  // operand stored MN-major ([K rows][M or N cols] row-major)
  uint32_t bm;          // tile rows: BM x CTAs per tile
  uint32_t a_stream, b_stream;  // operand read once per GEMM (row-sized): L2 evict-first loads
  uint32_t b_lo_tma;            // 3xTF32: B residual precomputed, TMA-loaded per stage
  GemmEpi epi;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

// Parity wait with a watchdog: a pipeline bug traps (kernel error) instead of
// hanging the GPU.
#ifdef GEMM_WAIT_PROFILE
// diagnostics build: nanoseconds each wait site spent blocked, summed over CTAs
__device__ unsigned long long g_gemm_wait_ns[8];
#endif
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase, int site = -1) {
  uint32_t done = 0;
  uint64_t t0 = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
#ifdef GEMM_WAIT_PROFILE
  struct Acc {
    uint64_t t0; int site;
    __device__ ~Acc() {
      uint64_t t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      if (site >= 0 && (threadIdx.x & 31) == 0) atomicAdd(&g_gemm_wait_ns[site], (unsigned long long)(t1 - t0));
    }
  } acc{t0, site};
#endif
  while (true) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(phase)
        : "memory");
    if (done) return;
    uint64_t t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (t1 - t0 > 2000000000ull) __trap();  // 2 s
  }
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}

// Same with an L2 eviction policy (createpolicy): row-sized activation
// operands are streamed once per GEMM and loaded evict-first, so the output
// the next kernel consumes stays in L2.
__device__ __forceinline__ void tma_load_2d_hint(uint32_t dst, const CUtensorMap* map, int x, int y,
                                                 uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// UMMA shared-memory descriptor, K-major, SWIZZLE_128B: rows of 128 bytes,
// 8-row core groups 1024 bytes apart (SBO), LBO unused (1), version 1.
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr) {
  return (uint64_t)((addr & 0x3FFFFu) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) |
         (2ull << 61);
}

// MN-major tf32 operands use the SWIZZLE_128B_BASE32B layout (layout type 1:
// 32-byte chunks swizzled within 128-byte rows, 4-row period; filled by TMA's
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B): 32-element (128 B) atoms along M/N,
// LBO = 4 KB between M/N atoms (one 32 x 32 TMA box each), SBO = 512 B between
// 4-row K groups; one MMA (K = 8) spans two K groups, so k-steps advance 1 KB.
__device__ __forceinline__ uint64_t umma_desc_mn(uint32_t addr) {
  return (uint64_t)((addr & 0x3FFFFu) >> 4) | (256ull << 16) | (32ull << 32) | (1ull << 46) |
         (1ull << 61);
}

// MN-major 16-bit operands (bf16x3 path): canonical SWIZZLE_128B layout —
// 64-element (128 B) atoms along M/N, one {64 x 64} TMA box each, LBO = 8 KB
// between M/N atoms, SBO = 1 KB between 8-row K groups; one MMA (K = 16) spans
// two K groups, so k-steps advance 2 KB.
__device__ __forceinline__ uint64_t umma_desc_mn16(uint32_t addr) {
  return (uint64_t)((addr & 0x3FFFFu) >> 4) | (512ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
// descriptor of k-step ks (K = 16 bf16) of a bf16 stage tile (K-major rows of
// 64 elements = 128 B, SWIZZLE_128B: +32 B per k-step as for tf32)
__device__ __forceinline__ uint64_t op_desc16(uint32_t base, int ks, bool mn) {
  return mn ? umma_desc_mn16(base + ks * 2048) : umma_desc(base + ks * 32);
}

// descriptor of k-step ks (K = 8 elements) of a stage tile in either layout
__device__ __forceinline__ uint64_t op_desc(uint32_t base, int ks, bool mn) {
  return mn ? umma_desc_mn(base + ks * 1024) : umma_desc(base + ks * 32);
}

// TMA fill of one operand stage: K-major = one {32 x rows} box; MN-major =
// rows/32 boxes of {32 (M/N) x 32 (K)} placed 4 KB apart.
// policy != 0: load with that L2 cache hint.
__device__ __forceinline__ void load_operand(uint32_t dst, const CUtensorMap* map, bool mn, int k0, int r0,
                                             uint32_t rows, uint32_t bar, uint64_t policy) {
  if (!mn) {
    if (policy) tma_load_2d_hint(dst, map, k0, r0, bar, policy);
    else tma_load_2d(dst, map, k0, r0, bar);
  } else {
    for (uint32_t a = 0; a < rows / 32; ++a) {
      if (policy) tma_load_2d_hint(dst + a * 4096, map, r0 + (int)(32 * a), k0, bar, policy);
      else tma_load_2d(dst + a * 4096, map, r0 + (int)(32 * a), k0, bar);
    }
  }
}

// bf16 x bf16 -> f32 (kind::f16, K = 16 per instruction)
template <int NCTA>
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
  if (NCTA == 2)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// TMA fill of one bf16 operand half (hi or lo) of a stage: K-major = one
// {64 x rows} box; MN-major = rows/64 boxes of {64 (M/N) x 64 (K)} 8 KB apart.
__device__ __forceinline__ void load_operand16(uint32_t dst, const CUtensorMap* map, bool mn, int k0, int r0,
                                               uint32_t rows, uint32_t bar) {
  if (!mn) {
    tma_load_2d(dst, map, k0, r0, bar);
  } else {
    for (uint32_t a = 0; a < rows / 64; ++a) tma_load_2d(dst + a * 8192, map, r0 + (int)(64 * a), k0, bar);
  }
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
// CTA pair: arrive on the barrier at this offset in both CTAs
__device__ __forceinline__ void mma_commit_pair(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}
template <int NCTA>
__device__ __forceinline__ void commit_to(uint32_t bar) {
  if (NCTA == 2) mma_commit_pair(bar);
  else mma_commit(bar);
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the barrier at local offset `bar` in CTA `cta` of the cluster
__device__ __forceinline__ void mbar_arrive_cta(uint32_t bar, uint32_t cta) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(bar), "r"(cta));
  // default .release.cta semantics (as CUTLASS's ClusterBarrier::arrive): a
  // .cluster-scope release costs a MEMBAR.GPU per arrival
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float tf32_residual(float x) {
  return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}
__device__ __forceinline__ float4 tf32_residual4(float4 v) {
  return make_float4(tf32_residual(v.x), tf32_residual(v.y), tf32_residual(v.z), tf32_residual(v.w));
}

__device__ __forceinline__ float apply_epi(const GemmEpi& e, uint32_t row, uint32_t col, float v) {
  if (e.rowscale && col >= e.scale_col_begin) v *= __ldg(e.rowscale + row);
  if (e.bias) v += __ldg(e.bias + col);
  if (e.relu) v = fmaxf(v, 0.f);
  if (e.mask_bits && !((__ldg(e.mask_bits + (size_t)row * e.mask_words + col / 32) >> (col % 32)) & 1u)) v = 0.f;
  return v * e.out_scale;
}
__device__ __forceinline__ void store_epi(const GemmEpi& e, uint32_t row, uint32_t col, float v) {
  if (e.out_h) e.out_h[(size_t)row * (e.ld_h ? e.ld_h : e.ld_out) + e.out_col + col] = __float2half_rn(v);
  if (e.out_bhi) {
    const size_t o = (size_t)row * (e.ld_h ? e.ld_h : e.ld_out) + e.out_col + col;
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    e.out_bhi[o] = h;
    e.out_blo[o] = __float2bfloat16_rn(v - __bfloat162float(h));
  }
  if (e.out) e.out[(size_t)row * e.ld_out + e.out_col + col] = v;
}
__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

__device__ __forceinline__ void tile_coords(const GemmArgs& a, uint32_t t, uint32_t& m0, uint32_t& n0,
                                            uint32_t& kb0, uint32_t& nkb) {
  // n fastest: CTAs working on the same M block at the same time share A in L2
  const uint32_t n = t % a.nt, m = (t / a.nt) % a.mt, z = t / (a.nt * a.mt);
  m0 = m * a.bm;
  n0 = n * a.BN;
  const uint32_t nkb_total = (a.K + a.bk - 1) / a.bk;
  kb0 = z * a.kb_per_split;
  const uint32_t kb1 = min(nkb_total, kb0 + a.kb_per_split);
  nkb = kb1 > kb0 ? kb1 - kb0 : 0;
}

__device__ __forceinline__ float4 lds4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts4(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

// lo = x - tf32(x) over n16 16-byte words of a stage tile; 128 converter
// threads, 8 words in flight per thread (element-wise, so the SW128 layout of
// the source carries over to the residual tile).
__device__ __forceinline__ void convert_tile(uint32_t src, uint32_t dst, uint32_t n16, uint32_t t) {
  constexpr uint32_t NT = 32 * kConvWarps;
  for (uint32_t k0 = t; k0 < n16; k0 += NT * 8) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t k = k0 + u * NT;
      if (k < n16) v[u] = lds4(src + k * 16);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t k = k0 + u * NT;
      if (k < n16) sts4(dst + k * 16, tf32_residual4(v[u]));
    }
  }
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// Persistent warp-specialised kernel (one CTA per SM; NCTA = 2: CTA pairs on
// the two SMs of a TPC, cta_group::2, 256-row tiles):
//   warp 0     TMA producer over every tile's k-blocks (S-stage ring); in a
//              pair each CTA loads its own 128 rows of A and its half of B
//   warp 1     TMEM allocator + MMA issuer (the pair's rank-0 CTA only);
//              accumulators double-buffered in TMEM (2 x acc_cols columns) so
//              tile i's epilogue overlaps tile i+1's MMAs
//   warps 2-5  3xTF32 converters (lo = x - tf32(x) tiles); in a pair they also
//              relay "stage ready" to the rank-0 CTA's barrier
//   warps 6-9 (6-13) epilogue: tcgen05.ld -> fused epilogue -> 128-bit stores
// Pair protocol: full[s] / empty[s] are per CTA (local TMA, multicast MMA
// commit); conv[s] and tempty[b] live in the rank-0 CTA and count the arrivals
// of both CTAs' converter / epilogue warps; tfull[b] is multicast.
// BF = true: the bf16x3 path — operands arrive pre-split as bf16 (hi, lo)
// pairs (tmA / tmAl, tmB / tmBl), each stage holds the hi and lo halves of A
// and B (64 K-elements = 128-byte rows), the MMA warp issues lo*hi + hi*lo +
// hi*hi with kind::f16 (K = 16) and no converter pass exists (the converter
// warps only relay "stage ready" in a CTA pair).
template <int NCTA, int EPIW, bool BF>
__global__ void __launch_bounds__(threads_for<EPIW>(), 1)
    gemm_tf32_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmBl, const __grid_constant__ CUtensorMap tmAl,
                     const GemmArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t BN = args.BN;
  const uint32_t BNh = BN / NCTA;  // B rows (N) held by this CTA
  const uint32_t B_STAGE = BNh * BK * 4;  // BNh rows of 128 B (bf16: one of the two halves)
  const uint32_t A_STG = BF ? 2 * A_STAGE : A_STAGE;  // stage strides: bf16 stages hold hi and lo
  const uint32_t B_STG = BF ? 2 * B_STAGE : B_STAGE;
  const uint32_t S = args.stages;
  const bool split3 = args.split3 != 0;
  uint8_t* sA = smem;
  uint8_t* sB = smem + (size_t)S * A_STG;
  // 3xTF32 residual tiles (same swizzled layout) in a ring of L slots: the
  // converters of stage `it` write slot it % L once the MMAs of stage it - L
  // have drained it, so the TMA ring keeps S full stages in flight with only L
  // residual copies (the skinny GEMMs are bound by that TMA round trip)
  // With b_lo_tma the B residual (a small weight operand, reused by every
  // tile) is precomputed once per GEMM and TMA-loaded with each stage
  // (sBt[s]); the converters then only split A.
  const uint32_t L = split3 ? args.lo_slots : 0;
  const bool blt = split3 && args.b_lo_tma;
  uint8_t* sBt = sB + (size_t)S * B_STG;
  uint8_t* sAl = sBt + (blt ? (size_t)S * B_STAGE : 0);
  uint8_t* sBl = sAl + (size_t)L * A_STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sBl + (blt ? 0 : (size_t)L * B_STAGE));
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* conv = bars + 2 * S;
  uint64_t* tfull = bars + 3 * S;    // [2] accumulator ready
  uint64_t* tempty = bars + 3 * S + 2;  // [2] accumulator drained
  uint64_t* lo_empty = bars + 3 * S + 4;  // [L] residual slot drained by the MMAs
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 3 * S + 4 + kMaxLo);
  // epilogue staging: per epilogue warp a 32-row x 32-column tile, rows 144 B
  // apart (conflict-free 128-bit row and column-chunk accesses)
  float4* epi_tiles = reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(bars) + kBarBytes(S));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = NCTA == 2 ? cluster_rank() : 0;
  const uint32_t cid = blockIdx.x / NCTA, ncl = gridDim.x / NCTA;  // pair index / count
  // stage-ready signal the MMA waits on: the TMA barrier itself for a single
  // CTA in plain TF32, else the converters' (relay) barrier
  const bool via_conv = split3 || NCTA == 2;

  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < S; ++i) {
      mbar_init(smem_u32(full + i), 1);
      mbar_init(smem_u32(empty + i), 1);
      mbar_init(smem_u32(conv + i), kConvWarps * NCTA);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(tfull + b), 1);
      mbar_init(smem_u32(tempty + b), EPIW * NCTA);
    }
    for (uint32_t j = 0; j < L; ++j) mbar_init(smem_u32(lo_empty + j), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    if (NCTA == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                   "r"(args.tmem_cols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                   "r"(args.tmem_cols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (NCTA == 2) cluster_sync();  // barriers of both CTAs initialised before any remote arrive
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_holder;
  const uint32_t acc_cols = args.tmem_cols / 2;

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t bytes = BF ? A_STG + B_STG : A_STAGE + B_STAGE * (blt ? 2 : 1);
      const uint64_t ef = policy_evict_first();
      const uint64_t pol_a = args.a_stream ? ef : 0, pol_b = args.b_stream ? ef : 0;
      uint32_t it = 0;
      for (uint32_t t = cid; t < args.tiles; t += ncl) {
        uint32_t m0, n0, kb0, nkb;
        tile_coords(args, t, m0, n0, kb0, nkb);
        m0 += crank * BM;
        n0 += crank * BNh;
        for (uint32_t i = 0; i < nkb; ++i, ++it) {
          const uint32_t s = it % S, ph = (it / S) & 1;
          mbar_wait(smem_u32(empty + s), ph ^ 1, 0);
          mbar_expect_tx(smem_u32(full + s), bytes);
          const int kx = (int)((kb0 + i) * args.bk);
          if constexpr (BF) {
            const uint32_t fb = smem_u32(full + s);
            const uint32_t a0 = smem_u32(sA + (size_t)s * A_STG), b0 = smem_u32(sB + (size_t)s * B_STG);
            load_operand16(a0, &tmA, args.a_mn, kx, (int)m0, BM, fb);
            load_operand16(a0 + A_STAGE, &tmAl, args.a_mn, kx, (int)m0, BM, fb);
            load_operand16(b0, &tmB, args.b_mn, kx, (int)n0, BNh, fb);
            load_operand16(b0 + B_STAGE, &tmBl, args.b_mn, kx, (int)n0, BNh, fb);
          } else {
            load_operand(smem_u32(sA + (size_t)s * A_STAGE), &tmA, args.a_mn, kx, (int)m0, BM, smem_u32(full + s), pol_a);
            load_operand(smem_u32(sB + (size_t)s * B_STAGE), &tmB, args.b_mn, kx, (int)n0, BNh, smem_u32(full + s), pol_b);
            if (blt) load_operand(smem_u32(sBt + (size_t)s * B_STAGE), &tmBl, args.b_mn, kx, (int)n0, BNh, smem_u32(full + s), 0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && crank == 0) {
      uint32_t it = 0, j = 0;
      for (uint32_t t = cid; t < args.tiles; t += ncl, ++j) {
        uint32_t m0, n0, kb0, nkb;
        tile_coords(args, t, m0, n0, kb0, nkb);
        const uint32_t b = j & 1;
        mbar_wait(smem_u32(tempty + b), ((j >> 1) & 1) ^ 1, 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + b * acc_cols;
        const bool amn = args.a_mn != 0, bmn = args.b_mn != 0;
        for (uint32_t i = 0; i < nkb; ++i, ++it) {
          const uint32_t s = it % S, ph = (it / S) & 1;
          mbar_wait(smem_u32(via_conv ? conv + s : full + s), ph, 2);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a0 = smem_u32(sA + (size_t)s * A_STG);
          const uint32_t b0 = smem_u32(sB + (size_t)s * B_STG);
          if constexpr (BF) {  // small terms first: lo*hi, hi*lo, then hi*hi
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {  // K = 16 bf16 (32 bytes) per instruction
              const uint32_t first = (i > 0 || ks > 0) ? 1u : 0u;
              mma_bf16<NCTA>(acc, op_desc16(a0 + A_STAGE, ks, amn), op_desc16(b0, ks, bmn), args.idesc, first);
              mma_bf16<NCTA>(acc, op_desc16(a0, ks, amn), op_desc16(b0 + B_STAGE, ks, bmn), args.idesc, 1u);
              mma_bf16<NCTA>(acc, op_desc16(a0, ks, amn), op_desc16(b0, ks, bmn), args.idesc, 1u);
            }
            commit_to<NCTA>(smem_u32(empty + s));
            continue;
          }
          const uint32_t lj = split3 ? it % L : 0;
          const uint32_t al = smem_u32(sAl + (size_t)lj * A_STAGE);
          const uint32_t bl = blt ? smem_u32(sBt + (size_t)s * B_STAGE) : smem_u32(sBl + (size_t)lj * B_STAGE);
#pragma unroll
          for (int ks = 0; ks < BK / 8; ++ks) {  // K = 8 tf32 (32 bytes) per instruction
            const uint32_t first = (i > 0 || ks > 0) ? 1u : 0u;
            if (NCTA == 2) {
              if (split3) {  // small terms first
                mma_tf32_pair(acc, op_desc(al, ks, amn), op_desc(b0, ks, bmn), args.idesc, first);
                mma_tf32_pair(acc, op_desc(a0, ks, amn), op_desc(bl, ks, bmn), args.idesc, 1u);
                mma_tf32_pair(acc, op_desc(a0, ks, amn), op_desc(b0, ks, bmn), args.idesc, 1u);
              } else {
                mma_tf32_pair(acc, op_desc(a0, ks, amn), op_desc(b0, ks, bmn), args.idesc, first);
              }
            } else {
              if (split3) {
                mma_tf32(acc, op_desc(al, ks, amn), op_desc(b0, ks, bmn), args.idesc, first);
                mma_tf32(acc, op_desc(a0, ks, amn), op_desc(bl, ks, bmn), args.idesc, 1u);
                mma_tf32(acc, op_desc(a0, ks, amn), op_desc(b0, ks, bmn), args.idesc, 1u);
              } else {
                mma_tf32(acc, op_desc(a0, ks, amn), op_desc(b0, ks, bmn), args.idesc, first);
              }
            }
          }
          commit_to<NCTA>(smem_u32(empty + s));
          if (split3) commit_to<NCTA>(smem_u32(lo_empty + lj));
        }
        if (nkb) {
          commit_to<NCTA>(smem_u32(tfull + b));
        } else {  // empty K range: the epilogue writes zeros
          mbar_arrive(smem_u32(tfull + b));
          if (NCTA == 2) mbar_arrive_cta(smem_u32(tfull + b), 1);
        }
      }
    }
    __syncwarp();
  } else if (warp < kEpiWarp0) {
    if (via_conv) {
      const uint32_t tt = threadIdx.x - 64;
      const uint32_t a4 = A_STAGE / 16, b4 = B_STAGE / 16;
      uint32_t it = 0;
      for (uint32_t t = cid; t < args.tiles; t += ncl) {
        uint32_t m0, n0, kb0, nkb;
        tile_coords(args, t, m0, n0, kb0, nkb);
        for (uint32_t i = 0; i < nkb; ++i, ++it) {
          const uint32_t s = it % S, ph = (it / S) & 1;
          mbar_wait(smem_u32(full + s), ph, 3);
          if (split3) {
            const uint32_t lj = it % L, lph = (it / L) & 1;
            mbar_wait(smem_u32(lo_empty + lj), lph ^ 1, 4);  // the MMAs of stage it - L are done with slot lj
            convert_tile(smem_u32(sA + (size_t)s * A_STAGE), smem_u32(sAl + (size_t)lj * A_STAGE), a4, tt);
            if (!blt) convert_tile(smem_u32(sB + (size_t)s * B_STAGE), smem_u32(sBl + (size_t)lj * B_STAGE), b4, tt);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          }
          __syncwarp();
          if (lane == 0) {
            if (NCTA == 2) mbar_arrive_cta(smem_u32(conv + s), 0);
            else mbar_arrive(smem_u32(conv + s));
          }
        }
      }
    }
  } else {
    const uint32_t q = warp & 3;  // TMEM lane quarter this warp may access
    const uint32_t ew = warp - kEpiWarp0;  // epilogue warp index
    const uint32_t chalf = ew / 4;          // with 8 warps: chunks c = 32*(chalf + 2i)
    constexpr uint32_t kCStep = 32 * (EPIW / 4);
    const GemmEpi& e = args.epi;
    uint32_t j = 0;
    for (uint32_t t = cid; t < args.tiles; t += ncl, ++j) {
      uint32_t m0, n0, kb0, nkb;
      tile_coords(args, t, m0, n0, kb0, nkb);
      m0 += crank * BM;
      const uint32_t b = j & 1;
      mbar_wait(smem_u32(tfull + b), (j >> 1) & 1, 5);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t row = m0 + q * 32 + lane;
      const bool row_ok = row < args.M;
      const float rs = (row_ok && e.rowscale) ? __ldg(e.rowscale + row) : 1.f;
      const uint32_t z = t / (args.nt * args.mt);
      float4* T = epi_tiles + ew * (32 * kTileLd4);
      const uint32_t r8 = lane >> 3, c4 = lane & 7;
      const uint32_t rbase = m0 + q * 32;
      // ReLU-backward mask words are fetched one 32-column chunk ahead, so the
      // global load latency overlaps the previous chunk's TMEM drain and stores
      // (a whole-tile prefetch with the chunk loop unrolled measured slower)
      const uint32_t* mrow = (e.mask_bits && row_ok) ? e.mask_bits + (size_t)row * e.mask_words : nullptr;
      const uint32_t cfirst = 32 * chalf;
      float rmax = 0.f;  // max |v| of this row over the chunks this warp stores (e.rowmax)
      uint32_t mw_next = (mrow && cfirst < BN && n0 + cfirst < args.N) ? __ldg(mrow + (n0 + cfirst) / 32) : 0xffffffffu;
      for (uint32_t c = cfirst; c < BN; c += kCStep) {
        const uint32_t mw_cur = mw_next;
        if (mrow && n0 + c + kCStep < args.N && c + kCStep < BN) mw_next = __ldg(mrow + (n0 + c + kCStep) / 32);
        float v[32];
        if (nkb) {
          tmem_ld32(tmem + b * acc_cols + ((q * 32u) << 16) + c, v);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0.f;
        }
        const uint32_t col0 = n0 + c;
        if (col0 >= args.N) continue;  // warp-uniform
        // Outputs are staged through shared memory so a warp writes whole
        // 128-byte lines (its lanes own 32 different rows); the ReLU-backward
        // mask is one 32-bit word per row and chunk, and ReLU layers emit the
        // same word for their own backward (bits_out).
        // columns this chunk stores through the staging tile: a whole chunk, or
        // the ragged tail when the caller lets the padding up to store_cols be
        // written (a multiple of 4 columns)
        const uint32_t ns = max(args.N, e.store_cols);
        const uint32_t nc = min(32u, ns - col0);
        if (!e.partial && (nc == 32 || (e.store_cols && nc % ((e.out_h || e.out_bhi) ? 8 : 4) == 0))) {
          const uint32_t mw = mrow ? mw_cur : 0xffffffffu;
          uint32_t bw = 0;
          // fp16-only output of a whole chunk: each lane's row segment is 64
          // contiguous bytes (two sectors), stored straight from registers —
          // no staging round trip (the skinny-K GEMMs are epilogue bound)
          // (the residual output only in the 4-epilogue-warp kernels: the 8-warp
          // ones are capped at 128 registers)
          const bool direct = e.out_h && !e.out && !e.out_bhi && nc % 8 == 0 && (EPIW == 4 || !e.out_hl);
          uint32_t hw[16];
          uint32_t lw[EPIW == 4 ? 16 : 1];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float4 o = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
            if (e.rowscale && col0 + 4 * i >= e.scale_col_begin) { o.x *= rs; o.y *= rs; o.z *= rs; o.w *= rs; }
            if (e.bias) {
              const float4 bb = __ldg(reinterpret_cast<const float4*>(e.bias + col0) + i);
              o.x += bb.x; o.y += bb.y; o.z += bb.z; o.w += bb.w;
            }
            if (e.relu) {
              o.x = fmaxf(o.x, 0.f); o.y = fmaxf(o.y, 0.f); o.z = fmaxf(o.z, 0.f); o.w = fmaxf(o.w, 0.f);
            }
            if (e.mask_bits) {
              const uint32_t nib = mw >> (4 * i);
              o.x = (nib & 1u) ? o.x : 0.f; o.y = (nib & 2u) ? o.y : 0.f;
              o.z = (nib & 4u) ? o.z : 0.f; o.w = (nib & 8u) ? o.w : 0.f;
            }
            o.x *= e.out_scale; o.y *= e.out_scale; o.z *= e.out_scale; o.w *= e.out_scale;
            bw |= ((o.x > 0.f) | ((o.y > 0.f) << 1) | ((o.z > 0.f) << 2) | ((o.w > 0.f) << 3)) << (4 * i);
            if (e.rowmax && 4 * i < nc)
              rmax = fmaxf(rmax, fmaxf(fmaxf(fabsf(o.x), fabsf(o.y)), fmaxf(fabsf(o.z), fabsf(o.w))));
            if (direct) {
              hw[2 * i] = pack_h2(o.x, o.y);
              hw[2 * i + 1] = pack_h2(o.z, o.w);
              if constexpr (EPIW == 4) {
                if (e.out_hl) {  // rounding residual, scaled into the fp16 normal range
                  const float2 h0 = __half22float2(*reinterpret_cast<const __half2*>(&hw[2 * i]));
                  const float2 h1 = __half22float2(*reinterpret_cast<const __half2*>(&hw[2 * i + 1]));
                  lw[2 * i] = pack_h2((o.x - h0.x) * 2048.f, (o.y - h0.y) * 2048.f);
                  lw[2 * i + 1] = pack_h2((o.z - h1.x) * 2048.f, (o.w - h1.y) * 2048.f);
                }
              }
            } else {
              T[lane * kTileLd4 + i] = o;
            }
          }
          if (direct) {
            if (nc < 32) bw &= (1u << nc) - 1u;
            if (e.bits_out && row_ok) e.bits_out[(size_t)row * e.bits_words + col0 / 32] = bw;
            if (row_ok) {
              const size_t o = (size_t)row * (e.ld_h ? e.ld_h : e.ld_out) + e.out_col + col0;
              uint4* dst = reinterpret_cast<uint4*>(e.out_h + o);
#pragma unroll
              for (int k = 0; k < 4; ++k)
                if (8 * k < (int)nc) dst[k] = make_uint4(hw[4 * k], hw[4 * k + 1], hw[4 * k + 2], hw[4 * k + 3]);
              if constexpr (EPIW == 4) {
                if (e.out_hl) {
                  uint4* dl = reinterpret_cast<uint4*>(e.out_hl + o);
#pragma unroll
                  for (int k = 0; k < 4; ++k)
                    if (8 * k < (int)nc) dl[k] = make_uint4(lw[4 * k], lw[4 * k + 1], lw[4 * k + 2], lw[4 * k + 3]);
                }
              }
            }
            continue;
          }
          if (nc < 32) bw &= (1u << nc) - 1u;  // staged columns past the stored ones are not results
          if (e.bits_out && row_ok) e.bits_out[(size_t)row * e.bits_words + col0 / 32] = bw;
          __syncwarp();
          if (e.out_h) {  // fp16 rows: nc/8 16-byte vectors per row, consecutive lanes along the row
            const uint32_t n8 = nc / 8;
            for (uint32_t f = lane; f < 32 * n8; f += 32) {
              const uint32_t rr = f / n8, cc = f % n8, grow = rbase + rr;
              if (grow < args.M) {
                const float4 a = T[rr * kTileLd4 + 2 * cc], b = T[rr * kTileLd4 + 2 * cc + 1];
                const uint4 h = make_uint4(pack_h2(a.x, a.y), pack_h2(a.z, a.w), pack_h2(b.x, b.y), pack_h2(b.z, b.w));
                const size_t o = (size_t)grow * (e.ld_h ? e.ld_h : e.ld_out) + e.out_col + col0;
                reinterpret_cast<uint4*>(e.out_h + o)[cc] = h;
                if (e.out_hl) {  // rounding residual, scaled into the fp16 normal range
                  const __half2* hh = reinterpret_cast<const __half2*>(&h);
                  const float2 h0 = __half22float2(hh[0]), h1 = __half22float2(hh[1]);
                  const float2 h2 = __half22float2(hh[2]), h3 = __half22float2(hh[3]);
                  reinterpret_cast<uint4*>(e.out_hl + o)[cc] =
                      make_uint4(pack_h2((a.x - h0.x) * 2048.f, (a.y - h0.y) * 2048.f),
                                 pack_h2((a.z - h1.x) * 2048.f, (a.w - h1.y) * 2048.f),
                                 pack_h2((b.x - h2.x) * 2048.f, (b.y - h2.y) * 2048.f),
                                 pack_h2((b.z - h3.x) * 2048.f, (b.w - h3.y) * 2048.f));
                }
              }
            }
          }
          if (e.out_bhi) {  // bf16x3 pair rows: nc/8 16-byte vectors per row and half
            const uint32_t n8 = nc / 8;
            for (uint32_t f = lane; f < 32 * n8; f += 32) {
              const uint32_t rr = f / n8, cc = f % n8, grow = rbase + rr;
              if (grow < args.M) {
                const float4 a = T[rr * kTileLd4 + 2 * cc], b = T[rr * kTileLd4 + 2 * cc + 1];
                const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
                uint32_t hw[4], lw[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  const __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
                  const __nv_bfloat162 l = __floats2bfloat162_rn(v[2 * k] - __low2float(h), v[2 * k + 1] - __high2float(h));
                  hw[k] = *reinterpret_cast<const uint32_t*>(&h);
                  lw[k] = *reinterpret_cast<const uint32_t*>(&l);
                }
                const size_t o = (size_t)grow * (e.ld_h ? e.ld_h : e.ld_out) + e.out_col + col0;
                reinterpret_cast<uint4*>(e.out_bhi + o)[cc] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                reinterpret_cast<uint4*>(e.out_blo + o)[cc] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
              }
            }
          }
          if (e.out && nc == 32) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const uint32_t rr = 4 * i + r8, grow = rbase + rr;
              if (grow < args.M)
                reinterpret_cast<float4*>(e.out + (size_t)grow * e.ld_out + e.out_col + col0)[c4] = T[rr * kTileLd4 + c4];
            }
          } else if (e.out) {  // ragged tail: nc/4 float4 per row, consecutive lanes along the row
            const uint32_t n4 = nc / 4;
            for (uint32_t f = lane; f < 32 * n4; f += 32) {
              const uint32_t rr = f / n4, cc = f % n4, grow = rbase + rr;
              if (grow < args.M)
                reinterpret_cast<float4*>(e.out + (size_t)grow * e.ld_out + e.out_col + col0)[cc] = T[rr * kTileLd4 + cc];
            }
          }
          __syncwarp();
          continue;
        }
        if (!row_ok) continue;
        if (e.partial) {
          float* dst = e.partial + ((size_t)z * args.M + row) * args.N + col0;
          if (col0 + 32 <= args.N && (args.N & 3) == 0) {
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
            continue;
          }
        }
        if (!row_ok) continue;
        if (e.partial) {
          float* dst = e.partial + ((size_t)z * args.M + row) * args.N + col0;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (col0 + i < args.N) dst[i] = v[i];
          continue;
        }
        uint32_t bw = 0;
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (col0 + i < args.N) {
            const float o = apply_epi(e, row, col0 + i, v[i]);
            store_epi(e, row, col0 + i, o);
            bw |= (uint32_t)(o > 0.f) << i;
          }
        if (e.bits_out) e.bits_out[(size_t)row * e.bits_words + col0 / 32] = bw;
      }
      if (e.rowmax && row_ok && rmax > 0.f) atomicMax(reinterpret_cast<int*>(e.rowmax) + row, __float_as_int(rmax));
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if (NCTA == 2) mbar_arrive_cta(smem_u32(tempty + b), 0);
        else mbar_arrive(smem_u32(tempty + b));
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (NCTA == 2) cluster_sync();  // the peer's MMAs / remote arrivals are done
  else __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (NCTA == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(args.tmem_cols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(args.tmem_cols));
  }
}
__global__ void gemm_reduce_kernel(const float* __restrict__ partial, uint32_t splits, uint32_t M,
                                   uint32_t N, GemmEpi e) {
  const uint64_t total = (uint64_t)M * N;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (uint32_t z = 0; z < splits; ++z) acc += partial[(uint64_t)z * total + i];
    const uint32_t row = (uint32_t)(i / N), col = (uint32_t)(i % N);
    store_epi(e, row, col, apply_epi(e, row, col, acc));
  }
}
// Split-K sums of a plain fp32 output (the weight gradients: no epilogue ops),
// four columns per thread, four splits' loads in flight, summed in split order
// (the same order as gemm_reduce_kernel: deterministic, identical results).
__global__ void gemm_reduce4_kernel(const float4* __restrict__ partial, uint32_t splits, uint32_t M, uint32_t N,
                                    float* __restrict__ out, uint32_t ld_out, uint32_t out_col) {
  const uint64_t total4 = (uint64_t)M * N / 4;
  const uint32_t n4 = N / 4;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total4;
       i += (uint64_t)gridDim.x * blockDim.x) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    uint32_t z = 0;
    for (; z + 3 < splits; z += 4) {
      const float4 a = __ldcg(partial + (uint64_t)z * total4 + i), b = __ldcg(partial + (uint64_t)(z + 1) * total4 + i);
      const float4 c = __ldcg(partial + (uint64_t)(z + 2) * total4 + i), d = __ldcg(partial + (uint64_t)(z + 3) * total4 + i);
      acc.x += a.x; acc.y += a.y; acc.z += a.z; acc.w += a.w;
      acc.x += b.x; acc.y += b.y; acc.z += b.z; acc.w += b.w;
      acc.x += c.x; acc.y += c.y; acc.z += c.z; acc.w += c.w;
      acc.x += d.x; acc.y += d.y; acc.z += d.z; acc.w += d.w;
    }
    for (; z < splits; ++z) {
      const float4 a = __ldcg(partial + (uint64_t)z * total4 + i);
      acc.x += a.x; acc.y += a.y; acc.z += a.z; acc.w += a.w;
    }
    const uint32_t row = (uint32_t)(i / n4), c4 = (uint32_t)(i % n4);
    *reinterpret_cast<float4*>(out + (size_t)row * ld_out + out_col + c4 * 4) = acc;
  }
}
// the split-K reduction: the vectorised kernel when the output is a plain
// 16-byte aligned fp32 matrix, else the general one
void launch_reduce(catgnn_ctx ctx, const float* partial, uint32_t splits, uint32_t M, uint32_t N, const GemmEpi& epi) {
  const bool plain = epi.out && !epi.out_h && !epi.out_bhi && !epi.rowscale && !epi.bias && !epi.relu &&
                     !epi.mask_bits && !epi.bits_out && !epi.rowmax && epi.out_scale == 1.0f && N % 4 == 0 &&
                     epi.ld_out % 4 == 0 && epi.out_col % 4 == 0;
  const uint64_t total = (uint64_t)M * N;
  if (plain) {
    const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((total / 4 + 255) / 256, 148 * 16));
    gemm_reduce4_kernel<<<g, 256, 0, ctx->stream>>>(reinterpret_cast<const float4*>(partial), splits, M, N, epi.out,
                                                    epi.ld_out, epi.out_col);
  } else {
    const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((total + 255) / 256, 148 * 16));
    gemm_reduce_kernel<<<g, 256, 0, ctx->stream>>>(partial, splits, M, N, epi);
  }
  CG_CHECK_LAUNCH();
  ctx->launches++;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  if (!fn) throw InternalError("cuTensorMapEncodeTiled unavailable");
  return fn;
}

CUtensorMap make_map(const float* ptr, uint64_t rows, uint64_t K, uint32_t ld, uint32_t box_rows) {
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (ld * 4) % 16)
    throw ConfigError("GEMM operand must be 16-byte aligned with a row stride multiple of 4 floats");
  CUtensorMap m;
  cuuint64_t dims[2] = {K, rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {BK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides,
                           box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw InternalError("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return m;
}

// MN-major operand stored row-major as [K rows][MN cols]: inner dim = MN,
// {32 x 32} boxes (128-byte inner rows for SWIZZLE_128B); OOB zero-filled.
CUtensorMap make_map_mn(const float* ptr, uint64_t mn, uint64_t K, uint32_t ld) {
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (ld * 4) % 16)
    throw ConfigError("GEMM operand must be 16-byte aligned with a row stride multiple of 4 floats");
  CUtensorMap m;
  cuuint64_t dims[2] = {mn, K};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {32, BK};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides,
                           box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw InternalError("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return m;
}

uint32_t pow2_cols(uint32_t n) {
  uint32_t c = 32;
  while (c < n) c <<= 1;
  return c;
}

}  // namespace

void check_epi_output(const GemmEpi& epi) {
  if (!epi.out && !epi.out_h && !epi.out_bhi) throw ConfigError("GEMM needs an output");
  if (epi.out_bhi && (!epi.out_blo || !epi.store_cols || epi.store_cols % 8 || ((epi.ld_h ? epi.ld_h : epi.ld_out) % 8)))
    throw ConfigError("GEMM bf16 pair output: hi and lo, store_cols and row stride multiples of 8");
  if (epi.out && epi.out_h && !epi.store_cols) throw ConfigError("GEMM fp32 + fp16 outputs need store_cols");
  if (epi.rowmax && !epi.store_cols) throw ConfigError("GEMM row max needs store_cols (staged epilogue)");
  if (epi.out_hl && (!epi.out_h || !epi.store_cols)) throw ConfigError("GEMM fp16 residual needs out_h and store_cols");
  if ((epi.ld_out % 4) || (epi.out_col % 4)) throw ConfigError("GEMM output stride must be a multiple of 4");
  if (epi.out_h && (((epi.ld_h ? epi.ld_h : epi.ld_out) % 8) || (epi.out_col % 8) || (epi.store_cols % 8)))
    throw ConfigError("GEMM fp16 output: stride, column and store_cols must be multiples of 8");
  if (!(epi.out_scale > 0.f)) throw ConfigError("GEMM out_scale must be positive");
}

void gemm_tn(catgnn_ctx ctx, const float* A, uint32_t lda, const float* B, uint32_t ldb, uint32_t M,
             uint32_t N, uint32_t K, const GemmEpi& epi_in, uint32_t split_k, int precision) {
  gemm(ctx, GemmOperand{A, lda, false}, GemmOperand{B, ldb, false}, M, N, K, epi_in, split_k, precision);
}

void gemm(catgnn_ctx ctx, GemmOperand a, GemmOperand b, uint32_t M, uint32_t N, uint32_t K,
          const GemmEpi& epi_in, uint32_t split_k, int precision) {
  const float* A = a.ptr;
  const float* B = b.ptr;
  const uint32_t lda = a.ld, ldb = b.ld;
  if (M == 0 || N == 0) return;
  GemmEpi epi = epi_in;
  check_epi_output(epi);
  if (epi.store_cols && (epi.store_cols % 4 || epi.store_cols < N || epi.out_col + epi.store_cols > epi.ld_out))
    throw ConfigError("GEMM store_cols must be a multiple of 4 in [N, ld_out - out_col]");
  if (K == 0) {  // empty contraction: the epilogue of a zero accumulator
    const uint64_t total = (uint64_t)M * N;
    unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((total + 255) / 256, 148 * 16));
    gemm_reduce_kernel<<<g, 256, 0, ctx->stream>>>(nullptr, 0, M, N, epi);
    CG_CHECK_LAUNCH();
    ctx->launches++;
    return;
  }
  const bool split3 = precision == 3;
  // CTA pairs (cta_group::2, 256-row tiles) halve each SM's operand traffic —
  // the SMEM port, not the tensor pipe, bounds the 3xTF32 main loop
  static const int pair_env = [] {
    const char* v = std::getenv("CATGNN_GEMM_PAIR");
    return v ? std::atoi(v) : 1;
  }();
  // (skinny N: the pair's per-tile handshakes outweigh the halved B traffic)
  const bool pair = pair_env != 0 && M >= 256 && N >= 128;
  const uint32_t ncta = pair ? 2 : 1;
  // 3xTF32 doubles the stage (lo tiles): single-CTA 128-wide N tiles keep 3 stages in flight
  const uint32_t bn_max = (split3 && !pair) ? 128 : 256;
  // per-CTA B rows must be whole 8-row swizzle groups (K-major) or 32-wide atoms (MN-major)
  const uint32_t bn_q = (b.mn_major ? 32 : 16) * ncta;
  const uint32_t BN = N >= bn_max ? bn_max : round_up(N, bn_q);
  const uint32_t BNh = BN / ncta;
  const uint32_t nkb = (K + BK - 1) / BK;
  const uint32_t bm = BM * ncta;
  const uint32_t mt = (M + bm - 1) / bm, nt = (N + BN - 1) / BN;
  const uint32_t gsms = ctx->gemm_sms ? std::max<uint32_t>(ncta, (uint32_t)ctx->gemm_sms) : (uint32_t)ctx->num_sms;
  const uint32_t units = gsms / ncta;  // persistent CTAs (pairs)
  uint32_t splits = 1;
  if (split_k == 0) {
    // fill the SMs when the tile grid is small and K is long
    const uint32_t tiles = mt * nt;
    if (tiles < units && nkb >= 8)
      splits = std::min<uint32_t>(std::max<uint32_t>(1, units / tiles), nkb / 4);
  } else {
    splits = std::min<uint32_t>(split_k, std::max<uint32_t>(1, nkb));
  }
  splits = std::max<uint32_t>(1, splits);
  const uint32_t kbps = std::max<uint32_t>(1, (nkb + splits - 1) / splits);
  splits = std::max<uint32_t>(1, (nkb + kbps - 1) / kbps);
  if ((epi.bits_out || epi.rowmax) && splits > 1) throw ConfigError("GEMM bit / row-max output needs an unsplit K");
  if (epi.bias && (reinterpret_cast<uintptr_t>(epi.bias) & 15))
    throw ConfigError("GEMM epilogue operands must be 16-byte aligned");

  const uint32_t b_stage = BNh * BK * 4;
  // (a precomputed, TMA-loaded B residual — b_lo_tma — measured no faster on
  // reddit and is not used by the host: the converters split both operands)
  const bool blt = false;
  const size_t stage_bytes = (size_t)A_STAGE + (size_t)b_stage * (blt ? 2 : 1);
  const size_t lo_bytes = (size_t)A_STAGE + (blt ? 0 : (size_t)b_stage);  // one residual slot
  static const int lo_env = [] {
    const char* v = std::getenv("CATGNN_GEMM_LO_SLOTS");
    return v ? std::atoi(v) : 2;
  }();
  // short K loops (<= 4 k-blocks per tile, no split-K partials) are bound by the
  // accumulator drain: 8 epilogue warps; otherwise 4 (more warps slow the
  // compute-bound GEMMs through issue contention)
  static const int epi_env = [] {
    const char* v = std::getenv("CATGNN_GEMM_EPI_WARPS");
    return v ? std::atoi(v) : 0;
  }();
  const int epiw = epi_env == 4 || epi_env == 8 ? epi_env : (nkb <= 4 && splits == 1 ? 8 : 4);
  const size_t kEpiSmem = epi_smem(epiw);
  const size_t budget = 227 * 1024 - 1024 - kBarBytes(kMaxStages) - kEpiSmem;
  uint32_t stages, lo_slots = 0;
  if (split3 && lo_env > 0) {
    lo_slots = (uint32_t)std::min<int>(lo_env, (int)kMaxLo);
    stages = (uint32_t)std::min<size_t>(kMaxStages, (budget - lo_slots * lo_bytes) / stage_bytes);
  } else if (split3) {  // CATGNN_GEMM_LO_SLOTS=0: one residual copy per stage (previous layout)
    stages = (uint32_t)std::min<size_t>(6, budget / (stage_bytes + lo_bytes));
    lo_slots = stages;
  } else {
    stages = (uint32_t)std::min<size_t>(kMaxStages, budget / stage_bytes);
  }
  if (stages < 2) throw InternalError("GEMM tile does not fit in shared memory");
  const size_t smem = 1024 + (size_t)stages * stage_bytes + (size_t)lo_slots * lo_bytes + kBarBytes(stages) + kEpiSmem;

  GemmArgs args{};
  args.M = M;
  args.N = N;
  args.K = K;
  args.BN = BN;
  args.stages = stages;
  args.lo_slots = lo_slots;
  args.b_lo_tma = blt ? 1u : 0u;
  args.kb_per_split = kbps;
  args.tmem_cols = pow2_cols(2 * round_up(BN, 32));  // two accumulator buffers
  args.split3 = split3 ? 1u : 0u;
  args.bk = BK;
  args.mt = mt;
  args.nt = nt;
  args.splits = splits;
  args.tiles = mt * nt * splits;
  args.a_mn = a.mn_major ? 1u : 0u;
  args.b_mn = b.mn_major ? 1u : 0u;
  args.bm = bm;
  args.a_stream = args.b_stream = 0u;  // evict-first operand loads measured slower on the reddit step
  // instruction descriptor: D f32, A/B tf32, A/B major (bit 15/16), N>>3, M>>4
  args.idesc = (1u << 4) | (2u << 7) | (2u << 10) | (args.a_mn << 15) | (args.b_mn << 16) | ((BN >> 3) << 17) |
               ((bm >> 4) << 24);
  float* partial = nullptr;
  if (splits > 1) {
    partial = ctx->scratch_buf<float>("gemm_partial", (size_t)splits * M * N);
    args.epi = epi;
    args.epi.partial = partial;
  } else {
    args.epi = epi;
    args.epi.partial = nullptr;
  }
  CUtensorMap ta = a.mn_major ? make_map_mn(A, M, K, lda) : make_map(A, M, K, lda, BM);
  CUtensorMap tb = b.mn_major ? make_map_mn(B, N, K, ldb) : make_map(B, N, K, ldb, BNh);
  const CUtensorMap& tbl = tb;
  // cudaFuncSetAttribute is per device: one flag set per device ordinal
  static std::mutex attr_mu;
  static std::map<int, std::array<bool, 4>> attr_set;
  auto kern = pair ? (epiw == 8 ? gemm_tf32_kernel<2, 8, false> : gemm_tf32_kernel<2, 4, false>)
                   : (epiw == 8 ? gemm_tf32_kernel<1, 8, false> : gemm_tf32_kernel<1, 4, false>);
  const int kThreads = epiw == 8 ? threads_for<8>() : threads_for<4>();
  {
    std::lock_guard<std::mutex> lk(attr_mu);
    bool& done = attr_set[ctx->device][(ncta - 1) * 2 + (epiw == 8)];
    if (!done) {
      CG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      done = true;
    }
  }
  // timing label: the GEMM's shape class (row-sized extents as "rows")
  auto dim = [](uint32_t x) { return x > 4096 ? std::string("rows") : std::to_string(x); };
  int t = ctx->begin_timed(1, ctx->timing ? "K3 gemm M=" + dim(M) + " N=" + dim(N) + " K=" + dim(K) +
                                             (pair ? " pair" : "") + (splits > 1 ? " split-K" : "")
                                       : std::string());
  const unsigned grid = std::min<unsigned>(args.tiles, units) * ncta;  // persistent
  if (pair) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CG_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, tbl, ta, args));
  } else {
    kern<<<grid, kThreads, smem, ctx->stream>>>(ta, tb, tbl, ta, args);
  }
  CG_CHECK_LAUNCH();
  ctx->launches++;
  if (splits > 1) launch_reduce(ctx, partial, splits, M, N, epi);
  ctx->end_timed(t);
}

namespace {

CUtensorMap make_map16(const __nv_bfloat16* ptr, uint64_t rows, uint64_t K, uint32_t ld, uint32_t box_rows) {
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (ld * 2) % 16)
    throw ConfigError("bf16 GEMM operand must be 16-byte aligned with a row stride multiple of 8 elements");
  CUtensorMap m;
  cuuint64_t dims[2] = {K, rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16*>(ptr), dims, strides,
                           box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw InternalError("cuTensorMapEncodeTiled (bf16) failed: " + std::to_string((int)r));
  return m;
}

// MN-major bf16 operand stored [K rows][MN cols]: {64 (MN) x 64 (K)} boxes, 128-byte
// inner rows, SWIZZLE_128B; OOB zero-filled.
CUtensorMap make_map16_mn(const __nv_bfloat16* ptr, uint64_t mn, uint64_t K, uint32_t ld) {
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (ld * 2) % 16)
    throw ConfigError("bf16 GEMM operand must be 16-byte aligned with a row stride multiple of 8 elements");
  CUtensorMap m;
  cuuint64_t dims[2] = {mn, K};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64, 64};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16*>(ptr), dims, strides,
                           box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw InternalError("cuTensorMapEncodeTiled (bf16, MN-major) failed: " + std::to_string((int)r));
  return m;
}

// hi = bf16(x) (round to nearest), lo = bf16(x - hi): x = hi + lo to ~2^-17
__global__ void split_bf16_kernel(const float* __restrict__ in, uint32_t ld_in, uint64_t rows, uint32_t cols,
                                  __nv_bfloat16* __restrict__ hi, __nv_bfloat16* __restrict__ lo, uint32_t ld_out) {
  const uint32_t q = ld_out / 2;  // bf16 pairs per output row
  const uint64_t total = rows * q;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = i / q;
    const uint32_t c = (uint32_t)(i % q) * 2;
    const float x0 = c < cols ? in[r * ld_in + c] : 0.f;
    const float x1 = c + 1 < cols ? in[r * ld_in + c + 1] : 0.f;
    const __nv_bfloat162 h = __floats2bfloat162_rn(x0, x1);
    const __nv_bfloat162 l = __floats2bfloat162_rn(x0 - __low2float(h), x1 - __high2float(h));
    reinterpret_cast<__nv_bfloat162*>(hi + r * ld_out)[c / 2] = h;
    reinterpret_cast<__nv_bfloat162*>(lo + r * ld_out)[c / 2] = l;
  }
}

}  // namespace

void split_bf16(catgnn_ctx ctx, const float* in, uint32_t ld_in, uint64_t rows, uint32_t cols, __nv_bfloat16* hi,
                __nv_bfloat16* lo, uint32_t ld_out) {
  if (ld_out % 2 || cols > ld_out) throw ConfigError("split_bf16: output stride must be even and >= cols");
  const uint64_t total = rows * (ld_out / 2);
  if (!total) return;
  const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((total + 255) / 256, (uint64_t)ctx->num_sms * 16));
  split_bf16_kernel<<<g, 256, 0, ctx->stream>>>(in, ld_in, rows, cols, hi, lo, ld_out);
  CG_CHECK_LAUNCH();
  ctx->launches++;
}

void gemm_bf16x3(catgnn_ctx ctx, SplitOperand a, SplitOperand b, uint32_t M, uint32_t N, uint32_t K,
                 const GemmEpi& epi_in, uint32_t split_k) {
  if (M == 0 || N == 0) return;
  GemmEpi epi = epi_in;
  check_epi_output(epi);
  if (epi.store_cols && (epi.store_cols % 4 || epi.store_cols < N || epi.out_col + epi.store_cols > epi.ld_out))
    throw ConfigError("GEMM store_cols must be a multiple of 4 in [N, ld_out - out_col]");
  if (K == 0) {
    const uint64_t total = (uint64_t)M * N;
    unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((total + 255) / 256, 148 * 16));
    gemm_reduce_kernel<<<g, 256, 0, ctx->stream>>>(nullptr, 0, M, N, epi);
    CG_CHECK_LAUNCH();
    ctx->launches++;
    return;
  }
  constexpr uint32_t BKE = 64;  // bf16 elements per k-block (128-byte rows)
  static const int pair_env = [] {
    const char* v = std::getenv("CATGNN_GEMM_PAIR");
    return v ? std::atoi(v) : 1;
  }();
  const bool pair = pair_env != 0 && M >= 256 && N >= 128;
  const uint32_t ncta = pair ? 2 : 1;
  // per-CTA B rows: whole 8-row swizzle groups (K-major) or 64-wide atoms (MN-major)
  const uint32_t bn_q = (b.mn_major ? 64 : 16) * ncta;
  const uint32_t BN = N >= 256 ? 256 : round_up(N, bn_q);
  const uint32_t BNh = BN / ncta;
  const uint32_t nkb = (K + BKE - 1) / BKE;
  const uint32_t bm = BM * ncta;
  const uint32_t mt = (M + bm - 1) / bm, nt = (N + BN - 1) / BN;
  const uint32_t gsms = ctx->gemm_sms ? std::max<uint32_t>(ncta, (uint32_t)ctx->gemm_sms) : (uint32_t)ctx->num_sms;
  const uint32_t units = gsms / ncta;
  uint32_t splits = 1;
  if (split_k == 0) {
    const uint32_t tiles = mt * nt;
    if (tiles < units && nkb >= 8) splits = std::min<uint32_t>(std::max<uint32_t>(1, units / tiles), nkb / 4);
  } else {
    splits = std::min<uint32_t>(split_k, std::max<uint32_t>(1, nkb));
  }
  splits = std::max<uint32_t>(1, splits);
  const uint32_t kbps = std::max<uint32_t>(1, (nkb + splits - 1) / splits);
  splits = std::max<uint32_t>(1, (nkb + kbps - 1) / kbps);
  if ((epi.bits_out || epi.rowmax) && splits > 1) throw ConfigError("GEMM bit / row-max output needs an unsplit K");
  if (epi.bias && (reinterpret_cast<uintptr_t>(epi.bias) & 15))
    throw ConfigError("GEMM epilogue operands must be 16-byte aligned");
  static const int epi_env = [] {
    const char* v = std::getenv("CATGNN_GEMM_EPI_WARPS");
    return v ? std::atoi(v) : 0;
  }();
  const int epiw = epi_env == 4 || epi_env == 8 ? epi_env : (nkb <= 2 && splits == 1 ? 8 : 4);
  const size_t kEpiSmem = epi_smem(epiw);
  const size_t budget = 227 * 1024 - 1024 - kBarBytes(kMaxStages) - kEpiSmem;
  const size_t stage_bytes = 2 * (size_t)A_STAGE + 2 * (size_t)BNh * 128;
  const uint32_t stages = (uint32_t)std::min<size_t>(kMaxStages, budget / stage_bytes);
  if (stages < 2) throw InternalError("GEMM tile does not fit in shared memory");
  const size_t smem = 1024 + (size_t)stages * stage_bytes + kBarBytes(stages) + kEpiSmem;

  GemmArgs args{};
  args.M = M;
  args.N = N;
  args.K = K;
  args.BN = BN;
  args.bk = BKE;
  args.stages = stages;
  args.kb_per_split = kbps;
  args.tmem_cols = pow2_cols(2 * round_up(BN, 32));
  args.split3 = 0;
  args.mt = mt;
  args.nt = nt;
  args.splits = splits;
  args.tiles = mt * nt * splits;
  args.a_mn = a.mn_major ? 1u : 0u;
  args.b_mn = b.mn_major ? 1u : 0u;
  args.bm = bm;
  // instruction descriptor: D f32, A/B bf16 (kind::f16), majors, N>>3, M>>4
  args.idesc = (1u << 4) | (1u << 7) | (1u << 10) | (args.a_mn << 15) | (args.b_mn << 16) | ((BN >> 3) << 17) |
               ((bm >> 4) << 24);
  float* partial = nullptr;
  args.epi = epi;
  args.epi.partial = nullptr;
  if (splits > 1) {
    partial = ctx->scratch_buf<float>("gemm_partial", (size_t)splits * M * N);
    args.epi.partial = partial;
  }
  const CUtensorMap tah = a.mn_major ? make_map16_mn(a.hi, M, K, a.ld) : make_map16(a.hi, M, K, a.ld, BM);
  const CUtensorMap tal = a.mn_major ? make_map16_mn(a.lo, M, K, a.ld) : make_map16(a.lo, M, K, a.ld, BM);
  const CUtensorMap tbh = b.mn_major ? make_map16_mn(b.hi, N, K, b.ld) : make_map16(b.hi, N, K, b.ld, BNh);
  const CUtensorMap tbl = b.mn_major ? make_map16_mn(b.lo, N, K, b.ld) : make_map16(b.lo, N, K, b.ld, BNh);
  static std::mutex attr_mu;
  static std::map<int, std::array<bool, 4>> attr_set;
  auto kern = pair ? (epiw == 8 ? gemm_tf32_kernel<2, 8, true> : gemm_tf32_kernel<2, 4, true>)
                   : (epiw == 8 ? gemm_tf32_kernel<1, 8, true> : gemm_tf32_kernel<1, 4, true>);
  const int kThreads = epiw == 8 ? threads_for<8>() : threads_for<4>();
  {
    std::lock_guard<std::mutex> lk(attr_mu);
    bool& done = attr_set[ctx->device][(ncta - 1) * 2 + (epiw == 8)];
    if (!done) {
      CG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      done = true;
    }
  }
  auto dim = [](uint32_t x) { return x > 4096 ? std::string("rows") : std::to_string(x); };
  int t = ctx->begin_timed(1, ctx->timing ? "K3 gemm bf16x3 M=" + dim(M) + " N=" + dim(N) + " K=" + dim(K) +
                                             (pair ? " pair" : "") + (splits > 1 ? " split-K" : "")
                                       : std::string());
  const unsigned grid = std::min<unsigned>(args.tiles, units) * ncta;
  if (pair) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CG_CUDA(cudaLaunchKernelEx(&cfg, kern, tah, tbh, tbl, tal, args));
  } else {
    kern<<<grid, kThreads, smem, ctx->stream>>>(tah, tbh, tbl, tal, args);
  }
  CG_CHECK_LAUNCH();
  ctx->launches++;
  if (splits > 1) launch_reduce(ctx, partial, splits, M, N, epi);
  ctx->end_timed(t);
}

}  // namespace catgnn

// Diagnostics (GEMM_WAIT_PROFILE builds): per wait site, the nanoseconds
// warps spent blocked since the last call (0 producer empty, 1 MMA tempty,
// 2 MMA conv/full, 3 converter full, 4 converter lo slot, 5 epilogue tfull).
extern "C" int catgnn_debug_gemm_waits(unsigned long long* out8) {
  using namespace catgnn;
  return guarded([&] {
#ifdef GEMM_WAIT_PROFILE
    CG_CUDA(cudaDeviceSynchronize());
    CG_CUDA(cudaMemcpyFromSymbol(out8, g_gemm_wait_ns, 8 * sizeof(unsigned long long)));
    const unsigned long long z[8] = {0};
    CG_CUDA(cudaMemcpyToSymbol(g_gemm_wait_ns, z, sizeof(z)));
#else
    (void)out8;
    throw ConfigError("library built without GEMM_WAIT_PROFILE");
#endif
  });
}

// General test hook: A is M x K (a_mn = 0) or K x M (a_mn = 1), B is N x K or
// K x N, all host row-major; C = A . B^T in the logical (M x K).(N x K)^T sense.
extern "C" int catgnn_gemm(catgnn_ctx ctx, uint32_t M, uint32_t N, uint32_t K, const float* A, int a_mn,
                           const float* B, int b_mn, float* Cout, uint32_t split_k, int precision) {
  using namespace catgnn;
  return guarded([&] {
    if (!ctx) throw ConfigError("null context");
    if (precision != 1 && precision != 3 && precision != 4)
      throw ConfigError("precision must be 1 (TF32), 3 (3xTF32) or 4 (bf16x3)");
    CG_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    auto upload = [&](const char* name, const float* h, uint32_t r, uint32_t c) {
      const uint32_t ld = round_up(std::max(c, 1u), 4);
      float* d = ctx->scratch_buf<float>(name, (size_t)std::max(r, 1u) * ld + 64);
      CG_CUDA(cudaMemsetAsync(d, 0, ((size_t)std::max(r, 1u) * ld + 64) * 4, st));
      if (r && c) CG_CUDA(cudaMemcpy2DAsync(d, ld * 4, h, c * 4, c * 4, r, cudaMemcpyHostToDevice, st));
      return GemmOperand{d, ld, false};
    };
    GemmOperand ga = a_mn ? upload("g_A", A, K, M) : upload("g_A", A, M, K);
    GemmOperand gb = b_mn ? upload("g_B", B, K, N) : upload("g_B", B, N, K);
    ga.mn_major = a_mn != 0;
    gb.mn_major = b_mn != 0;
    const uint32_t ldc = round_up(N, 4);
    float* dC = ctx->scratch_buf<float>("g_C", (size_t)std::max(M, 1u) * ldc);
    GemmEpi e{};
    e.out = dC;
    e.ld_out = ldc;
    if (precision == 4) {  // bf16x3: split both operands on the device, then the pre-split GEMM
      auto split = [&](const char* name, const GemmOperand& o, uint32_t rows, uint32_t cols) {
        const uint32_t ld8 = round_up(std::max(cols, 1u), 8);
        __nv_bfloat16* p = ctx->scratch_buf<__nv_bfloat16>(name, 2 * (size_t)std::max(rows, 1u) * ld8 + 64);
        __nv_bfloat16* lo = p + (size_t)std::max(rows, 1u) * ld8;
        split_bf16(ctx, o.ptr, o.ld, rows, cols, p, lo, ld8);
        return SplitOperand{p, lo, ld8, o.mn_major};
      };
      SplitOperand sa = a_mn ? split("g_As", ga, K, M) : split("g_As", ga, M, K);
      SplitOperand sb = b_mn ? split("g_Bs", gb, K, N) : split("g_Bs", gb, N, K);
      gemm_bf16x3(ctx, sa, sb, M, N, K, e, split_k);
    } else {
      gemm(ctx, ga, gb, M, N, K, e, split_k, precision);
    }
    CG_CUDA(cudaMemcpy2DAsync(Cout, N * 4, dC, ldc * 4, N * 4, M, cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaStreamSynchronize(st));
  });
}

extern "C" int catgnn_gemm_tn(catgnn_ctx ctx, uint32_t M, uint32_t N, uint32_t K, const float* A,
                              const float* B, float* Cout, uint32_t split_k, int precision) {
  using namespace catgnn;
  return guarded([&] {
    if (!ctx) throw ConfigError("null context");
    CG_CUDA(cudaSetDevice(ctx->device));
    const uint32_t lda = round_up(std::max(K, 1u), 4), ldc = round_up(N, 4);
    float* dA = ctx->scratch_buf<float>("gt_A", (size_t)std::max(M, 1u) * lda);
    float* dB = ctx->scratch_buf<float>("gt_B", (size_t)std::max(N, 1u) * lda);
    float* dC = ctx->scratch_buf<float>("gt_C", (size_t)std::max(M, 1u) * ldc);
    cudaStream_t st = ctx->stream;
    CG_CUDA(cudaMemsetAsync(dA, 0, (size_t)std::max(M, 1u) * lda * 4, st));
    CG_CUDA(cudaMemsetAsync(dB, 0, (size_t)std::max(N, 1u) * lda * 4, st));
    if (K) {
      CG_CUDA(cudaMemcpy2DAsync(dA, lda * 4, A, K * 4, K * 4, M, cudaMemcpyHostToDevice, st));
      CG_CUDA(cudaMemcpy2DAsync(dB, lda * 4, B, K * 4, K * 4, N, cudaMemcpyHostToDevice, st));
    }
    GemmEpi e{};
    e.out = dC;
    e.ld_out = ldc;
    if (precision != 1 && precision != 3) throw ConfigError("precision must be 1 (TF32) or 3 (3xTF32)");
    gemm_tn(ctx, dA, lda, dB, lda, M, N, K, e, split_k, precision);
    CG_CUDA(cudaMemcpy2DAsync(Cout, N * 4, dC, ldc * 4, N * 4, M, cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaStreamSynchronize(st));
  });
}

// Diagnostics hook (scripts/gemm_micro.py): one K3 GEMM on caller-owned DEVICE
// buffers, enqueued on ctx's stream without a host sync (timed by the caller
// with events on that stream).  Not part of the drop-in boundary.
extern "C" int catgnn_debug_gemm_dev(catgnn_ctx ctx, uint32_t M, uint32_t N, uint32_t K, const float* A,
                                     uint32_t lda, int a_mn, const float* B, uint32_t ldb, int b_mn, float* C,
                                     uint32_t ldc, uint32_t split_k, int precision, const float* rowscale,
                                     const float* bias, int relu, const uint32_t* mask_bits, uint32_t mask_words,
                                     uint32_t* bits_out, uint32_t bits_words, uint32_t store_cols) {
  using namespace catgnn;
  return guarded([&] {
    if (!ctx) throw ConfigError("null context");
    CG_CUDA(cudaSetDevice(ctx->device));
    GemmEpi e{};
    e.store_cols = store_cols;
    e.out = C;
    e.ld_out = ldc;
    e.rowscale = rowscale;
    e.bias = bias;
    e.relu = relu;
    e.mask_bits = mask_bits;
    e.mask_words = mask_words;
    e.bits_out = bits_out;
    e.bits_words = bits_words;
    gemm(ctx, GemmOperand{A, lda, a_mn != 0}, GemmOperand{B, ldb, b_mn != 0}, M, N, K, e, split_k, precision);
  });
}

// Diagnostics hook: one bf16x3 GEMM on caller-owned pre-split DEVICE operands.
extern "C" int catgnn_debug_gemm16_dev(catgnn_ctx ctx, uint32_t M, uint32_t N, uint32_t K, const void* A_hi,
                                       const void* A_lo, uint32_t lda, int a_mn, const void* B_hi, const void* B_lo,
                                       uint32_t ldb, int b_mn, float* C, uint32_t ldc, uint32_t split_k,
                                       const float* rowscale, const float* bias, int relu, const uint32_t* mask_bits,
                                       uint32_t mask_words, uint32_t store_cols) {
  using namespace catgnn;
  return guarded([&] {
    if (!ctx) throw ConfigError("null context");
    CG_CUDA(cudaSetDevice(ctx->device));
    GemmEpi e{};
    e.out = C;
    e.ld_out = ldc;
    e.rowscale = rowscale;
    e.bias = bias;
    e.relu = relu;
    e.mask_bits = mask_bits;
    e.mask_words = mask_words;
    e.store_cols = store_cols;
    auto bf = [](const void* p) { return static_cast<const __nv_bfloat16*>(p); };
    gemm_bf16x3(ctx, SplitOperand{bf(A_hi), bf(A_lo), lda, a_mn != 0}, SplitOperand{bf(B_hi), bf(B_lo), ldb, b_mn != 0},
                M, N, K, e, split_k);
  });
}
