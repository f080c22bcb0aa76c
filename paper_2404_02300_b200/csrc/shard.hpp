// Device-resident shard: the B200 restatement of gnnpart::Shard
// (proj/include/gnnpart/train.hpp:84-91) plus the aggregation work plan.
//
// HBM layout (all row-major, 16-byte aligned rows):
//   row_ptr  int64[rows+1]      CSR offsets (LocalAdjacency.offsets, widened to
//                               64 bit: train.hpp:19 is u32 and overflows past
//                               4.29e9 nnz at papers100M scale)
//   col      int32[nnz]         neighbours, per-row order = build_adjacency's
//                               cursor order (train.cpp:41-45)
//   x        f32[rows][ld]      input features, ld = round_up(dim, 4)
//   xprop    f32[rows][ld]      SGC-propagated features (sgc_propagate output)
//   dinv     f32[rows]          (1+deg)^-1/2  (GCN normalisation)
//   inv_deg  f32[rows]          1/deg, 0 for deg 0 (SAGE mean)
//   inv_deg1 f32[rows]          1/(1+deg)     (SGC normalisation, train.cpp:60)
//   units    int4[n_units]      aggregation work units (see aggregate.cu)
//   heavy    int4[n_heavy]      split rows: {row, first partial slot, chunks, 0}
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "common.hpp"

struct catgnn_shard_s {
  catgnn_ctx ctx = nullptr;  // retained (ctx_retain) for the shard's lifetime
  uint64_t rows = 0;
  uint64_t nnz = 0;
  uint64_t num_edges = 0;
  catgnn::DevBuf<int64_t> row_ptr;
  catgnn::DevBuf<int32_t> col;
  catgnn::DevBuf<float> dinv, inv_deg, inv_deg1;
  // aggregation plan (built once per shard, reused by every pass)
  catgnn::DevBuf<int4> units;
  catgnn::DevBuf<int4> heavy;
  uint64_t n_units = 0, n_heavy = 0, n_chunks = 0;
  uint64_t n_big_heavy = 0;  // split rows with more than 16 chunks (block-per-row fix-up)
  uint32_t unit_cost = 0;
  // features
  uint32_t dim = 0, ld = 0;
  catgnn::DevBuf<float> x, xprop;
  // bf16x3 copy of x (hi / lo, row stride xs_ld = round8(dim)) for the tensor-core
  // GEMMs of the GNN layers, re-split whenever x changes (x_version)
  catgnn::DevBuf<uint16_t> xs_hi, xs_lo;
  uint32_t xs_ld = 0;
  uint64_t x_version = 1, xs_version = 0;
  // catgnn_shard_set_feature_layout(split_only): feature gathers write only the
  // bf16x3 copy; fp32 x is then stale (x_fp32_valid) until the next upload
  bool x_split_only = false, x_fp32_valid = true;
  // labels / roles (host copies + device copies)
  std::vector<int32_t> h_labels;
  std::vector<uint32_t> h_train, h_val, h_test;
  catgnn::DevBuf<int32_t> labels;
  catgnn::DevBuf<uint32_t> d_train, d_val, d_test;
  uint32_t classes = 1;
  int32_t train_label_min = 0, train_label_max = -1;  // over the train rows (model class-range check)
  // replica map (only for shards created from a partition)
  std::vector<uint64_t> ext_ids;
  std::vector<uint8_t> owner, role;
  catgnn::DevBuf<uint64_t> d_ext;  // device copy of ext_ids (feature gathers)
  uint64_t ext_max = 0;
  // Train-row views of the CSR for the lean train step (gnn.cu): the last
  // layer's logits matter only on train rows (train_sub: those rows' full
  // neighbour lists, row_map = their rows here) and its gradient is non-zero
  // only on them (train_nbr: every row, neighbours restricted to train rows, in
  // order).  Built on first use, dropped when the labels or the CSR change.
  std::unique_ptr<catgnn_shard_s> train_sub, train_nbr;
  catgnn::DevBuf<int32_t> row_map;  // a view's rows in its parent (train_sub)
};

namespace catgnn {

// Post-scale of the aggregated sum, computed from the local CSR degree.
enum AggNorm : int {
  kNormNone = 0,  // 1
  kNormSgc = 1,   // 1/(1+deg)          (train.cpp:60)
  kNormGcn = 2,   // (1+deg)^-1/2
  kNormMean = 3,  // deg>0 ? 1/deg : 0  (SAGE mean)
};

struct AggArgs {
  const float* in = nullptr;  // rows x in_ld, columns [in_col, in_col+width)
  // fp16 input rows instead of `in` (in_ld, in_col in halves, multiples of 8;
  // columns up to round8(width) readable, padding zero); the values are stored
  // multiplied by 1/in_scale (a power of two), in_scale is folded into the post
  // scale.  No per-source scale: the producer applies it before rounding.
  // Row `rows` must exist and be zero (idle gather slots load it instead of
  // being predicated off).
  const void* in_h = nullptr;
  float in_scale = 1.0f;
  // the shard is a row view (train_sub): output / self / mask rows are
  // row_map[r]; post_arr: per-row post scale (a filtered view's rows keep their
  // full degree's scale); zero_row: the input's zero row when the view has
  // fewer rows than the input (default: the shard's rows)
  const int32_t* row_map = nullptr;
  const float* post_arr = nullptr;
  int64_t zero_row = -1;
  bool in_zero_row = false;  // fp32 input: row `rows` exists and is zero (fp16: always required)
  // guarded fp16 forward of a ReLU layer (aggregate.cu epilogue_row GUARD):
  // per-row max |T| of the rounded rows (rows + 1 entries, the zero row 0),
  // flag bits (rows x bits_words), and the fp16 rounding residual of in_h
  // times 2^11 (same layout) the flagged elements are recomputed with
  const float* guard_smax = nullptr;
  uint32_t* guard_flags = nullptr;
  const void* guard_lo = nullptr;
  uint32_t in_ld = 0, in_col = 0;
  float* out = nullptr;  // rows x out_ld, columns [out_col, out_col+width)
  uint32_t out_ld = 0, out_col = 0;
  uint32_t width = 0;              // multiple of 4
  const float* pre = nullptr;      // per-source-row scale (applied to self term too)
  int self = 0;                    // add the row's own (pre-scaled) input
  int norm = kNormNone;            // post scale
  const float* bias = nullptr;     // [width]
  const float* residual = nullptr; // rows x res_ld at res_col
  uint32_t res_ld = 0, res_col = 0;
  int relu = 0;
  const uint32_t* mask_bits = nullptr;  // ReLU backward: keep where bit (r, c) is set
  uint32_t mask_words = 0;              // 32-bit words per row
  uint32_t* bits_out = nullptr;         // write out > 0 as bits (forward ReLU layers)
  uint32_t bits_words = 0;
  // bf16x3 output: out[r][c] also (or, with out == nullptr, only) written as the
  // pair hi = bf16(v), lo = bf16(v - hi) at column c of rows out_s_ld apart — the
  // pre-split operand of the next tensor-core GEMM (gemm_bf16x3)
  void* out_hi = nullptr;
  void* out_lo = nullptr;
  uint32_t out_s_ld = 0;
};

// K1: CSR builder (stable radix sort by source row, bit-exact with
// build_adjacency) + aggregation plan + degree scales.  pairs are device
// local-id pairs in edge order.
void build_csr(catgnn_shard_s* s, const uint32_t* d_pairs, uint64_t num_edges);
// home partition of every shard row (owner ids / parts: every partition's owned
// ids and their partition, host arrays, n_owned entries): device radix sort of
// the owner table + binary search of the shard's d_ext.  Returns the halo rows.
uint64_t halo_map(catgnn_shard_s* s, const uint32_t* owner_ids, const uint32_t* owner_parts, uint64_t n_owned,
                  uint64_t num_ids, uint32_t* home_host);
// Device mapping of external-id edges to local rows by binary search over the
// ascending node table (load_training_data's local[] map, train.cpp:258-271).
void map_ext_edges(catgnn_ctx ctx, const uint64_t* d_ext_ids, uint64_t rows,
                   const uint64_t* d_edges_ext, uint64_t num_edges, uint32_t* d_pairs);
// K2: neighbourhood aggregation over the shard CSR.
void aggregate(catgnn_shard_s* s, const AggArgs& a);
// The train-row views (built on first use; nullptr when the shard has no train rows).
catgnn_shard_s* train_rows_view(catgnn_shard_s* s);
catgnn_shard_s* train_nbr_view(catgnn_shard_s* s);
// Copy rows x width between strided buffers (hops = 0 propagate).
void copy_rows(catgnn_ctx ctx, const float* in, uint32_t in_ld, float* out, uint32_t out_ld,
               uint64_t rows, uint32_t width);

}  // namespace catgnn
