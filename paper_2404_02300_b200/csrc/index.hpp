// Device graph index (index.cu): compute_degrees' GraphIndex plus the sorted
// unique-id table used to route arbitrary 64-bit external ids on the device.
#pragma once

#include <cstdint>
#include <vector>

#include "common.hpp"

struct catgnn_index_s {
  catgnn_ctx ctx = nullptr;
  uint64_t n = 0, m = 0, self_loops = 0;
  std::vector<uint64_t> dense_to_ext;  // first-seen order (GraphIndex::dense_to_ext)
  std::vector<uint32_t> degree;        // self-loops count 2
  catgnn::DevBuf<uint64_t> sorted_ext;    // unique ext ids, ascending ("runs")
  catgnn::DevBuf<uint32_t> dense_of_run;  // run -> dense id
};

namespace catgnn {
void build_index(catgnn_ctx ctx, const uint64_t* d_edges, uint64_t m, catgnn_index_s* idx);
__global__ void map_to_runs_kernel(const uint64_t* __restrict__ sorted_ext, uint64_t n, const uint64_t* __restrict__ ids,
                                   uint64_t m, uint32_t* __restrict__ runs, int* missing);
}  // namespace catgnn
