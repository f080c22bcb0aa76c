#pragma once

#include "common.hpp"

namespace catgnn {

// Stable LSD radix sort of n (key, value) uint32 pairs by the low `bits` key
// bits (radix.cu).  (keys, vals) hold the input, (keys_alt, vals_alt) are
// same-sized scratch; passes ping-pong between the two and *keys_result /
// *vals_result point at whichever pair holds the sorted output.
void radix_sort_pairs(catgnn_ctx ctx, uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt,
                      uint64_t n, int bits, uint32_t** keys_result, uint32_t** vals_result);

}  // namespace catgnn
