// fallback.cuh — small helpers of the sort driver (the depth-cap fallback
// itself, hot-path step a9, is in loop.cuh).
#pragma once

#include "common.cuh"

namespace bq {

// A single leaf [0, n) in the user buffer (sorts with n <= S).
static __global__ void k_single_leaf(Leaf *leaves, uint32_t n) { leaves[0] = Leaf{0, n, 0, 0}; }

}  // namespace bq
