// fallback.cuh — hot-path step a9: the depth-cap fallback (H6).
//
// The paper's Introsort switches a sub-array to Heapsort once the recursion
// depth exceeds 2 log n + 3, guaranteeing
// O(n log n).  Heapsort is inherently serial, so on the GPU a depth-capped
// segment is instead finished by a merge sort: its S-element chunks are
// sorted by the leaf kernel in place, then log2(len/S) merge passes ping-pong
// between the two buffers.  Each merge thread locates its first output by a
// merge-path binary search (O(log w)) and then emits IPT outputs serially, so
// a pass costs O(len) work and the fallback O(len log len) in total.  Ties
// take the left run first (stable merge).
#pragma once

#include "common.cuh"

namespace bq {

template <class KT, int NT, int IPT>
__global__ void __launch_bounds__(NT) k_merge(const typename KT::T *X, typename KT::T *Y, uint64_t b,
                                               uint32_t len, uint32_t w) {
    using T = typename KT::T;
    const uint64_t o = ((uint64_t)blockIdx.x * NT + threadIdx.x) * IPT;
    if (o >= len) return;
    const uint64_t pair0 = (o / (2ull * w)) * (2ull * w);
    const uint64_t a0 = pair0;
    const uint64_t a1 = pair0 + w < len ? pair0 + w : len;
    const uint64_t b1 = pair0 + 2ull * w < len ? pair0 + 2ull * w : len;
    const uint64_t na = a1 - a0, nb = b1 - a1;
    const uint64_t d = o - pair0;
    const T *A = X + b + a0;
    const T *B = X + b + a1;
    uint64_t lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (!(KT::key(B[d - 1 - mid]) < KT::key(A[mid]))) lo = mid + 1;   // A[mid] <= B[d-1-mid]
        else hi = mid;
    }
    uint64_t i = lo, j = d - lo;
    const uint64_t end = (o + IPT) < b1 ? (o + IPT) : b1;
    for (uint64_t r = o; r < end; r++) {
        const bool takeA = j >= nb || (i < na && !(KT::key(B[j]) < KT::key(A[i])));
        Y[b + r] = takeA ? A[i++] : B[j++];
    }
}

// Leaf descriptors for the S-element chunks of a fallback segment.
static __global__ void k_chunk_leaves(Leaf *leaves, uint32_t b, uint32_t len, uint32_t parity, uint32_t S) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t nch = (len + S - 1) / S;
    if (c >= nch) return;
    const uint32_t cb = b + c * S;
    const uint32_t cl = (len - c * S) < S ? (len - c * S) : S;
    leaves[c] = Leaf{cb, cl, parity, 0};
}

// A single leaf [0, n) in the user buffer (sorts with n <= S).
static __global__ void k_single_leaf(Leaf *leaves, uint32_t n) { leaves[0] = Leaf{0, n, 0, 0}; }

}  // namespace bq
