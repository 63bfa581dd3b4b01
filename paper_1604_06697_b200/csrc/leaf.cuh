// leaf.cuh — hot-path step a8: segments of at most S elements are finished on
// one CTA in shared memory by a bitonic sorting network (north_star (5):
// "small segments finished in shared memory by a sorting network").  This is
// the role Insertionsort plays below 17 elements in the paper (P:300-310,
// P:1257-1258); the threshold is retuned for the on-chip memory of an SM.
//
// Keys are sorted as their comparison keys (H0 codec for float64) and decoded
// on the way out.  Records are sorted as (key, index) pairs and gathered from
// a shared-memory copy, so a leaf may be sorted in place.  Padding to the next
// power of two uses (KMAX, index >= len), which orders after every real
// element.
#pragma once

#include "common.cuh"

namespace bq {

template <class KT>
struct LeafParams {
    using T = typename KT::T;
    const Leaf *leaves;
    T *bufs[2];
    T *out;            // destination buffer (the user buffer, or in-place for fallback chunks)
    int out_inplace;   // 1: write back into bufs[parity] (fallback chunk sort)
};

template <class KT>
constexpr size_t leaf_smem_bytes() {
    using K = typename KT::K;
    if constexpr (KT::is_record)
        return (size_t)Tune<KT>::LEAF * (sizeof(K) + sizeof(uint32_t) + sizeof(typename KT::T));
    else
        return (size_t)Tune<KT>::LEAF * sizeof(K);
}

template <class KT, int NT>
__global__ void __launch_bounds__(NT) k_leaf(LeafParams<KT> P) {
    using T = typename KT::T;
    using K = typename KT::K;
    constexpr int S = Tune<KT>::LEAF;
    constexpr bool REC = KT::is_record;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K *sk = reinterpret_cast<K *>(smem_raw);
    uint32_t *si = reinterpret_cast<uint32_t *>(smem_raw + S * sizeof(K));
    T *sr = reinterpret_cast<T *>(smem_raw + S * (sizeof(K) + sizeof(uint32_t)));

    const Leaf lf = P.leaves[blockIdx.x];
    const uint32_t len = lf.len;
    T *srcbuf = lf.parity ? P.bufs[1] : P.bufs[0];
    const T *src = srcbuf;
    T *out = P.out_inplace ? srcbuf : P.out;
    const uint64_t b = lf.begin;
    uint32_t pw = 1;
    while (pw < len) pw <<= 1;

    for (uint32_t i = threadIdx.x; i < pw; i += NT) {
        if (i < len) {
            const T x = src[b + i];
            sk[i] = KT::key(x);
            if constexpr (REC) { si[i] = i; sr[i] = x; }
        } else {
            sk[i] = KT::KMAX;
            if constexpr (REC) si[i] = i;
        }
    }
    __syncthreads();

    // bitonic network: for k = 2..pw, j = k/2..1, compare-exchange (i, i^j)
    for (uint32_t kk = 2; kk <= pw; kk <<= 1) {
        for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
            for (uint32_t q = threadIdx.x; q < (pw >> 1); q += NT) {
                const uint32_t i = 2 * q - (q & (j - 1));   // i has bit j clear
                const uint32_t l = i + j;
                const bool up = (i & kk) == 0;
                const K a = sk[i], c = sk[l];
                bool gt;
                if constexpr (REC) {
                    const uint32_t ia = si[i], ic = si[l];
                    gt = (c < a) || (!(a < c) && ic < ia);
                    const bool sw = up ? gt : !gt;
                    if (sw) { sk[i] = c; sk[l] = a; si[i] = ic; si[l] = ia; }
                } else {
                    gt = c < a;
                    const bool sw = up ? gt : (a < c);
                    sk[i] = sw ? c : a;
                    sk[l] = sw ? a : c;
                }
            }
            __syncthreads();
        }
    }

    for (uint32_t i = threadIdx.x; i < len; i += NT) {
        if constexpr (REC) out[b + i] = sr[si[i]];
        else out[b + i] = KT::from_key(sk[i]);
    }
}

}  // namespace bq
