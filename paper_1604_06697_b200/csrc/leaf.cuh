// leaf.cuh — hot-path step a8: segments of at most S elements are finished on
// one CTA by a bitonic sorting network (north_star (5): "small segments
// finished in shared memory by a sorting network").  This is the role
// Insertionsort plays below 17 elements in the paper (P:300-310,
// P:1257-1258); the threshold is retuned for the on-chip memory of an SM.
//
// Design (register-resident network, shared memory only for transposes).
// A leaf of len keys is padded to a network of NET = 2^L >= len elements
// (padding = the largest key, so it sorts last) and held in registers:
// NT = 2^(L-R) threads x IPT = 2^R keys.  Element index i is spread over
// (thread, register) by a *layout*: layout 0 puts index bits [0, R) in the
// register number (thread t holds i = t*IPT + r), layout s >= 5 puts bits
// [s, s+R) there.  Every compare-exchange of the network (stage bit b: i vs
// i ^ 2^b) is done between two registers of one thread in a layout whose
// register bits contain b; between stages whose bits live in different
// layouts the keys are transposed through shared memory ("remap").  For
// L = 13, R = 5 that is 19 remaps for the 91 stages of the network (the
// previous version did all 91 stages in shared memory).  The few stages with
// R <= b < 5 (records, R = 4) exchange between lanes with shuffles.
//
// Directions: instead of alternating ascending/descending compare-exchanges,
// every compare-exchange is ascending on keys that are complemented (~x, an
// order-reversing bijection) where the classic network sorts descending:
// before merge m the keys whose index has bit m set are complemented, which
// costs one LOP per key per merge.
//
// Shared memory: one plane per key component, element i at a swizzled byte
// offset (16-byte chunk index XOR row bits) so that both the vector
// (layout 0, 16-byte) and the scalar (layout s >= 5) accesses are free of
// bank conflicts.  Records are sorted as (key, index) pairs (the index
// breaks ties, so padding stays behind real keys) and gathered from a
// shared-memory copy of the leaf at the end.
#pragma once

#include "common.cuh"

namespace bq {

template <class KT>
struct LeafParams {
    using T = typename KT::T;
    const Leaf *leaves;
    const uint32_t *count_dev;   // non-null: persistent grid over *count_dev leaves; else one leaf per CTA
    T *bufs[2];
    T *out;            // destination buffer (the user buffer, or in-place for fallback chunks)
    int out_inplace;   // 1: write back into bufs[parity] (fallback chunk sort)
};

// ---- register element types and their compare-exchange --------------------
struct RecKI {
    uint64_t k;
    uint32_t i;
};

#ifndef BQ_LEAF_R32
#define BQ_LEAF_R32 5
#endif
// 64-bit keys: 16 per thread at up to 1024 resident threads per SM (measured
// on c3: 32 keys per thread at 256 threads left the SM latency-bound)
#ifndef BQ_LEAF_R64
#define BQ_LEAF_R64 4
#endif
#ifndef BQ_LEAF_OCC64
#define BQ_LEAF_OCC64 1024
#endif
#ifndef BQ_LEAF_RREC
#define BQ_LEAF_RREC 3
#endif
#ifndef BQ_LEAF_OCC32
#define BQ_LEAF_OCC32 512
#endif
#ifndef BQ_LEAF_OCCREC
#define BQ_LEAF_OCCREC 1024
#endif
template <class KT>
struct LeafTraits {
    using E = typename KT::K;
    static constexpr int R = sizeof(E) == 4 ? BQ_LEAF_R32 : BQ_LEAF_R64;   // log2(keys per thread)
    static constexpr int OCC = sizeof(E) == 4 ? BQ_LEAF_OCC32 : BQ_LEAF_OCC64;   // resident threads/SM the registers target
};
template <>
struct LeafTraits<KRec> {
    using E = RecKI;
    static constexpr int R = BQ_LEAF_RREC;
    static constexpr int OCC = BQ_LEAF_OCCREC;
};

template <>
struct LeafTraits<KPair> : LeafTraits<KRec> {};   // pairs sort as (key, leaf index) like records

template <class KT>
constexpr int leaf_lmin() { return LeafTraits<KT>::R + 5; }   // one warp
template <class KT>
constexpr int leaf_lmax() {
    int l = 0;
    while ((1 << l) < Tune<KT>::LEAF) l++;
    return l;
}
template <class KT>
constexpr int leaf_nclass() { return leaf_lmax<KT>() - leaf_lmin<KT>() + 1; }
constexpr int MAX_LEAF_CLASSES = 8;   // LevelCtrl::nleaf_cls, leaf-count words per set

// network-size class of a leaf of `len` keys: NET = 2^(lmin + class)
template <class KT>
__host__ __device__ inline uint32_t leaf_class(uint32_t len) {
    uint32_t c = 0;
    while ((1u << (leaf_lmin<KT>() + c)) < len) c++;
    return c;
}

__device__ __forceinline__ void ce(int32_t &a, int32_t &b) {
    const int32_t lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}
__device__ __forceinline__ void ce(uint64_t &a, uint64_t &b) {
    const bool s = b < a;
    const uint64_t lo = s ? b : a, hi = s ? a : b;
    a = lo;
    b = hi;
}
__device__ __forceinline__ bool e_less(const RecKI &a, const RecKI &b) {
    return a.k < b.k || (a.k == b.k && a.i < b.i);
}
__device__ __forceinline__ bool e_less(int32_t a, int32_t b) { return a < b; }
__device__ __forceinline__ bool e_less(uint64_t a, uint64_t b) { return a < b; }
__device__ __forceinline__ void ce(RecKI &a, RecKI &b) {
    const bool s = e_less(b, a);
    const RecKI lo = s ? b : a, hi = s ? a : b;
    a = lo;
    b = hi;
}
// w ^ m for m in {0, ~0}, computed as w * (2m + 1) + m (m = ~0: -w - 1 = ~w)
// with IMADs, which issue on the FMA pipe: the network's compare-exchanges
// keep the ALU pipe busy, the FMA pipe is idle
__device__ __forceinline__ uint32_t flip_w(uint32_t w, uint32_t m) {
    uint32_t s, r;
    asm("mad.lo.u32 %0, %1, 2, 1;" : "=r"(s) : "r"(m));
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(w), "r"(s), "r"(m));
    return r;
}
__device__ __forceinline__ void flip_if(int32_t &a, uint32_t m) { a = (int32_t)flip_w((uint32_t)a, m); }
__device__ __forceinline__ void flip_if(uint64_t &a, uint32_t m) {
    a = ((uint64_t)flip_w((uint32_t)(a >> 32), m) << 32) | flip_w((uint32_t)a, m);
}
__device__ __forceinline__ void flip_if(RecKI &a, uint32_t m) {
    flip_if(a.k, m);
    a.i = flip_w(a.i, m);
}
__device__ __forceinline__ int32_t shfl_x(int32_t v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }
__device__ __forceinline__ uint64_t shfl_x(uint64_t v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }
__device__ __forceinline__ RecKI shfl_x(RecKI v, int m) {
    return RecKI{__shfl_xor_sync(0xffffffffu, v.k, m), (uint32_t)__shfl_xor_sync(0xffffffffu, v.i, m)};
}

// ---- shared-memory planes -----------------------------------------------------
// byte offset of element i in a plane of W-byte components whose layout-0
// owner writes TB = IPT*W bytes: 16-byte chunk index XOR (row >> RS) & 7
template <int W, int TB>
__device__ __forceinline__ uint32_t swz(uint32_t i) {
    constexpr int RS = TB >= 256 ? 1 + (TB >= 512) + (TB >= 1024) : 0;
    const uint32_t b = i * W;
    return b ^ ((((b >> 7) >> RS) & 7u) << 4);
}

template <int L, int R, int S>
__device__ __forceinline__ uint32_t lidx(uint32_t t, uint32_t r) {
    if constexpr (S == 0)
        return (t << R) + r;
    else
        return ((t >> S) << (S + R)) | (r << S) | (t & ((1u << S) - 1));
}

// store / load one plane (component C of E) in layout S
template <class KT>
struct Planes;

template <class KT>
struct Planes {   // keys: one plane of K
    using E = typename LeafTraits<KT>::E;
    static constexpr int R = LeafTraits<KT>::R, IPT = 1 << R, W = sizeof(E), TB = IPT * W;
    template <int NET>
    static constexpr int bytes() { return NET * W; }
    template <int L, int S>
    static __device__ __forceinline__ void store(const E (&x)[IPT], unsigned char *sm, uint32_t t) {
        if constexpr (S == 0) {
            constexpr int PER = 16 / W;
#pragma unroll
            for (int c = 0; c < IPT / PER; c++) {
                E tmp[PER];
#pragma unroll
                for (int j = 0; j < PER; j++) tmp[j] = x[c * PER + j];
                uint4 v;
                memcpy(&v, tmp, 16);
                *reinterpret_cast<uint4 *>(sm + swz<W, TB>((t << R) + c * PER)) = v;
            }
        } else {
#pragma unroll
            for (int r = 0; r < IPT; r++) *reinterpret_cast<E *>(sm + swz<W, TB>(lidx<L, R, S>(t, r))) = x[r];
        }
    }
    template <int L, int S>
    static __device__ __forceinline__ void load(E (&x)[IPT], const unsigned char *sm, uint32_t t) {
        if constexpr (S == 0) {
            constexpr int PER = 16 / W;
#pragma unroll
            for (int c = 0; c < IPT / PER; c++) {
                const uint4 v = *reinterpret_cast<const uint4 *>(sm + swz<W, TB>((t << R) + c * PER));
                E tmp[PER];
                memcpy(tmp, &v, 16);
#pragma unroll
                for (int j = 0; j < PER; j++) x[c * PER + j] = tmp[j];
            }
        } else {
#pragma unroll
            for (int r = 0; r < IPT; r++) x[r] = *reinterpret_cast<const E *>(sm + swz<W, TB>(lidx<L, R, S>(t, r)));
        }
    }
};

template <>
struct Planes<KRec> {   // records: key plane (8 B) + index plane (4 B)
    using E = RecKI;
    static constexpr int R = LeafTraits<KRec>::R, IPT = 1 << R;
    template <int NET>
    static constexpr int bytes() { return NET * 12; }
    template <int L, int S>
    static __device__ __forceinline__ void store(const E (&x)[IPT], unsigned char *sm, uint32_t t) {
        constexpr int NET = 1 << L;
        unsigned char *pk = sm, *pi = sm + NET * 8;
        if constexpr (S == 0) {
#pragma unroll
            for (int c = 0; c < IPT / 2; c++) {
                const uint4 v = make_uint4((uint32_t)x[2 * c].k, (uint32_t)(x[2 * c].k >> 32),
                                           (uint32_t)x[2 * c + 1].k, (uint32_t)(x[2 * c + 1].k >> 32));
                *reinterpret_cast<uint4 *>(pk + swz<8, IPT * 8>((t << R) + 2 * c)) = v;
            }
#pragma unroll
            for (int c = 0; c < IPT / 4; c++) {
                const uint4 v = make_uint4(x[4 * c].i, x[4 * c + 1].i, x[4 * c + 2].i, x[4 * c + 3].i);
                *reinterpret_cast<uint4 *>(pi + swz<4, IPT * 4>((t << R) + 4 * c)) = v;
            }
        } else {
#pragma unroll
            for (int r = 0; r < IPT; r++) {
                const uint32_t i = lidx<L, R, S>(t, r);
                *reinterpret_cast<uint64_t *>(pk + swz<8, IPT * 8>(i)) = x[r].k;
                *reinterpret_cast<uint32_t *>(pi + swz<4, IPT * 4>(i)) = x[r].i;
            }
        }
    }
    template <int L, int S>
    static __device__ __forceinline__ void load(E (&x)[IPT], const unsigned char *sm, uint32_t t) {
        constexpr int NET = 1 << L;
        const unsigned char *pk = sm, *pi = sm + NET * 8;
        if constexpr (S == 0) {
#pragma unroll
            for (int c = 0; c < IPT / 2; c++) {
                const uint4 v = *reinterpret_cast<const uint4 *>(pk + swz<8, IPT * 8>((t << R) + 2 * c));
                x[2 * c].k = (uint64_t)v.x | ((uint64_t)v.y << 32);
                x[2 * c + 1].k = (uint64_t)v.z | ((uint64_t)v.w << 32);
            }
#pragma unroll
            for (int c = 0; c < IPT / 4; c++) {
                const uint4 v = *reinterpret_cast<const uint4 *>(pi + swz<4, IPT * 4>((t << R) + 4 * c));
                x[4 * c].i = v.x;
                x[4 * c + 1].i = v.y;
                x[4 * c + 2].i = v.z;
                x[4 * c + 3].i = v.w;
            }
        } else {
#pragma unroll
            for (int r = 0; r < IPT; r++) {
                const uint32_t i = lidx<L, R, S>(t, r);
                x[r].k = *reinterpret_cast<const uint64_t *>(pk + swz<8, IPT * 8>(i));
                x[r].i = *reinterpret_cast<const uint32_t *>(pi + swz<4, IPT * 4>(i));
            }
        }
    }
};

template <>
struct Planes<KPair> : Planes<KRec> {};

// ---- the network ---------------------------------------------------------------
template <class KT, int L>
struct Net {
    using E = typename LeafTraits<KT>::E;
    using PL = Planes<KT>;
    static constexpr int R = LeafTraits<KT>::R, IPT = 1 << R;
    static_assert(L - R >= 5, "a network spans at least one warp");

    template <int S1, int S2>
    static __device__ __forceinline__ void remap(E (&x)[IPT], unsigned char *sm, uint32_t t) {
        __syncthreads();   // previous readers of the plane are done
        PL::template store<L, S1>(x, sm, t);
        __syncthreads();
        PL::template load<L, S2>(x, sm, t);
    }

    // compare-exchange of register pairs differing in register bit RB
    template <int RB>
    static __device__ __forceinline__ void regs(E (&x)[IPT]) {
#pragma unroll
        for (int r = 0; r < IPT; r++)
            if (!(r & (1 << RB))) ce(x[r], x[r | (1 << RB)]);
    }
    // compare-exchange across lanes (layout 0, R <= B < 5)
    template <int B>
    static __device__ __forceinline__ void lanes(E (&x)[IPT], uint32_t t) {
        constexpr int LB = B - R;
        const bool upper = (t >> LB) & 1;
#pragma unroll
        for (int r = 0; r < IPT; r++) {
            const E y = shfl_x(x[r], 1 << LB);
            x[r] = (e_less(y, x[r]) != upper) ? y : x[r];
        }
    }

    // stages for bits HB..0 of one merge, starting in layout CUR, ending in layout 0
    template <int HB, int CUR>
    static __device__ __forceinline__ void phase(E (&x)[IPT], unsigned char *sm, uint32_t t) {
        if constexpr (HB < 0) {
            if constexpr (CUR != 0) remap<CUR, 0>(x, sm, t);
        } else if constexpr (HB >= 5 && HB >= R) {
            constexpr int S = (HB - R + 1) > 5 ? (HB - R + 1) : 5;
            if constexpr (S != CUR) remap<CUR, S>(x, sm, t);
            bits_in<HB, S>(x);
            phase<S - 1, S>(x, sm, t);
        } else {
            if constexpr (CUR != 0) remap<CUR, 0>(x, sm, t);
            low_bits<HB>(x, t);
        }
    }
    template <int B, int S>
    static __device__ __forceinline__ void bits_in(E (&x)[IPT]) {   // B down to S, register bits of layout S
        regs<B - S>(x);
        if constexpr (B > S) bits_in<B - 1, S>(x);
    }
    template <int B>
    static __device__ __forceinline__ void low_bits(E (&x)[IPT], uint32_t t) {   // B down to 0 in layout 0
        if constexpr (B >= R)
            lanes<B>(x, t);
        else
            regs<B>(x);
        if constexpr (B > 0) low_bits<B - 1>(x, t);
    }

    // bit K of the index of (t, r) in layout 0, as a 0 / ~0 mask
    template <int K>
    static __device__ __forceinline__ uint32_t bitmask(uint32_t t, int r) {
        if constexpr (K >= L) return 0u;
        else if constexpr (K < R) return ((r >> K) & 1) ? ~0u : 0u;
        else return ((t >> (K - R)) & 1) ? ~0u : 0u;
    }
    // merges M..L: during merge M the keys are complemented where index bit M
    // is set (M < L), i.e. in the classic network's descending blocks; the
    // transition from merge M-1 is an XOR with (bit M-1) ^ (bit M)
    template <int M>
    static __device__ __forceinline__ void merges(E (&x)[IPT], unsigned char *sm, uint32_t t) {
#pragma unroll
        for (int r = 0; r < IPT; r++) {
            uint32_t m = bitmask<M>(t, r);
            if constexpr (M > 1) m ^= bitmask<M - 1>(t, r);
            flip_if(x[r], m);
        }
        phase<M - 1, 0>(x, sm, t);
        if constexpr (M < L) merges<M + 1>(x, sm, t);
    }

    // sorts the NET keys held in layout S0 = L-R (thread t, register r: index
    // r*NT + t); returns them sorted, in the same layout
    static __device__ __forceinline__ void sort(E (&x)[IPT], unsigned char *sm, uint32_t t) {
        constexpr int S0 = L - R;
        __syncthreads();
        PL::template store<L, S0>(x, sm, t);
        __syncthreads();
        PL::template load<L, 0>(x, sm, t);
        merges<1>(x, sm, t);
        remap<0, S0>(x, sm, t);
    }
};

template <class KT>
constexpr bool leaf_classes_fit() { return leaf_nclass<KT>() <= MAX_LEAF_CLASSES; }

template <class KT, int L>
constexpr size_t leaf_smem_bytes() {
    static_assert(leaf_classes_fit<KT>(), "S / 2^(R+5) network classes exceed MAX_LEAF_CLASSES");
    constexpr int NET = 1 << L;
    size_t b = (size_t)Planes<KT>::template bytes<NET>();
    if constexpr (KT::is_record) b += (size_t)NET * sizeof(typename KT::T);
    return b;
}

// One leaf, by the whole CTA.  For keys it is called out of line from the
// persistent loop below: inlined, the compiler hoists the transposes'
// per-thread addresses out of the loop and spills.
template <class KT, int L>
__device__ __forceinline__ void leaf_body(const LeafParams<KT> &P, const Leaf lf, unsigned char *smem_raw) {
    using T = typename KT::T;
    using K = typename KT::K;
    using E = typename LeafTraits<KT>::E;
    constexpr int R = LeafTraits<KT>::R, IPT = 1 << R, NT = 1 << (L - R), NET = 1 << L;
    unsigned char *planes = smem_raw;
    const uint32_t t = threadIdx.x;
    const uint32_t len = lf.len;
    T *srcbuf = lf.parity ? P.bufs[1] : P.bufs[0];
    T *out = P.out_inplace ? srcbuf : P.out;
    const uint64_t b = lf.begin;

    E x[IPT];
    if constexpr (KT::is_record) {
        // leaf copy in shared memory (the output is gathered from it, so the
        // leaf may be sorted in place)
        T *sr = reinterpret_cast<T *>(smem_raw + Planes<KT>::template bytes<NET>());
        constexpr uint32_t V = sizeof(T) / 16;   // 16-byte vectors per record
        const uint4 *g = reinterpret_cast<const uint4 *>(srcbuf + b);
        uint4 *s4 = reinterpret_cast<uint4 *>(sr);
        for (uint32_t q = t; q < V * len; q += NT) s4[q] = g[q];
        __syncthreads();
#pragma unroll
        for (int r = 0; r < IPT; r++) {
            const uint32_t i = (uint32_t)r * NT + t;
            x[r] = RecKI{i < len ? sr[i].key : ~0ull, i};
        }
        Net<KT, L>::sort(x, planes, t);
#pragma unroll
        for (int r = 0; r < IPT; r++) {
            const uint32_t i = (uint32_t)r * NT + t;
            if (i < len) {
                const uint4 *s = reinterpret_cast<const uint4 *>(sr + x[r].i);
                uint4 *d = reinterpret_cast<uint4 *>(out + b + i);
                uint4 v[V];
#pragma unroll
                for (uint32_t c = 0; c < V; c++) v[c] = s[c];
#pragma unroll
                for (uint32_t c = 0; c < V; c++) d[c] = v[c];
            }
        }
    } else {
#pragma unroll
        for (int r = 0; r < IPT; r++) {
            const uint32_t i = (uint32_t)r * NT + t;
            x[r] = i < len ? (E)KT::key(srcbuf[b + i]) : (E)KT::KMAX;
        }
        Net<KT, L>::sort(x, planes, t);
#pragma unroll
        for (int r = 0; r < IPT; r++) {
            const uint32_t i = (uint32_t)r * NT + t;
            if (i < len) out[b + i] = KT::from_key((K)x[r]);
        }
    }
}

template <class KT, int L>
__device__ __noinline__ void leaf_one(const LeafParams<KT> &P, const Leaf lf, unsigned char *smem_raw) {
    leaf_body<KT, L>(P, lf, smem_raw);
}

template <class KT, int L>
__global__ void __launch_bounds__(1 << (L - LeafTraits<KT>::R), (LeafTraits<KT>::OCC >> (L - LeafTraits<KT>::R)) > 0 ? (LeafTraits<KT>::OCC >> (L - LeafTraits<KT>::R)) : 1) k_leaf(LeafParams<KT> P) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const uint32_t nleaves = P.count_dev ? *P.count_dev : gridDim.x;
    for (uint32_t li = blockIdx.x; li < nleaves; li += gridDim.x) {
        if (li != blockIdx.x) __syncthreads();   // the previous leaf's shared-memory readers are done
        // (keys: out of line, see leaf_one; records measured faster inlined)
        if constexpr (KT::is_record) leaf_body<KT, L>(P, P.leaves[li], smem_raw);
        else leaf_one<KT, L>(P, P.leaves[li], smem_raw);
    }
}

// host: launch the leaf kernel of class c (NET = 2^(lmin + c)) over `count` leaves
// count > 0: one CTA per leaf; count == 0: persistent grid (resident CTAs)
// over LP.count_dev leaves
template <class KT, int L>
cudaError_t launch_leaf_l(const LeafParams<KT> &LP, uint32_t count, cudaStream_t s) {
    constexpr size_t smem = leaf_smem_bytes<KT, L>();
    constexpr int NT = 1 << (L - LeafTraits<KT>::R);
    static CapCache cc;
    int cap = 0;
#ifdef BQ_LEAF_CTAS_PER_SM
    constexpr int per_sm_max = BQ_LEAF_CTAS_PER_SM;   // leave room for co-resident partition CTAs
#else
    constexpr int per_sm_max = 0;
#endif
    cudaError_t e = resident_ctas(k_leaf<KT, L>, NT, smem, cc, &cap, per_sm_max);
    if (e != cudaSuccess) return e;
    k_leaf<KT, L><<<count ? count : (uint32_t)cap, NT, smem, s>>>(LP);
    return cudaGetLastError();
}

template <class KT, int C = 0>
cudaError_t launch_leaf_class(int cls, const LeafParams<KT> &LP, uint32_t count, cudaStream_t s) {
    if constexpr (C >= leaf_nclass<KT>()) {
        return cudaErrorInvalidValue;
    } else {
        if (cls == C) return launch_leaf_l<KT, leaf_lmin<KT>() + C>(LP, count, s);
        return launch_leaf_class<KT, C + 1>(cls, LP, count, s);
    }
}

}  // namespace bq
