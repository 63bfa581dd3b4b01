// leaf.cuh — hot-path step a8: segments of at most S elements are finished on
// one CTA in shared memory (north_star (5); "register
// network for <= 32, then merge").  This is the role Insertionsort plays below
// 17 elements in the paper; the threshold is retuned
// to the on-chip memory of an SM (S = 31 Ki int32 keys, 15 Ki 64-bit keys,
// 9 Ki key+index pairs), which removes the partition levels below it.
//
// Algorithm (a merge sort whose base case is a sorting network):
//   1. the leaf is loaded into a shared-memory plane (1D TMA bulk copy);
//   2. thread t sorts the IPT keys at positions [t*IPT, (t+1)*IPT) in
//      registers with Batcher's odd-even merge sort (a fixed network of
//      compare-exchanges: no data-dependent branches);
//   3. merge rounds: the runs of length RL = IPT * 2^r are merged pairwise
//      until one run remains.  Every thread produces IPT consecutive outputs
//      of its pair's merged run: it finds where its output range starts with
//      a binary search on the "merge path" (the number of A keys among the
//      first d outputs), then emits IPT outputs serially.  Runs are stored
//      alternately ascending and descending, so the two runs of a pair form
//      one bitonic sequence A-ascending | B-descending and every output is
//      min(front of A, back of B): when one run is exhausted its pointer
//      walks into the other run from that run's largest end, so the serial
//      merge needs no bounds checks (a bitonic sequence's minimum is at one of
//      its ends).  Outputs are written back in place after a barrier;
//   4. the sorted plane is written to the user buffer with a TMA bulk store
//      (keys), or the records are gathered by their leaf index (records and
//      key+index pairs sort (key, index) and then move each record once).
// Work per key: ~log2(IPT) network levels + ceil(log2(len / IPT)) merge
// rounds of a handful of instructions, against the L(L+1)/2 compare-exchange
// stages of a bitonic network of 2^L keys.
//
// IPT is odd: thread t's keys sit at a stride of IPT words, so the per-thread
// loads and stores of steps 2 and 3 are free of bank conflicts.
#pragma once

#include <utility>

#include "common.cuh"

namespace bq {

template <class KT>
struct LeafParams {
    using T = typename KT::T;
    const Leaf *leaves;
    const uint32_t *count_dev;   // non-null: persistent grid over *count_dev leaves; else one leaf per CTA
    T *bufs[2];
    T *out;            // destination buffer (the user buffer)
    int out_other;     // 1: write into bufs[parity ^ 1] instead (fallback chunk sort)
    uint64_t n_total;  // length of each data buffer (bounds the TMA reads)
    int aligned;       // both data buffers (and out) 16-byte aligned -> TMA bulk copies
    // level loop: non-null -> the leaves of the previous batch of levels, list
    // lsets[*set ^ 1] (+ class offset lcls), count csets[..] + cls
    const uint32_t *set;
    const Leaf *lsets[2];
    const uint32_t *csets[2];
    size_t lcls;
    int cls;
};

// ---- register element types -------------------------------------------------
struct RecKI {   // record key + the record's position in its leaf
    uint64_t k;
    uint32_t i;
};

template <class KT>
struct LeafTraits {
    using E = typename KT::K;
    static constexpr int IPT = Tune<KT>::LEAF_IPT, NTMAX = Tune<KT>::LEAF_NT;
};
template <>
struct LeafTraits<KRec> {
    using E = RecKI;
    static constexpr int IPT = Tune<KRec>::LEAF_IPT, NTMAX = Tune<KRec>::LEAF_NT;
};
template <>
struct LeafTraits<KPair> {
    using E = RecKI;
    static constexpr int IPT = Tune<KPair>::LEAF_IPT, NTMAX = Tune<KPair>::LEAF_NT;
};

// Leaf classes: class c runs CTAs of 32 << c threads and takes leaves of up to
// IPT * (32 << c) keys.
template <class KT>
constexpr int leaf_nclass() {
    int c = 0;
    while ((32 << c) < LeafTraits<KT>::NTMAX) c++;
    return c + 1;
}
constexpr int MAX_LEAF_CLASSES = 8;   // LevelCtrl::nleaf_cls, leaf-count words per set
template <class KT>
__host__ __device__ inline uint32_t leaf_class(uint32_t len) {
    uint32_t c = 0;
    while ((uint32_t)LeafTraits<KT>::IPT * (32u << c) < len) c++;
    return c;
}

__device__ __forceinline__ bool e_less(int32_t a, int32_t b) { return a < b; }
__device__ __forceinline__ bool e_less(uint64_t a, uint64_t b) { return a < b; }
__device__ __forceinline__ bool e_less(const RecKI &a, const RecKI &b) {
    return a.k < b.k || (a.k == b.k && a.i < b.i);
}
__device__ __forceinline__ int32_t e_min(int32_t a, int32_t b) { return min(a, b); }
__device__ __forceinline__ int32_t e_max(int32_t a, int32_t b) { return max(a, b); }
__device__ __forceinline__ uint64_t e_min(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint64_t e_max(uint64_t a, uint64_t b) { return a < b ? b : a; }
__device__ __forceinline__ RecKI e_min(const RecKI &a, const RecKI &b) { return e_less(b, a) ? b : a; }
__device__ __forceinline__ RecKI e_max(const RecKI &a, const RecKI &b) { return e_less(b, a) ? a : b; }
__device__ __forceinline__ void ce(int32_t &a, int32_t &b) {
    const int32_t lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}
template <class E>
__device__ __forceinline__ void ce(E &a, E &b) {
    const bool s = e_less(b, a);
    const E lo = s ? b : a, hi = s ? a : b;
    a = lo;
    b = hi;
}

// Batcher's odd-even merge sort on NP = 2^k >= N virtual elements, elements
// N..NP-1 being +infinity: every comparator that touches them is a no-op and
// is pruned at compile time (all comparators put the minimum at the lower
// index, so an infinite element never moves).  The comparator list is built
// by a constexpr function and applied by template recursion, so every
// register index is a compile-time constant.
constexpr int oem_np(int n) { return n <= 1 ? 1 : 2 * oem_np((n + 1) / 2); }
struct OemNet {
    int n;
    short lo[640], hi[640];
};
constexpr OemNet oem_make(int N) {
    OemNet r{};
    const int NP = oem_np(N);
    for (int p = 1; p < NP; p += p)
        for (int k = p; k > 0; k /= 2)
            for (int j = k % p; j + k < NP; j += k + k)
                for (int i = 0; i < k && i + j + k < NP; i++) {
                    const int lo = i + j, hi = i + j + k;
                    if (hi < N && (lo / (p + p)) == (hi / (p + p))) {
                        r.lo[r.n] = (short)lo;
                        r.hi[r.n] = (short)hi;
                        r.n++;
                    }
                }
    return r;
}
template <int N>
struct OemConst {
    static constexpr OemNet net = oem_make(N);
};
template <class E, int N, size_t... I>
__device__ __forceinline__ void oem_apply(E (&x)[N], std::index_sequence<I...>) {
    (ce(x[OemConst<N>::net.lo[I]], x[OemConst<N>::net.hi[I]]), ...);
}
template <class E, int N>
__device__ __forceinline__ void oem_sort(E (&x)[N]) {
    static_assert(N <= 64, "per-thread network size");
    oem_apply<E, N>(x, std::make_index_sequence<(size_t)OemConst<N>::net.n>{});
}

// ---- shared-memory planes ----------------------------------------------------
// Slots are element indices of the leaf; a plane has SLACK slots of room on
// both sides (the serial merge's pointers may run up to IPT + 1 slots past a
// run's ends in outputs that are discarded) and VW more for the 16-byte
// alignment offset of the TMA copies.
constexpr int LEAF_SLACK = 64;
#ifndef BQ_LEAF_PRED_ADV
#define BQ_LEAF_PRED_ADV 1
#endif

template <class KT, int NT>
struct LeafSmem {
    using E = typename LeafTraits<KT>::E;
    static constexpr int IPT = LeafTraits<KT>::IPT;
    static constexpr int CAP = IPT * NT + 16 + 2 * LEAF_SLACK;   // slots per plane incl. slack
    static constexpr bool REC = KT::is_record;
    static constexpr size_t KEY_BYTES = (size_t)CAP * (REC ? 8 : sizeof(E));
    static constexpr size_t bytes() { return 128 + KEY_BYTES + (REC ? (size_t)CAP * 4 : 0); }
    // plane pointers at slot 0 (slots may be negative down to -LEAF_SLACK)
    static __device__ __forceinline__ unsigned char *keyp(unsigned char *sm) { return sm + 128 + (size_t)LEAF_SLACK * (REC ? 8 : sizeof(E)); }
    static __device__ __forceinline__ uint32_t *idxp(unsigned char *sm) { return reinterpret_cast<uint32_t *>(sm + 128 + KEY_BYTES) + LEAF_SLACK; }
};

// 32-bit shared-window accesses (explicit ld/st.shared: the loops below
// walk byte addresses, with no generic-address conversion per access)
__device__ __forceinline__ int32_t lds_e(uint32_t a, int32_t *) {
    int32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint64_t lds_e(uint32_t a, uint64_t *) {
    uint64_t v;
    asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_e(uint32_t a, uint32_t *) {
    uint32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_e(uint32_t a, int32_t v) { asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }
__device__ __forceinline__ void sts_e(uint32_t a, uint32_t v) { asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }
__device__ __forceinline__ void sts_e(uint32_t a, uint64_t v) { asm volatile("st.shared.b64 [%0], %1;" ::"r"(a), "l"(v) : "memory"); }

// A plane seen through "cursors": keys walk byte addresses (cursor = address
// of the slot, step W), records walk slot numbers over their two planes.
template <class E>
struct LPlane {   // keys: one plane of E
    uint32_t k0;   // shared address of slot 0
    static constexpr int STEP = (int)sizeof(E);
    __device__ __forceinline__ uint32_t cur(int slot) const { return k0 + (uint32_t)(slot * STEP); }
    __device__ __forceinline__ E ldc(uint32_t c) const { return lds_e(c, (E *)nullptr); }
    __device__ __forceinline__ void stc(uint32_t c, E v) const { sts_e(c, v); }
};
template <>
struct LPlane<RecKI> {   // records: key plane (8 B) + index plane (4 B)
    uint32_t k0, i0;
    static constexpr int STEP = 1;
    __device__ __forceinline__ uint32_t cur(int slot) const { return (uint32_t)slot; }
    __device__ __forceinline__ RecKI ldc(uint32_t c) const {
        return RecKI{lds_e(k0 + c * 8u, (uint64_t *)nullptr), lds_e(i0 + c * 4u, (uint32_t *)nullptr)};
    }
    __device__ __forceinline__ void stc(uint32_t c, RecKI v) const {
        sts_e(k0 + c * 8u, v.k);
        sts_e(i0 + c * 4u, v.i);
    }
};

template <class KT>
__device__ __forceinline__ typename LeafTraits<KT>::E leaf_pad() {
    if constexpr (KT::is_record) return RecKI{~0ull, 0xffffffffu};   // after every real (key, index)
    else return (typename LeafTraits<KT>::E)KT::KMAX;
}

// x[0, cnt) -> slots base + k * dir (dir = +1 ascending, -1 descending).
template <class E, int IPT, class PL>
__device__ __forceinline__ void store_run(const PL &pl, const E (&x)[IPT], int cnt, int base, int dir) {
    BQ_CHECK(cnt >= 0 && cnt <= IPT);
    if (cnt == 0) return;
    if (cnt == IPT) {
        // the address walks in the run's direction (an IMAD per key on the
        // FMA pipe; a select of x[m] or x[IPT-1-m] would take the ALU pipe
        // the merge loop saturates)
        const uint32_t c0 = pl.cur(base), step = (uint32_t)(dir * PL::STEP);
#pragma unroll
        for (int m = 0; m < IPT; m++) pl.stc(c0 + (uint32_t)m * step, x[m]);
    } else {
#pragma unroll
        for (int k = 0; k < IPT; k++)
            if (k < cnt) pl.stc(pl.cur(base + k * dir), x[k]);
    }
}

// Barrier over the threads that share the runs of merge round r: a group of
// G = 2^(r+1) threads reads and rewrites only its own slots, so rounds whose
// groups fit a warp synchronise the warp, and larger groups their own slice
// of 128, 256 or 512 threads on named barriers with ids of their own (every
// use of an id is by the same threads with the same count, so instances of
// different rounds cannot mix); a group of the whole CTA uses barrier 0.
template <int NT>
__device__ __forceinline__ void group_sync(int r, int t) {
    const int G = 2 << r;
    if (G <= 32) __syncwarp();
    else if (G >= NT) __syncthreads();
    else if (G <= 128) named_bar_sync(1u + ((uint32_t)t >> 7), 128u);            // ids 1..8
    else if (G == 256) named_bar_sync(9u + ((uint32_t)t >> 8), 256u);            // ids 9..12
    else named_bar_sync(13u + ((uint32_t)t >> 9), 512u);                         // ids 13..14
}

// One leaf, by the whole CTA of NT threads.
template <class KT, int NT>
__device__ __forceinline__ void leaf_body(const LeafParams<KT> &P, const Leaf lf, unsigned char *sm, uint64_t *bar,
                                          uint32_t &phase) {
    using T = typename KT::T;
    using K = typename KT::K;
    using E = typename LeafTraits<KT>::E;
    using SM = LeafSmem<KT, NT>;
    using PL = LPlane<E>;
    constexpr int IPT = LeafTraits<KT>::IPT;
    constexpr bool REC = KT::is_record;
    constexpr uint32_t VW = REC ? 1u : 16u / (uint32_t)sizeof(T);
    unsigned char *kp = SM::keyp(sm);
    PL pl;
    pl.k0 = smem_u32(kp);
    if constexpr (REC) pl.i0 = smem_u32(SM::idxp(sm));
    const int t = (int)threadIdx.x;
    const int len = (int)lf.len;
    BQ_CHECK(len >= 0 && len <= IPT * NT && lf.begin + (uint64_t)len <= P.n_total);
    T *src = lf.parity ? P.bufs[1] : P.bufs[0];
    T *out = P.out_other ? (lf.parity ? P.bufs[0] : P.bufs[1]) : P.out;
    const uint64_t b = lf.begin;

    // ---- 1. load ------------------------------------------------------------
    int off = 0;   // slot of leaf element 0 (keys: 16-byte alignment offset)
    const T *gsrc = src;   // records: where the final gather reads from
    if constexpr (!REC) {
        off = (int)(b % VW);
        const uint64_t lo16 = b - (uint64_t)off, hi16 = (b + (uint64_t)len + VW - 1) / VW * VW;
        if (P.aligned && hi16 <= P.n_total) {
            if (t == 0) {
                fence_proxy_async_smem();   // earlier generic accesses of the plane precede the async write
                const uint32_t bytes = (uint32_t)((hi16 - lo16) * sizeof(T));
                mbar_arrive_expect_tx(bar, bytes);
                tma_load_1d(kp, src + lo16, bytes, bar);
            }
            mbar_wait(bar, phase);
            phase ^= 1;
        } else {
            for (int q = t; q < len; q += NT) reinterpret_cast<T *>(kp)[off + q] = src[b + q];
            __syncthreads();
        }
    } else {
        // keys into the key plane; the gather reads the records from `src`,
        // or, when the leaf already sits in the output buffer, from a copy of
        // them in the same range of the other buffer (free: the segment owns
        // [b, b + len) in both buffers)
        T *other = lf.parity ? P.bufs[0] : P.bufs[1];
        const bool copy = src == out;
        if (copy) gsrc = other;
        for (int q = t; q < len; q += NT) {
            const T v = src[b + q];
            reinterpret_cast<uint64_t *>(kp)[q] = KT::key(v);
            if (copy) other[b + q] = v;
        }
        __syncthreads();
    }

    // ---- 2. per-thread network ---------------------------------------------------
    E x[IPT];
    const int nruns = (len + IPT - 1) / IPT;
    {
        const int s0 = t * IPT;
        if constexpr (REC) {
#pragma unroll
            for (int k = 0; k < IPT; k++) {
                const int slot = s0 + k;
                x[k] = slot < len ? RecKI{lds_e(pl.k0 + (uint32_t)slot * 8u, (uint64_t *)nullptr), (uint32_t)slot}
                                  : leaf_pad<KT>();
            }
        } else {
            const uint32_t c0 = pl.cur(off + s0);
            if (s0 + IPT <= len) {
#pragma unroll
                for (int k = 0; k < IPT; k++) x[k] = (E)KT::key((T)pl.ldc(c0 + (uint32_t)(k * PL::STEP)));
            } else {
#pragma unroll
                for (int k = 0; k < IPT; k++)
                    x[k] = s0 + k < len ? (E)KT::key((T)pl.ldc(c0 + (uint32_t)(k * PL::STEP))) : leaf_pad<KT>();
            }
        }
        oem_sort<E, IPT>(x);
    }

    // ---- 3. merge rounds ---------------------------------------------------------
    // outputs of the current step: x[0, cnt) go to slots base + k * dir
    int cnt = t < nruns ? min(IPT, len - t * IPT) : 0;
    int base = t * IPT, dir = 1;
    bool fin = nruns <= 1;
    if (!fin && (t & 1)) {   // odd runs descending
        base = t * IPT + cnt - 1;
        dir = -1;
    }
    for (int r = 0; !fin; r++) {
        // (the initial runs: each thread owns its slots, no barrier needed before)
        store_run<E, IPT>(pl, x, cnt, off + base, dir);
        group_sync<NT>(r, t);
        const int RL = IPT << r;
        const int g = t >> (r + 1), j = t & ((2 << r) - 1);
        const int a0 = g * 2 * RL;
        fin = 2 * RL >= len;
        cnt = 0;
        if (a0 < len) {
            const int na = min(RL, len - a0), tot = min(2 * RL, len - a0), nb = tot - na;
            const int d = j * IPT;
            if (d < tot) {
                cnt = min(IPT, tot - d);
                // merge path: ai = #A keys among the first d outputs (ties: A first);
                // B[q] sits at slot a0 + tot - 1 - q (descending): A[m] at cursor
                // ca + m, B[d-1-m] at cursor cb + m
                int lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
                const uint32_t ca = pl.cur(off + a0), cb = pl.cur(off + a0 + tot - d);
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    const uint32_t o = (uint32_t)(mid * PL::STEP);
                    const E av = pl.ldc(ca + o), bv = pl.ldc(cb + o);
                    if (e_less(bv, av)) hi = mid;
                    else lo = mid + 1;
                }
                BQ_CHECK(lo >= 0 && lo <= na && d - lo >= 0 && d - lo <= nb && a0 + tot <= len);
                uint32_t pa = ca + (uint32_t)(lo * PL::STEP);
                uint32_t pb = pl.cur(off + a0 + tot - 1 - (d - lo));
                // serial merge: out = min(head kept, head just loaded), keep the
                // max, advance the side of the output (tA: side A)
                const E ka = pl.ldc(pa), kb = pl.ldc(pb);
                bool tA = !e_less(kb, ka);
                x[0] = e_min(ka, kb);
                E hv = e_max(ka, kb), nv;
                if (tA) pa += (uint32_t)PL::STEP;
                else pb -= (uint32_t)PL::STEP;
                nv = pl.ldc(tA ? pa : pb);
#pragma unroll
                for (int k = 1; k < IPT; k++) {
                    x[k] = e_min(hv, nv);
                    const bool keep_side = e_less(nv, hv);   // the output is nv: same side again
                    hv = e_max(hv, nv);
                    tA = tA == keep_side;
                    if (k + 1 < IPT) {
#if BQ_LEAF_PRED_ADV
                        // predicated pointer advances (one add each, on the
                        // FMA pipe) instead of both advanced values computed
                        // and the kept ones selected (two more ALU selects)
                        asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t"
                            "@q add.u32 %0, %0, %3;\n\t@!q sub.u32 %1, %1, %3;\n\t}"
                            : "+r"(pa), "+r"(pb)
                            : "r"((uint32_t)tA), "n"((int)PL::STEP));
#else
                        if (tA) pa += (uint32_t)PL::STEP;
                        else pb -= (uint32_t)PL::STEP;
#endif
                        nv = pl.ldc(tA ? pa : pb);
                    }
                }
                if (!fin && (g & 1)) {
                    base = a0 + tot - 1 - d;
                    dir = -1;
                } else {
                    base = a0 + d;
                    dir = 1;
                }
            }
        }
        group_sync<NT>(r, t);   // the group has read its inputs before its slots are overwritten
    }
    __syncthreads();

    // ---- 4. write out --------------------------------------------------------------
    // x[0, cnt) are the outputs [base, base + cnt) of the sorted leaf (ascending)
    if constexpr (REC) {
#pragma unroll
        for (int k = 0; k < IPT; k++) {
            if (k < cnt) {
                const uint32_t pos = (uint32_t)(base + k);
                BQ_CHECK(pos < (uint32_t)len && x[k].i < (uint32_t)len);
                constexpr uint32_t V = sizeof(T) / 16;
                const uint4 *s4 = reinterpret_cast<const uint4 *>(gsrc + b + x[k].i);
                uint4 *d4 = reinterpret_cast<uint4 *>(out + b + pos);
                uint4 v[V];
#pragma unroll
                for (uint32_t c = 0; c < V; c++) v[c] = s4[c];
#pragma unroll
                for (uint32_t c = 0; c < V; c++) d4[c] = v[c];
            }
        }
    } else {
        T *plane = reinterpret_cast<T *>(kp);
        E y[IPT];
#pragma unroll
        for (int k = 0; k < IPT; k++) y[k] = (E)KT::from_key((K)x[k]);
        store_run<E, IPT>(pl, y, cnt, off + base, 1);
        if (P.aligned) {
            fence_proxy_async_smem();
            __syncthreads();
            const uint64_t e = b + (uint64_t)len;
            const uint64_t ls = (b + VW - 1) / VW * VW, le = e / VW * VW;
            if (t == 0 && le > ls) {
                tma_store_1d(out + ls, plane + off + (ls - b), (uint32_t)((le - ls) * sizeof(T)));
                bulk_commit();
            }
            // head and tail (< 16 bytes each) outside the bulk body
            if (t < 2 * (int)VW) {   // (NT may be a single warp)
                const int u = t;
                const bool tail = u >= (int)VW;
                const uint64_t pos = tail ? (le > ls ? le : ls) + (uint64_t)(u - VW) : b + (uint64_t)u;
                const bool ok = tail ? pos < e : pos < (ls < e ? ls : e);
                if (ok) out[pos] = plane[off + (pos - b)];
            }
            if (t == 0) bulk_wait_read0();   // the plane may be reused once the store has read it
        } else {
            __syncthreads();
            for (int q = t; q < len; q += NT) out[b + q] = plane[off + q];
        }
    }
}

template <class KT, int NT>
__global__ void __launch_bounds__(NT, (LeafTraits<KT>::NTMAX / NT) > 0 ? LeafTraits<KT>::NTMAX / NT : 1)
    k_leaf(const LeafParams<KT> Pin) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw);
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t phase = 0;
    __shared__ LeafParams<KT> sP;
    if (threadIdx.x == 0) {
        sP = Pin;
        if (sP.set) {
            const uint32_t set = *sP.set ^ 1u;
            sP.leaves = sP.lsets[set] + sP.lcls;
            sP.count_dev = sP.csets[set] + sP.cls;
        }
    }
    __syncthreads();
    const LeafParams<KT> &P = sP;
    const uint32_t nleaves = P.count_dev ? *P.count_dev : gridDim.x;
    for (uint32_t li = blockIdx.x; li < nleaves; li += gridDim.x) {
        if (li != blockIdx.x) __syncthreads();   // the previous leaf's readers of the planes are done
        if (threadIdx.x == 0 && li + gridDim.x < nleaves) {
            // warm L2 with this CTA's next leaf while this one is sorted
            const Leaf nx = P.leaves[li + gridDim.x];
            const typename KT::T *nsrc = nx.parity ? P.bufs[1] : P.bufs[0];
            const uint64_t a = (uint64_t)(nsrc + nx.begin) & ~15ull;
            const uint64_t z = ((uint64_t)(nsrc + nx.begin + nx.len) + 15) & ~15ull;
            if (P.aligned && z > a)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)(z - a)) : "memory");
        }
        leaf_body<KT, NT>(P, P.leaves[li], smem_raw, bar, phase);
    }
    if (threadIdx.x == 0) bulk_wait0();
}

template <class KT, int NT>
constexpr size_t leaf_smem_bytes() {
    return LeafSmem<KT, NT>::bytes();
}

// host: launch the leaf kernel of class c (NT = 32 << c) over `count` leaves
// count > 0: one CTA per leaf; count == 0: persistent grid (resident CTAs)
// over LP.count_dev leaves
template <class KT, int NT>
cudaError_t launch_leaf_nt(const LeafParams<KT> &LP, uint32_t count, cudaStream_t s) {
    constexpr size_t smem = leaf_smem_bytes<KT, NT>();
    static CapCache cc;
    int cap = 0;
    cudaError_t e = resident_ctas(k_leaf<KT, NT>, NT, smem, cc, &cap);
    if (e != cudaSuccess) return e;
    // persistent grids: at most 2 CTAs per SM (small classes hold few keys)
    const uint32_t pgrid = (uint32_t)cap < 296u ? (uint32_t)cap : 296u;
    k_leaf<KT, NT><<<count ? count : pgrid, NT, smem, s>>>(LP);
    return cudaGetLastError();
}

template <class KT, int C = 0>
cudaError_t launch_leaf_class(int cls, const LeafParams<KT> &LP, uint32_t count, cudaStream_t s) {
    if constexpr (C >= leaf_nclass<KT>()) {
        return cudaErrorInvalidValue;
    } else {
        if (cls == C) return launch_leaf_nt<KT, (32 << C)>(LP, count, s);
        return launch_leaf_class<KT, C + 1>(cls, LP, count, s);
    }
}

}  // namespace bq
