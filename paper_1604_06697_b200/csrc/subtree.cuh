// subtree.cuh — SURVEY §8(f) N1, second half: the deep levels of the
// recursion moved off HBM.  A segment of S < len <= SUB elements (SUB = the
// elements of 128 KB) is not partitioned by the breadth-first level passes;
// one CTA loads it into shared memory and finishes its subtree depth-first
// there — the paper's explicit stack ("push the larger side,
// continue with the smaller") with three-way block partitions
// in shared memory — down to pieces of <= S elements, which go to the leaf
// lists (a8), and equal bands, which are final.
//
// One partition step over A[o, o+m) of the shared-memory copy: every thread
// holds up to IPT elements in registers (index tid + k*NT), classifies them
// against the pivot with branch-free counters (Alg. 3 l.8-9), a CTA scan of
// the (<, =, >) counts gives every thread its offsets, and after a barrier
// the elements are written back to A in [< | = | >] order.  The pivot is the
// same sampled rule as the level passes (a1), read from shared memory.
#pragma once

namespace bq {

constexpr int SUB_THREADS = 1024;
constexpr int SUB_BYTES = 96 * 1024;   // per buffer; two buffers (A, B) per CTA
constexpr int SUB_STACK = 48;

template <class KT>
constexpr uint32_t sub_elems() { return (uint32_t)(SUB_BYTES / sizeof(typename KT::T)); }
template <class KT>
constexpr bool sub_enabled() { return sub_elems<KT>() > (uint32_t)Tune<KT>::LEAF; }

template <class KT>
struct SubParams {
    using T = typename KT::T;
    T *bufs[2];                  // [0]: the user buffer (final), [1]: scratch
    const Leaf *jobs;            // subtree segments of this batch: begin, len, parity, depth (pad)
    const uint32_t *job_count;
    Leaf *leaves;                // leaf lists of this batch (one per class, leaf_cap each)
    uint32_t *leaf_counts;
    uint32_t leaf_cap;
    Leaf *fallback;
    uint32_t *fallback_count;
    LevelCtrl *ctrl;             // statistics (element passes, bands, leaves)
    uint32_t *overflow;          // set when a leaf list would overflow (the call then fails)
    int aligned;                 // both buffers 16-byte aligned: bulk (TMA) copies
    uint32_t leaf_max;
    int32_t depth_limit;
    int32_t pivot_rule;
};

template <class KT>
struct SubSmem {
    using T = typename KT::T;
    static constexpr uint32_t CAP = sub_elems<KT>() + 16;   // + the job's 16-byte phase; a 16-byte multiple
    alignas(128) T buf[2][CAP];
    uint64_t bar;
    uint32_t wl[SUB_THREADS / 32], we[SUB_THREADS / 32], wg[SUB_THREADS / 32];
    uint32_t so[SUB_STACK], sm[SUB_STACK], sd[SUB_STACK], sb[SUB_STACK];   // offset, length, depth, buffer
    uint32_t sp, tot_l, tot_e;
    uint64_t piv;
    uint64_t passes, band;
    uint32_t nleaf;
};

template <class KT>
constexpr int sub_smem_bytes() { return (int)sizeof(SubSmem<KT>); }

// a final range dst[0, m) <- X[0, m) (same 16-byte phase).  Bulk: thread 0
// alone (TMA body + the < 16-byte head and tail); the range is never written
// again in this job, so the store is not waited for until the next job's
// load.  Otherwise: plain stores by the whole CTA.
template <class T, int NT>
__device__ __forceinline__ void sub_store(T *dst, const T *X, uint32_t m, bool bulk) {
    constexpr uint32_t W = sizeof(T), VW = W >= 16 ? 1 : 16 / W;
    if (!bulk) {
        for (uint32_t i = threadIdx.x; i < m; i += NT) dst[i] = X[i];
        return;
    }
    if (threadIdx.x != 0) return;
    const uint32_t ph = (uint32_t)(((uintptr_t)dst & 15) / W);
    const uint32_t hb = ph ? (VW - ph < m ? VW - ph : m) : 0;
    const uint32_t nb = (m - hb) / VW * VW;
    if (nb) {
        tma_store_1d(dst + hb, X + hb, nb * W);
        bulk_commit();
    }
    for (uint32_t i = 0; i < hb; i++) dst[i] = X[i];
    for (uint32_t i = hb + nb; i < m; i++) dst[i] = X[i];
}

template <class KT, int NT>
__global__ void __launch_bounds__(NT, 1) k_subtree(SubParams<KT> P) {
    using T = typename KT::T;
    using K = typename KT::K;
    constexpr uint32_t NW = NT / 32;
    constexpr uint32_t W = sizeof(T);
    constexpr uint32_t VW = W >= 16 ? 1 : 16 / W;   // elements per 16 bytes
    extern __shared__ __align__(128) unsigned char smraw[];
    SubSmem<KT> &sm = *reinterpret_cast<SubSmem<KT> *>(smraw);
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t njobs = *P.job_count;
    T *const out = P.bufs[0];
    const int prule = P.pivot_rule == BQ_PIVOT_MO3 ? BQ_PIVOT_MO3 : BQ_PIVOT_NINTHER;   // R20
    if (tid == 0) {
        sm.passes = 0;
        sm.band = 0;
        sm.nleaf = 0;
        mbar_init(&sm.bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async_smem();
    }
    uint32_t phase = 0;

    for (uint32_t j = blockIdx.x; j < njobs; j += gridDim.x) {
        const Leaf jb = P.jobs[j];
        const T *src = P.bufs[jb.parity & 1] + jb.begin;
        const uint32_t len = jb.len;
        // X[ph + i] <-> element i: the job's 16-byte phase in both buffers
        const uint32_t ph = (uint32_t)(((uintptr_t)src & 15) / W);
        const uint32_t hb = ph ? (VW - ph < len ? VW - ph : len) : 0;   // head before the first 16 B
        const uint32_t nb = (len - hb) / VW * VW;                         // aligned body
        if (tid == 0) bulk_wait_read0();   // the previous job's bulk stores have read the buffers
        __syncthreads();                   // ... and its readers of the buffers and the stack are done
        T *const X0 = sm.buf[0] + ph;
        T *const X1 = sm.buf[1] + ph;
        if (P.aligned) {
            if (tid == 0) {
                if (nb) {
                    mbar_arrive_expect_tx(&sm.bar, nb * W);
                    tma_load_1d(X0 + hb, src + hb, nb * W, &sm.bar);
                } else {
                    mbar_arrive(&sm.bar);
                }
            }
            for (uint32_t i = tid; i < hb; i += NT) X0[i] = src[i];
            for (uint32_t i = hb + nb + tid; i < len; i += NT) X0[i] = src[i];
            mbar_wait(&sm.bar, phase);
            phase ^= 1;
        } else {
            for (uint32_t i = tid; i < len; i += NT) X0[i] = src[i];
        }
        if (tid == 0) {
            sm.so[0] = 0;
            sm.sm[0] = len;
            sm.sd[0] = jb.pad;
            sm.sb[0] = 0;
            sm.sp = 1;
        }
        __syncthreads();
        for (;;) {
            const uint32_t sp = sm.sp;
            if (sp == 0) break;
            const uint32_t o = sm.so[sp - 1], m = sm.sm[sp - 1], d = sm.sd[sp - 1], b = sm.sb[sp - 1];
            const T *S = (b ? X1 : X0) + o;
            T *D = (b ? X0 : X1) + o;
            if (m <= P.leaf_max || (int)d >= P.depth_limit) {
                // a piece: stored when the job ends, then sorted by the leaf
                // kernels (or the depth-capped fallback)
                __syncthreads();   // everyone has read the top
                if (tid == 0) {
                    sm.sp = sp - 1;
                    const Leaf lf{jb.begin + o, m, 0, 0};
                    if (m <= P.leaf_max) {
                        const uint32_t lc = leaf_class<KT>(m);
                        const uint32_t li = atomicAdd(&P.leaf_counts[lc], 1u);
                        if (li < P.leaf_cap) P.leaves[lc * P.leaf_cap + li] = lf;
                        else *P.overflow = 1;
                        sm.nleaf++;
                    } else {
                        P.fallback[atomicAdd(P.fallback_count, 1u)] = lf;
                        atomicAdd(&P.ctrl->nfallback, 1u);
                    }
                }
                sub_store<T, NT>(out + jb.begin + o, S, m, P.aligned != 0);
                __syncthreads();
                continue;
            }
            // a1: ninther (Mo3 for the Mo3 rule) of S[0, m), lane 0 of warp 0
            if (tid == 0) sm.piv = (uint64_t)select_pivot<KT>(S, 0, m, prule);
            __syncthreads();
            const K pk = (K)sm.piv;
            // count (branch-free counters, Alg. 3 l.8-9)
            uint32_t cl = 0, ce = 0;
            for (uint32_t i = tid; i < m; i += NT) {
                const K kk = KT::key(S[i]);
                cl += kk < pk;
                ce += !(kk < pk) && !(pk < kk);
            }
            const uint32_t mine = (m > tid) ? (m - tid + NT - 1) / NT : 0;
            const uint32_t cg = mine - cl - ce;
            // CTA scan of the three counts
            uint32_t il = cl, ie = ce, ig = cg;
#pragma unroll
            for (int dd = 1; dd < 32; dd <<= 1) {
                const uint32_t a1 = __shfl_up_sync(0xffffffffu, il, dd);
                const uint32_t a2 = __shfl_up_sync(0xffffffffu, ie, dd);
                const uint32_t a3 = __shfl_up_sync(0xffffffffu, ig, dd);
                if (lane >= (uint32_t)dd) {
                    il += a1;
                    ie += a2;
                    ig += a3;
                }
            }
            if (lane == 31) {
                sm.wl[warp] = il;
                sm.we[warp] = ie;
                sm.wg[warp] = ig;
            }
            __syncthreads();
            if (warp == 0) {
                const uint32_t vl = lane < NW ? sm.wl[lane] : 0, ve = lane < NW ? sm.we[lane] : 0;
                const uint32_t vg = lane < NW ? sm.wg[lane] : 0;
                uint32_t sl = vl, se = ve, sg = vg;
#pragma unroll
                for (int dd = 1; dd < 32; dd <<= 1) {
                    const uint32_t a1 = __shfl_up_sync(0xffffffffu, sl, dd);
                    const uint32_t a2 = __shfl_up_sync(0xffffffffu, se, dd);
                    const uint32_t a3 = __shfl_up_sync(0xffffffffu, sg, dd);
                    if (lane >= (uint32_t)dd) {
                        sl += a1;
                        se += a2;
                        sg += a3;
                    }
                }
                if (lane < NW) {
                    sm.wl[lane] = sl - vl;
                    sm.we[lane] = se - ve;
                    sm.wg[lane] = sg - vg;
                }
                if (lane == 31) {
                    sm.tot_l = sl;
                    sm.tot_e = se;
                }
            }
            __syncthreads();
            const uint32_t LT = sm.tot_l, EQ = sm.tot_e;
            uint32_t rl = sm.wl[warp] + il - cl;
            uint32_t re = LT + sm.we[warp] + ie - ce;
            uint32_t rg = LT + EQ + sm.wg[warp] + ig - cg;
            // rearrangement: the same elements in the same order, into the other buffer
            for (uint32_t i = tid; i < m; i += NT) {
                const T x = S[i];
                const K kk = KT::key(x);
                const bool lt = kk < pk, gt = pk < kk;
                D[lt ? rl : (gt ? rg : re)] = x;
                rl += lt;
                rg += gt;
                re += !lt && !gt;
            }
            if (P.aligned) fence_proxy_async_smem();   // D becomes visible to the bulk stores
            __syncthreads();
            // the equal band is final (a6)
            if (EQ) sub_store<T, NT>(out + jb.begin + o + LT, D + LT, EQ, P.aligned != 0);
            if (tid == 0) {
                sm.passes += m;
                sm.band += EQ;
                const uint32_t G = m - LT - EQ;
                uint32_t s = sp - 1;
                // children: the larger one below, the smaller one on top
                const uint32_t bo = o + LT + EQ;
                const bool gfirst = G >= LT;
                const uint32_t o1 = gfirst ? bo : o, m1 = gfirst ? G : LT;
                const uint32_t o2 = gfirst ? o : bo, m2 = gfirst ? LT : G;
                if (m1 && s < SUB_STACK) {
                    sm.so[s] = o1;
                    sm.sm[s] = m1;
                    sm.sd[s] = d + 1;
                    sm.sb[s] = b ^ 1;
                    s++;
                }
                if (m2 && s < SUB_STACK) {
                    sm.so[s] = o2;
                    sm.sm[s] = m2;
                    sm.sd[s] = d + 1;
                    sm.sb[s] = b ^ 1;
                    s++;
                }
                sm.sp = s;
            }
            __syncthreads();
        }
    }
    if (tid == 0) bulk_wait0();
    __syncthreads();
    if (tid == 0) {
        if (sm.passes) atomicAdd(&P.ctrl->element_passes, (unsigned long long)sm.passes);
        if (sm.band) atomicAdd(&P.ctrl->band_elems, (unsigned long long)sm.band);
        if (sm.nleaf) atomicAdd(&P.ctrl->nleaf, sm.nleaf);
    }
}

}  // namespace bq
