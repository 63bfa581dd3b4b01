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
constexpr int SUB_BYTES = 128 * 1024;
constexpr int SUB_STACK = 48;

template <class KT>
constexpr uint32_t sub_elems() { return (uint32_t)(SUB_BYTES / sizeof(typename KT::T)); }
// the subtree path pays off when a subtree spans at least two leaf sizes
template <class KT>
constexpr bool sub_enabled() { return sub_elems<KT>() >= 2u * (uint32_t)Tune<KT>::LEAF; }

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
    alignas(128) T a[sub_elems<KT>() + 16 / sizeof(T) + 1];   // + the job's 16-byte phase
    uint64_t bar;
    uint32_t wl[SUB_THREADS / 32], we[SUB_THREADS / 32], wg[SUB_THREADS / 32];
    uint32_t so[SUB_STACK], sm[SUB_STACK], sd[SUB_STACK];
    uint32_t sp, tot_l, tot_e;
    uint64_t piv;
    uint64_t passes, band;
    uint32_t nleaf;
};

template <class KT>
constexpr int sub_smem_bytes() { return (int)sizeof(SubSmem<KT>); }

template <class KT, int NT>
__global__ void __launch_bounds__(NT, 1) k_subtree(SubParams<KT> P) {
    using T = typename KT::T;
    using K = typename KT::K;
    constexpr uint32_t SUB = sub_elems<KT>();
    constexpr uint32_t IPT = SUB / NT;
    constexpr uint32_t NW = NT / 32;
    static_assert(SUB % NT == 0 && IPT <= 32, "elements per thread");
    extern __shared__ __align__(128) unsigned char smraw[];
    SubSmem<KT> &sm = *reinterpret_cast<SubSmem<KT> *>(smraw);
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t njobs = *P.job_count;
    constexpr uint32_t W = sizeof(T);
    constexpr uint32_t VW = W >= 16 ? 1 : 16 / W;   // elements per 16 bytes
    T *const out = P.bufs[0];
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
        // A[ph + i] <-> element i: the same 16-byte phase as the job in memory
        const uint32_t ph = (uint32_t)(((uintptr_t)src & 15) / W);
        const uint32_t hb = ph ? (VW - ph < len ? VW - ph : len) : 0;   // head before the first 16 B
        const uint32_t nb = (len - hb) / VW * VW;                         // aligned body
        if (tid == 0) bulk_wait_read0();   // the previous job's bulk store has read A
        __syncthreads();   // ... and its readers of A and the stack are done
        T *const A = sm.a + ph;
        if (P.aligned) {
            if (tid == 0) {
                if (nb) {
                    mbar_arrive_expect_tx(&sm.bar, nb * W);
                    tma_load_1d(A + hb, src + hb, nb * W, &sm.bar);
                } else {
                    mbar_arrive(&sm.bar);
                }
            }
            for (uint32_t i = tid; i < hb; i += NT) A[i] = src[i];
            for (uint32_t i = hb + nb + tid; i < len; i += NT) A[i] = src[i];
            mbar_wait(&sm.bar, phase);
            phase ^= 1;
        } else {
            for (uint32_t i = tid; i < len; i += NT) A[i] = src[i];
        }
        if (tid == 0) {
            sm.so[0] = 0;
            sm.sm[0] = len;
            sm.sd[0] = jb.pad;
            sm.sp = 1;
        }
        __syncthreads();
        for (;;) {
            const uint32_t sp = sm.sp;
            if (sp == 0) break;
            const uint32_t o = sm.so[sp - 1], m = sm.sm[sp - 1], d = sm.sd[sp - 1];
            __syncthreads();   // everyone has read the top before it changes
            if (m <= P.leaf_max || (int)d >= P.depth_limit) {
                // a piece: to the leaf lists (or the depth-capped fallback list,
                // P:293-299); A is written to the user buffer when the job ends
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
                __syncthreads();
                continue;
            }
            // a1: the pivot of A[o, o+m) (warp 0; generic loads from shared memory)
            if (warp == 0) {
                const K p = select_pivot_warp<KT>(A + o, 0, m, P.pivot_rule, lane);
                if (lane == 0) sm.piv = (uint64_t)p;
            }
            __syncthreads();
            const K pk = (K)sm.piv;
            // classify (branch-free counters) with the elements held in registers
            T x[IPT];
            uint32_t cl = 0, ce = 0, cg = 0, cls = 0, ceq = 0;
#pragma unroll
            for (uint32_t k = 0; k < IPT; k++) {
                const uint32_t i = tid + k * NT;
                if (i < m) {
                    x[k] = A[o + i];
                    const K kk = KT::key(x[k]);
                    const bool lt = kk < pk, gt = pk < kk;
                    cls |= (uint32_t)lt << k;
                    ceq |= (uint32_t)(!lt && !gt) << k;
                    cl += lt;
                    ce += !lt && !gt;
                    cg += gt;
                }
            }
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
            __syncthreads();   // also: every element of A[o, o+m) is in registers
            if (warp == 0) {
                uint32_t vl = lane < NW ? sm.wl[lane] : 0, ve = lane < NW ? sm.we[lane] : 0;
                uint32_t vg = lane < NW ? sm.wg[lane] : 0;
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
            uint32_t rl = o + sm.wl[warp] + il - cl;
            uint32_t re = o + LT + sm.we[warp] + ie - ce;
            uint32_t rg = o + LT + EQ + sm.wg[warp] + ig - cg;
#pragma unroll
            for (uint32_t k = 0; k < IPT; k++) {
                const uint32_t i = tid + k * NT;
                if (i < m) {
                    const bool lt = (cls >> k) & 1, eq = (ceq >> k) & 1;
                    const uint32_t dst = lt ? rl : (eq ? re : rg);
                    A[dst] = x[k];
                    rl += lt;
                    re += eq;
                    rg += !lt && !eq;
                }
            }
            __syncthreads();
            if (tid == 0) {
                sm.passes += m;
                sm.band += EQ;
                const uint32_t G = m - LT - EQ;
                // children: the larger one below, the smaller one on top
                uint32_t s = sp - 1;
                const uint32_t bo = o + LT + EQ;
                const bool gfirst = G >= LT;   // push the larger first
                const uint32_t o1 = gfirst ? bo : o, m1 = gfirst ? G : LT;
                const uint32_t o2 = gfirst ? o : bo, m2 = gfirst ? LT : G;
                if (m1 && s < SUB_STACK) {
                    sm.so[s] = o1;
                    sm.sm[s] = m1;
                    sm.sd[s] = d + 1;
                    s++;
                }
                if (m2 && s < SUB_STACK) {
                    sm.so[s] = o2;
                    sm.sm[s] = m2;
                    sm.sd[s] = d + 1;
                    s++;
                }
                sm.sp = s;
            }
            __syncthreads();
        }
        // the job's final layout (pieces for the leaves, finished equal bands)
        T *dst = out + jb.begin;
        if (P.aligned) {
            fence_proxy_async_smem();
            __syncthreads();
            if (tid == 0 && nb) {
                tma_store_1d(dst + hb, A + hb, nb * W);
                bulk_commit();
            }
            for (uint32_t i = tid; i < hb; i += NT) dst[i] = A[i];
            for (uint32_t i = hb + nb + tid; i < len; i += NT) dst[i] = A[i];
        } else {
            for (uint32_t i = tid; i < len; i += NT) dst[i] = A[i];
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
