// loop.cuh — device-side control of the sort's level loop (hot-path step a7)
// and the depth-cap fallback (a9) over every capped segment of a sort.
//
// The paper drives its partitioner with an explicit stack.  Here
// one breadth-first level of that recursion is a fixed sequence of launches
// (multiway count/scan/scatter/post when enabled, binary partition, k_post,
// k_fill, k_level_end) that reads the current level from device memory
// (LoopPtrs, partition.cuh).  The sequence is the body of a CUDA-graph WHILE
// node whose condition k_level_end sets from the level's child count, so a
// sort is enqueued without any host round trip; leaves are sorted by an IF
// node inside the loop whenever their lists fill up, and at the end.
#pragma once

#include "common.cuh"
#include "partition.cuh"

namespace bq {

// misc words of a sort's workspace (driver.cuh): counts that live across levels
struct LoopMisc {
    uint32_t fb_count;                          // depth-capped segments
    uint32_t level;                             // current level of the loop
    uint32_t nflush;                            // leaf flushes executed
    uint32_t overflow;                          // a leaf or copy list was full (the call fails)
    uint32_t leaf_counts[2][MAX_LEAF_CLASSES];  // fill of each leaf-class list, by set
    uint32_t copy_count[2];                     // records: finished equal runs to copy, by set
    uint32_t set;                               // list set of the current batch of levels
    uint32_t pad[9];
};
static_assert(sizeof(LoopMisc) == 128, "LoopMisc layout");

// End of one level: advance the level counter and continue while the level
// had children (a level without segments runs as no-ops: its kernels find
// zero tiles and segments).  In graph mode this sets the WHILE condition (and, at the
// end, the IF condition of the fallback); the host-driven mode reads the
// control blocks instead.
template <class KT>
__global__ void k_level_end(LoopPtrs<KT> lp, LoopMisc *misc, uint32_t batch, int use_cond,
                            cudaGraphConditionalHandle h_loop, cudaGraphConditionalHandle h_fb) {
    const uint32_t lv = misc->level;
    const LevelCtrl &c = lp.ctrl[lv];
    const bool more = (c.nseg_next + c.nmseg_next) > 0 && lv + LOOP_BATCH + 1 < (uint32_t)MAX_LEVELS;
    misc->level = lv + 1;
    misc->set = ((lv + 1) / batch) & 1u;
    if (use_cond) {
        cudaGraphSetConditional(h_loop, more ? 1u : 0u);
        cudaGraphSetConditional(h_fb, (!more && misc->fb_count > 0) ? 1u : 0u);
    }
}

// after the previous level's leaves are sorted: their set is empty again
static __global__ void k_flush_reset(LoopMisc *misc) {
    const uint32_t set = misc->set ^ 1u;
    for (int k = 0; k < MAX_LEAF_CLASSES; k++) misc->leaf_counts[set][k] = 0;
    misc->copy_count[set] = 0;
    misc->nflush++;
}

// ---- a9: the depth-cap fallback over all capped segments ----------------------
// Each capped segment [b, b+len) (data in bufs[parity]) is cut into S-element
// chunks sorted by the leaf kernel into the other buffer, then merged pairwise
// (runs of S, 2S, ...) until one run remains, and copied to the user buffer if
// it ended in the scratch buffer.  The paper's Introsort uses Heapsort here
// (P:64-70): both guarantee O(len log len).
constexpr int MERGE_THREADS = 256, MERGE_IPT = 8;
constexpr uint32_t MERGE_TILE = MERGE_THREADS * MERGE_IPT;

struct FbState {
    uint32_t nseg;     // capped segments
    uint32_t nchunk;   // their S-element chunks (the chunk leaf list's count)
    uint32_t ntiles;   // merge tiles over all segments
    uint32_t npass;    // merge passes (enough for the longest segment)
    uint32_t pass;     // passes done
    uint32_t pad;
    uint64_t w;        // current run width
};

// one CTA of 1024 threads: chunk leaves, merge-tile prefix, pass count
static __global__ void __launch_bounds__(1024) k_fb_setup(const Leaf *fb, const uint32_t *fb_count, Leaf *chunks,
                                                          uint32_t *tprefix, FbState *st, uint32_t S, int use_cond,
                                                          cudaGraphConditionalHandle h) {
    __shared__ uint32_t s_c[1024], s_t[1024];
    __shared__ uint32_t s_cbase, s_tbase, s_max;
    const uint32_t F = *fb_count, tid = threadIdx.x;
    if (tid == 0) {
        s_cbase = 0;
        s_tbase = 0;
        s_max = 0;
    }
    __syncthreads();
    for (uint32_t f0 = 0; f0 < F; f0 += 1024) {
        const uint32_t f = f0 + tid;
        const Leaf lf = f < F ? fb[f] : Leaf{0, 0, 0, 0};
        const uint32_t nc = (lf.len + S - 1) / S, nt = (lf.len + MERGE_TILE - 1) / MERGE_TILE;
        s_c[tid] = nc;
        s_t[tid] = nt;
        if (f < F) atomicMax(&s_max, lf.len);
        __syncthreads();
        for (uint32_t d = 1; d < 1024; d <<= 1) {   // inclusive scans
            const uint32_t a = tid >= d ? s_c[tid - d] : 0, b = tid >= d ? s_t[tid - d] : 0;
            __syncthreads();
            s_c[tid] += a;
            s_t[tid] += b;
            __syncthreads();
        }
        if (f < F) {
            const uint32_t c0 = s_cbase + s_c[tid] - nc;
            for (uint32_t c = 0; c < nc; c++) {
                const uint32_t cb = lf.begin + c * S;
                chunks[c0 + c] = Leaf{cb, (lf.len - c * S) < S ? (lf.len - c * S) : S, lf.parity, 0};
            }
            tprefix[f] = s_tbase + s_t[tid] - nt;
        }
        __syncthreads();
        if (tid == 1023) {
            s_cbase += s_c[1023];
            s_tbase += s_t[1023];
        }
        __syncthreads();
    }
    if (tid == 0) {
        tprefix[F] = s_tbase;
        uint32_t np = 0;
        for (uint64_t w = S; w < s_max; w *= 2) np++;
        st->nseg = F;
        st->nchunk = s_cbase;
        st->ntiles = s_tbase;
        st->npass = np;
        st->pass = 0;
        st->w = S;
        if (use_cond) cudaGraphSetConditional(h, np > 0 ? 1u : 0u);
    }
}

// the capped segment owning merge tile t
__device__ __forceinline__ uint32_t fb_owner(const uint32_t *tprefix, uint32_t F, uint32_t t) {
    uint32_t lo = 0, hi = F;   // largest f with tprefix[f] <= t
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (tprefix[mid] <= t) lo = mid;
        else hi = mid;
    }
    return lo;
}

// One merge pass over every capped segment: runs of width w are merged
// pairwise from the buffer the previous pass wrote into the other one.  Each
// thread locates its first output by a merge-path binary search and emits
// MERGE_IPT outputs serially (ties take the left run: stable).
template <class KT>
__global__ void __launch_bounds__(MERGE_THREADS) k_fb_merge(const Leaf *fb, const uint32_t *tprefix, const FbState *st,
                                                            typename KT::T *buf0, typename KT::T *buf1) {
    using T = typename KT::T;
    const uint32_t F = st->nseg, ntiles = st->ntiles, pass = st->pass;
    const uint64_t w = st->w;
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint32_t f = fb_owner(tprefix, F, t);
        const Leaf lf = fb[f];
        const uint32_t srcp = lf.parity ^ 1u ^ (pass & 1u);
        const T *X = (srcp ? buf1 : buf0) + lf.begin;
        T *Y = (srcp ? buf0 : buf1) + lf.begin;
        const uint64_t len = lf.len;
        const uint64_t o = (uint64_t)(t - tprefix[f]) * MERGE_TILE + (uint64_t)threadIdx.x * MERGE_IPT;
        if (o >= len) continue;
        const uint64_t pair0 = (o / (2 * w)) * (2 * w);
        const uint64_t a1 = pair0 + w < len ? pair0 + w : len;
        const uint64_t b1 = pair0 + 2 * w < len ? pair0 + 2 * w : len;
        const uint64_t na = a1 - pair0, nb = b1 - a1;
        const uint64_t d = o - pair0;
        const T *A = X + pair0;
        const T *B = X + a1;
        uint64_t lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (!(KT::key(B[d - 1 - mid]) < KT::key(A[mid]))) lo = mid + 1;   // A[mid] <= B[d-1-mid]
            else hi = mid;
        }
        uint64_t i = lo, j = d - lo;
        BQ_CHECK(i <= na && j <= nb && pair0 + na + nb <= len);
        const uint64_t end = (o + MERGE_IPT) < b1 ? (o + MERGE_IPT) : b1;
        for (uint64_t r = o; r < end; r++) {
            const bool takeA = j >= nb || (i < na && !(KT::key(B[j]) < KT::key(A[i])));
            Y[r] = takeA ? A[i++] : B[j++];
        }
    }
}

static __global__ void k_fb_next(FbState *st, int use_cond, cudaGraphConditionalHandle h) {
    st->pass++;
    st->w *= 2;
    if (use_cond) cudaGraphSetConditional(h, st->pass < st->npass ? 1u : 0u);
}

// segments whose last pass wrote the scratch buffer: copy to the user buffer
template <class KT>
__global__ void __launch_bounds__(MERGE_THREADS) k_fb_finish(const Leaf *fb, const uint32_t *tprefix, const FbState *st,
                                                             typename KT::T *user, const typename KT::T *scratch) {
    const uint32_t F = st->nseg, ntiles = st->ntiles, np = st->npass;
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint32_t f = fb_owner(tprefix, F, t);
        const Leaf lf = fb[f];
        if ((lf.parity ^ 1u ^ (np & 1u)) == 0) continue;   // already in the user buffer
        const uint64_t o = (uint64_t)(t - tprefix[f]) * MERGE_TILE;
        for (uint64_t q = o + threadIdx.x; q < o + MERGE_TILE && q < lf.len; q += MERGE_THREADS)
            user[lf.begin + q] = scratch[lf.begin + q];
    }
}

}  // namespace bq
