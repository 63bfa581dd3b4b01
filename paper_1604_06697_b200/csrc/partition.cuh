// partition.cuh — the tile-partition pass (hot-path steps a2-a6) and the
// per-level bookkeeping kernels (a1 pivot, a6 equal band, a7 segment queue).
//
// GPU analogue of Alg. 3.  The paper scans a block of B=128
// elements, stores *every* offset and advances a counter by the comparison
// outcome (Alg. 3 l.8-9, 15-16), then swaps buffered pairs.  Here
// one CTA owns a tile of TILE elements:
//   a2  coalesced 128-bit loads of the tile (tiles laid out from the
//       segment's 16-byte-aligned begin, common.cuh seg_tiles; slots outside
//       the segment masked);
//   a3  three-way classification against the pivot; `__ballot_sync` per item
//       slot + `__popc(mask & lanemask_lt)` give every key its rank among the
//       < (resp. >, =) keys of its warp chunk — the offsets buffers — and one
//       warp scans the per-warp counts into tile-local offsets;
//   a4  decoupled look-back over packed 64-bit status words assigns the
//       tile's global ranges (the start/num cursors of P:379);
//   a5  branch-free scatter: keys are staged in shared memory as
//       [< run | > run (| = run)] and written out coalesced: the < run to
//       [b+Lprefix, ...), the > run element-reversed ending at e-1-Gprefix;
//   a6  keys equal to the pivot are not moved: the band [b+L, b+L+E) is
//       filled with the pivot's bits afterwards (k_post); records' equal
//       elements are compacted into a staging area and copied into the band.
// The pass is out-of-place (src -> dst), one HBM read + one HBM write per
// element; see DESIGN.md for why the paper's in-place swap does not stream.
#pragma once

#include "common.cuh"
#include "leaf.cuh"

namespace bq {

template <class KT>
struct PassParams;
template <class KT>
__device__ __forceinline__ uint32_t pass_ntiles(const PassParams<KT> &P);

// Device-resident level state of the sort's level loop (the paper's explicit
// stack, as breadth-first level arrays).  A kernel launched by
// the loop reads the current level and picks that level's arrays (segment
// lists and tile maps ping-pong by level parity), so one fixed sequence of
// launches — the body of a CUDA-graph loop — serves every level.
template <class KT>
struct LoopPtrs {
    const uint32_t *level;   // nullptr: the params are static (standalone pass, root)
    const uint32_t *set;     // list set of the current batch of levels (LoopMisc::set)
    Seg *segs[2];
    uint32_t *tile_map[2];
    unsigned long long *cursor[2];
    uint32_t *ecursor[2];
    void *msegs[2];          // MSeg<KT> (multiway.cuh)
    uint32_t *mtile_map[2], *mhist[2], *mcursor[2];
    LevelCtrl *ctrl;         // one control block per level
    LevelCtrl *root;         // the root's counts (level -1)
    // leaves (and finished equal-record runs) of a batch of levels go to list
    // set `*set`: one iteration of the loop partitions a batch while it sorts
    // the previous batch's leaves (loop.cuh)
    Leaf *leaves[2];
    uint32_t *leaf_counts[2];
    Leaf *copies[2];
    uint32_t *copy_count[2];
};
template <class KT>
__device__ __forceinline__ const LevelCtrl *loop_prev(const LoopPtrs<KT> &lp, uint32_t lv) {
    return lv == 0 ? lp.root : lp.ctrl + lv - 1;
}

template <class KT>
struct PassParams {
    using T = typename KT::T;
    T *bufs[2];            // [parity]: segment data; the pass writes bufs[parity^1]
    T *stage[2];           // records: equal-element staging base, by parity
    T *final_buf;          // where equal bands are materialised (user buffer / dst)
    const Seg *segs;       // segment descriptors of this level
    const uint32_t *tile_map;  // tile -> segment (nullptr: single segment `seg0`)
    Seg seg0;
    uint64_t *status;      // one look-back word per tile, zeroed before the pass (ordered mode)
    unsigned long long *cursor;  // per segment: packed (lt | gt << 32) running offsets / totals
    uint32_t *ecursor;     // per segment: equal-record running offset (records, fast mode)
    LevelCtrl *ctrl;       // ticket + counters of this level
    uint32_t ntiles;
    const uint32_t *ntiles_dev;  // non-null: the level's tile count lives in device memory
    uint64_t n_total;      // length of each data buffer (bounds the TMA reads)
    int aligned;           // both data buffers 16-byte aligned -> TMA bulk copies
    int ordered;           // 1: decoupled look-back (deterministic layout), 0: atomic cursor
    LoopPtrs<KT> lp;       // lp.level != nullptr: segs .. ntiles_dev are the current level's
};

template <class KT>
__device__ __forceinline__ uint32_t pass_ntiles(const PassParams<KT> &P) {
    return P.ntiles_dev ? *P.ntiles_dev : P.ntiles;
}

// Kernels of the loop keep their parameters in shared memory, resolved once
// per CTA by thread 0 (a per-thread copy of a modified by-value parameter
// struct would live in local memory):  `const auto &P = cta_params(Pin, sP);`
// the level's control blocks before any parameter copy: loop kernels of a
// level without work (the trailing levels of a batch) exit at once
template <class KT>
__device__ __forceinline__ const LevelCtrl *loop_prev_ctrl(const LoopPtrs<KT> &lp) {
    return lp.level ? loop_prev(lp, *lp.level) : nullptr;
}
template <class KT>
__device__ __forceinline__ const LevelCtrl *loop_cur_ctrl(const LoopPtrs<KT> &lp) {
    return lp.level ? lp.ctrl + *lp.level : nullptr;
}

template <class PP>
__device__ __forceinline__ const PP &cta_params(const PP &in, PP &sm) {
    if (threadIdx.x == 0) {
        sm = in;
        loop_resolve(sm);
    }
    __syncthreads();
    return sm;
}

// the level's arrays (every kernel of the loop calls this first)
template <class KT>
__device__ __forceinline__ void loop_resolve(PassParams<KT> &P) {
    if (!P.lp.level) return;
    const uint32_t lv = *P.lp.level, cp = lv & 1;
    P.segs = P.lp.segs[cp];
    P.tile_map = P.lp.tile_map[cp];
    P.cursor = P.lp.cursor[cp];
    P.ecursor = P.lp.ecursor[cp];
    P.ctrl = P.lp.ctrl + lv;
    P.ntiles_dev = &loop_prev(P.lp, lv)->ntiles_next;
}

}  // namespace bq

#include "partition_kernel.cuh"
#include "partition_fast.cuh"
#include "multiway.cuh"
#include "multiway8.cuh"
#include "multiway8w.cuh"
#include "inplace.cuh"

namespace bq {

// ---------------------------------------------------------------------------
// Level bookkeeping.
// ---------------------------------------------------------------------------
template <class KT>
struct PostParams {
    using T = typename KT::T;
    PassParams<KT> pass;    // the level just partitioned
    // children (a7): next-level segments with their tile map and cursors, leaves,
    // depth-capped segments
    Seg *next_segs;
    uint32_t *next_tile_map;
    unsigned long long *next_cursor;
    uint32_t *next_ecursor;
    Leaf *leaves;           // leaf lists (one per network-size class, leaf_cap each)
    uint32_t *leaf_counts;  // their fill counts
    Leaf *fallback;
    uint32_t *fallback_count;
    uint64_t *d_counts;     // pass mode: {split, n_equal, n_greater} per segment
    uint32_t nseg;          // segments of the level (nseg_dev == nullptr)
    const uint32_t *nseg_dev;  // non-null: the level's segment count lives in device memory
    uint32_t leaf_max;      // S
    uint32_t leaf_cap;      // capacity of each leaf-class list
    uint32_t band_inline_max;  // equal bands up to this size are filled by k_post, larger ones by k_fill
    int32_t depth_limit;
    int32_t pivot_rule;
    int emit_children;      // 0 in the standalone pass
    int ways;               // > 2: children may be split multiway (keys only)
    uint64_t *status;       // next level's look-back words (ordered placement), or nullptr
    LevelCtrl *child_ctrl;  // counters the children are appended to
    // multiway: the level just scattered, and the next level's lists
    MwParams<KT> mw;
    MSeg<KT> *next_msegs;
    uint32_t *next_mtile_map;
    uint32_t *next_mhist;   // [bucket * mhstride + segment], zeroed for new segments
    uint32_t mhstride;
    // records, two-way placement: finished runs of equal keys still in the
    // scratch buffer, copied to the user buffer by k_copy_runs
    Leaf *copies;
    uint32_t *copy_count;
    uint32_t copy_cap;
    // set to 1 when a leaf list would overflow (the call then fails)
    uint32_t *overflow;
    uint32_t nseg_cap, ntile_cap;   // list capacities (checked with -DBQ_CHECKS)
};

template <class KT>
__device__ __forceinline__ void loop_resolve(PostParams<KT> &Q) {
    loop_resolve(Q.pass);
    loop_resolve(Q.mw);
    const LoopPtrs<KT> &lp = Q.pass.lp;
    if (!lp.level) return;
    const uint32_t lv = *lp.level, np = (lv & 1) ^ 1;
    Q.next_segs = lp.segs[np];
    Q.next_tile_map = lp.tile_map[np];
    Q.next_cursor = lp.cursor[np];
    Q.next_ecursor = lp.ecursor[np];
    Q.next_msegs = static_cast<MSeg<KT> *>(lp.msegs[np]);
    Q.next_mtile_map = lp.mtile_map[np];
    Q.next_mhist = lp.mhist[np];
    Q.child_ctrl = lp.ctrl + lv;
    Q.nseg_dev = &loop_prev(lp, lv)->nseg_next;
    const uint32_t set = *lp.set;
    Q.leaves = lp.leaves[set];
    Q.leaf_counts = lp.leaf_counts[set];
    Q.copies = lp.copies[set];
    Q.copy_count = lp.copy_count[set];
}

template <class KT>
struct SegCounts {
    uint32_t L, G, E;
};
template <class KT>
__device__ __forceinline__ SegCounts<KT> seg_counts(const PassParams<KT> &P, uint32_t si, const Seg &sg) {
    const unsigned long long fin = P.cursor[si];
    SegCounts<KT> c;
    c.L = (uint32_t)fin;
    c.G = (uint32_t)(fin >> 32);
    c.E = sg.len - c.L - c.G;
    return c;
}

// a6 + a7: one CTA per segment of the level.  The CTA fills (keys) or copies
// (records) the segment's equal band when it is at most band_inline_max long
// (larger bands are counted in ctrl->nbig and left to k_fill), and pushes the
// children: the "push larger side / continue on smaller" of P:1238-1252
// becomes: both children are appended to the next level (with their pivot,
// a1, their slice of the next tile map and a reset cursor), small ones to the
// leaf lists, depth-capped ones to the fallback list.
// Per-CTA statistics of the bookkeeping kernels: counted with shared-memory
// atomics and added to the level's control block once per CTA (deep levels
// have tens of thousands of segments; one global atomic per segment and
// counter on the same address serialises in L2).
struct PostStats {
    unsigned long long passes, band_pass, band_child;
    uint32_t nleaf, nfallback, maxtiles;
    uint32_t nleaf_cls[MAX_LEAF_CLASSES];
};
__device__ __forceinline__ PostStats &post_stats() {
    __shared__ PostStats s;
    return s;
}
__device__ __forceinline__ void post_stats_init() {
    if (threadIdx.x == 0) {
        PostStats &st = post_stats();
        st.passes = st.band_pass = st.band_child = 0;
        st.nleaf = st.nfallback = st.maxtiles = 0;
        for (int c = 0; c < MAX_LEAF_CLASSES; c++) st.nleaf_cls[c] = 0;
    }
    __syncthreads();
}
template <class KT>
__device__ __forceinline__ void post_stats_flush(const PostParams<KT> &Q) {
    __syncthreads();
    if (threadIdx.x != 0 || !Q.emit_children) return;
    const PostStats &st = post_stats();
    LevelCtrl *P = Q.pass.ctrl, *C = Q.child_ctrl;
    if (P && st.passes) atomicAdd(&P->element_passes, st.passes);
    if (P && st.band_pass) atomicAdd(&P->band_elems, st.band_pass);
    if (st.band_child) atomicAdd(&C->band_elems, st.band_child);
    if (st.nleaf) atomicAdd(&C->nleaf, st.nleaf);
    if (st.nfallback) atomicAdd(&C->nfallback, st.nfallback);
    if (st.maxtiles) atomicMax(&C->maxtiles_next, st.maxtiles);
    for (int c = 0; c < MAX_LEAF_CLASSES; c++)
        if (st.nleaf_cls[c]) atomicAdd(&C->nleaf_cls[c], st.nleaf_cls[c]);
}

// a7 for up to MW_K children of one segment (or the root), by a whole CTA of
// NT threads: each child becomes nothing (empty), a leaf (<= S), a
// depth-capped fallback segment, or a next-level segment — multiway when
// allowed and its 256-key sample gives distinct splitters (multiway.cuh), else
// binary with the pivot of `pivot_rule` (the sample's median when multiway
// was tried).  Warps select pivots/splitters, one thread per child appends
// it, then the CTA writes the children's slices of the next tile maps.
// hint[c] (optional): 0 = choose a pivot; 1 = follow-up pass [<= p | > p]
// with p = hint_pivot; 2 = a finished run of equal keys (records)
#ifndef BQ_LEAF_AWARE
#define BQ_LEAF_AWARE 1
#endif
// duplicate check at the leaf boundary (keys): a leaf-sized child of at least
// BQ_DC_MIN keys whose 64-key sample holds at most BQ_DC_DISTINCT distinct
// keys is partitioned three-way once more (its repeated keys leave as an
// equal band) instead of merge-sorted; a pass costs a fraction of a leaf sort
// per key (R23)
#ifndef BQ_DC_MIN
#define BQ_DC_MIN 2048
#endif
#ifndef BQ_DC_DISTINCT
#define BQ_DC_DISTINCT 8
#endif
#ifndef BQ_LA_DIV
#define BQ_LA_DIV 16   // margin len / 16: one standard deviation of the sample's rank error
#endif
template <class KT, int NT>
__device__ __forceinline__ void emit_children(const PostParams<KT> &Q, int nch, const uint32_t *cb,
                                              const uint32_t *cl, uint8_t cp, uint16_t cd, bool dups,
                                              const uint8_t *hint = nullptr, uint64_t hint_pivot = 0) {
    using T = typename KT::T;
    using K = typename KT::K;
    constexpr uint32_t TILE = (uint32_t)tile_elems<KT>();
    constexpr int NW = NT / 32;
    enum { C_NONE = 0, C_LEAF, C_FALLBACK, C_BIN, C_MW, C_BAND };
    __shared__ uint32_t s_kind[MW_K], s_idx[MW_K], s_tb[MW_K], s_nt[MW_K], s_mode[MW_K];
    __shared__ uint64_t s_piv[MW_K];
    __shared__ K s_tree[MW_K][MW_K];
    LevelCtrl *C = Q.child_ctrl;
    const T *cbuf = cp ? Q.pass.bufs[1] : Q.pass.bufs[0];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();   // the previous segment's readers of s_* are done
    for (int c = warp; c < nch; c += NW) {
        const uint32_t len = cl[c];
        const uint8_t h = hint ? hint[c] : 0;
        uint32_t kind = C_NONE, mode = 0;
        if (len == 0) kind = C_NONE;
        else if (h == 2) kind = C_BAND;
        else if (len <= Q.leaf_max) {
            kind = C_LEAF;
            if constexpr (!KT::is_record) if (dups && len >= BQ_DC_MIN && (int)cd < Q.depth_limit) {
                uint32_t distinct = 64;
                const K piv = sample64_median_distinct<KT>(cbuf, cb[c], len, lane, &distinct);
                if (distinct <= BQ_DC_DISTINCT) {
                    kind = C_BIN;
                    if (lane == 0) s_piv[c] = (uint64_t)piv;
                }
            }
        }
        else if ((int)cd >= Q.depth_limit) kind = C_FALLBACK;
        else if (h == 1) {
            kind = C_BIN;
            mode = 1;
            if (lane == 0) s_piv[c] = hint_pivot;
        } else if (mw_capable<KT>() && Q.ways > 2 && !(KT::is_record && Q.pass.ordered)) {
            K node, piv;
            const bool ok = mw_splitters<KT>(cbuf, cb[c], len, Q.leaf_max, lane, node, piv, (uint32_t)Q.ways);
            kind = ok ? C_MW : C_BIN;
            if (lane == 0) s_piv[c] = (uint64_t)piv;
            if (lane < MW_K) s_tree[c][lane] = node;
            // records falling back to the binary pass: their sample showed
            // duplicates, so the two-way pass gets its follow-up (mode bit 1)
            if (KT::is_record && !ok) mode = 2;
        } else if (KT::is_record && !Q.pass.ordered) {
            // two-way records: a pivot repeated in its sample gets a follow-up pass
            bool dup = false;
            const K piv = select_pivot_warp<KT>(cbuf, cb[c], len, Q.pivot_rule, lane, &dup);
            if (lane == 0) s_piv[c] = (uint64_t)piv;
            kind = C_BIN;
            mode = dup ? 2 : 0;
        } else {
            // Leaf-aware split of a segment that is one pass from its leaves
            // (S < len <= 2 (S - m)): instead of the median, the sample
            // quantile that leaves ~S - m keys on the left, m = len / 16 (one
            // standard deviation of the 64-key sample's rank error, at most
            // len sqrt(1/4 / 64)); both children then fit one leaf network, the
            // left one nearly full, where two halves of ~len/2 would each pad
            // an S network by up to half (R22)
            uint32_t q = 31;
#if BQ_LEAF_AWARE
            if (Q.pivot_rule == BQ_PIVOT_SAMPLE64 && len > Q.leaf_max && len < 2 * Q.leaf_max) {
                const uint32_t m = len / BQ_LA_DIV, t = Q.leaf_max - m;   // m < S / 4 here
                if (len <= 2 * t) {
                    const uint32_t k = (uint32_t)(((uint64_t)t * 64) / len);
                    q = k < 1 ? 0 : (k > 63 ? 62 : k - 1);
                }
            }
#endif
            const K piv = select_pivot_warp<KT>(cbuf, cb[c], len, Q.pivot_rule, lane, nullptr, q);
            if (lane == 0) s_piv[c] = (uint64_t)piv;
            kind = C_BIN;
        }
        if (lane == 0) {
            s_kind[c] = kind;
            s_mode[c] = mode;
        }
    }
    __syncthreads();
    if ((int)threadIdx.x < nch) {
        const int c = threadIdx.x;
        const uint32_t kind = s_kind[c], len = cl[c];
        s_nt[c] = 0;
        if (kind == C_LEAF) {
            // leaf lists are binned by sorting-network size (leaf.cuh)
            const uint32_t lc = leaf_class<KT>(len);
            const uint32_t li = atomicAdd(&Q.leaf_counts[lc], 1u);
            atomicAdd(&post_stats().nleaf_cls[lc], 1u);
            atomicAdd(&post_stats().nleaf, 1u);
            if (li < Q.leaf_cap) Q.leaves[lc * Q.leaf_cap + li] = Leaf{cb[c], len, cp, 0};
            else if (Q.overflow) *Q.overflow = 1u;
        } else if (kind == C_FALLBACK) {
            const uint32_t fi = atomicAdd(Q.fallback_count, 1u);
            atomicAdd(&post_stats().nfallback, 1u);
            BQ_CHECK(fi < Q.nseg_cap);
            Q.fallback[fi] = Leaf{cb[c], len, cp, 0};
        } else if (kind == C_BAND) {
            atomicAdd(&post_stats().band_child, (unsigned long long)len);
            if (cp != 0)   // in the scratch buffer: copy to the user buffer in chunks
                for (uint32_t off = 0; off < len; off += 65536) {
                    const uint32_t ci = atomicAdd(Q.copy_count, 1u);
                    if (ci < Q.copy_cap) Q.copies[ci] = Leaf{cb[c] + off, (len - off) < 65536u ? (len - off) : 65536u, cp, 0};
                    else if (Q.overflow) *Q.overflow = 1u;
                }
        } else if (kind == C_BIN || kind == C_MW) {
            Seg ch;
            ch.pivot = s_piv[c];
            ch.begin = cb[c];
            ch.len = len;
            ch.ntiles = seg_tiles<KT>(cb[c], len);
            ch.depth = cd;
            ch.parity = cp;
            ch.pad0 = (uint8_t)s_mode[c];   // records: bit 0 = [<= p | > p] pass, bit 1 = pivot duplicated
            ch.pad1 = 0;
            uint32_t ci;
            if (kind == C_BIN) {
                ch.tile_base = atomicAdd(&C->ntiles_next, ch.ntiles);
                atomicMax(&post_stats().maxtiles, ch.ntiles);
                ci = atomicAdd(&C->nseg_next, 1u);
                BQ_CHECK(ci < Q.nseg_cap && ch.tile_base + ch.ntiles <= Q.ntile_cap);
                Q.next_segs[ci] = ch;
                Q.next_cursor[ci] = 0;
                Q.next_ecursor[ci] = 0;
            } else {
                ch.tile_base = atomicAdd(&C->nmtiles_next, ch.ntiles);
                ci = atomicAdd(&C->nmseg_next, 1u);
                BQ_CHECK(ci < Q.nseg_cap && ch.tile_base + ch.ntiles <= Q.ntile_cap);
                MSeg<KT> &m = Q.next_msegs[ci];
                m.s = ch;
#pragma unroll
                for (int q = 0; q < MW_K; q++) m.tree[q] = s_tree[c][q];
            }
            s_idx[c] = ci;
            s_tb[c] = ch.tile_base;
            s_nt[c] = ch.ntiles;
        }
    }
    __syncthreads();
    // the children's slices of the next level's tile maps (and resets)
    for (int c = 0; c < nch; c++) {
        const uint32_t kind = s_kind[c];
        if (kind != C_BIN && kind != C_MW) continue;
        const uint32_t nt = s_nt[c], tb = s_tb[c], ci = s_idx[c];
        if (kind == C_BIN) {
            for (uint32_t j = threadIdx.x; j < nt; j += NT) {
                Q.next_tile_map[tb + j] = ci;
                if (Q.status) Q.status[tb + j] = 0;
            }
        } else {
            for (uint32_t j = threadIdx.x; j < nt; j += NT) Q.next_mtile_map[tb + j] = ci;
            if (threadIdx.x < MW_K) Q.next_mhist[threadIdx.x * Q.mhstride + ci] = 0;
        }
    }
}

template <class KT, int NT>
__device__ __forceinline__ void post_segment(const PostParams<KT> &Q, uint32_t si);

// A key segment made of copies of its pivot only (L = G = 0) whose source is
// the final buffer already is its own equal band: nothing to write (the key
// codecs are bijections on bit patterns, so equal keys are equal bits).
// The all-equal input of c4 and the single-value segments that end a
// few-distinct-values sort take this exit.
template <class KT>
__device__ __forceinline__ bool band_in_place(const PassParams<KT> &P, const Seg &sg, uint32_t L, uint32_t G) {
    if (KT::is_record) return false;
    return L == 0 && G == 0 && (sg.parity ? P.bufs[1] : P.bufs[0]) == P.final_buf;
}

template <class KT, int NT>
__global__ void __launch_bounds__(NT) k_post(const PostParams<KT> Qin) {
    if (const LevelCtrl *pv = loop_prev_ctrl(Qin.pass.lp)) if (pv->nseg_next == 0) return;
    __shared__ PostParams<KT> sQ;
    const PostParams<KT> &Q = cta_params(Qin, sQ);
    const uint32_t nseg = Q.nseg_dev ? *Q.nseg_dev : Q.nseg;
    post_stats_init();
    for (uint32_t si = blockIdx.x; si < nseg; si += gridDim.x) post_segment<KT, NT>(Q, si);
    post_stats_flush(Q);
}

template <class KT, int NT>
__device__ __forceinline__ void post_segment(const PostParams<KT> &Q, uint32_t si) {
    using T = typename KT::T;
    using K = typename KT::K;
    constexpr uint32_t TILE = (uint32_t)tile_elems<KT>();
    const PassParams<KT> &P = Q.pass;
    const Seg sg = P.segs ? P.segs[si] : P.seg0;
    const SegCounts<KT> cn = seg_counts(P, si, sg);
    const uint32_t L = cn.L, G = cn.G, E = cn.E;
    const uint64_t b = sg.begin;
    LevelCtrl *C = P.ctrl;

    const bool inplace = band_in_place<KT>(P, sg, L, G);
    if (E > 0 && E <= Q.band_inline_max && !inplace) {
        const uint64_t band0 = b + L;
        if constexpr (KT::is_record) {
            // staged equal records: stage[parity][b + j], j < E
            const T *stg = sg.parity ? P.stage[1] : P.stage[0];
            if (stg != P.final_buf) {
                for (uint32_t j = threadIdx.x; j < E; j += NT) P.final_buf[band0 + j] = stg[b + j];
            } else {
                // same buffer: move [b, b+E) right by L, last chunk first; a
                // chunk is read completely before any of it is written
                for (int64_t c0 = (int64_t)((E - 1) / NT) * NT; c0 >= 0; c0 -= NT) {
                    const uint32_t j = (uint32_t)c0 + threadIdx.x;
                    T v;
                    if (j < E) v = stg[b + j];
                    __syncthreads();
                    if (j < E) P.final_buf[band0 + j] = v;
                    __syncthreads();
                }
            }
        } else {
            const T pv = KT::from_key((K)sg.pivot);
            for (uint32_t j = threadIdx.x; j < E; j += NT) P.final_buf[band0 + j] = pv;
        }
    }
    if (threadIdx.x == 0 && E > Q.band_inline_max && Q.emit_children && !inplace) atomicAdd(&C->nbig, 1u);
    if (threadIdx.x == 0 && Q.d_counts) {
        Q.d_counts[3 * si + 0] = L;
        Q.d_counts[3 * si + 1] = E;
        Q.d_counts[3 * si + 2] = G;
    }
    if (!Q.emit_children) return;

    if (threadIdx.x == 0) {
        atomicAdd(&post_stats().passes, (unsigned long long)sg.len);
        atomicAdd(&post_stats().band_pass, (unsigned long long)E);
    }
    if (KT::is_record && !P.ordered) {
        // two-way records (E == 0): [< p | >= p], the right side followed up by
        // [<= p | > p] when p was duplicated in its sample; the left side of a
        // follow-up pass is a finished run of keys equal to p
        const uint32_t cb[2] = {sg.begin, sg.begin + L};
        const uint32_t cl[2] = {L, G};
        const uint8_t h[2] = {(uint8_t)((sg.pad0 & 1) ? 2 : 0), (uint8_t)((sg.pad0 & 1) ? 0 : ((sg.pad0 & 2) ? 1 : 0))};
        emit_children<KT, NT>(Q, 2, cb, cl, (uint8_t)(sg.parity ^ 1), (uint16_t)(sg.depth + 1), false, h, sg.pivot);
        return;
    }
    const uint32_t cb[2] = {sg.begin, sg.begin + L + E};
    const uint32_t cl[2] = {L, G};
    // R23's sample is drawn only below a pivot that was repeated (E >= 2):
    // few distinct keys in a child imply many copies of its parent's pivot
    emit_children<KT, NT>(Q, 2, cb, cl, (uint8_t)(sg.parity ^ 1), (uint16_t)(sg.depth + 1), E >= 2);
}

// Equal bands longer than band_inline_max, tile-parallel over the level
// (grid-stride): keys are filled with the pivot's bits; records are copied
// from their staging area — phase 0 copies into the final buffer, or, when
// the staging area is the final buffer itself (it may overlap the band), into
// the other buffer, from where phase 1 copies them into the final buffer.
template <class KT, int NT>
__global__ void __launch_bounds__(NT) k_fill(const PostParams<KT> Qin, int phase) {
    if (const LevelCtrl *cv = loop_cur_ctrl(Qin.pass.lp)) if (cv->nbig == 0) return;
    using T = typename KT::T;
    using K = typename KT::K;
    constexpr uint32_t TILE = (uint32_t)tile_elems<KT>();
    __shared__ PostParams<KT> sQ;
    const PostParams<KT> &Q = cta_params(Qin, sQ);
    const PassParams<KT> &P = Q.pass;
    if (Q.emit_children && P.ctrl->nbig == 0) return;   // sort: no long band this level
    const uint32_t ntiles = pass_ntiles(P);
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint32_t si = P.tile_map ? P.tile_map[t] : 0;
        const Seg sg = P.segs ? P.segs[si] : P.seg0;
        const SegCounts<KT> cn = seg_counts(P, si, sg);
        if (cn.E <= Q.band_inline_max || band_in_place<KT>(P, sg, cn.L, cn.G)) continue;
        const uint64_t b = sg.begin;
        const uint64_t tbeg = b / tile_vw<KT>() * tile_vw<KT>() + (uint64_t)(t - sg.tile_base) * TILE;
        const uint64_t band0 = b + cn.L, band1 = band0 + cn.E;
        const uint64_t x0 = tbeg > band0 ? tbeg : band0;
        const uint64_t x1 = (tbeg + TILE) < band1 ? (tbeg + TILE) : band1;
        if constexpr (KT::is_record) {
            const T *stg = sg.parity ? P.stage[1] : P.stage[0];
            T *other = sg.parity ? P.bufs[0] : P.bufs[1];
            if (phase == 0) {
                T *tgt = (stg == P.final_buf) ? other : P.final_buf;
                for (uint64_t i = x0 + threadIdx.x; i < x1; i += NT) tgt[i] = stg[b + (i - band0)];
            } else if (stg == P.final_buf) {
                for (uint64_t i = x0 + threadIdx.x; i < x1; i += NT) P.final_buf[i] = other[i];
            }
        } else {
            if (phase != 0) continue;
            // scalar head up to a 16-byte boundary, 16-byte stores, scalar tail
            const T pv = KT::from_key((K)sg.pivot);
            constexpr uint32_t V = 16 / sizeof(T);
            T *o = P.final_buf;
            if (x1 <= x0) continue;
            uint64_t head = ((16 - (reinterpret_cast<uintptr_t>(o + x0) & 15)) & 15) / sizeof(T);
            if (head > x1 - x0) head = x1 - x0;
            const uint64_t nb = (x1 - x0 - head) / V;
            T rep[V];
#pragma unroll
            for (uint32_t k = 0; k < V; k++) rep[k] = pv;
            uint4 vv;
            memcpy(&vv, rep, 16);
            for (uint64_t i = x0 + threadIdx.x; i < x0 + head; i += NT) o[i] = pv;
            uint4 *ov = reinterpret_cast<uint4 *>(o + x0 + head);
            for (uint64_t j = threadIdx.x; j < nb; j += NT) ov[j] = vv;
            for (uint64_t i = x0 + head + nb * V + threadIdx.x; i < x1; i += NT) o[i] = pv;
        }
    }
}

// Tile map + status reset for a level: tile_map[tile_base + j] = segment.
static __global__ void k_map(const Seg *segs, uint32_t *tile_map, uint64_t *status, unsigned long long *cursor,
                             uint32_t *ecursor) {
    const uint32_t s = blockIdx.x;
    const Seg sg = segs[s];
    if (blockIdx.y == 0 && threadIdx.x == 0) {
        cursor[s] = 0;
        ecursor[s] = 0;
    }
    for (uint32_t j = blockIdx.y * blockDim.x + threadIdx.x; j < sg.ntiles; j += gridDim.y * blockDim.x) {
        tile_map[sg.tile_base + j] = s;
        status[sg.tile_base + j] = 0;
    }
}

// Root segment of a sort: [0, n) in the user buffer becomes the first
// binary or multiway segment (a1 pivot / splitters, tile map, counts in
// Q.child_ctrl = the root's control block), exactly like a child.
template <class KT, int NT>
__global__ void __launch_bounds__(NT) k_init_root(PostParams<KT> Q, uint32_t n) {
    const uint32_t cb[1] = {0}, cl[1] = {n};
    post_stats_init();
    emit_children<KT, NT>(Q, 1, cb, cl, 0, 0, true);
    post_stats_flush(Q);
}

// a7 after a multiway scatter: the (up to) 16 buckets of every multiway
// segment become its children.
template <class KT, int NT>
__global__ void __launch_bounds__(NT) k_post_mw(const PostParams<KT> Qin) {
    __shared__ uint32_t cb[MW_K], cl[MW_K];
    if (const LevelCtrl *pv = loop_prev_ctrl(Qin.pass.lp)) if (pv->nmseg_next == 0) return;
    __shared__ PostParams<KT> sQ;
    const PostParams<KT> &Q = cta_params(Qin, sQ);
    const uint32_t nseg = *Q.mw.nseg_dev;
    post_stats_init();
    for (uint32_t si = blockIdx.x; si < nseg; si += gridDim.x) {
        const MSeg<KT> &m = Q.mw.msegs[si];
        if (Q.mw.tabmode) {   // 8-way levels (multiway8w.cuh): buckets from the tile-count table
            if (threadIdx.x < 32) {
                uint32_t tot, start, pf;
                const uint32_t U = mw8w_upt<KT>(*Q.mw.ntiles_dev);
                mw8w_seg_buckets(Q.mw, m.s.tile_base * U, m.s.ntiles * U, *Q.mw.ntiles_dev * U, threadIdx.x, tot, start,
                                 pf);
                if (threadIdx.x < MW_K) {
                    cb[threadIdx.x] = m.s.begin + start;
                    cl[threadIdx.x] = threadIdx.x < MW8 ? tot : 0;
                }
                BQ_CHECK(__shfl_sync(0xffffffffu, start + tot, MW8 - 1) == m.s.len);
            }
        } else if (threadIdx.x < MW_K) {
            cb[threadIdx.x] = m.s.begin + m.start[threadIdx.x];
            cl[threadIdx.x] = Q.mw.hist[threadIdx.x * Q.mw.hstride + si];
        }
        emit_children<KT, NT>(Q, MW_K, cb, cl, (uint8_t)(m.s.parity ^ 1), (uint16_t)(m.s.depth + 1), false);
    }
    post_stats_flush(Q);
}

// Finished runs of equal record keys still in the scratch buffer -> user
// buffer (persistent grid over one copy list; in the level loop the list of
// the previous batch of levels, loop_prev_set).
template <class KT, int NT>
__global__ void __launch_bounds__(NT) k_copy_runs(const LoopPtrs<KT> lp, const uint32_t *level, typename KT::T *user,
                                                  const typename KT::T *scratch) {
    const uint32_t set = *lp.set ^ 1u;
    const Leaf *list = set ? lp.copies[1] : lp.copies[0];
    const uint32_t n = set ? *lp.copy_count[1] : *lp.copy_count[0];
    for (uint32_t li = blockIdx.x; li < n; li += gridDim.x) {
        const Leaf l = list[li];
        for (uint32_t j = threadIdx.x; j < l.len; j += NT) user[(uint64_t)l.begin + j] = scratch[(uint64_t)l.begin + j];
    }
}

// bq_pivot_*: the pivot key of buf[0, n).
template <class KT>
__global__ void k_pivot(const typename KT::T *buf, uint32_t n, int rule, uint64_t *out) {
    const typename KT::K pk = select_pivot_warp<KT>(buf, 0, n, rule, threadIdx.x);   // one warp
    if (threadIdx.x == 0) *out = (uint64_t)pk;
}

}  // namespace bq
