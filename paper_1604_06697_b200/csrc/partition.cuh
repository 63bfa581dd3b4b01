// partition.cuh — the tile-partition pass (hot-path steps a2-a6) and the
// per-level bookkeeping kernels (a1 pivot, a6 equal band, a7 segment queue).
//
// GPU analogue of Alg. 3.  The paper scans a block of B=128
// elements, stores *every* offset and advances a counter by the comparison
// outcome (Alg. 3 l.8-9, 15-16), then swaps buffered pairs.  Here
// one CTA owns a tile of TILE elements:
//   a2  coalesced 128-bit loads of the tile (tiles anchored at absolute
//       multiples of TILE, masked at segment ends);
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
    uint64_t n_total;      // length of each data buffer (bounds the TMA reads)
    int aligned;           // both data buffers 16-byte aligned -> TMA bulk copies
    int ordered;           // 1: decoupled look-back (deterministic layout), 0: atomic cursor
};

}  // namespace bq

#include "partition_kernel.cuh"
#include "partition_fast.cuh"

namespace bq {

// ---------------------------------------------------------------------------
// Level bookkeeping.
// ---------------------------------------------------------------------------
template <class KT>
struct PostParams {
    using T = typename KT::T;
    PassParams<KT> pass;
    // children (a7): next-level segments, leaves, depth-capped segments
    Seg *next_segs;
    Leaf *leaves;
    Leaf *fallback;
    uint32_t *fallback_count;
    uint64_t *d_counts;     // pass mode: {split, n_equal, n_greater}
    uint32_t leaf_max;      // S
    uint32_t leaf_cap;      // capacity of each leaf-class list
    int32_t depth_limit;
    int32_t pivot_rule;
    int emit_children;      // 0 in the standalone pass
};

// a6 + a7: one CTA per tile of the level.  Every CTA fills (keys) or copies
// (records) the part of its segment's equal band that falls inside its tile;
// the CTA of a segment's first tile pushes the children (the "push larger
// side / continue on smaller" of P:1238-1252 becomes: both children are
// appended to the next level, small ones to the leaf list, depth-capped ones
// to the fallback list — P:293-299).
template <class KT, int NT>
__global__ void __launch_bounds__(NT) k_post(PostParams<KT> Q) {
    using T = typename KT::T;
    using K = typename KT::K;
    constexpr uint32_t TILE = (uint32_t)tile_elems<KT>();
    const PassParams<KT> &P = Q.pass;
    const uint32_t t = blockIdx.x;
    const Seg sg = P.tile_map ? P.segs[P.tile_map[t]] : P.seg0;
    const uint32_t k = t - sg.tile_base;
    const unsigned long long fin = P.cursor[P.tile_map ? P.tile_map[t] : 0];
    const uint32_t L = (uint32_t)fin, G = (uint32_t)(fin >> 32);
    const uint32_t E = sg.len - L - G;
    const uint64_t b = sg.begin;
    const uint64_t tbeg = (b / TILE) * TILE + (uint64_t)k * TILE;
    const uint64_t band0 = b + L, band1 = b + L + E;
    const uint64_t x0 = tbeg > band0 ? tbeg : band0;
    const uint64_t x1 = (tbeg + TILE) < band1 ? (tbeg + TILE) : band1;
    if constexpr (KT::is_record) {
        // staged equal records: stage[parity][b + j], j in [0, E)
        const T *stg = sg.parity ? P.stage[1] : P.stage[0];
        T *tgt = (stg == P.final_buf) ? (sg.parity ? P.bufs[0] : P.bufs[1]) : P.final_buf;
        for (uint64_t i = x0 + threadIdx.x; i < x1; i += NT) tgt[i] = stg[b + (i - band0)];
    } else {
        const T pv = KT::from_key((K)sg.pivot);
        for (uint64_t i = x0 + threadIdx.x; i < x1; i += NT) P.final_buf[i] = pv;
    }
    if (k != 0 || threadIdx.x != 0) return;

    if (Q.d_counts) {
        const uint32_t si = P.tile_map ? P.tile_map[t] : 0;
        Q.d_counts[3 * si + 0] = L;
        Q.d_counts[3 * si + 1] = E;
        Q.d_counts[3 * si + 2] = G;
    }
    if (!Q.emit_children) return;
    LevelCtrl *C = P.ctrl;
    atomicAdd(&C->element_passes, (unsigned long long)sg.len);
    atomicAdd(&C->band_elems, (unsigned long long)E);
    const uint8_t cp = sg.parity ^ 1;
    const T *cbuf = cp ? P.bufs[1] : P.bufs[0];
    const uint32_t cb[2] = {sg.begin, sg.begin + L + E};
    const uint32_t cl[2] = {L, G};
    const uint16_t cd = sg.depth + 1;
#pragma unroll
    for (int c = 0; c < 2; c++) {
        if (cl[c] == 0) continue;
        if (cl[c] <= Q.leaf_max) {
            // leaf lists are binned by sorting-network size (leaf.cuh)
            const uint32_t lc = leaf_class<KT>(cl[c]);
            const uint32_t li = atomicAdd(&C->nleaf_cls[lc], 1u);
            atomicAdd(&C->nleaf, 1u);
            Q.leaves[lc * Q.leaf_cap + li] = Leaf{cb[c], cl[c], cp, 0};
        } else if ((int)cd >= Q.depth_limit) {
            const uint32_t fi = atomicAdd(Q.fallback_count, 1u);
            atomicAdd(&C->nfallback, 1u);
            Q.fallback[fi] = Leaf{cb[c], cl[c], cp, 0};
        } else {
            Seg ch;
            ch.pivot = (uint64_t)select_pivot<KT>(cbuf, cb[c], cl[c], Q.pivot_rule);
            ch.begin = cb[c];
            ch.len = cl[c];
            ch.ntiles = seg_ntiles(cb[c], cl[c], TILE);
            ch.tile_base = atomicAdd(&C->ntiles_next, ch.ntiles);
            ch.depth = cd;
            ch.parity = cp;
            ch.pad0 = 0;
            ch.pad1 = 0;
            atomicMax(&C->maxtiles_next, ch.ntiles);
            const uint32_t si = atomicAdd(&C->nseg_next, 1u);
            Q.next_segs[si] = ch;
        }
    }
}

// Records whose equal band was staged in the user buffer itself were copied
// to the other buffer by k_post; move them into the user buffer.
template <class KT, int NT>
__global__ void __launch_bounds__(NT) k_band2(PassParams<KT> P) {
    using T = typename KT::T;
    constexpr uint32_t TILE = (uint32_t)tile_elems<KT>();
    const uint32_t t = blockIdx.x;
    const Seg sg = P.tile_map ? P.segs[P.tile_map[t]] : P.seg0;
    if ((sg.parity ? P.stage[1] : P.stage[0]) != P.final_buf) return;
    const uint32_t k = t - sg.tile_base;
    const unsigned long long fin = P.cursor[P.tile_map ? P.tile_map[t] : 0];
    const uint32_t L = (uint32_t)fin, G = (uint32_t)(fin >> 32);
    const uint32_t E = sg.len - L - G;
    const uint64_t b = sg.begin;
    const uint64_t tbeg = (b / TILE) * TILE + (uint64_t)k * TILE;
    const uint64_t band0 = b + L, band1 = b + L + E;
    const uint64_t x0 = tbeg > band0 ? tbeg : band0;
    const uint64_t x1 = (tbeg + TILE) < band1 ? (tbeg + TILE) : band1;
    const T *from = sg.parity ? P.bufs[0] : P.bufs[1];
    for (uint64_t i = x0 + threadIdx.x; i < x1; i += NT) P.final_buf[i] = from[i];
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

// Root segment of a sort: [0, n) in the user buffer with its pivot (a1).
template <class KT>
__global__ void k_init_root(Seg *segs, const typename KT::T *buf, uint32_t n, int rule) {
    constexpr uint32_t TILE = (uint32_t)tile_elems<KT>();
    Seg s;
    s.pivot = (uint64_t)select_pivot<KT>(buf, 0, n, rule);
    s.begin = 0;
    s.len = n;
    s.tile_base = 0;
    s.ntiles = seg_ntiles(0, n, TILE);
    s.depth = 0;
    s.parity = 0;
    s.pad0 = 0;
    s.pad1 = 0;
    segs[0] = s;
}

// bq_pivot_*: the pivot key of buf[0, n).
template <class KT>
__global__ void k_pivot(const typename KT::T *buf, uint32_t n, int rule, uint64_t *out) {
    *out = (uint64_t)select_pivot<KT>(buf, 0, n, rule);
}

}  // namespace bq
