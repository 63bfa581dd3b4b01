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
    uint64_t *status;      // one look-back word per tile, zeroed before the pass
    LevelCtrl *ctrl;       // ticket + counters of this level
    uint32_t ntiles;
    int aligned;           // both data buffers 16-byte aligned -> vector loads
};

// Swizzled staging index: items of consecutive lanes land in distinct banks
// for 4- and 8-byte keys.
template <class T>
__device__ __forceinline__ uint32_t stage_phys(uint32_t s) {
    if constexpr (sizeof(T) == 4) return s ^ ((s >> 5) & 3);
    else if constexpr (sizeof(T) == 8) return s ^ ((s >> 4) & 1);
    else return s;
}

template <class T>
__device__ __forceinline__ void store_stream(T *p, const T &v) {
    if constexpr (sizeof(T) == 32) {
        const uint4 *q = reinterpret_cast<const uint4 *>(&v);
        __stcs(reinterpret_cast<uint4 *>(p), q[0]);
        __stcs(reinterpret_cast<uint4 *>(p) + 1, q[1]);
    } else {
        __stcs(p, v);
    }
}

template <class KT, int NT, int IPT>
__global__ void __launch_bounds__(NT) k_partition(PassParams<KT> P) {
    using T = typename KT::T;
    using K = typename KT::K;
    constexpr bool REC = KT::is_record;
    constexpr int VEC = REC ? 1 : (int)(16 / sizeof(T));
    constexpr int V = IPT / VEC;
    constexpr int NW = NT / 32;
    constexpr int TILE = NT * IPT;
    constexpr int NE = V * NW;                 // warp chunks per tile
    constexpr int PER = (NE + 31) / 32;
    static_assert(IPT % VEC == 0, "IPT must be a multiple of the vector width");
    static_assert(IPT <= 32, "bitmasks hold 32 items");

    __shared__ __align__(16) T s_stage[TILE];
    __shared__ uint32_t s_wl[NE], s_wg[NE], s_we[REC ? NE : 1];
    __shared__ uint32_t s_tile, s_tl, s_tg, s_te, s_lp, s_gp;

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    // ordered tile claiming: every look-back predecessor is already running
    if (tid == 0) s_tile = atomicAdd(&P.ctrl->ticket, 1u);
    __syncthreads();
    const uint32_t t = s_tile;
    const Seg sg = P.tile_map ? P.segs[P.tile_map[t]] : P.seg0;
    const uint32_t k = t - sg.tile_base;
    const uint64_t b = sg.begin, e = b + sg.len;
    const uint64_t tbeg = (b / TILE) * TILE + (uint64_t)k * TILE;
    const uint64_t lo = tbeg > b ? tbeg : b;
    const uint64_t hi = (tbeg + TILE) < e ? (tbeg + TILE) : e;
    const T *src = sg.parity ? P.bufs[1] : P.bufs[0];
    T *dst = sg.parity ? P.bufs[0] : P.bufs[1];
    const K pk = (K)sg.pivot;

    // ---- a2: load ------------------------------------------------------------
    T it[V][VEC];
    uint32_t lt_bits = 0, gt_bits = 0, eq_bits = 0;
#pragma unroll
    for (int v = 0; v < V; v++) {
        const uint64_t i0 = tbeg + (uint64_t)(v * NT + tid) * VEC;
        if (P.aligned && i0 >= lo && i0 + VEC <= hi) {
            if constexpr (REC) {
                const uint4 *q = reinterpret_cast<const uint4 *>(src + i0);
                uint4 *d = reinterpret_cast<uint4 *>(&it[v][0]);
                d[0] = ldg_cs(q);
                d[1] = ldg_cs(q + 1);
            } else {
                uint4 r = ldg_stream(reinterpret_cast<const uint4 *>(src + i0));
                const T *rv = reinterpret_cast<const T *>(&r);
#pragma unroll
                for (int c = 0; c < VEC; c++) it[v][c] = rv[c];
            }
#pragma unroll
            for (int c = 0; c < VEC; c++) {
                const K kk = KT::key(it[v][c]);
                const int bit = v * VEC + c;
                lt_bits |= (uint32_t)(kk < pk) << bit;
                gt_bits |= (uint32_t)(pk < kk) << bit;
                if constexpr (REC) eq_bits |= (uint32_t)(!(kk < pk) && !(pk < kk)) << bit;
            }
        } else {
#pragma unroll
            for (int c = 0; c < VEC; c++) {
                const uint64_t i = i0 + c;
                const bool valid = i >= lo && i < hi;
                if (valid) it[v][c] = src[i];
                const K kk = valid ? KT::key(it[v][c]) : pk;
                const int bit = v * VEC + c;
                lt_bits |= (uint32_t)(valid && kk < pk) << bit;
                gt_bits |= (uint32_t)(valid && pk < kk) << bit;
                if constexpr (REC) eq_bits |= (uint32_t)(valid && !(kk < pk) && !(pk < kk)) << bit;
            }
        }
    }

    // ---- a3: offsets via ballot / popc ------------------------------------------
    const uint32_t lm = lanemask_lt();
    uint32_t rk_l[V][VEC], rk_g[V][VEC], rk_e[REC ? V : 1][VEC];
#pragma unroll
    for (int v = 0; v < V; v++) {
        uint32_t cl = 0, cg = 0, ce = 0, tl = 0, tg = 0, te = 0;
#pragma unroll
        for (int c = 0; c < VEC; c++) {
            const int bit = v * VEC + c;
            const uint32_t ml = __ballot_sync(0xffffffffu, (lt_bits >> bit) & 1);
            const uint32_t mg = __ballot_sync(0xffffffffu, (gt_bits >> bit) & 1);
            cl += __popc(ml & lm);
            cg += __popc(mg & lm);
            tl += __popc(ml);
            tg += __popc(mg);
            if constexpr (REC) {
                const uint32_t me = __ballot_sync(0xffffffffu, (eq_bits >> bit) & 1);
                ce += __popc(me & lm);
                te += __popc(me);
            }
        }
#pragma unroll
        for (int c = 0; c < VEC; c++) {
            const int bit = v * VEC + c;
            rk_l[v][c] = cl;
            cl += (lt_bits >> bit) & 1;
            rk_g[v][c] = cg;
            cg += (gt_bits >> bit) & 1;
            if constexpr (REC) {
                rk_e[v][c] = ce;
                ce += (eq_bits >> bit) & 1;
            }
        }
        if (lane == 0) {
            s_wl[v * NW + warp] = tl;
            s_wg[v * NW + warp] = tg;
            if constexpr (REC) s_we[v * NW + warp] = te;
        }
    }
    __syncthreads();

    // ---- warp 0: scan warp-chunk counts, then a4 look-back ------------------------
    if (warp == 0) {
        uint32_t al[PER], ag[PER], ae[PER];
        uint32_t sl = 0, sgt = 0, se = 0;
#pragma unroll
        for (int i = 0; i < PER; i++) {
            const int idx = lane * PER + i;
            const uint32_t xl = idx < NE ? s_wl[idx] : 0;
            const uint32_t xg = idx < NE ? s_wg[idx] : 0;
            uint32_t xe = 0;
            if constexpr (REC) xe = idx < NE ? s_we[idx] : 0;
            al[i] = sl; ag[i] = sgt; ae[i] = se;
            sl += xl; sgt += xg; se += xe;
        }
        uint32_t il = sl, ig = sgt, ie = se;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t ol = __shfl_up_sync(0xffffffffu, il, d);
            const uint32_t og = __shfl_up_sync(0xffffffffu, ig, d);
            const uint32_t oe = __shfl_up_sync(0xffffffffu, ie, d);
            if (lane >= (uint32_t)d) { il += ol; ig += og; ie += oe; }
        }
#pragma unroll
        for (int i = 0; i < PER; i++) {
            const int idx = lane * PER + i;
            if (idx < NE) {
                s_wl[idx] = il - sl + al[i];
                s_wg[idx] = ig - sgt + ag[i];
                if constexpr (REC) s_we[idx] = ie - se + ae[i];
            }
        }
        const uint32_t TL = __shfl_sync(0xffffffffu, il, 31);
        const uint32_t TG = __shfl_sync(0xffffffffu, ig, 31);
        const uint32_t TE = __shfl_sync(0xffffffffu, ie, 31);

        uint64_t *st = P.status;
        uint32_t accl = 0, accg = 0;
        if (k == 0) {
            if (lane == 0) st_release_u64(st + t, st_pack(ST_INC, TL, TG));
        } else {
            if (lane == 0) st_release_u64(st + t, st_pack(ST_AGG, TL, TG));
            int64_t pred = (int64_t)t - 1;
            const int64_t first_tile = sg.tile_base;
            while (true) {
                const int64_t idx = pred - (int64_t)lane;
                uint64_t w;
                if (idx >= first_tile) {
                    do { w = ld_acquire_u64(st + idx); } while (st_flag(w) == 0);
                } else {
                    w = ST_INC;   // before the segment start: inclusive zero
                }
                const uint32_t inc = __ballot_sync(0xffffffffu, st_flag(w) == 2);
                const int first = inc ? (__ffs(inc) - 1) : 31;
                uint32_t l = (int)lane <= first ? st_lt(w) : 0;
                uint32_t g = (int)lane <= first ? st_gt(w) : 0;
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) {
                    l += __shfl_xor_sync(0xffffffffu, l, d);
                    g += __shfl_xor_sync(0xffffffffu, g, d);
                }
                accl += l;
                accg += g;
                if (inc) break;
                pred -= 32;
            }
            if (lane == 0) st_release_u64(st + t, st_pack(ST_INC, accl + TL, accg + TG));
        }
        if (lane == 0) {
            s_tl = TL; s_tg = TG; s_te = TE;
            s_lp = accl; s_gp = accg;
        }
    }
    __syncthreads();

    // ---- a5: stage in shared memory as [< | > | =] ---------------------------------
    const uint32_t TL = s_tl, TG = s_tg;
    const uint32_t TE = REC ? s_te : 0;
#pragma unroll
    for (int v = 0; v < V; v++) {
        const uint32_t bl = s_wl[v * NW + warp];
        const uint32_t bg = TL + s_wg[v * NW + warp];
        uint32_t be = 0;
        if constexpr (REC) be = TL + TG + s_we[v * NW + warp];
#pragma unroll
        for (int c = 0; c < VEC; c++) {
            const int bit = v * VEC + c;
            if ((lt_bits >> bit) & 1) s_stage[stage_phys<T>(bl + rk_l[v][c])] = it[v][c];
            else if ((gt_bits >> bit) & 1) s_stage[stage_phys<T>(bg + rk_g[v][c])] = it[v][c];
            else if constexpr (REC) {
                if ((eq_bits >> bit) & 1) s_stage[stage_phys<T>(be + rk_e[v][c])] = it[v][c];
            }
        }
    }
    __syncthreads();

    // ---- coalesced write-out ----------------------------------------------------
    const uint64_t lp = s_lp, gp = s_gp;
    const uint32_t cnt = TL + TG + TE;
    const uint64_t lbase = b + lp;
    const uint64_t gtop = e - 1 - gp;
    T *estage = nullptr;
    uint64_t ebase = 0;
    if constexpr (REC) {
        estage = sg.parity ? P.stage[1] : P.stage[0];
        ebase = b + ((lo - b) - lp - gp);   // + Eprefix
    }
    for (uint32_t s = tid; s < cnt; s += NT) {
        const T x = s_stage[stage_phys<T>(s)];
        if (s < TL) store_stream(dst + lbase + s, x);
        else if (s < TL + TG) store_stream(dst + (gtop - (s - TL)), x);
        else if constexpr (REC) store_stream(estage + ebase + (s - TL - TG), x);
    }
}

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
    const uint64_t fin = P.status[sg.tile_base + sg.ntiles - 1];
    const uint32_t L = st_lt(fin), G = st_gt(fin);
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
        Q.d_counts[0] = L;
        Q.d_counts[1] = E;
        Q.d_counts[2] = G;
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
            const uint32_t li = atomicAdd(&C->nleaf, 1u);
            Q.leaves[li] = Leaf{cb[c], cl[c], cp, 0};
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
    const uint64_t fin = P.status[sg.tile_base + sg.ntiles - 1];
    const uint32_t L = st_lt(fin), G = st_gt(fin);
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
static __global__ void k_map(const Seg *segs, uint32_t *tile_map, uint64_t *status) {
    const uint32_t s = blockIdx.x;
    const Seg sg = segs[s];
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
