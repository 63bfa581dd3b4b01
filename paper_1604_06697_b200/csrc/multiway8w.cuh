// multiway8w.cuh — the 8-way multi-pivot level (N4) with warp-private tiles
// and exact output offsets: no block barriers and no atomics on the data path.
//
// The paper's block partition keeps, per block, the offsets of the elements to
// move and moves them in a second loop (Alg. 3); with k buckets the
// offsets become k counters (Super Scalar Sample Sort's "oracle").
// Here one warp owns a whole tile (TILE = tile_elems<KT>() keys, processed in
// rounds of 32 x IPT keys), and a level is three launches (+ k_post_mw):
//   k_mw8w_count    every tile's 8 bucket counts -> tab[t][b]      (read pass)
//   k_mw8w_scan     prefixes of tab over the tiles (blocks of MWS_BR tiles, the
//                   block prefixes by the CTA finishing last)
//   k_mw8w_scatter  per round: classify, rank inside the warp (packed counters
//                   and a byte-field warp scan), stage the round bucket by
//                   bucket in the warp's shared memory, store it coalesced;
//                   a segment's bucket b starts at its begin + the totals of
//                   buckets < b (mw8w_seg_buckets), and tile t's keys of b
//                   follow those of the segment's earlier tiles
// (k_post_mw derives the children from the same table.)
// Tiles of a segment are consecutive and a bucket receives them in tile
// order, so the layout of a level is deterministic.  Splitters, classification
// (float64 compares as doubles, R25) and counters are multiway8.cuh's.
#pragma once

namespace bq {

#ifndef BQ_MWS_BR
#define BQ_MWS_BR 512
#endif
constexpr uint32_t MWS_BR = BQ_MWS_BR;   // table rows per block of the row-count scan (256 threads)
constexpr uint32_t MWS_RPT = MWS_BR / 256;   // rows per thread
static_assert(MWS_BR % 256 == 0, "whole rows per thread");
constexpr int MW8W_WARPS = 8;       // warps per CTA of the count and scatter kernels
#ifndef BQ_MW8W_MINB
#define BQ_MW8W_MINB 2
#endif
#ifndef BQ_MW8W_MINB_PAIR
#define BQ_MW8W_MINB_PAIR 2
#endif

// A level with fewer tiles than MW8W_UNIT_WARPS splits each tile into U units
// (a power of two <= the rounds per tile) so that every warp has work; the
// unit is the row of the count table.  count, scan, scatter and k_post_mw
// derive the same U from the level's tile count.
constexpr uint32_t MW8W_UNIT_WARPS = 2048;
constexpr uint32_t MW8W_ROWS_EXTRA = 2 * MW8W_UNIT_WARPS;   // table rows beyond one per tile

template <class KT> struct Mw8wTune;
template <> struct Mw8wTune<KI32> { static constexpr int IPT = 8, MINB = BQ_MW8W_MINB; };
template <> struct Mw8wTune<KU64> { static constexpr int IPT = 8, MINB = BQ_MW8W_MINB; };
template <> struct Mw8wTune<KF64> { static constexpr int IPT = 8, MINB = BQ_MW8W_MINB; };
template <> struct Mw8wTune<KRec> { static constexpr int IPT = 2, MINB = BQ_MW8W_MINB; };
template <> struct Mw8wTune<KPair> { static constexpr int IPT = 4, MINB = BQ_MW8W_MINB_PAIR; };

template <class KT>
__host__ __device__ constexpr uint32_t mw8w_rounds() { return (uint32_t)tile_elems<KT>() / (32u * Mw8wTune<KT>::IPT); }
// Table rows per tile at least: the TMA-staged scatter (k_mw8t_scatter) stages
// a whole unit per warp, so units are at most BQ_MW8T_UNIT_BYTES (4 KB: four
// rows per 16 KB tile; 16 warps of double-buffered input and one staging plane
// per SM)
#ifndef BQ_MW8T
#define BQ_MW8T 1
#endif
#ifndef BQ_MW8T_UNIT_BYTES
#define BQ_MW8T_UNIT_BYTES 4096
#endif
template <class KT>
__host__ __device__ constexpr uint32_t mw8w_umin() {
    constexpr uint32_t tb = (uint32_t)(tile_elems<KT>() * sizeof(typename KT::T));
    return (BQ_MW8T && tb > BQ_MW8T_UNIT_BYTES) ? tb / BQ_MW8T_UNIT_BYTES : 1u;
}
template <class KT>
__device__ __forceinline__ uint32_t mw8w_upt(uint32_t ntiles) {
    static_assert(mw8w_umin<KT>() <= mw8w_rounds<KT>(), "a unit holds whole rounds");
    uint32_t u = mw8w_umin<KT>();
    while (u < mw8w_rounds<KT>() && ntiles * u < MW8W_UNIT_WARPS) u <<= 1;
    return u;
}

// per-warp staging of one round, double-buffered by round parity
template <class KT, int IPT>
struct Mw8wWarpSmem {
    static constexpr int RK = 32 * IPT;
    uint4 in[2][RK * sizeof(typename KT::T) / 16];   // the next round's keys (cp.async), by parity
    typename KT::T key[2][RK];
    uint8_t tag[2][RK];          // the staged key's bucket
    uint32_t ob[2][MW8];         // global index of staged slot 0 of each bucket's run
};
template <class KT>
constexpr int mw8w_smem_bytes() {
    return (int)(MW8W_WARPS * sizeof(Mw8wWarpSmem<KT, Mw8wTune<KT>::IPT>));
}

// the splitters of segment si as the 8-way classification compares them
template <class KT>
__device__ __forceinline__ void mw8w_load_cls(const MwParams<KT> &P, uint32_t si, Mw8Cls<KT> &cls) {
    typename KT::K tr[MW8];
#pragma unroll
    for (int q = 1; q < MW8; q++) tr[q] = mw8_tree_word<KT>(P.msegs[si].tree[q]);
    cls.load(tr);
}

// Round r0 (tile positions [r0, r0 + 32 IPT)) of the tile at src (= the
// buffer + tbeg): element c = v VW + e of lane L sits at position
// r0 + v 32 VW + L VW + e (VW elements per 16-byte vector: every vector load
// of the warp covers 512 contiguous bytes).  Returns the validity mask.
template <class KT, int IPT>
__device__ __forceinline__ uint32_t mw8w_load(const typename KT::T *src, uint32_t r0, uint32_t vlo, uint32_t vhi,
                                              uint32_t lane, bool vec, typename KT::T (&x)[IPT]) {
    using T = typename KT::T;
    constexpr uint32_t VW = sizeof(T) >= 16 ? 1u : 16u / (uint32_t)sizeof(T), NV = IPT / VW;
    static_assert(IPT % VW == 0, "whole vectors per thread");
    if (vec && r0 >= vlo && r0 + 32u * IPT <= vhi) {
#pragma unroll
        for (uint32_t v = 0; v < NV; v++) {
            const uint4 q = ldg_stream(reinterpret_cast<const uint4 *>(src + r0 + v * 32 * VW + lane * VW));
            memcpy(&x[v * VW], &q, 16);
        }
        return (1u << IPT) - 1;
    }
    uint32_t valid = 0;
#pragma unroll
    for (uint32_t v = 0; v < NV; v++)
#pragma unroll
        for (uint32_t e = 0; e < VW; e++) {
            const uint32_t pos = r0 + v * 32 * VW + lane * VW + e;
            const bool ok = pos >= vlo && pos < vhi;
            x[v * VW + e] = ok ? src[pos] : T{};
            valid |= (uint32_t)ok << (v * VW + e);
        }
    return valid;
}

__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// ---- the splitter tree in shared memory ---------------------------------------------
// Levels 1 and 2 of the three-compare bucket search read their splitter from
// a per-warp copy of the tree in shared memory, and the key's leaf value (the
// count kernel's one-hot counter increment) comes from a table there: per key
// three compares, three selects, three predicated adds and three shared loads,
// against the four register selects plus the increment's construction that
// kept the ALU pipe saturated (int32 count: 17 instructions per key, ALU 75 %).
// The addresses are built from p0 alone (selects issued beside the first
// load) plus the later predicates; a linked variant (each record holding its
// children's address) had fewer instructions but a longer dependent chain and
// ran slower (profiles/r02/mw8t.md).
template <class KT> struct Mw8CmpT { using type = typename KT::K; };
template <> struct Mw8CmpT<KF64> { using type = double; };
template <class KT>
struct Mw8Smt {
    typename Mw8CmpT<KT>::type node[MW8];   // node[j], j = 1..7 (heap order, mw_splitters)
    uint32_t leaf[MW8];                     // leaf value of bucket b
    uint2 l2[4];                            // 4-byte keys: level-2 node 4 + i as {splitter, leaf(2 i)}
};
__device__ __forceinline__ int32_t lds_ck(uint32_t a, int32_t *) { return (int32_t)lds32(a); }
__device__ __forceinline__ uint64_t lds_ck(uint32_t a, uint64_t *) {
    uint64_t v;
    asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ double lds_ck(uint32_t a, double *) { return __longlong_as_double((long long)lds_ck(a, (uint64_t *)nullptr)); }
// the key as the classification compares it (float64: the double)
template <class KT>
__device__ __forceinline__ typename Mw8CmpT<KT>::type mw8_ckey(const typename KT::T &x) {
    if constexpr (std::is_same<KT, KF64>::value) return __longlong_as_double((long long)x);
    else return KT::key(x);
}
// lanes 0..7 write the tree of segment si (leaf value of bucket b: leaf(b))
template <class KT, class F>
__device__ __forceinline__ void mw8_smt_write(const MwParams<KT> &P, uint32_t si, Mw8Smt<KT> &t, uint32_t lane, F leaf) {
    __syncwarp();   // the previous segment's readers are done
    if (lane < MW8) {
        const typename KT::K w = mw8_tree_word<KT>(P.msegs[si].tree[lane]);
        if constexpr (std::is_same<KT, KF64>::value) t.node[lane] = __longlong_as_double((long long)w);
        else t.node[lane] = w;
        t.leaf[lane] = leaf(lane);
        if constexpr (sizeof(typename Mw8CmpT<KT>::type) == 4)
            if (lane >= 4) t.l2[lane - 4] = make_uint2((uint32_t)w, leaf(2 * (lane - 4)));
    }
    __syncwarp();
}
// 4-byte keys, leaf values of buckets 2 i + 1 = those of 2 i << 4 (the count's
// one-hot increments): level 2 loads its splitter and the leaf value together
__device__ __forceinline__ uint32_t mw8_smt_inc32(uint32_t tb, uint32_t l2b, int32_t t1, int32_t k) {
    const bool p0 = t1 < k;
    const uint32_t a1 = p0 ? tb + 12u : tb + 8u;
    uint32_t a2 = p0 ? l2b + 16u : l2b;
    const int32_t n1 = (int32_t)lds32(a1);
    if (n1 < k) a2 += 8u;
    uint32_t n2, inc;
    asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(n2), "=r"(inc) : "r"(a2));
    return (int32_t)n2 < k ? inc << 4 : inc;
}
// the leaf value of key k: tb = the shared address of node[0], lb = of
// leaf[0], t1 = node[1] (in a register)
template <class CK>
__device__ __forceinline__ uint32_t mw8_smt_leaf(uint32_t tb, uint32_t lb, CK t1, CK k) {
    constexpr uint32_t SZ = sizeof(CK);
    const bool p0 = t1 < k;
    const uint32_t a1 = p0 ? tb + 3 * SZ : tb + 2 * SZ;
    uint32_t a2 = p0 ? tb + 6 * SZ : tb + 4 * SZ;
    uint32_t al = p0 ? lb + 16u : lb;
    const CK n1 = lds_ck(a1, (CK *)nullptr);
    const bool p1 = n1 < k;
    if (p1) a2 += SZ;
    if (p1) al += 8u;
    const CK n2 = lds_ck(a2, (CK *)nullptr);
    if (n2 < k) al += 4u;
    return lds32(al);
}

// ---- k_mw8w_count ------------------------------------------------------------------
template <class KT, int IPT>
__global__ void __launch_bounds__(MW8W_WARPS * 32) k_mw8w_count(const MwParams<KT> Pin) {
    if (const LevelCtrl *pv = loop_prev_ctrl(Pin.lp)) if (pv->nmseg_next == 0) return;
    __shared__ MwParams<KT> sP;
    const MwParams<KT> &P = cta_params(Pin, sP);
    using T = typename KT::T;
    constexpr uint32_t TILE = (uint32_t)tile_elems<KT>(), RK = 32u * IPT;
    static_assert(TILE % RK == 0 && (TILE / 32) <= 255, "rounds per tile; byte counters");
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t ntiles = *P.ntiles_dev, U = mw8w_upt<KT>(ntiles), lgU = __ffs(U) - 1, UL = TILE >> lgU;
    // a warp's item: a whole tile (its U rows) on large levels, one unit on
    // small ones (so that every warp has work)
    const uint32_t lgG = ntiles * U >= 8192 ? lgU : 0, nitems = (ntiles * U) >> lgG;
#ifndef BQ_MW8_NR
#define BQ_MW8_NR 4
#endif
    constexpr int NR = sizeof(T) <= 4 ? BQ_MW8_NR : 1;   // rounds loaded before the first is classified
    using CK = typename Mw8CmpT<KT>::type;
    __shared__ Mw8Smt<KT> s_tree[MW8W_WARPS];
    Mw8Smt<KT> &smt = s_tree[threadIdx.x >> 5];
    const uint32_t tb = smem_u32(smt.node), lb = smem_u32(smt.leaf), l2b = smem_u32(smt.l2);
    uint32_t cls_seg = 0xffffffffu;
    Mw8Cls<KT> cls;
    CK t1{};
    const bool aligned = P.aligned;
    for (uint32_t it = blockIdx.x * MW8W_WARPS + (threadIdx.x >> 5); it < nitems; it += gridDim.x * MW8W_WARPS) {
        const uint32_t u0 = it << lgG, t = u0 >> lgU;
        const uint32_t si = P.tile_map[t];
        const Seg sg = P.msegs[si].s;
        if (si != cls_seg) {
            mw8w_load_cls<KT>(P, si, cls);
            cls_seg = si;
            mw8_smt_write<KT>(P, si, smt, lane, [](uint32_t b) { return 1u << (4 * b); });
            t1 = cls.tr[1];
        }
        const TileGeom<KT, TILE> G(sg, t);
        const T *src = (sg.parity ? P.bufs[1] : P.bufs[0]) + G.tbeg;
        for (uint32_t u = u0; u < u0 + (1u << lgG); u++) {
            const uint32_t ub = (u & (U - 1)) * UL;
            const uint32_t lo = G.vlo > ub ? G.vlo : ub, hi = G.vhi < ub + UL ? G.vhi : ub + UL;   // the unit's keys
            uint32_t alo = 0, ahi = 0;   // byte counters: <= TILE / 32 per lane
            // one round's keys into the counters (valid: the keys inside the unit)
            auto tally = [&](const T (&xr)[IPT], uint32_t valid) {
                uint32_t inc[IPT];
                bool nan = false;
#pragma unroll
                for (int c = 0; c < IPT; c++) {
                    const CK k = mw8_ckey<KT>(xr[c]);
                    if constexpr (std::is_same<KT, KF64>::value) nan |= k != k;
                    if constexpr (std::is_same<KT, KI32>::value) inc[c] = mw8_smt_inc32(tb, l2b, t1, k);
                    else inc[c] = mw8_smt_leaf(tb, lb, t1, k);
                }
                if (nan)
#pragma unroll
                    for (int c = 0; c < IPT; c++) inc[c] = 1u << cls.fix4(xr[c], 31 - __clz(inc[c]));
                Mw8Ctr<IPT> ctr;
                if (valid == (1u << IPT) - 1) {
#pragma unroll
                    for (int c = 0; c < IPT; c++) ctr.c += inc[c];
                } else {
#pragma unroll
                    for (int c = 0; c < IPT; c++)
                        if ((valid >> c) & 1) ctr.c += inc[c];
                }
                uint32_t lo, hi;
                ctr.bytes(lo, hi);
                alo += lo;
                ahi += hi;
            };
            if (aligned && lo == ub && hi == ub + UL && UL % (NR * RK) == 0) {
                // a whole unit (the common case): one base pointer, no per-round checks
                constexpr uint32_t VW = sizeof(T) >= 16 ? 1u : 16u / (uint32_t)sizeof(T), NV = IPT / VW;
                const uint4 *p4 = reinterpret_cast<const uint4 *>(src + ub) + lane;
                for (uint32_t s0 = 0; s0 < UL; s0 += NR * RK) {
                    T x[NR][IPT];
#pragma unroll
                    for (int h = 0; h < NR; h++)
#pragma unroll
                        for (uint32_t v = 0; v < NV; v++) {
                            const uint4 q = ldg_stream(p4 + (s0 + h * RK) / VW + v * 32);
                            memcpy(&x[h][v * VW], &q, 16);
                        }
#pragma unroll
                    for (int h = 0; h < NR; h++) tally(x[h], (1u << IPT) - 1);
                }
            } else {
                for (uint32_t r0 = lo / RK * RK; r0 < hi; r0 += NR * RK) {
                    T x[NR][IPT];
                    uint32_t valid[NR];
#pragma unroll
                    for (int h = 0; h < NR; h++) valid[h] = mw8w_load<KT, IPT>(src, r0 + h * RK, lo, hi, lane, aligned, x[h]);
#pragma unroll
                    for (int h = 0; h < NR; h++) tally(x[h], valid[h]);
                }
            }
            uint32_t q[MW8 / 2];
            mw8_widen((uint64_t)alo | ((uint64_t)ahi << 32), q);
#pragma unroll
            for (int k = 0; k < MW8 / 2; k++) q[k] = __reduce_add_sync(0xffffffffu, q[k]);   // (16-bit fields <= 4096)
            // (selects with constant indices: a run-time index put q in local memory)
            const uint32_t mine = (lane & 4) ? ((lane & 2) ? q[3] : q[2]) : ((lane & 2) ? q[1] : q[0]);
            if (lane < MW8) P.mtab[(size_t)u * MW8 + lane] = (lane & 1) ? (mine >> 16) : (mine & 0xffff);
        }
    }
}

// exclusive scan of 8 columns over the 256 threads of a CTA: ex = this
// thread's prefix, the return value's columns = the totals (every thread)
__device__ __forceinline__ void mw8w_cta_scan8(const uint32_t (&v)[MW8], uint32_t (&ex)[MW8], uint32_t (&tot)[MW8],
                                               uint32_t (*s_w)[MW8]) {
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t inc[MW8];
#pragma unroll
    for (int k = 0; k < MW8; k++) inc[k] = v[k];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1)
#pragma unroll
        for (int k = 0; k < MW8; k++) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, inc[k], d);
            if (lane >= (uint32_t)d) inc[k] += o;
        }
    __syncthreads();   // s_w of a previous use read
    if (lane == 31)
#pragma unroll
        for (int k = 0; k < MW8; k++) s_w[warp][k] = inc[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < MW8; k++) {
        uint32_t w = 0, all = 0;
#pragma unroll
        for (uint32_t w2 = 0; w2 < 8; w2++) {
            w += w2 < warp ? s_w[w2][k] : 0;
            all += s_w[w2][k];
        }
        ex[k] = w + inc[k] - v[k];
        tot[k] = all;
    }
}

// ---- k_mw8w_scan: prefix of the tile counts --------------------------------------
// Blocks of MWS_BR tiles: tab[t] becomes the prefix of t inside its block and
// blk[i] the total of block i; the CTA that completes the last block turns
// blk into exclusive block prefixes (row nblk: the grand total).  The global
// prefix of tile t is then tab[t] + blk[t / MWS_BR].
template <class KT>
__global__ void __launch_bounds__(256) k_mw8w_scan(const MwParams<KT> Pin) {
    if (const LevelCtrl *pv = loop_prev_ctrl(Pin.lp)) if (pv->nmseg_next == 0) return;
    __shared__ MwParams<KT> sP;
    const MwParams<KT> &P = cta_params(Pin, sP);
    __shared__ uint32_t s_w[8][MW8];
    __shared__ uint32_t s_last;
    const uint32_t tid = threadIdx.x;
    const uint32_t ntiles = *P.ntiles_dev * mw8w_upt<KT>(*P.ntiles_dev);   // table rows
    const uint32_t nblk = (ntiles + MWS_BR - 1) / MWS_BR;
    uint32_t done = 0;
    for (uint32_t blk = blockIdx.x; blk < nblk; blk += gridDim.x, done++) {
        const uint32_t t0 = blk * MWS_BR + tid * MWS_RPT;
        uint32_t sum[MW8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (uint32_t t = t0; t < t0 + MWS_RPT && t < ntiles; t++) {
            const uint4 *row = reinterpret_cast<const uint4 *>(P.mtab + (size_t)t * MW8);
            const uint4 a = row[0], b = row[1];
            sum[0] += a.x; sum[1] += a.y; sum[2] += a.z; sum[3] += a.w;
            sum[4] += b.x; sum[5] += b.y; sum[6] += b.z; sum[7] += b.w;
        }
        uint32_t pre[MW8], all[MW8];
        mw8w_cta_scan8(sum, pre, all, s_w);
        if (tid == 0)
#pragma unroll
            for (int k = 0; k < MW8; k++) P.mblk[(size_t)blk * MW8 + k] = all[k];
        for (uint32_t t = t0; t < t0 + MWS_RPT && t < ntiles; t++) {
            uint4 *row = reinterpret_cast<uint4 *>(P.mtab + (size_t)t * MW8);
            const uint4 a = row[0], b = row[1];
            row[0] = make_uint4(pre[0], pre[1], pre[2], pre[3]);
            row[1] = make_uint4(pre[4], pre[5], pre[6], pre[7]);
            pre[0] += a.x; pre[1] += a.y; pre[2] += a.z; pre[3] += a.w;
            pre[4] += b.x; pre[5] += b.y; pre[6] += b.z; pre[7] += b.w;
        }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = done > 0 && atomicAdd(&P.ctrl->mw_scan_done, done) + done == nblk;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    uint32_t carry[MW8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (uint32_t b0 = 0; b0 < nblk; b0 += 256) {
        const uint32_t bi = b0 + tid;
        uint32_t v[MW8], ex[MW8], tot[MW8];
#pragma unroll
        for (int k = 0; k < MW8; k++) v[k] = bi < nblk ? __ldcg(&P.mblk[(size_t)bi * MW8 + k]) : 0;
        mw8w_cta_scan8(v, ex, tot, s_w);
#pragma unroll
        for (int k = 0; k < MW8; k++) {
            if (bi < nblk) P.mblk[(size_t)bi * MW8 + k] = carry[k] + ex[k];
            carry[k] += tot[k];
        }
    }
    if (tid == 0) {
        unsigned long long all = 0;
#pragma unroll
        for (int k = 0; k < MW8; k++) {
            P.mblk[(size_t)nblk * MW8 + k] = carry[k];
            all += carry[k];
        }
        atomicAdd(&P.ctrl->mw_element_passes, all);
    }
}

// Lanes b < 8 of a warp: the bucket b total (tot) and start (relative to the
// segment's begin) of the segment owning table rows [tile_base, tile_base +
// seg_tiles) of ntiles, and the global prefix of its first row (pf); every
// lane of the warp takes part (shuffles).
template <class KT>
__device__ __forceinline__ void mw8w_seg_buckets(const MwParams<KT> &P, uint32_t tile_base, uint32_t seg_tiles,
                                                 uint32_t ntiles, uint32_t lane, uint32_t &tot, uint32_t &start,
                                                 uint32_t &pf) {
    const uint32_t first = tile_base, end = tile_base + seg_tiles, nblk = (ntiles + MWS_BR - 1) / MWS_BR;
    tot = 0;
    pf = 0;
    if (lane < MW8) {
        pf = P.mtab[(size_t)first * MW8 + lane] + P.mblk[(size_t)(first / MWS_BR) * MW8 + lane];
        const uint32_t pe = end < ntiles ? P.mtab[(size_t)end * MW8 + lane] + P.mblk[(size_t)(end / MWS_BR) * MW8 + lane]
                                         : P.mblk[(size_t)nblk * MW8 + lane];
        tot = pe - pf;
    }
    uint32_t inc = tot;
#pragma unroll
    for (int d = 1; d < MW8; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= (uint32_t)d) inc += o;
    }
    start = inc - tot;
}

// per-lane asynchronous 16-byte copies global -> shared (LDGSTS), one group per round
__device__ __forceinline__ void cp_async16(void *sdst, const void *gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(sdst)),
                 "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// the tile a warp places next: its segment, source, destination and valid range
template <class KT>
struct Mw8wTile {
    uint32_t u, si, vlo, vhi, begin, tile_base, ntiles;   // unit, segment, the unit's keys, segment rows
    const typename KT::T *src;   // the buffer + the tile's first position
    typename KT::T *dst;
};
template <class KT>
__device__ __forceinline__ Mw8wTile<KT> mw8w_tile(const MwParams<KT> &P, uint32_t u, uint32_t U) {
    constexpr uint32_t TILE = (uint32_t)tile_elems<KT>();
    const uint32_t lgU = __ffs(U) - 1, t = u >> lgU, UL = TILE >> lgU, ub = (u & (U - 1)) * UL;
    Mw8wTile<KT> w;
    w.u = u;
    w.si = P.tile_map[t];
    const Seg sg = P.msegs[w.si].s;
    const TileGeom<KT, TILE> G(sg, t);
    w.vlo = G.vlo > ub ? G.vlo : ub;
    w.vhi = G.vhi < ub + UL ? G.vhi : ub + UL;
    w.begin = sg.begin;
    w.tile_base = sg.tile_base * U;
    w.ntiles = sg.ntiles * U;
    w.src = (sg.parity ? P.bufs[1] : P.bufs[0]) + G.tbeg;
    w.dst = sg.parity ? P.bufs[0] : P.bufs[1];
    return w;
}

// Round r0 of tile w into the lane's slots of a shared-memory input buffer
// (vector v of lane L at in[v * 32 + L]: the layout mw8w_load reads from
// global memory): whole valid vectors by asynchronous copies, vectors cut by
// the valid range element by element (zeros outside it).
template <class KT, int IPT>
__device__ __forceinline__ void mw8w_issue(const Mw8wTile<KT> &w, uint32_t r0, uint32_t lane, bool vec, uint4 *in) {
    using T = typename KT::T;
    constexpr uint32_t VW = sizeof(T) >= 16 ? 1u : 16u / (uint32_t)sizeof(T), NV = IPT / VW;
#pragma unroll
    for (uint32_t v = 0; v < NV; v++) {
        const uint32_t pos = r0 + v * 32 * VW + lane * VW;
        uint4 *d = &in[v * 32 + lane];
        if (vec && pos >= w.vlo && pos + VW <= w.vhi) {
            cp_async16(d, w.src + pos);
        } else {
            T e[VW];
#pragma unroll
            for (uint32_t k = 0; k < VW; k++) e[k] = (pos + k >= w.vlo && pos + k < w.vhi) ? w.src[pos + k] : T{};
            memcpy(d, e, 16);
        }
    }
}

// ---- k_mw8w_scatter ----------------------------------------------------------------
// Each warp runs one pipeline over its rounds (across its tiles): the next
// round's keys are copied into the other input buffer while the current
// round is classified, ranked, staged and stored.
template <class KT, int IPT>
__global__ void __launch_bounds__(MW8W_WARPS * 32, Mw8wTune<KT>::MINB) k_mw8w_scatter(const MwParams<KT> Pin) {
    if (const LevelCtrl *pv = loop_prev_ctrl(Pin.lp)) if (pv->nmseg_next == 0) return;
    __shared__ MwParams<KT> sP;
    const MwParams<KT> &P = cta_params(Pin, sP);
    using T = typename KT::T;
    using WS = Mw8wWarpSmem<KT, IPT>;
    constexpr uint32_t TILE = (uint32_t)tile_elems<KT>(), RK = 32u * IPT;
    constexpr uint32_t VW = sizeof(T) >= 16 ? 1u : 16u / (uint32_t)sizeof(T), NV = IPT / VW;
    static_assert(TILE % RK == 0 && IPT <= 8, "rounds per tile; byte-field scans");
    extern __shared__ __align__(128) unsigned char smraw[];
    WS &ws = reinterpret_cast<WS *>(smraw)[threadIdx.x >> 5];
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t U = mw8w_upt<KT>(*P.ntiles_dev), ntiles = *P.ntiles_dev * U;   // units (table rows)
    const uint32_t stride = gridDim.x * MW8W_WARPS;
    const uint32_t u0 = blockIdx.x * MW8W_WARPS + (threadIdx.x >> 5);
    if (u0 >= ntiles) return;
    const bool vec = P.aligned;
    Mw8wTile<KT> cur = mw8w_tile(P, u0, U);
    uint32_t r0 = cur.vlo / RK * RK, par = 0, cls_seg = 0xffffffffu, off = 0, seg_base = 0;
    bool new_tile = true;
    Mw8Cls<KT> cls;
    mw8w_issue<KT, IPT>(cur, r0, lane, vec, ws.in[0]);
    cp_async_commit();
    for (;;) {
        // the next round: of this tile, or the first of the warp's next tile
        Mw8wTile<KT> nxt = cur;
        uint32_t nr0 = r0 + RK;
        bool more = true;
        if (nr0 >= cur.vhi) {
            if (cur.u + stride < ntiles) {
                nxt = mw8w_tile(P, cur.u + stride, U);
                nr0 = nxt.vlo / RK * RK;
            } else {
                more = false;
            }
        }
        if (more) mw8w_issue<KT, IPT>(nxt, nr0, lane, vec, ws.in[par ^ 1]);
        cp_async_commit();
        if (new_tile) {
            if (cur.si != cls_seg) {
                mw8w_load_cls<KT>(P, cur.si, cls);
                uint32_t tot, start, pf;
                mw8w_seg_buckets(P, cur.tile_base, cur.ntiles, ntiles, lane, tot, start, pf);
                seg_base = cur.begin + start - pf;   // lane b: bucket b's output base minus its tiles' prefix
                cls_seg = cur.si;
            }
            // lane b < 8: the global index of this tile's next key of bucket b
            if (lane < MW8)
                off = seg_base + P.mtab[(size_t)cur.u * MW8 + lane] + P.mblk[(size_t)(cur.u / MWS_BR) * MW8 + lane];
        }
        cp_async_wait1();   // this round's copies (the lane reads only its own slots)
        T x[IPT];
#pragma unroll
        for (uint32_t v = 0; v < NV; v++) {
            const uint4 q = ws.in[par][v * 32 + lane];
            memcpy(&x[v * VW], &q, 16);
        }
        uint32_t valid = 0;
#pragma unroll
        for (uint32_t v = 0; v < NV; v++)
#pragma unroll
            for (uint32_t e = 0; e < VW; e++) {
                const uint32_t pos = r0 + v * 32 * VW + lane * VW + e;
                valid |= (uint32_t)(pos >= cur.vlo && pos < cur.vhi) << (v * VW + e);
            }
        T *dst = cur.dst;
        // (full rounds, the common case, skip every validity test)
        auto round = [&](auto full_tag) {
            constexpr bool FULL = decltype(full_tag)::value;
            uint32_t bk[IPT], rk[IPT];
            mw8_classify<KT, IPT>(cls, x, bk);
            Mw8Ctr<IPT> ctr;
#pragma unroll
            for (int c = 0; c < IPT; c++) rk[c] = ctr.take(bk[c], FULL ? 1u : (valid >> c) & 1);
            uint32_t ex[MW8 / 2], tot[MW8 / 2];
            mw8_scan<IPT>(ctr, lane, ex, tot);
            // the round's bucket starts rs (16-bit pairs: word k = buckets 2k, 2k+1)
            uint32_t rs[MW8 / 2], run = 0;
#pragma unroll
            for (int k = 0; k < MW8 / 2; k++) {
                tot[k] = __shfl_sync(0xffffffffu, tot[k], 31);
                const uint32_t lo = tot[k] & 0xffff;
                rs[k] = run | ((run + lo) << 16);
                run += lo + (tot[k] >> 16);
                ex[k] += rs[k];   // slot base of this lane's keys of each bucket
            }
            if (lane < MW8) {
                const uint32_t wb = (lane & 4) ? ((lane & 2) ? rs[3] : rs[2]) : ((lane & 2) ? rs[1] : rs[0]);
                const uint32_t tw = (lane & 4) ? ((lane & 2) ? tot[3] : tot[2]) : ((lane & 2) ? tot[1] : tot[0]);
                const uint32_t rsb = (lane & 1) ? (wb >> 16) : (wb & 0xffff);
                ws.ob[par][lane] = off - rsb;
                off += (lane & 1) ? (tw >> 16) : (tw & 0xffff);
            }
            // stage the round bucket by bucket
#pragma unroll
            for (int c = 0; c < IPT; c++) {
                if (FULL || ((valid >> c) & 1)) {
                    const uint32_t b = bk[c];
                    const uint32_t w01 = (b & 2) ? ex[1] : ex[0], w23 = (b & 2) ? ex[3] : ex[2];
                    const uint32_t w = (b & 4) ? w23 : w01;
                    const uint32_t slot = ((b & 1) ? (w >> 16) : (w & 0xffff)) + rk[c];
                    BQ_CHECK(slot < RK);
                    ws.key[par][slot] = x[c];
                    ws.tag[par][slot] = (uint8_t)b;
                }
            }
            __syncwarp();
            // store: slot j of bucket b goes to ob[b] + j (contiguous per bucket)
#pragma unroll
            for (uint32_t m = 0; m < (uint32_t)IPT; m++) {
                const uint32_t j = m * 32 + lane;
                if (FULL || j < run) {
                    const uint32_t g = ws.ob[par][ws.tag[par][j]] + j;
                    BQ_CHECK(g < P.n_total);
                    dst[g] = ws.key[par][j];
                }
            }
        };
        if (__all_sync(0xffffffffu, valid == (1u << IPT) - 1)) round(std::true_type{});
        else round(std::false_type{});
        par ^= 1;
        if (!more) break;
        new_tile = nxt.u != cur.u;
        cur = nxt;
        r0 = nr0;
    }
}

// ---- k_mw8t_scatter: bucket runs staged per unit, stored by TMA --------------------
// The scatter of the 8-way level with the output moved like k_part_fast's: a
// warp stages a whole unit (<= BQ_MW8T_UNIT_BYTES) bucket by bucket in its own
// shared-memory plane, each bucket's run placed at a slot congruent to its
// global destination modulo 16 bytes, and lanes 0..7 write the 16-byte aligned
// body of their bucket's run with one bulk copy each (heads and tails < 16
// bytes by plain stores).  The unit's input arrives by one bulk copy into a
// double buffer (the next unit's copy is in flight while this one is placed).
// Per key: classify, rank (packed counters, byte-field warp scan per round),
// one shared-memory store; no per-key global store, no tags, no block barrier.
// The layout is the one the count table fixes (unit u's keys of bucket b
// follow those of the segment's earlier units), the order inside a unit's run
// the (round, lane, key) order.
template <class KT, int IPT>
struct Mw8tWarpSmem {
    using T = typename KT::T;
    static constexpr uint32_t VW = tile_vw<KT>();
    static constexpr uint32_t UNIT = (uint32_t)tile_elems<KT>() / mw8w_umin<KT>();   // largest unit
    static constexpr uint32_t SCAP = (UNIT + MW8 * VW + VW + VW - 1) / VW * VW;     // runs + alignment gaps
    alignas(16) T in[2][UNIT];
    alignas(16) T stage[SCAP];
    uint32_t exs[MW8 * 32];   // lane L's first slot of bucket b this round at [32 b + L] (conflict-free)
    uint64_t bar[2];
};
template <class KT>
constexpr int mw8t_smem_bytes() {
    return (int)(MW8W_WARPS * sizeof(Mw8tWarpSmem<KT, Mw8wTune<KT>::IPT>));
}
template <class KT> struct Mw8tTune { static constexpr int MINB = 2; };

// unit u: segment, the unit's valid tile positions [lo, hi), its first tile
// position ub, the tile's buffers and whether its keys come by one bulk copy
template <class KT>
struct Mw8tUnit {
    uint32_t u, si, ub, lo, hi, begin, row0, nrows;
    bool tma;
    const typename KT::T *src;   // the buffer + the tile's first position
    typename KT::T *dst;
};
template <class KT>
__device__ __forceinline__ Mw8tUnit<KT> mw8t_unit(const MwParams<KT> &P, uint32_t u, uint32_t U) {
    constexpr uint32_t TILE = (uint32_t)tile_elems<KT>(), VW = tile_vw<KT>();
    const uint32_t lgU = __ffs(U) - 1, t = u >> lgU, UL = TILE >> lgU;   // (U: a power of two)
    Mw8tUnit<KT> w;
    w.u = u;
    w.ub = (u & (U - 1)) * UL;
    w.si = P.tile_map[t];
    const Seg sg = P.msegs[w.si].s;
    const TileGeom<KT, TILE> G(sg, t);
    w.lo = G.vlo > w.ub ? G.vlo : w.ub;
    w.hi = G.vhi < w.ub + UL ? G.vhi : w.ub + UL;
    w.begin = sg.begin;
    w.row0 = sg.tile_base * U;
    w.nrows = sg.ntiles * U;
    w.src = (sg.parity ? P.bufs[1] : P.bufs[0]) + G.tbeg;
    w.dst = sg.parity ? P.bufs[0] : P.bufs[1];
    if (w.hi <= w.lo) w.lo = w.hi = w.ub;   // a unit outside the segment
    w.tma = w.hi > w.lo && P.aligned && G.tbeg + (w.hi + VW - 1) / VW * VW <= P.n_total;
    return w;
}

// the keys of unit w into in[] (slot i = tile position ub + i): one bulk copy
// by lane 0 completing on bar, or plain loads by the warp
template <class KT>
__device__ __forceinline__ void mw8t_issue(const Mw8tUnit<KT> &w, typename KT::T *in, uint64_t *bar, uint32_t lane) {
    using T = typename KT::T;
    constexpr uint32_t VW = tile_vw<KT>();
    if (w.tma) {
        if (lane == 0) {
            const uint32_t a = w.lo / VW * VW, z = (w.hi + VW - 1) / VW * VW;
            const uint32_t bytes = (z - a) * (uint32_t)sizeof(T);
            constexpr uint32_t UNIT = (uint32_t)tile_elems<KT>() / mw8w_umin<KT>();
            BQ_CHECK(a >= w.ub && z - w.ub <= UNIT);
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(bar, bytes);
            tma_load_1d(in + (a - w.ub), w.src + a, bytes, bar);
        }
    } else {
        for (uint32_t p = w.lo + lane; p < w.hi; p += 32) in[p - w.ub] = w.src[p];
    }
}

__device__ __forceinline__ void sts_t(uint32_t a, uint32_t v) { sts32(a, v); }
__device__ __forceinline__ void sts_t(uint32_t a, int32_t v) { sts32(a, (uint32_t)v); }
__device__ __forceinline__ void sts_t(uint32_t a, uint64_t v) {
    asm volatile("st.shared.b64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ void sts_t(uint32_t a, const uint4 &v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
template <class T, class = typename std::enable_if<sizeof(T) == 16>::type>
__device__ __forceinline__ void sts_t(uint32_t a, const T &v) {   // (after the uint4 overload it calls)
    uint4 q;
    memcpy(&q, &v, 16);
    sts_t(a, q);
}

template <class KT, int IPT>
__global__ void __launch_bounds__(MW8W_WARPS * 32, Mw8tTune<KT>::MINB) k_mw8t_scatter(const MwParams<KT> Pin) {
    if (const LevelCtrl *pv = loop_prev_ctrl(Pin.lp)) if (pv->nmseg_next == 0) return;
    __shared__ MwParams<KT> sP;
    const MwParams<KT> &P = cta_params(Pin, sP);
    using T = typename KT::T;
    using WS = Mw8tWarpSmem<KT, IPT>;
    constexpr uint32_t RK = 32u * IPT, VW = tile_vw<KT>(), NV = IPT / VW;
    static_assert(IPT % VW == 0 && IPT <= 8 && WS::SCAP < 65536, "whole vectors; byte-field scans; 16-bit slots");
    extern __shared__ __align__(128) unsigned char smraw[];
    WS &ws = reinterpret_cast<WS *>(smraw)[threadIdx.x >> 5];
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nt = *P.ntiles_dev, U = mw8w_upt<KT>(nt), rows = nt * U;
    const uint32_t nblk = (rows + MWS_BR - 1) / MWS_BR;
    const uint32_t stride = gridDim.x * MW8W_WARPS;
    const uint32_t u0 = blockIdx.x * MW8W_WARPS + (threadIdx.x >> 5);
    if (u0 >= rows) return;
    if (lane == 0) {
        mbar_init(&ws.bar[0], 1);
        mbar_init(&ws.bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const uint32_t exrow = smem_u32(&ws.exs[lane]), stage0 = smem_u32(ws.stage);
    Mw8tUnit<KT> cur = mw8t_unit(P, u0, U);
    mw8t_issue<KT>(cur, ws.in[0], &ws.bar[0], lane);
    uint32_t par = 0, ph = 0, cls_seg = 0xffffffffu, seg_base = 0;
    bool stores_out = false;   // lanes 0..7: a bulk store of the stage may still read it
    Mw8Cls<KT> cls;
    // global prefix of table row r, lane b < 8: bucket b (as the two words
    // it sums, loaded a unit before they are added)
    // (every lane loads, lanes >= 8 the words of bucket 7, so no branch
    // divides the warp around the loads)
    const uint32_t lb7 = lane < MW8 ? lane : MW8 - 1;
    auto prefix2 = [&](uint32_t r) -> uint2 {
        return r < rows ? make_uint2(P.mtab[(size_t)r * MW8 + lb7], P.mblk[(size_t)(r / MWS_BR) * MW8 + lb7])
                        : make_uint2(P.mblk[(size_t)nblk * MW8 + lb7], 0u);
    };
    uint2 pu = prefix2(cur.u), pe = prefix2(cur.u + 1);   // global prefixes of the unit's row and the next row
    for (;;) {
        const bool more = cur.u + stride < rows;
        Mw8tUnit<KT> nxt = cur;
        uint2 pu_n = make_uint2(0, 0), pe_n = pu_n;
        if (more) {
            nxt = mw8t_unit(P, cur.u + stride, U);
            mw8t_issue<KT>(nxt, ws.in[par ^ 1], &ws.bar[par ^ 1], lane);
            pu_n = prefix2(nxt.u);   // (loaded a unit ahead)
            pe_n = prefix2(nxt.u + 1);
        }
        if (cur.si != cls_seg) {
            mw8w_load_cls<KT>(P, cur.si, cls);
            uint32_t tot, start, pf;
            mw8w_seg_buckets(P, cur.row0, cur.nrows, rows, lane, tot, start, pf);
            seg_base = cur.begin + start - pf;   // lane b: bucket b's output base minus its rows' prefix
            cls_seg = cur.si;
        }
        // lanes b < 8: the unit's run of bucket b: global start G, length nb,
        // stage slot S (S = G modulo VW)
        const uint32_t p0 = pu.x + pu.y;
        const uint32_t nb = lane < MW8 ? pe.x + pe.y - p0 : 0u, G = lane < MW8 ? seg_base + p0 : 0u;
        uint32_t S = nb + VW - 1;
#pragma unroll
        for (int d = 1; d < MW8; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, S, d);
            if (lane >= (uint32_t)d) S += o;
        }
        S -= nb + VW - 1;
        S += (G - S) & (VW - 1);
        BQ_CHECK(lane >= MW8 || (G + nb <= P.n_total && S + nb <= WS::SCAP));
        uint32_t cw[MW8 / 2];   // the lane's next slot of each bucket, 16-bit pairs
#pragma unroll
        for (int k = 0; k < MW8 / 2; k++)
            cw[k] = __shfl_sync(0xffffffffu, S, 2 * k) | (__shfl_sync(0xffffffffu, S, 2 * k + 1) << 16);
        if (cur.tma) {
            mbar_wait(&ws.bar[par], (ph >> par) & 1);
            ph ^= 1u << par;
        } else {
            __syncwarp();
        }
        const T *in = ws.in[par];
        const uint32_t lo = cur.lo - cur.ub, hi = cur.hi - cur.ub;
        for (uint32_t r0 = lo / RK * RK; r0 < hi; r0 += RK) {
            T x[IPT];
#pragma unroll
            for (uint32_t v = 0; v < NV; v++) {
                const uint4 q = *reinterpret_cast<const uint4 *>(in + r0 + v * 32 * VW + lane * VW);
                memcpy(&x[v * VW], &q, 16);
            }
            const bool full = r0 >= lo && r0 + RK <= hi;
            // (full rounds, the common case, skip every validity test)
            auto round = [&](auto full_tag) {
                constexpr bool FULL = decltype(full_tag)::value;
                uint32_t valid = (1u << IPT) - 1;
                if (!FULL) {
                    valid = 0;
#pragma unroll
                    for (uint32_t v = 0; v < NV; v++)
#pragma unroll
                        for (uint32_t e = 0; e < VW; e++) {
                            const uint32_t pos = r0 + v * 32 * VW + lane * VW + e;
                            valid |= (uint32_t)(pos >= lo && pos < hi) << (v * VW + e);
                        }
                }
                uint32_t b4[IPT], rk[IPT], ra[IPT];   // ra: the key's bucket entry of the lane's row
                {
                    bool nan = false;
#pragma unroll
                    for (int c = 0; c < IPT; c++) ra[c] = cls.a128(x[c], exrow, nan);
                    if (nan)
#pragma unroll
                        for (int c = 0; c < IPT; c++) ra[c] = exrow + 32u * cls.fix4(x[c], (ra[c] - exrow) >> 5);
                }
#pragma unroll
                for (int c = 0; c < IPT; c++) b4[c] = (ra[c] - exrow) >> 5;
                Mw8Ctr<IPT> ctr;
#pragma unroll
                for (int c = 0; c < IPT; c++) {
                    if (FULL) rk[c] = ctr.take4(b4[c]);
                    else rk[c] = ((valid >> c) & 1) ? ctr.take4(b4[c]) : 0u;
                }
                uint32_t ex[MW8 / 2], tot[MW8 / 2];
                mw8_scan<IPT>(ctr, lane, ex, tot);
#pragma unroll
                for (int k = 0; k < MW8 / 2; k++) {
                    tot[k] = __shfl_sync(0xffffffffu, tot[k], 31);
                    const uint32_t f = ex[k] + cw[k];   // this lane's first slots of buckets 2k, 2k+1
                    cw[k] += tot[k];
                    sts32(exrow + 256u * k, f & 0xffffu);
                    sts32(exrow + 256u * k + 128u, f >> 16);
                }
                if (stores_out) {   // the previous unit's bulk stores have read the stage
                    bulk_wait_read0();
                    stores_out = false;
                }
                __syncwarp();
                uint32_t slot[IPT];   // (every base load issued before the first store)
#pragma unroll
                for (int c = 0; c < IPT; c++) slot[c] = lds32(ra[c]) + rk[c];
#pragma unroll
                for (int c = 0; c < IPT; c++) {
                    if (FULL || ((valid >> c) & 1)) {
                        BQ_CHECK(slot[c] < WS::SCAP);
                        sts_t(stage0 + slot[c] * (uint32_t)sizeof(T), x[c]);
                    }
                }
            };
            if (full) round(std::true_type{});
            else round(std::false_type{});
        }
        // the unit's runs -> dst: aligned bodies by bulk copies (lanes 0..7),
        // heads and tails by plain stores (lane 4b + j: element j of bucket b's)
        fence_proxy_async_smem();
        __syncwarp();
        {
            const uint32_t b = lane >> 2, j = lane & 3;
            const uint32_t Gb = __shfl_sync(0xffffffffu, G, b), nbb = __shfl_sync(0xffffffffu, nb, b);
            const uint32_t Sb = __shfl_sync(0xffffffffu, S, b);
            const uint32_t e = Gb + nbb, gs = (Gb + VW - 1) / VW * VW, ge = e / VW * VW;
            const uint32_t hend = gs < e ? gs : e, tbeg = ge > hend ? ge : hend;
            if (VW > 1) {
                if (Gb + j < hend) cur.dst[Gb + j] = ws.stage[Sb + j];
                if (tbeg + j < e) cur.dst[tbeg + j] = ws.stage[Sb + (tbeg - Gb) + j];
            }
        }
        if (lane < MW8) {   // lane b: bucket b's body
            const uint32_t e = G + nb, gs = (G + VW - 1) / VW * VW, ge = e / VW * VW;
            if (ge > gs && gs < e) {
                BQ_CHECK(((S + (gs - G)) % VW) == 0 && ge <= P.n_total);
                tma_store_1d(cur.dst + gs, &ws.stage[S + (gs - G)], (ge - gs) * (uint32_t)sizeof(T));
                bulk_commit();
                stores_out = true;
            }
        }
        if (!more) break;
        __syncwarp();   // every lane is done with in[par] before it is refilled
        cur = nxt;
        pu = pu_n;
        pe = pe_n;
        par ^= 1;
    }
    if (lane < MW8) bulk_wait0();
}

}  // namespace bq
