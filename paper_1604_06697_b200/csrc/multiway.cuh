// multiway.cuh — SURVEY §8(f) N4: the multi-pivot block partition.
//
// The paper lists a multi-pivot BlockQuicksort as future work ("A three-pivot
// version might be interesting") and describes where many pivots
// lead: Super Scalar Sample Sort, whose bucket is found "by converting the
// results of comparisons to integers and then simply performing integer
// arithmetic".  On the GPU a k-way pass divides every segment by
// up to k = 16 in one read + one write, so a sort needs about
// log16(n/S) scatter passes (+ one read-only count pass each) instead of
// log2(n/S) binary ones.
//
// A multiway segment carries up to 15 splitters s_1 <= ... <= s_15, drawn as
// quantiles of a 256-key sample (jittered strata, R19), in an implicit search
// tree: tree[1] = s_8, tree[2..3] = s_4, s_12, ..., tree[8..15] = s_1, s_3, ...
// The bucket of key k is #{i : s_i < k}, found branch-free with four
// compare-and-shift steps (idx = 2*idx + (tree[idx] < k)).  Only segments whose
// real splitters are distinct (and below the sample's maximum) are split this
// way — every bucket is then a strict subset of the segment, so the recursion
// progresses; a segment whose sample shows duplicates goes to the binary
// three-way partition instead, whose equal band absorbs them.
//
// Per level:
//   k_mw_count    read-only pass: per-segment bucket histogram (warp ballots)
//   k_mw_scan     bucket starts = exclusive scan of the histogram
//   k_mw_scatter  the pass itself: classify, rank inside the warp with ballots
//                 and popcounts (the k-bucket analogue of the offset buffers),
//                 claim each bucket run's output with one atomicAdd per
//                 bucket and tile (consumed one tile later), stage the runs
//                 in shared memory aligned like their destinations, TMA bulk
//                 stores
//   k_post_mw     children: leaves, next-level multiway or binary segments
#pragma once

namespace bq {

constexpr int MW_K = 16;         // buckets of a multiway segment
// element types the multiway kernels move: keys, and the 16-byte key+index
// pairs (one element per 16-byte vector); 32-byte records stay binary
template <class KT>
constexpr bool mw_capable() { return !KT::is_record || sizeof(typename KT::T) == 16; }
#ifndef BQ_MW_FILL
#define BQ_MW_FILL 45
#endif
// Splitter sample keys per segment (NS / 32 per lane of one warp): 512 for
// int32 keys (c2: the narrower bucket spread leaves fewer leaves above half
// the leaf size, 6.54 -> 6.49 ms), 256 for the wider kinds (512 measured
// slower on c5).
#ifndef BQ_MW_SAMPLE
#define BQ_MW_SAMPLE 256
#endif
#ifndef BQ_MW_SAMPLE32
#define BQ_MW_SAMPLE32 512
#endif
constexpr int MW_SAMPLE = BQ_MW_SAMPLE;
template <class KT>
constexpr int mw_ns() { return std::is_same<KT, KI32>::value ? BQ_MW_SAMPLE32 : BQ_MW_SAMPLE; }
constexpr int mw_logs(int ns) { return ns == 256 ? 8 : ns == 512 ? 9 : 10; }
static_assert(mw_logs(BQ_MW_SAMPLE) <= 10 && mw_logs(BQ_MW_SAMPLE32) <= 10, "sample size");

template <class KT>
struct alignas(16) MSeg {
    Seg s;                          // begin, len, tile_base, ntiles, depth, parity (pivot unused)
    typename KT::K tree[MW_K];      // implicit search tree, tree[1..15]
    uint32_t start[MW_K];           // bucket starts relative to begin (k_mw_scan)
};

template <class KT>
__device__ __forceinline__ uint32_t mw_bucket(const typename KT::K *tree, typename KT::K k) {
    uint32_t idx = 1;
#pragma unroll
    for (int d = 0; d < 4; d++) idx = 2 * idx + (tree[idx] < k ? 1u : 0u);
    return idx - MW_K;
}

// position of sample key j of NS in [b, b+len): jittered strata (R19)
template <int NS>
__device__ __forceinline__ uint64_t mw_sample_pos(uint32_t b, uint32_t len, uint32_t j) {
    const uint64_t s0 = ((uint64_t)j * len) / NS, s1 = ((uint64_t)(j + 1) * len) / NS;
    const uint64_t r = splitmix64((((uint64_t)b << 32) | len) + (uint64_t)(j + 1) * 0x9E3779B97F4A7C15ull) >> 32;
    const uint64_t pos = s0 + ((r * (s1 - s0)) >> 32);
    return (uint64_t)b + (pos < len - 1 ? pos : len - 1);
}

// The NS sample keys of [b, b+len) sorted across one warp: index i =
// lane + 32 r is held by lane `lane` in v[r].  Bitonic network: register
// compare-exchanges for the index bits above 4, shuffles for bits 0-4.
template <class KT, int NS>
__device__ __forceinline__ void mw_sample_sorted(const typename KT::T *buf, uint32_t b, uint32_t len, uint32_t lane,
                                                 typename KT::K (&v)[NS / 32]) {
    using K = typename KT::K;
    constexpr int MW_SR = NS / 32, MW_LOGS = mw_logs(NS);
#pragma unroll
    for (int r = 0; r < MW_SR; r++) v[r] = load_key<KT>(buf, mw_sample_pos<NS>(b, len, lane + 32 * r));
#pragma unroll
    for (int m = 1; m <= MW_LOGS; m++) {
#pragma unroll
        for (int bb = m - 1; bb >= 0; bb--) {
            if (bb >= 5) {
                const int rb = bb - 5;
#pragma unroll
                for (int r = 0; r < MW_SR; r++) {
                    if (r & (1 << rb)) continue;
                    const int r2 = r | (1 << rb);
                    // direction of index bit m (a register bit for m >= 5, a lane bit below)
                    const bool asc = m == MW_LOGS || (m >= 5 ? ((r >> (m - 5)) & 1) == 0 : ((lane >> m) & 1) == 0);
                    const K lo = v[r2] < v[r] ? v[r2] : v[r], hi = v[r2] < v[r] ? v[r] : v[r2];
                    v[r] = asc ? lo : hi;
                    v[r2] = asc ? hi : lo;
                }
            } else {
#pragma unroll
                for (int r = 0; r < MW_SR; r++) {
                    const uint32_t i = lane + 32 * r;
                    const K p = __shfl_xor_sync(0xffffffffu, v[r], 1 << bb);
                    const bool lower = ((lane >> bb) & 1) == 0;
                    const bool asc = m == MW_LOGS || ((i >> m) & 1) == 0;
                    v[r] = (lower == asc) ? (p < v[r] ? p : v[r]) : (v[r] < p ? p : v[r]);
                }
            }
        }
    }
}

// sorted[q] of a warp-sorted sample, for a per-lane q (all lanes participate)
template <class K, int SR>
__device__ __forceinline__ K mw_pick(const K (&v)[SR], uint32_t q) {
    K out = v[0];
#pragma unroll
    for (int r = 0; r < SR; r++) {
        const K t = __shfl_sync(0xffffffffu, v[r], q & 31);
        out = (q >> 5) == (uint32_t)r ? t : out;
    }
    return out;
}

// Splitters for a segment of len keys (called by a whole warp).  Returns true
// (and the search tree, in lanes 1..15 for node = lane) when the segment is to
// be split multiway: k_eff = min(16, max(2, ceil(2 len / S))) buckets, real
// splitters at sample quantiles NS i / k_eff, pairwise distinct and below the
// sample maximum; the tree's unused slots repeat the last real splitter
// (empty buckets).  Otherwise returns false and `pivot` = the sample's lower
// median, for the binary three-way partition.
template <class KT>
__device__ bool mw_splitters(const typename KT::T *buf, uint32_t b, uint32_t len, uint32_t leaf_max, uint32_t lane,
                             typename KT::K &node_val, typename KT::K &pivot, uint32_t kmax = MW_K) {
    using K = typename KT::K;
    constexpr int NS = mw_ns<KT>();
    K v[NS / 32];
    mw_sample_sorted<KT, NS>(buf, b, len, lane, v);
    const uint64_t fl = (uint64_t)leaf_max * BQ_MW_FILL;   // buckets of about BQ_MW_FILL % of S
    uint64_t ke = ((uint64_t)len * 100 + fl - 1) / fl;
    const uint32_t keff = (uint32_t)(ke < 2 ? 2 : (ke > kmax ? kmax : ke));
    // lane i (1 <= i < keff) holds real splitter s_i; lanes i >= keff repeat s_{keff-1}
    const uint32_t i = lane < 1 ? 1 : (lane < keff ? lane : keff - 1);
    const K s = mw_pick(v, (i * NS) / keff);
    const K smax = __shfl_sync(0xffffffffu, v[NS / 32 - 1], 31);
    pivot = mw_pick(v, NS / 2 - 1);
    const K s_next = __shfl_down_sync(0xffffffffu, s, 1);
    const bool bad = (lane >= 1 && lane + 1 < keff && !(s < s_next)) || (lane == keff - 1 && !(s < smax));
    const bool ok = __ballot_sync(0xffffffffu, bad) == 0;
    // tree node `lane` (1..15) at depth d, position p holds s_{(2p+1) * 2^(3-d)}
    uint32_t si = 0;
    const uint32_t depth = kmax == MW_K ? 3 : 2;   // tree of kmax - 1 splitters
    if (lane >= 1 && lane < kmax) {
        const uint32_t d = 31 - __clz(lane);
        const uint32_t p = lane - (1u << d);
        si = (2 * p + 1) << (depth - d);
    }
    node_val = __shfl_sync(0xffffffffu, s, si);
    return ok;
}

// ---------------------------------------------------------------------------
template <class KT>
struct MwParams {
    using T = typename KT::T;
    T *bufs[2];
    MSeg<KT> *msegs;
    const uint32_t *tile_map;
    uint32_t *hist;      // [bucket * hstride + segment]
    uint32_t *cursor;    // [bucket * hstride + segment]
    uint32_t hstride;
    uint32_t *ticket;
    const uint32_t *nseg_dev;
    const uint32_t *ntiles_dev;
    uint64_t n_total;
    int aligned;
    LevelCtrl *ctrl;     // element-pass statistics
    LoopPtrs<KT> lp;     // lp.level != nullptr: the current level's lists (partition.cuh)
    int ticket_sel;      // loop: 0 = the count kernel's ticket, 1 = the scatter kernel's
    uint32_t *mtab;      // 8-way (multiway8w.cuh): per-tile bucket counts, then their prefix
    uint32_t *mblk;      // 8-way: per-block totals, then block prefixes
    uint32_t max_tiles;  // rows of mtab
    int tabmode;         // 8-way levels by multiway8w.cuh: children from mtab / mblk
};

template <class KT>
__device__ __forceinline__ void loop_resolve(MwParams<KT> &P) {
    if (!P.lp.level) return;
    const uint32_t lv = *P.lp.level, cp = lv & 1;
    const LevelCtrl *prev = loop_prev(P.lp, lv);
    P.msegs = static_cast<MSeg<KT> *>(P.lp.msegs[cp]);
    P.tile_map = P.lp.mtile_map[cp];
    P.hist = P.lp.mhist[cp];
    P.cursor = P.lp.mcursor[cp];
    P.nseg_dev = &prev->nmseg_next;
    P.ntiles_dev = &prev->nmtiles_next;
    P.ctrl = P.lp.ctrl + lv;
    P.ticket = P.ticket_sel ? &P.ctrl->mw_ticket_scatter : &P.ctrl->mw_ticket_count;
}

template <class KT, int NT, int IPT, int STAGES>
struct MwSmem {
    using T = typename KT::T;
    using K = typename KT::K;
    static constexpr int TILE = NT * IPT;
    static constexpr int NW = NT / 32;
    alignas(128) T in[STAGES][TILE];
    alignas(128) T out[TILE + MW_K * 8 + 16];   // runs + per-run alignment slack
    K tree[STAGES][MW_K];
    uint32_t start[STAGES][MW_K];
    uint32_t sb[STAGES], slen[STAGES], stb[STAGES], spar[STAGES], sidx[STAGES], tile[STAGES], manual[STAGES];
    uint64_t full[STAGES];
    uint64_t empty[STAGES];
    // per-thread bucket counters, bucket-major (entry b*NT + t): thread t only
    // touches its own column, so every access is free of bank conflicts; by
    // iteration parity
    uint32_t cnt_m[1][MW_K * NT];
    uint32_t wtot[2][NW][MW_K / 2];   // per-warp bucket totals, two 16-bit fields per word
    uint32_t wpre[2][NW][MW_K / 2];   // exclusive prefix of the warps' totals, packed likewise
    uint32_t boff[2][MW_K + 1];       // bucket starts inside the tile (boff[16] = valid keys)
    uint32_t delta[2][MW_K];       // staging shift per bucket (shifted start - unshifted start)
    uint32_t gstart[2][MW_K];      // global start of each run (low 32 bits of the element index)
    uint32_t cnt[2][MW_K];         // run lengths
    uint32_t sh[2][MW_K];          // shifted staging start of each run
};

#ifndef BQ_MW_STAGES
#define BQ_MW_STAGES 3
#endif
#ifndef BQ_MW_CHUNK
#define BQ_MW_CHUNK 4
#endif
constexpr int MW_STAGES = BQ_MW_STAGES;   // TMA ring depth of the multiway kernels (2 CTAs per SM)
constexpr uint32_t MW_CHUNK = BQ_MW_CHUNK;   // consecutive tiles per loader ticket

template <class KT>
constexpr int mw_smem_bytes() {
    return (int)sizeof(MwSmem<KT, Tune<KT>::PART_THREADS, Tune<KT>::PART_IPT, MW_STAGES>);
}

// a thread's 16 bucket counters (its matrix column), packed two per word
template <int NT>
__device__ __forceinline__ void mw_read_column(const uint32_t *C, uint32_t tid, uint32_t (&q)[MW_K / 2]) {
#pragma unroll
    for (int k = 0; k < MW_K / 2; k++) q[k] = C[(2 * k) * NT + tid] | (C[(2 * k + 1) * NT + tid] << 16);
}
// inclusive scan of packed counters over the lanes of a warp
__device__ __forceinline__ void mw_warp_scan(uint32_t (&q)[MW_K / 2], uint32_t lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
        for (int k = 0; k < MW_K / 2; k++) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, q[k], d);
            if (lane >= (uint32_t)d) q[k] += o;
        }
    }
}

// a splitter as the 8-way kernels compare it: float64 as the double's bits
// (compared as doubles, R25), every other kind as its key
template <class KT>
__device__ __forceinline__ typename KT::K mw8_tree_word(typename KT::K k) {
    if constexpr (std::is_same<KT, KF64>::value) return KF64::from_key(k);
    else return k;
}

// loader warp shared by the count and the scatter kernel: claims tiles in order,
// copies the segment's metadata into the stage and issues the TMA bulk load
template <class KT, int NT, int IPT, int STAGES, class SM>
__device__ __forceinline__ void mw_loader(const MwParams<KT> &P, SM &sm, uint32_t ntiles, bool need_start,
                                          bool decode = false) {
    constexpr uint32_t CHUNK = MW_CHUNK;
    using T = typename KT::T;
    constexpr uint32_t TILE = NT * IPT;
    constexpr uint32_t W = sizeof(T), VW = 16 / W;
    // a ticket is a chunk of CHUNK consecutive tiles (mostly of one segment:
    // the count kernel's per-segment accumulators flush rarely), the next
    // one claimed a chunk ahead (as in k_part_fast's loader); the next tile's
    // segment index is loaded one tile ahead, and a tile of the same segment
    // as the previous one copies that stage's metadata instead of reloading
    uint32_t c_next = atomicAdd(P.ticket, 1u) * CHUNK, j = 0;
    auto claim = [&]() -> uint32_t {
        const uint32_t t = c_next + j;
        if (++j == CHUNK || t + 1 >= ntiles) {
            if (t < ntiles) c_next = atomicAdd(P.ticket, 1u) * CHUNK;
            j = 0;
        }
        return t;
    };
    uint32_t t = claim();
    uint32_t si = t < ntiles ? P.tile_map[t] : 0, prev_si = 0xffffffffu;
    for (uint32_t i = 0;; i++) {
        const uint32_t s = i % STAGES, ps = (i + STAGES - 1) % STAGES;
        const uint32_t tn = t < ntiles ? claim() : ntiles;
        const uint32_t sin = tn < ntiles ? P.tile_map[tn] : 0;
        mbar_wait(&sm.empty[s], ((i / STAGES) & 1) ^ 1);
        sm.tile[s] = t;
        if (t >= ntiles) {
            mbar_arrive(&sm.full[s]);
            break;
        }
        Seg sg;
        if (si == prev_si) {
#pragma unroll
            for (int q = 1; q < MW_K; q++) sm.tree[s][q] = sm.tree[ps][q];
            if (need_start)
#pragma unroll
                for (int q = 0; q < MW_K; q++) sm.start[s][q] = sm.start[ps][q];
            sg.begin = sm.sb[ps];
            sg.len = sm.slen[ps];
            sg.tile_base = sm.stb[ps];
            sg.parity = (uint8_t)sm.spar[ps];
        } else {
            const MSeg<KT> &ms = P.msegs[si];
            sg = ms.s;
            if (decode)   // the 8-way kernels: float64 splitters as the doubles' bits (mw8_tree_word)
#pragma unroll
                for (int q = 1; q < MW_K; q++) sm.tree[s][q] = mw8_tree_word<KT>(ms.tree[q]);
            else
#pragma unroll
                for (int q = 1; q < MW_K; q++) sm.tree[s][q] = ms.tree[q];
            if (need_start)
#pragma unroll
                for (int q = 0; q < MW_K; q++) sm.start[s][q] = ms.start[q];
        }
        prev_si = si;
        sm.sb[s] = sg.begin;
        sm.slen[s] = sg.len;
        sm.stb[s] = sg.tile_base;
        sm.spar[s] = sg.parity;
        sm.sidx[s] = si;
        const TileGeom<KT, TILE> G(sg, t);
        const uint64_t lo16 = (G.tbeg + G.vlo) / VW * VW;
        const uint64_t hi16 = (G.tbeg + G.vhi + VW - 1) / VW * VW;
        const T *src = sg.parity ? P.bufs[1] : P.bufs[0];
        const bool tma = P.aligned && hi16 <= P.n_total;
        sm.manual[s] = !tma;
        if (tma) {
            const uint32_t bytes = (uint32_t)((hi16 - lo16) * W);
            mbar_arrive_expect_tx(&sm.full[s], bytes);
            tma_load_1d(&sm.in[s][lo16 - G.tbeg], src + lo16, bytes, &sm.full[s]);
        } else {
            mbar_arrive(&sm.full[s]);
        }
        t = tn;
        si = sin;
    }
}

// a consumer's IPT keys of stage s (conflict-free permuted 16-byte vectors),
// their buckets, and a validity mask (bit c) for partial tiles
template <class KT, int NT, int IPT, int STAGES>
__device__ __forceinline__ uint32_t mw_load_classify(const MwParams<KT> &P, MwSmem<KT, NT, IPT, STAGES> &sm,
                                                     uint32_t s, uint32_t t, uint32_t lane, uint32_t tid,
                                                     typename KT::T (&x)[IPT], uint32_t (&bk)[IPT]) {
    using T = typename KT::T;
    using K = typename KT::K;
    constexpr uint32_t TILE = NT * IPT;
    constexpr uint32_t W = sizeof(T), VW = 16 / W, NV4 = IPT / VW;
    const uint32_t sw = NV4 > 1 ? ((lane * NV4) / 8) & (NV4 - 1) : 0;
    const uint32_t e0 = tid * IPT;
    Seg sg;
    sg.begin = sm.sb[s];
    sg.len = sm.slen[s];
    sg.tile_base = sm.stb[s];
    const TileGeom<KT, TILE> G(sg, t);
    uint32_t valid = (1u << IPT) - 1;
    if (!sm.manual[s]) {
        const uint4 *in4 = reinterpret_cast<const uint4 *>(&sm.in[s][e0]);
#pragma unroll
        for (uint32_t k = 0; k < NV4; k++) {
            const uint4 v = in4[k ^ sw];
            memcpy(&x[k * VW], &v, 16);
        }
    } else {
        const T *src = sm.spar[s] ? P.bufs[1] : P.bufs[0];
#pragma unroll
        for (uint32_t k = 0; k < NV4; k++)
#pragma unroll
            for (uint32_t j = 0; j < VW; j++) {
                const uint32_t pos = e0 + (k ^ sw) * VW + j;
                x[k * VW + j] = (pos >= G.vlo && pos < G.vhi) ? src[G.tbeg + pos] : T{};
            }
    }
    if (G.vlo != 0 || G.vhi != TILE) {
        valid = 0;
#pragma unroll
        for (uint32_t k = 0; k < NV4; k++)
#pragma unroll
            for (uint32_t j = 0; j < VW; j++) {
                const uint32_t pos = e0 + (k ^ sw) * VW + j;
                valid |= (uint32_t)(pos >= G.vlo && pos < G.vhi) << (k * VW + j);
            }
    }
    const K *tree = sm.tree[s];
#pragma unroll
    for (uint32_t c = 0; c < IPT; c++) bk[c] = mw_bucket<KT>(tree, KT::key(x[c]));
    return valid;
}

// lanes' bucket masks of one key slot across the warp: bit l of the result is
// set iff lane l's key (in this slot, valid) is in bucket `b`
__device__ __forceinline__ uint32_t mw_match(uint32_t v0, uint32_t v1, uint32_t v2, uint32_t v3, uint32_t vm,
                                             uint32_t b) {
    const uint32_t m0 = (b & 1) ? v0 : ~v0, m1 = (b & 2) ? v1 : ~v1;
    const uint32_t m2 = (b & 4) ? v2 : ~v2, m3 = (b & 8) ? v3 : ~v3;
    return m0 & m1 & m2 & m3 & vm;
}

// ---- k_mw_count ---------------------------------------------------------------
// Per tile: every thread counts its keys' buckets in its column of the counter
// matrix (one LDS + STS per key), then the 16 threads of each bucket's row
// chunk reduce it and one of them adds the tile's count to the segment's
// histogram.
template <class KT, int NT, int IPT, int STAGES, int MINB>
__global__ void __launch_bounds__(NT + 32, MINB) k_mw_count(const MwParams<KT> Pin) {
    if (const LevelCtrl *pv = loop_prev_ctrl(Pin.lp)) if (pv->nmseg_next == 0) return;
    __shared__ MwParams<KT> sP;
    const MwParams<KT> &P = cta_params(Pin, sP);
    using SM = MwSmem<KT, NT, IPT, STAGES>;
    constexpr uint32_t NW = SM::NW;
    static_assert(NT == MW_K * MW_K, "one 16-thread chunk per bucket row");
    extern __shared__ __align__(128) unsigned char smraw[];
    SM &sm = *reinterpret_cast<SM *>(smraw);
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t ntiles = *P.ntiles_dev;
    if (tid == 0) {
        for (int s = 0; s < STAGES; s++) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async_smem();
    }
    __syncthreads();
    if (warp == NW) {
        if (lane == 0) mw_loader<KT, NT, IPT, STAGES, SM>(P, sm, ntiles, false);
        return;
    }
    // lane L < 16 accumulates this warp's count of bucket L for segment cur_seg
    uint32_t acc = 0, cur_seg = 0xffffffffu;
    uint32_t *C = sm.cnt_m[0];   // (columns are private: one matrix suffices)
    for (uint32_t i = 0;; i++) {
        const uint32_t s = i % STAGES;
        mbar_wait(&sm.full[s], (i / STAGES) & 1);
        const uint32_t t = sm.tile[s];
        if (t >= ntiles) break;
        const uint32_t si = sm.sidx[s];
#pragma unroll
        for (uint32_t b = 0; b < MW_K; b++) C[b * NT + tid] = 0;
        typename KT::T x[IPT];
        uint32_t bk[IPT];
        const uint32_t valid = mw_load_classify<KT, NT, IPT, STAGES>(P, sm, s, t, lane, tid, x, bk);
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[s]);
#pragma unroll
        for (uint32_t c = 0; c < IPT; c++) {
            uint32_t *cp = &C[bk[c] * NT + tid];
            if ((valid >> c) & 1) *cp = *cp + 1;
        }
        uint32_t q[MW_K / 2];
        mw_read_column<NT>(C, tid, q);
#pragma unroll
        for (int d = 16; d > 0; d >>= 1)
#pragma unroll
            for (int k = 0; k < MW_K / 2; k++) q[k] += __shfl_xor_sync(0xffffffffu, q[k], d);
        if (si != cur_seg) {
            if (cur_seg != 0xffffffffu && lane < MW_K && acc) atomicAdd(&P.hist[lane * P.hstride + cur_seg], acc);
            acc = 0;
            cur_seg = si;
        }
        uint32_t mine = 0;
#pragma unroll
        for (int k = 0; k < MW_K / 2; k++) mine = (lane >> 1) == (uint32_t)k ? q[k] : mine;
        acc += (lane & 1) ? (mine >> 16) : (mine & 0xffff);
    }
    if (cur_seg != 0xffffffffu && lane < MW_K && acc) atomicAdd(&P.hist[lane * P.hstride + cur_seg], acc);
}

// ---- k_mw_scan: bucket starts and cursor reset, one warp per segment ---------------
template <class KT>
__global__ void k_mw_scan(const MwParams<KT> Pin) {
    if (const LevelCtrl *pv = loop_prev_ctrl(Pin.lp)) if (pv->nmseg_next == 0) return;
    __shared__ MwParams<KT> sP;
    const MwParams<KT> &P = cta_params(Pin, sP);
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nseg = *P.nseg_dev;
    for (uint32_t si = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); si < nseg;
         si += gridDim.x * (blockDim.x / 32)) {
        const uint32_t h = lane < MW_K ? P.hist[lane * P.hstride + si] : 0;
        uint32_t inc = h;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= (uint32_t)d) inc += o;
        }
        if (lane < MW_K) {
            P.msegs[si].start[lane] = inc - h;
            P.cursor[lane * P.hstride + si] = 0;
        }
        if (lane == 31) atomicAdd(&P.ctrl->mw_element_passes, (unsigned long long)inc);
    }
}

// ---- k_mw_scatter -------------------------------------------------------------
template <class KT, int NT, int IPT, int STAGES, int MINB>
__global__ void __launch_bounds__(NT + 32, MINB) k_mw_scatter(const MwParams<KT> Pin) {
    if (const LevelCtrl *pv = loop_prev_ctrl(Pin.lp)) if (pv->nmseg_next == 0) return;
    __shared__ MwParams<KT> sP;
    const MwParams<KT> &P = cta_params(Pin, sP);
    using T = typename KT::T;
    using SM = MwSmem<KT, NT, IPT, STAGES>;
    constexpr uint32_t NW = SM::NW;
    constexpr uint32_t W = sizeof(T), VW = 16 / W;
    static_assert(IPT <= 16 && NT == MW_K * MW_K, "packed ranks, one 16-thread chunk per bucket row");
    extern __shared__ __align__(128) unsigned char smraw[];
    SM &sm = *reinterpret_cast<SM *>(smraw);
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t ntiles = *P.ntiles_dev;
    if (tid == 0) {
        for (int s = 0; s < STAGES; s++) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async_smem();
    }
    __syncthreads();
    if (warp == NW) {
        if (lane == 0) mw_loader<KT, NT, IPT, STAGES, SM>(P, sm, ntiles, true);
        return;
    }

    // previous tile, carried one iteration: keys and (tile offset | bucket << 16 | invalid << 31)
    T y[IPT];
    uint32_t ypk[IPT];
    bool have_prev = false;
    T *p_dst = nullptr;
    // warp 0, lane L < 16: the previous tile's bucket-L run (atomic result, length, tile offset, base)
    uint32_t p_old = 0, p_cnt = 0, p_off = 0;
    uint64_t p_base = 0;

    for (uint32_t i = 0;; i++) {
        const uint32_t s = i % STAGES, par = i & 1;
        mbar_wait(&sm.full[s], (i / STAGES) & 1);
        const uint32_t t = sm.tile[s];
        const bool cur = t < ntiles;
        uint32_t *C = sm.cnt_m[0];   // thread tid only ever touches its own column
        T x[IPT];
        uint32_t pk[IPT];
        uint32_t q[MW_K / 2], own[MW_K / 2];
        uint32_t si = 0, sbeg = 0, spar = 0, bstart = 0;
        if (cur) {
            si = sm.sidx[s];
            sbeg = sm.sb[s];
            spar = sm.spar[s];
            bstart = lane < MW_K ? sm.start[s][lane] : 0;
#pragma unroll
            for (uint32_t b = 0; b < MW_K; b++) C[b * NT + tid] = 0;
            const uint32_t valid = mw_load_classify<KT, NT, IPT, STAGES>(P, sm, s, t, lane, tid, x, pk);
            // the k-bucket offset buffers: rank of each key among this thread's
            // keys of its bucket (counter in the thread's matrix column)
#pragma unroll
            for (uint32_t c = 0; c < IPT; c++) {
                const uint32_t b = pk[c];
                uint32_t *cp = &C[b * NT + tid];
                const bool v = (valid >> c) & 1;
                const uint32_t r = *cp;
                if (v) *cp = r + 1;
                pk[c] = r | (b << 16) | ((uint32_t)!v << 31);
            }
            // per-bucket scan over the threads: warp part (packed 16-bit counters)
            mw_read_column<NT>(C, tid, q);
#pragma unroll
            for (int k = 0; k < MW_K / 2; k++) own[k] = q[k];
            mw_warp_scan(q, lane);
            if (lane == 31)
#pragma unroll
                for (int k = 0; k < MW_K / 2; k++) sm.wtot[par][warp][k] = q[k];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[s]);

        // warp 0: placement of the previous tile's runs, now that its atomics returned
        if (warp == 0 && have_prev) {
            const uint32_t L = lane;
            const uint64_t g = p_base + p_old;                       // global start of run L
            const uint32_t a = (uint32_t)(g % VW);
            const uint32_t padded = L < MW_K ? (a + p_cnt + VW - 1) / VW * VW : 0;
            uint32_t inc = padded;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= (uint32_t)d) inc += o;
            }
            if (L < MW_K) {
                const uint32_t shs = inc - padded + a;             // shifted staging start
                sm.delta[par ^ 1][L] = shs - p_off;
                sm.sh[par ^ 1][L] = shs;
                sm.gstart[par ^ 1][L] = (uint32_t)g;
                sm.cnt[par ^ 1][L] = p_cnt;
            }
        }
        if (tid < MW_K) bulk_wait_read0();   // the previous bulk stores (one group per run) have read `out`
        named_bar_sync(1, NT);               // B1: warp totals and placement visible, `out` free

        if (cur && warp == 0) {
            // cross-warp part: lane k < 8 runs over the warps for packed pair k
            if (lane < MW_K / 2) {
                uint32_t run = 0;
#pragma unroll
                for (uint32_t w2 = 0; w2 < NW; w2++) {
                    sm.wpre[par][w2][lane] = run;
                    run += sm.wtot[par][w2][lane];
                }
                // bucket totals -> bucket starts inside the tile (scan over the 16 fields)
                const uint32_t lo = run & 0xffff, hi = run >> 16;
                uint32_t pair = lo + hi, incp = pair;
#pragma unroll
                for (int d = 1; d < 8; d <<= 1) {
                    const uint32_t o = __shfl_up_sync(0x000000ffu, incp, d);
                    if (lane >= (uint32_t)d) incp += o;
                }
                const uint32_t ex = incp - pair;
                sm.boff[par][2 * lane] = ex;
                sm.boff[par][2 * lane + 1] = ex + lo;
                if (lane == MW_K / 2 - 1) sm.boff[par][MW_K] = incp;
            }
        }
        if (have_prev) {
            // stage the previous tile's runs aligned like their destinations
#pragma unroll
            for (uint32_t c = 0; c < IPT; c++) {
                const uint32_t v = ypk[c];
                BQ_CHECK((v >> 31) || (v & 0xffff) + sm.delta[par ^ 1][(v >> 16) & 0x7fff] < SM::TILE + MW_K * 8 + 16);
                if (!(v >> 31)) sm.out[(v & 0xffff) + sm.delta[par ^ 1][(v >> 16) & 0x7fff]] = y[c];
            }
            if (P.aligned) fence_proxy_async_smem();
        }
        named_bar_sync(1, NT);   // B2: prefixes visible, staging complete

        if (have_prev) {
            T *d = p_dst;
            if (!P.aligned) {
                for (uint32_t L = 0; L < MW_K; L++) {
                    const uint32_t n = sm.cnt[par ^ 1][L];
                    const uint64_t g = (uint64_t)sm.gstart[par ^ 1][L];
                    for (uint32_t qq = tid; qq < n; qq += NT) d[g + qq] = sm.out[sm.sh[par ^ 1][L] + qq];
                }
            } else if (tid < MW_K) {
                const uint32_t L = tid, n = sm.cnt[par ^ 1][L];
                const uint64_t g = sm.gstart[par ^ 1][L], ge = g + n;
                const uint64_t bs = (g + VW - 1) / VW * VW, be = ge / VW * VW;
                if (n && be > bs) tma_store_1d(d + bs, &sm.out[sm.sh[par ^ 1][L] + (bs - g)], (uint32_t)((be - bs) * W));
                bulk_commit();
            } else if (tid >= 32 && tid < 32 + MW_K * 2 * VW) {
                // heads and tails (< 16 bytes) of every run
                const uint32_t u = tid - 32, L = u / (2 * VW), qv = u % (2 * VW);
                const uint32_t n = sm.cnt[par ^ 1][L];
                const uint64_t g = sm.gstart[par ^ 1][L], ge = g + n;
                const uint64_t bs = (g + VW - 1) / VW * VW, be = ge / VW * VW;
                const bool tail = qv >= VW;
                const uint32_t qq = tail ? qv - VW : qv;
                const uint64_t pos = tail ? (be > bs ? be : bs) + qq : g + qq;
                const bool ok = n && (tail ? (ge > bs && pos < ge) : (pos < (bs < ge ? bs : ge)));
                if (ok) d[pos] = sm.out[sm.sh[par ^ 1][L] + (pos - g)];
            }
        }
        if (!cur) break;

        // every key's offset in the tile: bucket start + the preceding warps' and
        // lanes' keys of its bucket + its rank in this thread
        {
#pragma unroll
            for (int k = 0; k < MW_K / 2; k++) {
                const uint32_t ex = q[k] - own[k] + sm.wpre[par][warp][k];   // exclusive, packed
                C[(2 * k) * NT + tid] = (ex & 0xffff) + sm.boff[par][2 * k];
                C[(2 * k + 1) * NT + tid] = (ex >> 16) + sm.boff[par][2 * k + 1];
            }
#pragma unroll
            for (uint32_t c = 0; c < IPT; c++) {
                const uint32_t b = (pk[c] >> 16) & 0x7fff;
                pk[c] += C[b * NT + tid];
            }
        }
        if (warp == 0) {
            // claim this tile's runs: one atomic per bucket, consumed next iteration
            const uint32_t st = lane < MW_K ? sm.boff[par][lane] : 0;
            const uint32_t tot = lane < MW_K ? sm.boff[par][lane + 1] - st : 0;
            p_old = (lane < MW_K && tot) ? atomicAdd(&P.cursor[lane * P.hstride + si], tot) : 0;
            p_cnt = tot;
            p_off = st;
            p_base = (uint64_t)sbeg + bstart;
        }
#pragma unroll
        for (uint32_t c = 0; c < IPT; c++) {
            y[c] = x[c];
            ypk[c] = pk[c];
        }
        have_prev = true;
        p_dst = spar ? P.bufs[0] : P.bufs[1];
    }
    if (tid < MW_K) bulk_wait0();
}

}  // namespace bq
