// multiway8.cuh — the 8-way variant of the multi-pivot block partition (N4),
// sized so that every per-key step stays in registers.
//
// Segment metadata, splitter choice, bucket scan and children are shared with
// the 16-way form (multiway.cuh: MSeg, mw_splitters(kmax = 8), k_mw_scan,
// k_post_mw); the tree uses nodes 1..7: tree[1] = s_4, tree[2..3] = s_2, s_6,
// tree[4..7] = s_1, s_3, s_5, s_7.
//   classify  the 7 splitters of the tile's segment are read once per tile
//             into registers; a key's bucket (#{s_i < k}) is three compares
//             with register selects in between — the paper's "converting the
//             results of comparisons to integers";
//   rank      each thread keeps 8-bit counters of its keys' buckets in one
//             64-bit register (<= 16 keys per thread): rank = field b, then
//             field b += 1 — the k-bucket form of the offset buffers and
//             their branch-free counters (Alg. 3 l.8-9);
//   scan      the counters, widened to 16-bit pairs, are scanned over the
//             warp with shuffles and over the warps through shared memory;
//   place     one atomicAdd per bucket and tile claims the runs (consumed one
//             tile later), runs staged aligned like their destinations, TMA
//             bulk stores.
#pragma once

namespace bq {

constexpr int MW8 = 8;

template <class KT, int NT, int IPT, int STAGES>
struct Mw8Smem {
    using T = typename KT::T;
    using K = typename KT::K;
    static constexpr int TILE = NT * IPT;
    static constexpr int NW = NT / 32;
    alignas(128) T in[STAGES][TILE];
    alignas(128) T out[TILE + MW8 * 8 + 16];
    K tree[STAGES][MW_K];
    uint32_t start[STAGES][MW_K];
    uint32_t sb[STAGES], slen[STAGES], stb[STAGES], spar[STAGES], sidx[STAGES], tile[STAGES], manual[STAGES];
    uint64_t full[STAGES];
    uint64_t empty[STAGES];
    uint32_t wtot[2][NW][MW8 / 2];   // per-warp bucket totals, 16-bit pairs
    uint32_t wpre[2][NW][MW8 / 2];   // exclusive prefix over the warps, packed likewise
    uint32_t boff[2][MW8 + 1];       // bucket starts inside the tile
    uint32_t delta[2][MW8], gstart[2][MW8], cnt[2][MW8], sh[2][MW8];
};

template <class KT>
constexpr int mw8_smem_bytes() {
    return (int)sizeof(Mw8Smem<KT, Tune<KT>::PART_THREADS, Tune<KT>::PART_IPT, MW_STAGES>);
}

// the keys of stage s for this thread (permuted conflict-free vectors) and
// their validity mask
template <class KT, int NT, int IPT, int STAGES, class SM>
__device__ __forceinline__ uint32_t mw8_load(const MwParams<KT> &P, SM &sm, uint32_t s, uint32_t t, uint32_t lane,
                                             uint32_t tid, typename KT::T (&x)[IPT]) {
    using T = typename KT::T;
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
    return valid;
}

// bucket of key k: #{s_i < k} over the register-resident tree t[1..7]
template <class K>
__device__ __forceinline__ uint32_t mw8_bucket(const K (&tr)[MW8], K k) {
    const bool p0 = tr[1] < k;
    const K n1 = p0 ? tr[3] : tr[2];
    const bool p1 = n1 < k;
    const K lo = p1 ? tr[5] : tr[4], hi = p1 ? tr[7] : tr[6];
    const K n2 = p0 ? hi : lo;
    const bool p2 = n2 < k;
    return ((uint32_t)p0 << 2) | ((uint32_t)p1 << 1) | (uint32_t)p2;
}

// base + 4 x the bucket of key k, the offset added by predicated adds (the
// FMA pipe) instead of built from the predicates on the ALU pipe
template <class K, uint32_t M = 1>
__device__ __forceinline__ uint32_t mw8_a4(const K (&tr)[MW8], K k, uint32_t base) {
    const bool p0 = tr[1] < k;
    const K n1 = p0 ? tr[3] : tr[2];
    const K c1 = p0 ? tr[7] : tr[5], c0 = p0 ? tr[6] : tr[4];
    uint32_t a = p0 ? base + 16u * M : base;
    const bool p1 = n1 < k;
    const K n2 = p1 ? c1 : c0;
    if (p1) a += 8u * M;
    const bool p2 = n2 < k;
    if (p2) a += 4u * M;
    return a;
}
// The classification of one key against the tile's splitters.  float64 keys
// are compared as doubles (DSETP, the FP64 pipe) against the splitters the
// loader decoded (mw8_tree_word): for non-NaN values the double order is the
// totalOrder with -0.0 and +0.0 merged, so #{s_i < k} still cuts the segment
// into contiguous ranges of the total order (both zeros always share a
// bucket; R25) and no key is encoded.  NaN keys (outside the
// contract) are only detected per key (one predicate OR); a thread that saw
// one re-classifies its keys with fix().  Other kinds compare their keys.
template <class KT>
struct Mw8Cls {
    using K = typename KT::K;
    K tr[MW8];
    __device__ __forceinline__ void load(const K *tree) {
#pragma unroll
        for (int q = 1; q < MW8; q++) tr[q] = tree[q];
    }
    __device__ __forceinline__ uint32_t bucket(const typename KT::T &x, bool &) const {
        return mw8_bucket(tr, KT::key(x));
    }
    __device__ __forceinline__ uint32_t fix(const typename KT::T &, uint32_t b) const { return b; }
    __device__ __forceinline__ uint32_t fix4(const typename KT::T &, uint32_t b4) const { return b4; }
    __device__ __forceinline__ uint32_t a128(const typename KT::T &x, uint32_t base, bool &) const {
        return mw8_a4<typename KT::K, 32>(tr, KT::key(x), base);
    }
};
template <>
struct Mw8Cls<KF64> {
    double tr[MW8];
    __device__ __forceinline__ void load(const uint64_t *tree) {
#pragma unroll
        for (int q = 1; q < MW8; q++) tr[q] = __longlong_as_double((long long)tree[q]);
    }
    __device__ __forceinline__ uint32_t bucket(const uint64_t &x, bool &nan) const {
        const double d = __longlong_as_double((long long)x);
        nan |= d != d;
        return mw8_bucket(tr, d);
    }
    // NaN keys keep their bit-pattern place: -NaN before every other key,
    // +NaN after (R9); a NaN splitter only merges two adjacent buckets (its
    // compares are constant)
    __device__ __forceinline__ uint32_t fix(const uint64_t &x, uint32_t b) const {
        const double d = __longlong_as_double((long long)x);
        return d != d ? ((x >> 63) ? 0u : MW8 - 1u) : b;
    }
    __device__ __forceinline__ uint32_t fix4(const uint64_t &x, uint32_t b4) const {
        const double d = __longlong_as_double((long long)x);
        return d != d ? ((x >> 63) ? 0u : 4u * (MW8 - 1u)) : b4;
    }
    __device__ __forceinline__ uint32_t a128(const uint64_t &x, uint32_t base, bool &nan) const {
        const double d = __longlong_as_double((long long)x);
        nan |= d != d;
        return mw8_a4<double, 32>(tr, d, base);
    }
};

// the buckets of a thread's IPT keys (bk[c]), NaN fix-up included
template <class KT, int IPT>
__device__ __forceinline__ void mw8_classify(const Mw8Cls<KT> &cls, const typename KT::T (&x)[IPT],
                                             uint32_t (&bk)[IPT]) {
    bool nan = false;
#pragma unroll
    for (int c = 0; c < IPT; c++) bk[c] = cls.bucket(x[c], nan);
    if (nan)
#pragma unroll
        for (int c = 0; c < IPT; c++) bk[c] = cls.fix(x[c], bk[c]);
}

// 8 counters of 8 bits -> 4 words of two 16-bit counters
__device__ __forceinline__ void mw8_widen(uint64_t c, uint32_t (&q)[MW8 / 2]) {
    const uint32_t lo = (uint32_t)c, hi = (uint32_t)(c >> 32);
    q[0] = __byte_perm(lo, 0, 0x4140);   // bytes 0, 1 -> 16-bit fields
    q[1] = __byte_perm(lo, 0, 0x4342);
    q[2] = __byte_perm(hi, 0, 0x4140);
    q[3] = __byte_perm(hi, 0, 0x4342);
}

// four 4-bit fields (bits 0..15) -> four bytes
__device__ __forceinline__ uint32_t nib_spread(uint32_t x) {
    x = (x | (x << 8)) & 0x00ff00ffu;
    return (x | (x << 4)) & 0x0f0f0f0fu;
}

// A thread's counters of its keys' buckets, the k-bucket form of the offset
// buffers' branch-free counters (Alg. 3 l.8-9): 4-bit fields of
// one word when a thread holds at most 15 keys, else 8-bit fields of two.
template <int IPT>
struct Mw8Ctr {
    static constexpr bool NIB = IPT <= 15;
    static_assert(IPT <= 255, "8-bit counters");
    using W = typename std::conditional<NIB, uint32_t, uint64_t>::type;
    W c = 0;
    // rank of the next key of bucket b among this thread's; counted if v
    __device__ __forceinline__ uint32_t take(uint32_t b, uint32_t v) {
        const uint32_t sh = NIB ? 4 * b : 8 * b;
        const uint32_t r = (uint32_t)(c >> sh) & (NIB ? 0xfu : 0xffu);
        c += (W)v << sh;
        return r;
    }
    __device__ __forceinline__ void add(uint32_t b, uint32_t v) { c += (W)v << (NIB ? 4 * b : 8 * b); }
    // the same with the shift 4 b given (4-bit counters only)
    __device__ __forceinline__ uint32_t take4(uint32_t b4) {
        static_assert(NIB, "4-bit counters");
        const uint32_t r = (c >> b4) & 0xfu;
        c += 1u << b4;
        return r;
    }

    // the counters as bytes: lo = buckets 0..3, hi = buckets 4..7
    __device__ __forceinline__ void bytes(uint32_t &lo, uint32_t &hi) const {
        if constexpr (NIB) {
            lo = nib_spread((uint32_t)c & 0xffffu);
            hi = nib_spread((uint32_t)c >> 16);
        } else {
            lo = (uint32_t)c;
            hi = (uint32_t)((uint64_t)c >> 32);
        }
    }
};

// Warp scan of the 8 counters: ex = exclusive prefix over the lanes (16-bit
// pairs: word k = buckets 2k, 2k+1), tot = the warp's totals (valid in lane
// 31).  At most 8 keys per thread: the scan runs on the two byte words (every
// exclusive prefix is <= 31 * 8 = 248; lane 31's inclusive one may reach 256
// and wrap, but the difference incl - own is exact modulo 2^32 and fits).
template <int IPT>
__device__ __forceinline__ void mw8_scan(const Mw8Ctr<IPT> &ctr, uint32_t lane, uint32_t (&ex)[MW8 / 2],
                                         uint32_t (&tot)[MW8 / 2]) {
    uint32_t lo, hi, ow[MW8 / 2];
    ctr.bytes(lo, hi);
    mw8_widen((uint64_t)lo | ((uint64_t)hi << 32), ow);
    if constexpr (IPT <= 8) {
        uint32_t il = lo, ih = hi;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t ol = __shfl_up_sync(0xffffffffu, il, d), oh = __shfl_up_sync(0xffffffffu, ih, d);
            if (lane >= (uint32_t)d) {
                il += ol;
                ih += oh;
            }
        }
        mw8_widen((uint64_t)(il - lo) | ((uint64_t)(ih - hi) << 32), ex);
#pragma unroll
        for (int k = 0; k < MW8 / 2; k++) tot[k] = ex[k] + ow[k];
    } else {
        uint32_t q[MW8 / 2];
#pragma unroll
        for (int k = 0; k < MW8 / 2; k++) q[k] = ow[k];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
            for (int k = 0; k < MW8 / 2; k++) {
                const uint32_t o = __shfl_up_sync(0xffffffffu, q[k], d);
                if (lane >= (uint32_t)d) q[k] += o;
            }
        }
#pragma unroll
        for (int k = 0; k < MW8 / 2; k++) {
            ex[k] = q[k] - ow[k];
            tot[k] = q[k];
        }
    }
}

// the warp's total counts of the 8 buckets (two bytes words, per-lane byte
// fields <= 248) added to hist[bucket][seg] by lanes 0..7
template <class KT>
__device__ __forceinline__ void mw8_count_flush(const MwParams<KT> &P, uint32_t lo, uint32_t hi, uint32_t seg,
                                                uint32_t lane) {
    uint32_t q[MW8 / 2];
    mw8_widen((uint64_t)lo | ((uint64_t)hi << 32), q);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1)
#pragma unroll
        for (int k = 0; k < MW8 / 2; k++) q[k] += __shfl_xor_sync(0xffffffffu, q[k], d);
    uint32_t mine = 0;
#pragma unroll
    for (int k = 0; k < MW8 / 2; k++) mine = (lane >> 1) == (uint32_t)k ? q[k] : mine;
    const uint32_t v = (lane & 1) ? (mine >> 16) : (mine & 0xffff);
    if (lane < MW8 && v) atomicAdd(&P.hist[lane * P.hstride + seg], v);
}

// ---- k_mw8_count -----------------------------------------------------------------
template <class KT, int NT, int IPT, int STAGES, int MINB>
__global__ void __launch_bounds__(NT + 32, MINB) k_mw8_count(const MwParams<KT> Pin) {
    if (const LevelCtrl *pv = loop_prev_ctrl(Pin.lp)) if (pv->nmseg_next == 0) return;
    __shared__ MwParams<KT> sP;
    const MwParams<KT> &P = cta_params(Pin, sP);
    using K = typename KT::K;
    using SM = Mw8Smem<KT, NT, IPT, STAGES>;
    constexpr uint32_t NW = SM::NW;
    static_assert(IPT <= 255, "8-bit counters");
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
        if (lane == 0) mw_loader<KT, NT, IPT, STAGES, SM>(P, sm, ntiles, false, true);
        return;
    }
    // Each thread accumulates its byte counters over the tiles of one segment
    // (a loader ticket is a chunk of consecutive tiles); the warp reduces and
    // flushes them when the segment changes or before a byte could overflow.
    constexpr uint32_t FLUSH = 255 / IPT;
    uint32_t alo = 0, ahi = 0, nacc = 0, cur_seg = 0xffffffffu, cls_seg = 0xffffffffu;
    Mw8Cls<KT> cls;
    for (uint32_t i = 0;; i++) {
        const uint32_t s = i % STAGES;
        mbar_wait(&sm.full[s], (i / STAGES) & 1);
        const uint32_t t = sm.tile[s];
        if (t >= ntiles) break;
        const uint32_t si = sm.sidx[s];
        if (si != cls_seg) {   // the splitters change with the segment only
            cls.load(sm.tree[s]);
            cls_seg = si;
        }
        typename KT::T x[IPT];
        const uint32_t valid = mw8_load<KT, NT, IPT, STAGES, SM>(P, sm, s, t, lane, tid, x);
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[s]);
        uint32_t bk[IPT];
        mw8_classify<KT, IPT>(cls, x, bk);
        Mw8Ctr<IPT> ctr;
#pragma unroll
        for (uint32_t c = 0; c < IPT; c++) ctr.add(bk[c], (valid >> c) & 1);
        if (si != cur_seg || nacc == FLUSH) {
            if (cur_seg != 0xffffffffu) mw8_count_flush(P, alo, ahi, cur_seg, lane);
            alo = ahi = nacc = 0;
            cur_seg = si;
        }
        uint32_t lo, hi;
        ctr.bytes(lo, hi);
        alo += lo;
        ahi += hi;
        nacc++;
    }
    if (cur_seg != 0xffffffffu) mw8_count_flush(P, alo, ahi, cur_seg, lane);
}

// ---- k_mw8_scatter ---------------------------------------------------------------
template <class KT, int NT, int IPT, int STAGES, int MINB>
__global__ void __launch_bounds__(NT + 32, MINB) k_mw8_scatter(const MwParams<KT> Pin) {
    if (const LevelCtrl *pv = loop_prev_ctrl(Pin.lp)) if (pv->nmseg_next == 0) return;
    __shared__ MwParams<KT> sP;
    const MwParams<KT> &P = cta_params(Pin, sP);
    using T = typename KT::T;
    using K = typename KT::K;
    using SM = Mw8Smem<KT, NT, IPT, STAGES>;
    constexpr uint32_t NW = SM::NW;
    constexpr uint32_t W = sizeof(T), VW = 16 / W;
    static_assert(IPT <= 16, "8-bit counters, packed ranks");
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
        if (lane == 0) mw_loader<KT, NT, IPT, STAGES, SM>(P, sm, ntiles, true, true);
        return;
    }

    T y[IPT];
    uint32_t ypk[IPT];   // previous tile: tile offset | bucket << 16 | invalid << 31
    bool have_prev = false;
    T *p_dst = nullptr;
    uint32_t p_old = 0, p_cnt = 0, p_off = 0;   // warp 0, lane L < 8: previous tile's run L
    uint64_t p_base = 0;

    for (uint32_t i = 0;; i++) {
        const uint32_t s = i % STAGES, par = i & 1;
        mbar_wait(&sm.full[s], (i / STAGES) & 1);
        const uint32_t t = sm.tile[s];
        const bool cur = t < ntiles;
        T x[IPT];
        uint32_t pk[IPT];
        uint32_t ex[MW8 / 2];
        uint32_t si = 0, sbeg = 0, spar = 0, bstart = 0;
        if (cur) {
            si = sm.sidx[s];
            sbeg = sm.sb[s];
            spar = sm.spar[s];
            bstart = lane < MW8 ? sm.start[s][lane] : 0;
            Mw8Cls<KT> cls;   // (reloaded per tile: kept live, it would spill)
            cls.load(sm.tree[s]);
            const uint32_t valid = mw8_load<KT, NT, IPT, STAGES, SM>(P, sm, s, t, lane, tid, x);
            uint32_t bk[IPT];
            mw8_classify<KT, IPT>(cls, x, bk);
            Mw8Ctr<IPT> ctr;
#pragma unroll
            for (uint32_t c = 0; c < IPT; c++) {
                const uint32_t v = (valid >> c) & 1;
                pk[c] = ctr.take(bk[c], v) | (bk[c] << 16) | ((v ^ 1) << 31);
            }
            uint32_t tot[MW8 / 2];
            mw8_scan<IPT>(ctr, lane, ex, tot);
            if (lane == 31)
#pragma unroll
                for (int k = 0; k < MW8 / 2; k++) sm.wtot[par][warp][k] = tot[k];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[s]);

        // warp 0: placement of the previous tile's runs, now that its atomics returned
        if (warp == 0 && have_prev) {
            const uint64_t g = p_base + p_old;
            const uint32_t a = (uint32_t)(g % VW);
            const uint32_t padded = lane < MW8 ? (a + p_cnt + VW - 1) / VW * VW : 0;
            uint32_t inc = padded;
#pragma unroll
            for (int d = 1; d < MW8; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= (uint32_t)d) inc += o;
            }
            if (lane < MW8) {
                const uint32_t shs = inc - padded + a;
                sm.delta[par ^ 1][lane] = shs - p_off;
                sm.sh[par ^ 1][lane] = shs;
                sm.gstart[par ^ 1][lane] = (uint32_t)g;
                sm.cnt[par ^ 1][lane] = p_cnt;
            }
        }
        if (tid < MW8) bulk_wait_read0();
        named_bar_sync(1, NT);   // B1: warp totals and placement visible, `out` free

        if (cur && warp == 0 && lane < MW8 / 2) {
            uint32_t run = 0;
#pragma unroll
            for (uint32_t w2 = 0; w2 < NW; w2++) {
                sm.wpre[par][w2][lane] = run;
                run += sm.wtot[par][w2][lane];
            }
            const uint32_t lo = run & 0xffff, hi = run >> 16;
            const uint32_t pair = lo + hi;
            uint32_t incp = pair;
#pragma unroll
            for (int d = 1; d < MW8 / 2; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0x0000000fu, incp, d);
                if (lane >= (uint32_t)d) incp += o;
            }
            const uint32_t ex = incp - pair;
            sm.boff[par][2 * lane] = ex;
            sm.boff[par][2 * lane + 1] = ex + lo;
            if (lane == MW8 / 2 - 1) sm.boff[par][MW8] = incp;
        }
        if (have_prev) {
#pragma unroll
            for (uint32_t c = 0; c < IPT; c++) {
                const uint32_t v = ypk[c];
                BQ_CHECK((v >> 31) || (v & 0xffff) + sm.delta[par ^ 1][(v >> 16) & 0x7fff] < SM::TILE + MW8 * 8 + 16);
                if (!(v >> 31)) sm.out[(v & 0xffff) + sm.delta[par ^ 1][(v >> 16) & 0x7fff]] = y[c];
            }
            if (P.aligned) fence_proxy_async_smem();
        }
        named_bar_sync(1, NT);   // B2: prefixes visible, staging complete

        if (have_prev) {
            T *d = p_dst;
            if (!P.aligned) {
                for (uint32_t L = 0; L < MW8; L++) {
                    const uint32_t n = sm.cnt[par ^ 1][L];
                    const uint64_t g = (uint64_t)sm.gstart[par ^ 1][L];
                    for (uint32_t qq = tid; qq < n; qq += NT) d[g + qq] = sm.out[sm.sh[par ^ 1][L] + qq];
                }
            } else if (tid < MW8) {
                const uint32_t L = tid, n = sm.cnt[par ^ 1][L];
                const uint64_t g = sm.gstart[par ^ 1][L], ge = g + n;
                const uint64_t bs = (g + VW - 1) / VW * VW, be = ge / VW * VW;
                if (n && be > bs) tma_store_1d(d + bs, &sm.out[sm.sh[par ^ 1][L] + (bs - g)], (uint32_t)((be - bs) * W));
                bulk_commit();
            } else if (tid >= 32 && tid < 32 + MW8 * 2 * VW) {
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

        // each key's offset in the tile: bucket start + preceding warps' and lanes'
        // keys of its bucket + its rank among this thread's keys of the bucket
        {
            uint32_t base[MW8 / 2];
#pragma unroll
            for (int k = 0; k < MW8 / 2; k++) {
                base[k] = ex[k] + sm.wpre[par][warp][k] + (sm.boff[par][2 * k] | (sm.boff[par][2 * k + 1] << 16));
            }
#pragma unroll
            for (uint32_t c = 0; c < IPT; c++) {
                const uint32_t b = (pk[c] >> 16) & 0x7fff;
                const uint32_t w01 = (b & 2) ? base[1] : base[0], w23 = (b & 2) ? base[3] : base[2];
                const uint32_t w = (b & 4) ? w23 : w01;
                pk[c] += (b & 1) ? (w >> 16) : (w & 0xffff);
            }
        }
        if (warp == 0) {
            const uint32_t st = lane < MW8 ? sm.boff[par][lane] : 0;
            const uint32_t tot = lane < MW8 ? sm.boff[par][lane + 1] - st : 0;
            p_old = (lane < MW8 && tot) ? atomicAdd(&P.cursor[lane * P.hstride + si], tot) : 0;
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
    if (tid < MW8) bulk_wait0();
}

}  // namespace bq
