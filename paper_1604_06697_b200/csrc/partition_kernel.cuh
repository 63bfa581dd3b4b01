// partition_kernel.cuh — k_partition, the tile-partition pass (a2-a5).
// Included by partition.cuh after PassParams.
//
// Persistent, warp-specialised CTAs: NT/32 consumer warps plus a loader, a
// counter and (ordered mode) a look-back warp, around a STAGES-deep ring of
// shared-memory tile buffers.  Two ways to assign the tiles' output ranges
// (SURVEY §8(a) a4 allows both):
//   fast (default)  one packed 64-bit atomicAdd per tile on a per-segment
//                   cursor: no cross-tile dependency chain; tiles of a segment
//                   are placed in completion order;
//   ordered         decoupled look-back in ticket order: deterministic layout
//                   (the < keys in input order, the > keys reversed).
//
//   loader   lane 0 claims tiles in order from an atomic ticket, looks up the
//            tile's segment and issues a 1D TMA bulk copy (cp.async.bulk ->
//            UBLKCP) of the tile into a free stage (mbarrier `loaded`); it
//            runs up to STAGES tiles ahead of the consumers.
//   counter  as soon as a tile lands: counts its < and > keys and publishes
//            the tile's aggregate (a4: decoupled look-back word; inclusive for
//            a segment's first tile) — never blocked by anything but data.
//   lookback in claim order, starting as soon as the tile is claimed (while
//            its data is still in flight): walks back over the predecessors'
//            words to the nearest inclusive prefix; once the tile is counted it
//            publishes the tile's inclusive word and leaves the tile's global
//            offsets in the stage's metadata (mbarrier `full`).  The look-back
//            latency thus overlaps the tile's own load.
//   consumers a2 read the tile from shared memory: thread tid owns the IPT
//            consecutive keys [tid*IPT, (tid+1)*IPT) (swizzled 128-bit loads);
//            a3 classify them three-way in order, advancing per-thread counters
//            by the comparison results (the paper's "store always, increment
//            by the comparison", Alg. 3 l.8-9); a warp scan and one barrier
//            over the warp totals give each thread its tile offsets;
//            a5 keys are staged in shared memory as the < run and the > run
//            (element-reversed, i.e. ascending in memory), each shifted so its
//            16-byte alignment matches the destination; one lane issues TMA
//            bulk stores of the aligned bodies, a few lanes store the heads
//            and tails (< 16 bytes each).
// Each CTA's counter handles its tiles in claim order and needs only their
// own data for the aggregate, so the smallest tile without an inclusive
// prefix can always finish its look-back: no deadlock.
#pragma once

namespace bq {

template <class KT, int NT, int IPT, int STAGES>
struct PartSmem {
    using T = typename KT::T;
    static constexpr int TILE = NT * IPT;
    static constexpr int NW = NT / 32;
    alignas(128) T in[STAGES][TILE];
    // [< run | > run | = run] plus up to 2*(VW-1) alignment shifts and a
    // round-up of the < run: at most TILE + 3*(VW-1) + 1 slots
    alignas(128) T out[TILE + 16];
    Seg seg[STAGES];
    uint64_t claimed[STAGES];
    uint64_t loaded[STAGES];
    uint64_t counted[STAGES];
    uint64_t full[STAGES];
    uint64_t empty[STAGES];
    uint32_t tile[STAGES];
    uint32_t manual[STAGES];
    uint32_t segidx[STAGES];
    uint32_t meta[STAGES][5];              // TL, TG, Lprefix, Gprefix, Eprefix (records)
    uint32_t wtot[NW];                     // packed (lt | gt << 16) per consumer warp
};

template <class KT>
constexpr int part_smem_bytes() {
    return (int)sizeof(PartSmem<KT, Tune<KT>::PART_THREADS, Tune<KT>::PART_IPT, Tune<KT>::PART_STAGES>);
}

template <class KT, int TILE>
struct TileGeom {
    uint64_t b, e, tbeg;
    uint32_t vlo, vhi;   // valid tile-local range [vlo, vhi)
    __device__ TileGeom(const Seg &sg, uint32_t t) {
        constexpr uint32_t VW = tile_vw<KT>();
        b = sg.begin;
        e = b + sg.len;
        tbeg = b / VW * VW + (uint64_t)(t - sg.tile_base) * TILE;   // common.cuh seg_tiles
        vlo = (uint32_t)((tbeg > b ? tbeg : b) - tbeg);
        vhi = (uint32_t)(((tbeg + TILE) < e ? (tbeg + TILE) : e) - tbeg);
    }
};

template <class KT, int NT, int IPT, int STAGES, int MINB, bool ORDERED>
__global__ void __launch_bounds__(NT + (ORDERED ? 96 : 64), MINB) k_partition(const PassParams<KT> Pin) {
    if (const LevelCtrl *pv = loop_prev_ctrl(Pin.lp)) if (pv->ntiles_next == 0) return;
    __shared__ PassParams<KT> sP;
    const PassParams<KT> &P = cta_params(Pin, sP);
    using T = typename KT::T;
    using K = typename KT::K;
    using SM = PartSmem<KT, NT, IPT, STAGES>;
    constexpr uint32_t TILE = SM::TILE;
    constexpr uint32_t NW = SM::NW;
    constexpr uint32_t WSPAN = IPT * 32;             // elements per consumer warp
    constexpr bool REC = KT::is_record;
    constexpr uint32_t W = sizeof(T);
    constexpr uint32_t VW = W >= 16 ? 1 : 16 / W;   // elements per 16 bytes

    extern __shared__ __align__(128) unsigned char smraw[];
    SM &sm = *reinterpret_cast<SM *>(smraw);
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t ntiles = pass_ntiles(P);   // device-resident in the sort's level loop

    if (tid == 0) {
        for (int s = 0; s < STAGES; s++) {
            mbar_init(&sm.claimed[s], 1);
            mbar_init(&sm.loaded[s], 1);
            mbar_init(&sm.counted[s], 1);
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async_smem();
    }
    __syncthreads();

    // -------------------------------------------------------------- loader ----
    if (warp == NW) {
        if (lane != 0) return;
        for (uint32_t i = 0;; i++) {
            const uint32_t s = i % STAGES;
            mbar_wait(&sm.empty[s], ((i / STAGES) & 1) ^ 1);
            const uint32_t t = atomicAdd(&P.ctrl->ticket, 1u);
            sm.tile[s] = t;
            if (t >= ntiles) {
                if (ORDERED) mbar_arrive(&sm.claimed[s]);
                mbar_arrive(&sm.loaded[s]);
                break;
            }
            BQ_TR(t, 6, gtime());
            BQ_TR(t, 7, blockIdx.x);
            const uint32_t si = P.tile_map ? P.tile_map[t] : 0;
            const Seg sg = P.tile_map ? P.segs[si] : P.seg0;
            sm.seg[s] = sg;
            sm.segidx[s] = si;
            if (ORDERED) mbar_arrive(&sm.claimed[s]);   // the look-back warp may start on t
            const TileGeom<KT, TILE> G(sg, t);
            const uint64_t lo16 = (G.tbeg + G.vlo) / VW * VW;
            const uint64_t hi16 = (G.tbeg + G.vhi + VW - 1) / VW * VW;
            const T *src = sg.parity ? P.bufs[1] : P.bufs[0];
            const bool tma = P.aligned && hi16 <= P.n_total;
            sm.manual[s] = !tma;
            if (tma) {
                const uint32_t bytes = (uint32_t)((hi16 - lo16) * W);
                mbar_arrive_expect_tx(&sm.loaded[s], bytes);
                tma_load_1d(&sm.in[s][lo16 - G.tbeg], src + lo16, bytes, &sm.loaded[s]);
            } else {
                mbar_arrive(&sm.loaded[s]);
            }
        }
        return;
    }

    // ------------------------------------------------------------- counter ----
    // warp NW+1: count each landed tile's < and > keys.
    //  fast mode (a4 "one packed atomicAdd per tile"): one 64-bit atomicAdd of
    //    (lt | gt << 32) on the segment's cursor returns the tile's global
    //    offsets directly.  The atomic's latency is hidden by software
    //    pipelining: its result is consumed one tile later.  Tiles of a
    //    segment are then placed in completion order (each run stays in
    //    input order inside a tile).
    //  ordered mode (a4 decoupled look-back): publish the tile's aggregate and
    //    let the look-back warp assign offsets in ticket order (deterministic
    //    layout).  The cursor is still advanced (fire-and-forget) so that the
    //    segment totals are available to k_post in both modes.
    if (warp == NW + 1) {
        uint32_t pend_s = 0, pend_t = 0xffffffffu;
        unsigned long long pend_old = 0;
        uint32_t pend_eold = 0;
        auto finalize = [&](uint32_t ps, uint32_t pt, unsigned long long old, uint32_t eold) {
            if (!ORDERED && lane == 0 && pt < ntiles) {
                sm.meta[ps][2] = (uint32_t)old;
                sm.meta[ps][3] = (uint32_t)(old >> 32);
                sm.meta[ps][4] = eold;
                BQ_TR(pt, 4, gtime());
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(ORDERED ? &sm.counted[ps] : &sm.full[ps]);
        };
        for (uint32_t i = 0;; i++) {
            const uint32_t s = i % STAGES;
            mbar_wait(&sm.loaded[s], (i / STAGES) & 1);
            const uint32_t t = sm.tile[s];
            unsigned long long old = 0;
            uint32_t eold = 0;
            if (t < ntiles) {
                const Seg sg = sm.seg[s];
                const TileGeom<KT, TILE> G(sg, t);
                const K pk = (K)sg.pivot;
                uint32_t cl = 0, cg = 0;
                if (sm.manual[s]) {
                    const T *src = sg.parity ? P.bufs[1] : P.bufs[0];
                    for (uint32_t idx = G.vlo + lane; idx < G.vhi; idx += 32) {
                        const K kk = KT::key(src[G.tbeg + idx]);
                        cl += kk < pk;
                        cg += pk < kk;
                    }
                } else if constexpr (VW > 1) {
                    // 16-byte vectors of VW keys; edge vectors masked
                    const uint4 *v4 = reinterpret_cast<const uint4 *>(sm.in[s]);
                    const uint32_t v0 = G.vlo / VW, v1 = (G.vhi + VW - 1) / VW;
#pragma unroll 4
                    for (uint32_t v = v0 + lane; v < v1; v += 32) {
                        const uint4 q = v4[v];
                        const T *e4 = reinterpret_cast<const T *>(&q);
#pragma unroll
                        for (uint32_t c = 0; c < VW; c++) {
                            const uint32_t idx = v * VW + c;
                            const bool ok = idx >= G.vlo && idx < G.vhi;
                            const K kk = KT::key(e4[c]);
                            cl += ok && kk < pk;
                            cg += ok && pk < kk;
                        }
                    }
                } else {
#pragma unroll 4
                    for (uint32_t idx = G.vlo + lane; idx < G.vhi; idx += 32) {
                        const K kk = KT::key(sm.in[s][idx]);
                        cl += kk < pk;
                        cg += pk < kk;
                    }
                }
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) {
                    cl += __shfl_xor_sync(0xffffffffu, cl, d);
                    cg += __shfl_xor_sync(0xffffffffu, cg, d);
                }
                if (lane == 0) {
                    const uint32_t si = sm.segidx[s];
                    const unsigned long long inc = (unsigned long long)cl | ((unsigned long long)cg << 32);
                    sm.meta[s][0] = cl;
                    sm.meta[s][1] = cg;
                    if constexpr (ORDERED) {
                        st_publish_u64(P.status + t, st_pack(t == sg.tile_base ? ST_INC : ST_AGG, cl, cg));
                        atomicAdd(P.cursor + si, inc);   // totals only (RED, no wait)
                    } else {
                        old = atomicAdd(P.cursor + si, inc);
                        if constexpr (REC) eold = atomicAdd(P.ecursor + si, (G.vhi - G.vlo) - cl - cg);
                    }
                    BQ_TR(t, 5, gtime());
                }
            }
            if (ORDERED) {
                finalize(s, t, 0, 0);
            } else {
                // hand over the previous tile now that its atomic has returned
                if (i > 0) finalize(pend_s, pend_t, pend_old, pend_eold);
                pend_s = s;
                pend_t = t;
                pend_old = old;
                pend_eold = eold;
                if (t >= ntiles) finalize(s, t, 0, 0);   // release the end marker
            }
            if (t >= ntiles) break;
        }
        return;
    }

    // ----------------------------------------------------------- look-back ----
    // warp NW+2, in claim order, starting as soon as a tile is claimed (while
    // its data is still in flight).  The exclusive prefix of tile t is the
    // inclusive prefix of this CTA's previous tile p of the same segment
    // (known here) plus the counts of the tiles p < u < t that other CTAs
    // claimed meanwhile.  Those words are read upward, 32*LBQ per round; an
    // inclusive word met on the way replaces the running sum.  The wait is
    // thus for the newest predecessors' aggregates (which land about when
    // t's own data does), not for a chain of other tiles' look-backs.  Once
    // the tile is counted its inclusive word is published and its global
    // offsets are handed to the consumers.
    if (ORDERED && warp == NW + 2) {
        constexpr int LBQ = 8;
        uint32_t prev_t = 0xffffffffu, prev_base = 0xffffffffu, prev_il = 0, prev_ig = 0;
        for (uint32_t i = 0;; i++) {
            const uint32_t s = i % STAGES, ph = (i / STAGES) & 1;
            mbar_wait(&sm.claimed[s], ph);
            const uint32_t t = sm.tile[s];
            if (t < ntiles) {
                const Seg sg = sm.seg[s];
                uint64_t *st = P.status;
                uint32_t accl = 0, accg = 0;
                if (t != sg.tile_base) {
                    // scan the words (lo .. t-1) upward, 32*LBQ per round, starting
                    // from the known prefix below lo; an inclusive word resets the sum
                    const bool have_prev = prev_base == sg.tile_base && prev_t < t;
                    int64_t lo = have_prev ? (int64_t)prev_t + 1 : (int64_t)sg.tile_base;
                    if (lane == 0) BQ_TR(t, 2, gtime());
#ifdef BQ_TRACE
                    uint32_t nret = 0, nround = 0;
#endif
                    accl = have_prev ? prev_il : 0u;
                    accg = have_prev ? prev_ig : 0u;
                    const int64_t hi = (int64_t)t;   // exclusive
                    while (lo < hi) {
                        uint64_t w[LBQ];
#pragma unroll
                        for (int q = 0; q < LBQ; q++) {
                            const int64_t idx = lo + (int64_t)(lane * LBQ + q);
                            w[q] = idx < hi ? ld_relaxed_u64(st + idx) : st_pack(ST_AGG, 0, 0);
                        }
                        int ql = -1;   // last inclusive word among this lane's
#pragma unroll
                        for (int q = 0; q < LBQ; q++) {
                            const int64_t idx = lo + (int64_t)(lane * LBQ + q);
                            while (st_flag(w[q]) == 0) {
                                __nanosleep(BQ_POLL_SLEEP_NS);
                                w[q] = ld_relaxed_u64(st + idx);
#ifdef BQ_TRACE
                                nret++;
#endif
                            }
                            if (st_flag(w[q]) == 2) ql = q;
                        }
                        const uint32_t incm = __ballot_sync(0xffffffffu, ql >= 0);
                        const int last = incm ? 31 - __clz(incm) : -1;   // highest lane with one
                        uint32_t l = 0, g = 0;
#pragma unroll
                        for (int q = 0; q < LBQ; q++) {
                            // the last inclusive word itself and every word after it count
                            const bool take = (int)lane > last || ((int)lane == last && q >= ql);
                            l += take ? st_lt(w[q]) : 0;
                            g += take ? st_gt(w[q]) : 0;
                        }
#pragma unroll
                        for (int d = 16; d > 0; d >>= 1) {
                            l += __shfl_xor_sync(0xffffffffu, l, d);
                            g += __shfl_xor_sync(0xffffffffu, g, d);
                        }
                        accl = (incm ? 0u : accl) + l;
                        accg = (incm ? 0u : accg) + g;
                        lo += 32 * LBQ;
#ifdef BQ_TRACE
                        nround++;
#endif
                    }
#ifdef BQ_TRACE
                    nret = __reduce_max_sync(0xffffffffu, nret);
                    if (lane == 0) g_trace[t][7] |= ((unsigned long long)nret << 40) | ((unsigned long long)nround << 32) | (1ull << 63);
#endif
                }
                if (lane == 0) BQ_TR(t, 1, gtime());   // (trace: reuse slot 1 = scan end)
                mbar_wait(&sm.counted[s], ph);
                const uint32_t il = accl + sm.meta[s][0], ig = accg + sm.meta[s][1];
                if (lane == 0) {
                    if (t != sg.tile_base) st_publish_u64(st + t, st_pack(ST_INC, il, ig));
                    sm.meta[s][2] = accl;
                    sm.meta[s][3] = accg;
                    if constexpr (REC) {
                        const TileGeom<KT, TILE> G(sg, t);
                        sm.meta[s][4] = (uint32_t)((G.tbeg + G.vlo - G.b) - accl - accg);   // Eprefix
                    }
                    BQ_TR(t, 4, gtime());
                }
                prev_t = t;
                prev_base = sg.tile_base;
                prev_il = il;
                prev_ig = ig;
            } else {
                mbar_wait(&sm.counted[s], ph);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.full[s]);
            if (t >= ntiles) break;
        }
        return;
    }

    // ----------------------------------------------------------- consumers ----
    // Thread tid owns the IPT consecutive keys [tid*IPT, (tid+1)*IPT) of the
    // tile and scans them in order with the paper's branch-free idiom: the
    // destination offset is always formed and the counter advances by the
    // comparison result (Alg. 3 l.8-9).  A warp scan of the packed
    // (lt | gt << 16) counts plus one barrier over the warp totals turns the
    // per-thread counters into tile offsets.
    constexpr uint32_t NV4 = IPT * W / 16;   // 16-byte vectors per thread
    static_assert((IPT * W) % 16 == 0 && NV4 >= 1 && NV4 <= 8 && (NV4 & (NV4 - 1)) == 0, "thread span");
    // lane L reads its vector k from position k ^ sw: the 8 lanes of one
    // 128-bit shared-memory wavefront then touch 8 distinct 16-byte bank groups
    const uint32_t sw = NV4 > 1 ? ((lane * NV4) / 8) & (NV4 - 1) : 0;
    for (uint32_t i = 0;; i++) {
        const uint32_t s = i % STAGES;
        mbar_wait(&sm.full[s], (i / STAGES) & 1);
        const uint32_t t = sm.tile[s];
        if (t >= ntiles) break;
        if (tid == 0) BQ_TR(t, 0, gtime());
        const Seg sg = sm.seg[s];
        const bool manual = sm.manual[s] != 0;
        const TileGeom<KT, TILE> G(sg, t);
        const uint64_t b = G.b, e = G.e, tbeg = G.tbeg;
        const uint32_t vlo = G.vlo, vhi = G.vhi;
        const T *src = sg.parity ? P.bufs[1] : P.bufs[0];
        T *dst = sg.parity ? P.bufs[0] : P.bufs[1];
        const K pk = (K)sg.pivot;
        const uint32_t TL = sm.meta[s][0], TG = sm.meta[s][1];
        const uint32_t lp = sm.meta[s][2], gp = sm.meta[s][3];
        const uint32_t e0 = tid * IPT;

        // ---- a2: load my keys (swizzled 128-bit loads, then un-swizzled) --------
        T x[IPT];
        if (!manual) {
            const uint4 *in4 = reinterpret_cast<const uint4 *>(&sm.in[s][e0]);
            uint4 v[NV4];
#pragma unroll
            for (uint32_t k = 0; k < NV4; k++) v[k] = in4[k ^ sw];
#pragma unroll
            for (uint32_t bit = 1; bit < NV4; bit <<= 1) {
                const bool flip = (sw & bit) != 0;
#pragma unroll
                for (uint32_t k = 0; k < NV4; k++) {
                    if (k & bit) continue;
                    const uint4 a0 = v[k], a1 = v[k | bit];
                    v[k] = flip ? a1 : a0;
                    v[k | bit] = flip ? a0 : a1;
                }
            }
            memcpy(x, v, sizeof x);
        } else {
#pragma unroll
            for (uint32_t c = 0; c < IPT; c++)
                if (e0 + c >= vlo && e0 + c < vhi) x[c] = src[tbeg + e0 + c];
        }

        // ---- a3: three-way classification, branch-free counters ------------------
        uint32_t ltb = 0, gtb = 0, vb = 0, cl = 0, cg = 0;
#pragma unroll
        for (uint32_t c = 0; c < IPT; c++) {
            const bool valid = (e0 + c - vlo) < (vhi - vlo);
            const K kk = KT::key(x[c]);
            const bool lt = valid && kk < pk, gt = valid && pk < kk;
            cl += lt;
            cg += gt;
            ltb |= (uint32_t)lt << c;
            gtb |= (uint32_t)gt << c;
            if constexpr (REC) vb |= (uint32_t)valid << c;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[s]);   // this warp is done with stage s
        const uint32_t cnt = cl | (cg << 16);
        uint32_t inc = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= (uint32_t)d) inc += o;
        }
        if (lane == 31) sm.wtot[warp] = inc;
#ifndef BQ_STG_OUT
        if (tid == 0) bulk_wait_read0();   // the previous tile's bulk stores have read `out`
#endif
        named_bar_sync(1, NT);             // B1: warp totals visible, `out` free
        uint32_t base = inc - cnt;
#pragma unroll
        for (uint32_t w2 = 0; w2 < NW; w2++) base += w2 < warp ? sm.wtot[w2] : 0;

        // ---- a5: stage [< run | > run (ascending in memory) | = run] --------------
        const uint64_t lbase = b + lp;                    // first < destination
        const uint64_t g0 = e - gp - TG;                  // lowest > destination
        const uint32_t aL = (uint32_t)(lbase % VW);
        const uint32_t oG = (aL + TL + VW - 1) / VW * VW;
        const uint32_t aG = (uint32_t)(g0 % VW);
        const uint32_t oE = oG + aG + TG;                 // records only (VW == 1)
        uint32_t rl = aL + (base & 0xffff);               // next < slot
        uint32_t rg = oG + aG + TG - 1 - (base >> 16);    // next > slot (descending)
#pragma unroll
        for (uint32_t c = 0; c < IPT; c++) {
            const bool lt = (ltb >> c) & 1, gt = (gtb >> c) & 1;
            BQ_CHECK(!(lt || gt) || (lt ? rl : rg) < sizeof(sm.out) / sizeof(sm.out[0]));
            if (lt || gt) sm.out[lt ? rl : rg] = x[c];
            rl += lt;
            rg -= gt;
            if constexpr (REC) {
                if (((vb >> c) & 1) && !lt && !gt) {
                    // equal record: valid keys before it in the tile minus the < and > ones
                    const uint32_t vbefore = min(max(e0 + c, vlo), vhi) - vlo;
                    const uint32_t lbefore = rl - aL, gbefore = oG + aG + TG - 1 - rg;
                    sm.out[oE + vbefore - lbefore - gbefore] = x[c];
                }
            }
        }
        uint32_t TE = 0;
        T *estage = nullptr;
        uint64_t ebase = 0;
        if constexpr (REC) {
            TE = (vhi - vlo) - TL - TG;
            estage = sg.parity ? P.stage[1] : P.stage[0];
            ebase = b + sm.meta[s][4];   // b + Eprefix
        }
#ifndef BQ_STG_OUT
        if (P.aligned) fence_proxy_async_smem();
#endif
        named_bar_sync(1, NT);   // B2: staging complete
        if (tid == 0) BQ_TR(t, 3, gtime());

        // ---- stores -----------------------------------------------------------------
        if (!P.aligned) {
            // unaligned buffers (rare): plain coalesced stores
            for (uint32_t q = tid; q < TL; q += NT) dst[lbase + q] = sm.out[aL + q];
            for (uint32_t q = tid; q < TG; q += NT) dst[g0 + q] = sm.out[oG + aG + q];
            if constexpr (REC)
                for (uint32_t q = tid; q < TE; q += NT) estage[ebase + q] = sm.out[oE + q];
            continue;
        }
        const uint64_t lend = lbase + TL, gend = g0 + TG;
        const uint64_t ls = (lbase + VW - 1) / VW * VW, le = lend / VW * VW;
        const uint64_t gs = (g0 + VW - 1) / VW * VW, ge = gend / VW * VW;
#ifdef BQ_STG_OUT
        {
            // 16-byte vector stores of the aligned bodies straight from `out`
            const uint32_t nl = (uint32_t)(le > ls ? (le - ls) / VW : 0);
            const uint32_t ng = (uint32_t)(ge > gs ? (ge - gs) / VW : 0);
            const uint4 *ol = reinterpret_cast<const uint4 *>(&sm.out[aL + (ls - lbase)]);
            const uint4 *og = reinterpret_cast<const uint4 *>(&sm.out[oG + aG + (gs - g0)]);
            uint4 *dl = reinterpret_cast<uint4 *>(dst + ls);
            uint4 *dg = reinterpret_cast<uint4 *>(dst + gs);
            const uint32_t per = REC ? 2 : 1;   // uint4 per element vector (records: 2)
            for (uint32_t q = tid; q < nl * per; q += NT) __stcs(dl + q, ol[q]);
            for (uint32_t q = tid; q < ng * per; q += NT) __stcs(dg + q, og[q]);
            if constexpr (REC) {
                const uint4 *oe = reinterpret_cast<const uint4 *>(&sm.out[oE]);
                uint4 *de = reinterpret_cast<uint4 *>(estage + ebase);
                for (uint32_t q = tid; q < TE * 2; q += NT) __stcs(de + q, oe[q]);
            }
        }
        if (false) {
#else
        if (tid == 0) {
#endif
            if (le > ls) tma_store_1d(dst + ls, &sm.out[aL + (ls - lbase)], (uint32_t)((le - ls) * W));
            if (ge > gs) tma_store_1d(dst + gs, &sm.out[oG + aG + (gs - g0)], (uint32_t)((ge - gs) * W));
            if constexpr (REC) {
                if (TE) tma_store_1d(estage + ebase, &sm.out[oE], TE * W);
            }
            bulk_commit();
        }
        if constexpr (VW > 1) {
            // heads and tails (< 16 bytes each) that the bulk bodies leave out
            if (tid < 2 * VW) {
                const bool tail = tid >= VW;
                const uint32_t q = tail ? tid - VW : tid;
                const uint64_t pos = tail ? (le > ls ? le : ls) + q : lbase + q;
                const bool ok = tail ? (lend > ls && pos < lend) : (pos < (ls < lend ? ls : lend));
                if (ok) dst[pos] = sm.out[aL + (pos - lbase)];
            } else if (tid >= 32 && tid < 32 + 2 * VW) {
                const uint32_t u = tid - 32;
                const bool tail = u >= VW;
                const uint32_t q = tail ? u - VW : u;
                const uint64_t pos = tail ? (ge > gs ? ge : gs) + q : g0 + q;
                const bool ok = tail ? (gend > gs && pos < gend) : (pos < (gs < gend ? gs : gend));
                if (ok) dst[pos] = sm.out[oG + aG + (pos - g0)];
            }
        }
    }
    if (tid == 0) bulk_wait0();
}

}  // namespace bq
