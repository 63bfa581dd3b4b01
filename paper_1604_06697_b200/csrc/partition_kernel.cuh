// partition_kernel.cuh — k_partition, the tile-partition pass (a2-a5).
// Included by partition.cuh after PassParams.
//
// Persistent, warp-specialised CTAs: NT/32 consumer warps + one producer warp.
//
//   producer warp   lane 0 claims tiles in order from an atomic ticket, looks
//                   up the tile's segment and issues a 1D TMA bulk copy
//                   (cp.async.bulk -> UBLKCP) of the tile into a STAGES-deep
//                   shared-memory ring (mbarrier `loaded`).  One claim later
//                   the whole warp counts the landed tile's < and > keys and
//                   publishes the tile's look-back word right away (aggregate,
//                   or inclusive for a segment's first tile), then releases the
//                   stage to the consumers (mbarrier `full`).  Publishing from
//                   the producer keeps a prefetched tile from holding up the
//                   look-back of its successors while its CTA is still busy.
//   consumers       a2  read the tile from shared memory (striped: element
//                       j*NT + tid), three-way classify against the pivot;
//                   a3  per item slot j one __ballot_sync for "<" and one for
//                       ">"; __popc(mask & lanemask_lt) is the key's offset in
//                       its 32-key chunk (the paper's offset buffers, Alg. 3
//                       l.8-9), __popc(mask) the chunk count; one warp scans
//                       the chunk counts into tile offsets;
//                   a4  decoupled look-back over the packed status words gives
//                       the tile's global < and > prefixes;
//                   a5  keys are staged in shared memory as the < run and the
//                       > run (element-reversed, i.e. stored ascending in
//                       memory), each shifted so that its 16-byte alignment
//                       matches the destination; one lane issues TMA bulk
//                       stores of the aligned bodies, a few lanes store the
//                       heads/tails (< 16 bytes each).
// Each CTA processes its tiles in claim order, and a tile's aggregate needs
// only its own data, so the smallest unfinished tile can always finish: the
// look-back cannot deadlock.
#pragma once

namespace bq {


template <class KT, int NT, int IPT, int STAGES>
struct PartSmem {
    using T = typename KT::T;
    static constexpr int TILE = NT * IPT;
    static constexpr int NW = NT / 32;
    static constexpr int NCH = IPT * NW;   // 32-key chunks per tile
    alignas(128) T in[STAGES][TILE];
    // [< run | > run | = run] plus up to 2*(VW-1) alignment shifts and a
    // round-up of the < run: at most TILE + 3*(VW-1) + 1 slots
    alignas(128) T out[TILE + 16];
    Seg seg[STAGES];
    uint64_t loaded[STAGES];
    uint64_t full[STAGES];
    uint64_t empty[STAGES];
    uint32_t tile[STAGES];
    uint32_t manual[STAGES];
    uint32_t cnt[NCH];                     // packed (lt | gt << 16) per chunk -> exclusive prefix
    uint32_t tl, tg, lp, gp;
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
        b = sg.begin;
        e = b + sg.len;
        tbeg = (b / TILE) * TILE + (uint64_t)(t - sg.tile_base) * TILE;
        vlo = (uint32_t)((tbeg > b ? tbeg : b) - tbeg);
        vhi = (uint32_t)(((tbeg + TILE) < e ? (tbeg + TILE) : e) - tbeg);
    }
};

template <class KT, int NT, int IPT, int STAGES, int MINB>
__global__ void __launch_bounds__(NT + 32, MINB) k_partition(PassParams<KT> P) {
    using T = typename KT::T;
    using K = typename KT::K;
    using SM = PartSmem<KT, NT, IPT, STAGES>;
    constexpr uint32_t TILE = SM::TILE;
    constexpr uint32_t NW = SM::NW;
    constexpr bool REC = KT::is_record;
    constexpr uint32_t W = sizeof(T);
    constexpr uint32_t VW = W >= 16 ? 1 : 16 / W;   // elements per 16 bytes
    constexpr uint32_t NCH = SM::NCH;
    constexpr uint32_t PER = (NCH + 31) / 32;
    static_assert(STAGES >= 2, "the producer counts one claim behind");

    extern __shared__ __align__(128) unsigned char smraw[];
    SM &sm = *reinterpret_cast<SM *>(smraw);
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    if (tid == 0) {
        for (int s = 0; s < STAGES; s++) {
            mbar_init(&sm.loaded[s], 1);
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async_smem();
    }
    __syncthreads();

    // ------------------------------------------------------------ producer ----
    if (warp == NW) {
        // count claim j's landed tile, publish its look-back word, hand it over
        auto count_publish = [&](uint32_t j) {
            const uint32_t s = j % STAGES;
            mbar_wait(&sm.loaded[s], (j / STAGES) & 1);
            const uint32_t t = sm.tile[s];
            if (t < P.ntiles) {
                const Seg sg = sm.seg[s];
                const TileGeom<KT, TILE> G(sg, t);
                const bool manual = sm.manual[s] != 0;
                const T *src = sg.parity ? P.bufs[1] : P.bufs[0];
                const K pk = (K)sg.pivot;
                uint32_t cl = 0, cg = 0;
#pragma unroll 4
                for (uint32_t idx = G.vlo + lane; idx < G.vhi; idx += 32) {
                    const K kk = KT::key(manual ? src[G.tbeg + idx] : sm.in[s][idx]);
                    cl += kk < pk;
                    cg += pk < kk;
                }
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) {
                    cl += __shfl_xor_sync(0xffffffffu, cl, d);
                    cg += __shfl_xor_sync(0xffffffffu, cg, d);
                }
                if (lane == 0)
                    st_publish_u64(P.status + t, st_pack(t == sg.tile_base ? ST_INC : ST_AGG, cl, cg));
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.full[s]);
        };
        for (uint32_t i = 0;; i++) {
            const uint32_t s = i % STAGES;
            uint32_t t = 0;
            if (lane == 0) {
                mbar_wait(&sm.empty[s], ((i / STAGES) & 1) ^ 1);
                t = atomicAdd(&P.ctrl->ticket, 1u);
                sm.tile[s] = t;
                if (t >= P.ntiles) {
                    mbar_arrive(&sm.loaded[s]);
                } else {
                    const Seg sg = P.tile_map ? P.segs[P.tile_map[t]] : P.seg0;
                    sm.seg[s] = sg;
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
            }
            t = __shfl_sync(0xffffffffu, t, 0);
            if (i >= 1) count_publish(i - 1);
            if (t >= P.ntiles) {
                count_publish(i);   // releases the end marker to the consumers
                break;
            }
        }
        return;
    }

    // ----------------------------------------------------------- consumers ----
    const uint32_t lm = lanemask_lt();
    for (uint32_t i = 0;; i++) {
        const uint32_t s = i % STAGES;
        mbar_wait(&sm.full[s], (i / STAGES) & 1);
        const uint32_t t = sm.tile[s];
        if (t >= P.ntiles) break;
        const Seg sg = sm.seg[s];
        const bool manual = sm.manual[s] != 0;
        const TileGeom<KT, TILE> G(sg, t);
        const uint32_t k = t - sg.tile_base;
        const uint64_t b = G.b, e = G.e, tbeg = G.tbeg;
        const uint32_t vlo = G.vlo, vhi = G.vhi;
        const T *src = sg.parity ? P.bufs[1] : P.bufs[0];
        T *dst = sg.parity ? P.bufs[0] : P.bufs[1];
        const K pk = (K)sg.pivot;

        // ---- a2 + a3: load, classify, per-chunk ranks --------------------------
        T x[IPT];
        uint32_t rk[IPT];            // packed in-chunk ranks (lt | gt << 16)
        uint32_t ltb = 0, gtb = 0, vb = 0;
#pragma unroll
        for (int j = 0; j < IPT; j++) {
            const uint32_t idx = j * NT + tid;
            const bool valid = idx >= vlo && idx < vhi;
            if (valid) x[j] = manual ? src[tbeg + idx] : sm.in[s][idx];
            const K kk = valid ? KT::key(x[j]) : pk;
            ltb |= (uint32_t)(valid && kk < pk) << j;
            gtb |= (uint32_t)(valid && pk < kk) << j;
            vb |= (uint32_t)valid << j;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[s]);   // this warp is done with stage s
#pragma unroll
        for (int j = 0; j < IPT; j++) {
            const uint32_t ml = __ballot_sync(0xffffffffu, (ltb >> j) & 1);
            const uint32_t mg = __ballot_sync(0xffffffffu, (gtb >> j) & 1);
            rk[j] = __popc(ml & lm) | (__popc(mg & lm) << 16);
            if (lane == 0) sm.cnt[j * NW + warp] = __popc(ml) | (__popc(mg) << 16);
        }
        named_bar_sync(1, NT);   // B1: chunk counts complete

        // ---- warp 0: chunk scan + a4 look-back ------------------------------------
        if (warp == 0) {
            uint32_t a[PER], sum = 0;
#pragma unroll
            for (int q = 0; q < (int)PER; q++) {
                a[q] = sum;
                if (lane * PER + q < NCH) sum += sm.cnt[lane * PER + q];
            }
            uint32_t inc = sum;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= (uint32_t)d) inc += o;
            }
            const uint32_t ex = inc - sum;
#pragma unroll
            for (int q = 0; q < (int)PER; q++)
                if (lane * PER + q < NCH) sm.cnt[lane * PER + q] = ex + a[q];
            const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
            const uint32_t TL = tot & 0xffff, TG = tot >> 16;

            uint64_t *st = P.status;
            uint32_t accl = 0, accg = 0;
            if (k != 0) {   // the producer already published this tile's aggregate
                int64_t pred = (int64_t)t - 1;
                const int64_t first_tile = sg.tile_base;
                while (true) {
                    const int64_t idx = pred - (int64_t)lane;
                    uint64_t w = ST_INC;      // before the segment start: inclusive zero
                    if (idx >= first_tile) {
                        do { w = ld_relaxed_u64(st + idx); } while (st_flag(w) == 0);
                    }
                    const uint32_t incm = __ballot_sync(0xffffffffu, st_flag(w) == 2);
                    const int first = incm ? (__ffs(incm) - 1) : 31;
                    uint32_t l = (int)lane <= first ? st_lt(w) : 0;
                    uint32_t g = (int)lane <= first ? st_gt(w) : 0;
#pragma unroll
                    for (int d = 16; d > 0; d >>= 1) {
                        l += __shfl_xor_sync(0xffffffffu, l, d);
                        g += __shfl_xor_sync(0xffffffffu, g, d);
                    }
                    accl += l;
                    accg += g;
                    if (incm) break;
                    pred -= 32;
                }
                if (lane == 0) st_publish_u64(st + t, st_pack(ST_INC, accl + TL, accg + TG));
            }
            if (lane == 0) {
                sm.tl = TL;
                sm.tg = TG;
                sm.lp = accl;
                sm.gp = accg;
                bulk_wait_read0();   // the previous tile's bulk stores have read `out`
            }
        }
        named_bar_sync(1, NT);   // B2: prefixes + global offsets visible

        // ---- a5: stage [< run | > run (ascending in memory) | = run] --------------
        const uint32_t TL = sm.tl, TG = sm.tg;
        const uint32_t lp = sm.lp, gp = sm.gp;
        const uint64_t lbase = b + lp;                    // first < destination
        const uint64_t g0 = e - gp - TG;                  // lowest > destination
        const uint32_t aL = (uint32_t)(lbase % VW);
        const uint32_t oG = (aL + TL + VW - 1) / VW * VW;
        const uint32_t aG = (uint32_t)(g0 % VW);
        const uint32_t oE = oG + aG + TG;                 // records only (VW == 1)
#pragma unroll
        for (int j = 0; j < IPT; j++) {
            const uint32_t pre = sm.cnt[j * NW + warp] + rk[j];   // < | > keys before this one in the tile
            if ((ltb >> j) & 1) {
                sm.out[aL + (pre & 0xffff)] = x[j];
            } else if ((gtb >> j) & 1) {
                sm.out[oG + aG + (TG - 1 - (pre >> 16))] = x[j];
            } else if constexpr (REC) {
                if ((vb >> j) & 1) {
                    // equal record: valid keys before it in the tile minus the < and > ones
                    const uint32_t pos = j * NT + tid;
                    const uint32_t vbefore = min(max(pos, vlo), vhi) - vlo;
                    sm.out[oE + vbefore - (pre & 0xffff) - (pre >> 16)] = x[j];
                }
            }
        }
        uint32_t TE = 0;
        T *estage = nullptr;
        uint64_t ebase = 0;
        if constexpr (REC) {
            TE = (vhi - vlo) - TL - TG;
            estage = sg.parity ? P.stage[1] : P.stage[0];
            ebase = b + (uint64_t)(tbeg + vlo - b) - lp - gp;   // b + Eprefix
        }
        if (P.aligned) fence_proxy_async_smem();
        named_bar_sync(1, NT);   // B3: staging complete

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
        if (tid == 0) {
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
