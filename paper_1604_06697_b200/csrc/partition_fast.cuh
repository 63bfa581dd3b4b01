// partition_fast.cuh — k_part_fast, the tile-partition pass (a2-a5) for keys
// with atomic-cursor placement (the sort's default).  Included by
// partition.cuh after PassParams.
//
// Persistent CTAs: NT consumer threads + one loader warp around a STAGES-deep
// ring of shared-memory tiles filled by 1D TMA bulk copies (cp.async.bulk ->
// UBLKCP), tiles claimed from an atomic ticket.
//
// The consumers run a two-tile software pipeline.  Iteration i:
//   a2  read tile i from the ring (thread tid owns the IPT keys
//       [tid*IPT, (tid+1)*IPT); the 16-byte vectors are visited in an
//       XOR-permuted order, which makes the reads free of bank conflicts —
//       the order of keys inside a tile does not matter for this placement);
//   a3  classify three-way with the paper's branch-free counters (Alg. 3
//       l.8-9: "store the offset always, advance the counter by the
//       comparison"), warp scan + one barrier over the warp
//       totals -> the tile's counts (TL, TG) and every thread's offsets;
//   a4  one thread claims the tile's output ranges with a single packed
//       64-bit atomicAdd (lt | gt << 32) on the segment's cursor — its result
//       is not needed until the next iteration, so its L2 round trip
//       overlaps the classification of the next tile;
//   a5  tile i-1 (its keys kept in registers) is staged in shared memory as
//       [< run | > run], each run shifted to the 16-byte alignment of its
//       destination, and written with TMA bulk stores (aligned bodies) plus
//       a few scalar head/tail stores.
// Keys equal to the pivot are dropped: k_post fills the equal band.  Keys
// outside the segment in a partial tile are replaced by the pivot on load,
// which drops them the same way.
// Records (32 B) are never dropped: the split is two-way by the segment's
// mode (Seg::pad0 bit 0): [< p | >= p], or [<= p | > p] for the follow-up pass
// of a pivot that was duplicated in its sample, whose left side is then a
// finished run of equal keys (k_post).  Positions outside the segment in a
// partial tile are masked.
#pragma once

namespace bq {

template <class KT, int NT, int IPT, int STAGES>
struct FastSmem {
    using T = typename KT::T;
    static constexpr int TILE = NT * IPT;
    static constexpr int NW = NT / 32;
    alignas(128) T in[STAGES][TILE];
    alignas(128) T out[TILE + 16];
    Seg seg[STAGES];
    uint64_t full[STAGES];
    uint64_t empty[STAGES];
    uint32_t tile[STAGES];
    uint32_t manual[STAGES];
    uint32_t segidx[STAGES];
    unsigned long long offs[2];           // atomic results, by iteration parity
    uint32_t wtot[2][NW];                 // packed (lt | gt << 16) per warp, by parity
};

template <class KT>
constexpr int fast_smem_bytes() {
    return (int)sizeof(FastSmem<KT, Tune<KT>::PART_THREADS, Tune<KT>::PART_IPT, Tune<KT>::PART_STAGES>);
}

template <class KT, int NT, int IPT, int STAGES, int MINB>
__global__ void __launch_bounds__(NT + 32, MINB) k_part_fast(const PassParams<KT> Pin) {
    if (const LevelCtrl *pv = loop_prev_ctrl(Pin.lp)) if (pv->ntiles_next == 0) return;
    __shared__ PassParams<KT> sP;
    const PassParams<KT> &P = cta_params(Pin, sP);
    using T = typename KT::T;
    using K = typename KT::K;
    using SM = FastSmem<KT, NT, IPT, STAGES>;
    constexpr bool REC = KT::is_record;
    constexpr uint32_t TILE = SM::TILE;
    constexpr uint32_t NW = SM::NW;
    constexpr uint32_t W = sizeof(T);
    constexpr uint32_t VW = W >= 16 ? 1 : 16 / W;   // elements per 16-byte vector
    constexpr uint32_t NV4 = IPT * W / 16;          // vectors per thread
    static_assert(REC || (IPT % VW == 0 && NV4 >= 1 && NV4 <= 8 && (NV4 & (NV4 - 1)) == 0), "thread span");

    extern __shared__ __align__(128) unsigned char smraw[];
    SM &sm = *reinterpret_cast<SM *>(smraw);
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t ntiles = pass_ntiles(P);   // device-resident in the sort's level loop

    if (tid == 0) {
        for (int s = 0; s < STAGES; s++) {
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
        // a ticket is a chunk of PART_CHUNK consecutive tiles, the next one
        // claimed a chunk ahead, so the atomic's L2 round trip overlaps the
        // tiles' metadata reads and the wait for a free stage (a claimed
        // ticket is always processed: the loop stops only on a tile >=
        // ntiles, and every later ticket is larger); the next tile's segment
        // index is read a tile ahead and a segment's metadata once per run of
        // its tiles
        uint32_t c_next = atomicAdd(&P.ctrl->ticket, 1u) * PART_CHUNK, j = 0;
        auto claim = [&]() -> uint32_t {
            const uint32_t t = c_next + j;
            if (++j == PART_CHUNK || t + 1 >= ntiles) {
                if (t < ntiles) c_next = atomicAdd(&P.ctrl->ticket, 1u) * PART_CHUNK;
                j = 0;
            }
            return t;
        };
        uint32_t t = claim();
        uint32_t si = (P.tile_map && t < ntiles) ? P.tile_map[t] : 0, prev_si = 0xffffffffu;
        Seg sg = P.seg0;
        for (uint32_t i = 0;; i++) {
            const uint32_t s = i % STAGES;
            const uint32_t tn = t < ntiles ? claim() : ntiles;
            const uint32_t sin = (P.tile_map && tn < ntiles) ? P.tile_map[tn] : 0;
            if (P.tile_map && si != prev_si) sg = P.segs[si];
            prev_si = si;
            mbar_wait(&sm.empty[s], ((i / STAGES) & 1) ^ 1);
            sm.tile[s] = t;
            if (t >= ntiles) {
                mbar_arrive(&sm.full[s]);
                break;
            }
            sm.seg[s] = sg;
            sm.segidx[s] = si;
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
        return;
    }

    // ----------------------------------------------------------- consumers ----
    // lane L visits its vector k at position k ^ sw: the 8 lanes of one
    // 128-bit shared-memory wavefront then touch 8 distinct 16-byte bank groups
    const uint32_t sw = NV4 > 1 ? ((lane * NV4) / 8) & (NV4 - 1) : 0;
    const uint32_t e0 = tid * IPT;

    // the previous tile, carried across one iteration
    T y[IPT];
    bool have_prev = false;
    uint32_t p_base = 0, p_TL = 0, p_TG = 0;
    uint64_t p_b = 0, p_e = 0;
    K p_pk = 0;
    T *p_dst = nullptr;
    uint32_t p_valid = 0, p_mode = 0;   // records: valid mask, split mode
    unsigned long long my_old = 0;   // thread 0: atomic result of the previous tile

    for (uint32_t i = 0;; i++) {
        const uint32_t s = i % STAGES, par = i & 1;
        mbar_wait(&sm.full[s], (i / STAGES) & 1);
        const uint32_t t = sm.tile[s];
        const bool cur = t < ntiles;
        // everything this iteration needs from the slot is read before the
        // slot is released to the loader
        const uint32_t si = sm.segidx[s];
        const bool manual = sm.manual[s] != 0;

        // ---- a2 + a3: load and classify tile i ---------------------------------
        T x[IPT];
        uint32_t cnt = 0, valid = (1u << IPT) - 1, mode = 0;
        Seg sg;
        uint64_t b = 0, e = 0;
        K pk = 0;
        if constexpr (REC) if (cur) {
            sg = sm.seg[s];
            const TileGeom<KT, TILE> G(sg, t);
            b = G.b;
            e = G.e;
            pk = (K)sg.pivot;
            mode = sg.pad0 & 1;
            const T *src = sg.parity ? P.bufs[1] : P.bufs[0];
#pragma unroll
            for (uint32_t c = 0; c < IPT; c++) {
                const uint32_t pos = e0 + c;
                const bool v = pos >= G.vlo && pos < G.vhi;
                if (!manual) x[c] = sm.in[s][pos];
                else if (v) x[c] = src[G.tbeg + pos];
                valid = v ? valid : (valid & ~(1u << c));
            }
            uint32_t cl = 0, cg = 0;
#pragma unroll
            for (uint32_t c = 0; c < IPT; c++) {
                const K kk = KT::key(x[c]);
                const bool v = (valid >> c) & 1;
                const bool lt = mode ? !(pk < kk) : (kk < pk);
                cl += v && lt;
                cg += v && !lt;
            }
            cnt = cl | (cg << 16);
        }
        if constexpr (!REC) if (cur) {
            sg = sm.seg[s];
            const TileGeom<KT, TILE> G(sg, t);
            b = G.b;
            e = G.e;
            pk = (K)sg.pivot;
            if (!manual) {
                const uint4 *in4 = reinterpret_cast<const uint4 *>(&sm.in[s][e0]);
#pragma unroll
                for (uint32_t k = 0; k < NV4; k++) {
                    const uint4 v = in4[k ^ sw];
                    memcpy(&x[k * VW], &v, 16);
                }
                if (G.vlo != 0 || G.vhi != TILE) {
                    // partial tile: keys outside the segment become the pivot
                    const T pv = KT::from_key(pk);
#pragma unroll
                    for (uint32_t k = 0; k < NV4; k++)
#pragma unroll
                        for (uint32_t j = 0; j < VW; j++) {
                            const uint32_t pos = e0 + (k ^ sw) * VW + j;
                            if (pos < G.vlo || pos >= G.vhi) x[k * VW + j] = pv;
                        }
                }
            } else {
                const T *src = sg.parity ? P.bufs[1] : P.bufs[0];
                const T pv = KT::from_key(pk);
#pragma unroll
                for (uint32_t k = 0; k < NV4; k++)
#pragma unroll
                    for (uint32_t j = 0; j < VW; j++) {
                        const uint32_t pos = e0 + (k ^ sw) * VW + j;
                        x[k * VW + j] = (pos >= G.vlo && pos < G.vhi) ? src[G.tbeg + pos] : pv;
                    }
            }
            uint32_t cl = 0, cg = 0;
#pragma unroll
            for (uint32_t c = 0; c < IPT; c++) {
                const K kk = KT::key(x[c]);
                cl += kk < pk;
                cg += pk < kk;
            }
            cnt = cl | (cg << 16);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[s]);   // this warp is done with stage s
        uint32_t inc = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= (uint32_t)d) inc += o;
        }
        if (lane == 31) sm.wtot[par][warp] = inc;
        if (tid == 0) {
            if (have_prev) sm.offs[par ^ 1] = my_old;   // waits for last iteration's atomic
            bulk_wait_read0();                          // the previous bulk stores have read `out`
        }
        named_bar_sync(1, NT);   // B1: warp totals and the previous tile's offsets visible

        uint32_t base = 0, TL = 0, TG = 0;
        if (cur) {
            uint32_t pre = 0, tot = 0;
#pragma unroll
            for (uint32_t w2 = 0; w2 < NW; w2++) {
                const uint32_t v = sm.wtot[par][w2];
                pre += w2 < warp ? v : 0;
                tot += v;
            }
            base = pre + inc - cnt;
            TL = tot & 0xffff;
            TG = tot >> 16;
            if (tid == 0) {
                my_old = atomicAdd(P.cursor + si, (unsigned long long)TL | ((unsigned long long)TG << 32));
            }
        }

        // ---- a5: stage and store the previous tile ------------------------------
        if (have_prev) {
            const unsigned long long old = sm.offs[par ^ 1];
            const uint64_t lbase = p_b + (uint32_t)old;                 // first < destination
            const uint64_t g0 = p_e - (uint32_t)(old >> 32) - p_TG;      // lowest > destination
            BQ_CHECK(lbase >= p_b && lbase + p_TL <= p_e && g0 >= p_b && g0 + p_TG <= p_e);
            const uint32_t aL = (uint32_t)(lbase % VW);
            const uint32_t oG = (aL + p_TL + VW - 1) / VW * VW;
            const uint32_t aG = (uint32_t)(g0 % VW);
            uint32_t rl = aL + (p_base & 0xffff);
            uint32_t rg = oG + aG + (p_base >> 16);
#pragma unroll
            for (uint32_t c = 0; c < IPT; c++) {
                const K kk = KT::key(y[c]);
                bool lt, gt;
                if constexpr (REC) {
                    const bool v = (p_valid >> c) & 1;
                    const bool l0 = p_mode ? !(p_pk < kk) : (kk < p_pk);
                    lt = v && l0;
                    gt = v && !l0;
                } else {
                    lt = kk < p_pk;
                    gt = p_pk < kk;
                }
                const uint32_t idx = lt ? rl : rg;
                BQ_CHECK(!(lt || gt) || idx < TILE + 16);
                if (lt || gt) sm.out[idx] = y[c];
                rl += lt;
                rg += gt;
            }
            if (P.aligned) fence_proxy_async_smem();
            named_bar_sync(1, NT);   // B2: staging complete
            T *d = p_dst;   // the other buffer of the previous tile's segment
            const uint64_t lend = lbase + p_TL, gend = g0 + p_TG;
            if (!P.aligned) {
                for (uint32_t q = tid; q < p_TL; q += NT) d[lbase + q] = sm.out[aL + q];
                for (uint32_t q = tid; q < p_TG; q += NT) d[g0 + q] = sm.out[oG + aG + q];
            } else {
                const uint64_t ls = (lbase + VW - 1) / VW * VW, le = lend / VW * VW;
                const uint64_t gs = (g0 + VW - 1) / VW * VW, ge = gend / VW * VW;
                if (tid == 0) {
                    if (le > ls) tma_store_1d(d + ls, &sm.out[aL + (ls - lbase)], (uint32_t)((le - ls) * W));
                    if (ge > gs) tma_store_1d(d + gs, &sm.out[oG + aG + (gs - g0)], (uint32_t)((ge - gs) * W));
                    bulk_commit();
                }
                // heads and tails (< 16 bytes each) that the bulk bodies leave out
                if (tid >= 32 && tid < 32 + 2 * VW) {
                    const uint32_t u = tid - 32;
                    const bool tail = u >= VW;
                    const uint32_t q = tail ? u - VW : u;
                    const uint64_t pos = tail ? (le > ls ? le : ls) + q : lbase + q;
                    const bool ok = tail ? (lend > ls && pos < lend) : (pos < (ls < lend ? ls : lend));
                    if (ok) d[pos] = sm.out[aL + (pos - lbase)];
                } else if (tid >= 64 && tid < 64 + 2 * VW) {
                    const uint32_t u = tid - 64;
                    const bool tail = u >= VW;
                    const uint32_t q = tail ? u - VW : u;
                    const uint64_t pos = tail ? (ge > gs ? ge : gs) + q : g0 + q;
                    const bool ok = tail ? (gend > gs && pos < gend) : (pos < (gs < gend ? gs : gend));
                    if (ok) d[pos] = sm.out[oG + aG + (pos - g0)];
                }
            }
        }
        if (!cur) break;
        // carry tile i to the next iteration
#pragma unroll
        for (uint32_t c = 0; c < IPT; c++) y[c] = x[c];
        have_prev = true;
        p_base = base;
        p_TL = TL;
        p_TG = TG;
        p_b = b;
        p_e = e;
        p_pk = pk;
        p_valid = valid;
        p_mode = mode;
        p_dst = sg.parity ? P.bufs[0] : P.bufs[1];
    }
    if (tid == 0) bulk_wait0();
}

}  // namespace bq
