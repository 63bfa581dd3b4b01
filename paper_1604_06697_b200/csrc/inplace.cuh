// inplace.cuh — SURVEY §8(f) N2: the in-place block partition, Alg. 3
// lifted to CTA granularity, with no n-element scratch buffer
// (the paper's in-place property).
//
// k_inplace: every CTA runs the paper's main loop on blocks of T elements
// claimed from both ends of the range: a left block from the left cursor, a
// right block from the right cursor (one 64-bit word, claimed atomically, so
// no block is taken twice and the two sides meet).  For each block the scan
// phase stores the offsets of its misplaced elements in a shared-memory
// offsets buffer — "the pointer is always stored, the counter advances by the
// comparison" (Alg. 3 l.8-9, 15-16) — the rearrangement phase swaps
// num = min(num_L, num_R) pairs (l.19-21), start/num advance (l.24-25), and a
// block whose buffer ran empty is neutralized: written back, and the next
// block on its side is claimed (l.26-27).  When one side is exhausted the CTA
// writes back the block it still holds and lists it as a leftover.
//
// The cleanup kernels that follow (k_ip_plan .. k_ip_fix, launched by
// run_partition_inplace_ip in driver.cuh without host round trips) swap the
// leftover blocks into the middle of the range and partition the middle
// (<= #CTAs + 1 blocks: "compare and rearrange remaining elements", l.29)
// out of place in a small buffer; pass 1 forms the equal band in the right
// part (from recorded positions, by compaction, or by a second block pass).
#pragma once

namespace bq {

constexpr uint32_t IP_GMAX = 148 * 8;   // bound on the resident k_inplace CTAs (and so on the leftovers)

// claim-word bias: lo and hi start at IP_BIAS and IP_BIAS + #blocks
constexpr uint32_t IP_BIAS = 1u << 30;
constexpr uint32_t IP_NONE = 0xffffffffu;

struct InplaceState {
    unsigned long long claim;        // lo: next left block, hi: end of the right blocks
    unsigned long long n_equal;      // keys equal to the pivot, over every block as loaded
    unsigned long long n_equal_held; // ... of them in the blocks held at the end (the middle)
    uint32_t nleftover;              // blocks a CTA held when its partner side ran out
    uint32_t left_ok;                // blocks claimed from the left (= the meeting point)
    uint32_t neqpos;                 // pass 0: positions recorded of keys equal to p in final right blocks
    uint32_t pad[7];
};
static_assert(sizeof(InplaceState) == 64, "InplaceState layout");

// One in-place pass over data[off, off + len), device-resident from set-up
// (k_ip_setup) to result (k_ip_fix): the host launches the whole sequence
// without reading anything back.
struct IpPass {
    InplaceState st;
    unsigned long long off, len, h;      // the range and its head (< 16 bytes, to align the blocks)
    unsigned long long o1, n1, o2, tail; // cleanup ranges, relative to off: middle [o1, o1+n1), tail [o2, len)
    unsigned long long v;                // elements the cleanup partitions: h + n1 + tail
    unsigned long long lcur, rcur, ev;   // k_vsplit: left / right cursors, keys equal to p
    unsigned long long n_left, n_eq;     // results: end of the left part (absolute), keys equal to p
    unsigned long long cnt_eq, cnt_gt;   // compaction (pass 1): keys = p past the band, keys > p inside it
    uint32_t nb, active, npairs, compact;
    uint32_t fast_eq, pad2;              // compaction from pass 0's recorded positions (no full scan)
};

template <class KT>
struct InplaceParams {
    using T = typename KT::T;
    T *data;                 // the caller's array
    IpPass *ps;              // this pass
    uint64_t pivot;          // pivot key (KT::K)
    int mode;                // 0: left <=> key < p; 1: left <=> key <= p
    uint32_t *leftover;      // [2 * k]: block index, side (0 left, 1 right)
    uint64_t *eqpos;         // mode 0: (block << 32 | offset) of keys equal to p in final right blocks
    uint32_t eqcap;          // its capacity (more: the equal band falls back to a full scan)
};

// Three block buffers: the left block, the right block and a spare that the
// next block of the side about to be neutralized streams into (TMA) while
// the current pair is rearranged.  Offsets buffers belong to the sides.
template <class KT, int NT, int IPT>
struct InplaceSmem {
    using T = typename KT::T;
    static constexpr int TILE = NT * IPT;
    static constexpr int NW = NT / 32;
    alignas(128) T buf[3][TILE];
    uint16_t off[2][TILE];            // offsets buffers of the misplaced elements (Alg. 3 offsets_L/R)
    uint64_t bar[3];                  // TMA completion, one per buffer
    uint32_t wsum[NW];
    uint32_t blk[3];                  // block index held by each buffer
    uint32_t slot[2];                 // buffer of each side (3: the side is finished)
    uint32_t spare;
    uint32_t start[2], num[2], dirty[2], fresh[2];
    uint32_t eqcnt[2];                // keys equal to p in each side's block (mode 0)
    uint32_t weq[NW];                 // per-warp equal counts of a fresh block
};

// blocks of the in-place partition: PART_THREADS x ip_ipt elements; keys use
// half the pass tile (8 KB blocks: more CTAs per SM to overlap the block
// loads with the swaps; measured 1-4 % faster), records the pass tile
#ifndef BQ_IP_IPT_DIV
#define BQ_IP_IPT_DIV 2
#endif
template <class KT>
constexpr int ip_ipt() {
    return KT::is_record ? Tune<KT>::PART_IPT
                         : (Tune<KT>::PART_IPT / BQ_IP_IPT_DIV < 1 ? 1 : Tune<KT>::PART_IPT / BQ_IP_IPT_DIV);
}
template <class KT>
constexpr uint32_t ip_tile() { return (uint32_t)(Tune<KT>::PART_THREADS * ip_ipt<KT>()); }

template <class KT>
constexpr int inplace_smem_bytes() {
    return (int)sizeof(InplaceSmem<KT, Tune<KT>::PART_THREADS, ip_ipt<KT>()>);
}

// one fetch-and-add on the packed word decides a claim; a failed claim moves
// lo past hi (or hi below lo), which keeps failing — IP_BIAS keeps both
// halves clear of wrap-around (at most one failure per CTA and side)
__device__ __forceinline__ uint32_t ip_claim(InplaceState *st, int side) {
    const unsigned long long old = atomicAdd(&st->claim, side == 0 ? 1ull : 0xffffffff00000000ull);
    const uint32_t lo = (uint32_t)old, hi = (uint32_t)(old >> 32);
    if (lo >= hi) return IP_NONE;
    if (side == 0) atomicAdd(&st->left_ok, 1u);
    return (side == 0 ? lo : hi - 1) - IP_BIAS;
}

#ifndef BQ_IP_MINB
#define BQ_IP_MINB 6
#endif
template <class KT, int NT, int IPT>
__global__ void __launch_bounds__(NT, BQ_IP_MINB) k_inplace(InplaceParams<KT> P) {
    using T = typename KT::T;
    using K = typename KT::K;
    using SM = InplaceSmem<KT, NT, IPT>;
    constexpr uint32_t TILE = SM::TILE, NW = SM::NW;
    constexpr uint32_t W = sizeof(T);
    constexpr uint32_t BYTES = TILE * W;
    constexpr uint32_t VW = W >= 16 ? 1 : 16 / W;   // keys per 16-byte vector
    static_assert(TILE <= 65536, "16-bit offsets");
    static_assert(IPT <= 32 && IPT % VW == 0, "misplaced flags in one word");
    static_assert(BYTES % 16 == 0, "bulk copies move 16-byte multiples");
    extern __shared__ __align__(128) unsigned char smraw[];
    SM &sm = *reinterpret_cast<SM *>(smraw);
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const K pk = (K)P.pivot;
    if (!P.ps->active) return;
    InplaceState *const st = &P.ps->st;
    T *const base = P.data + P.ps->off + P.ps->h;   // 16-byte aligned first block

    if (tid == 0) {
        for (int b = 0; b < 3; b++) mbar_init(&sm.bar[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async_smem();
        sm.spare = 2;
        for (int side = 0; side < 2; side++) {
            const uint32_t got = ip_claim(st, side);
            sm.dirty[side] = 0;
            sm.num[side] = sm.start[side] = 0;
            if (got == IP_NONE) {
                sm.slot[side] = 3;
                sm.fresh[side] = 0;
            } else {
                sm.slot[side] = side;
                sm.blk[side] = got;
                sm.fresh[side] = 1;
                mbar_arrive_expect_tx(&sm.bar[side], BYTES);
                tma_load_1d(sm.buf[side], base + (uint64_t)got * TILE, BYTES, &sm.bar[side]);
            }
        }
    }
    __syncthreads();

    uint32_t phase = 0;   // mbarrier parity per buffer (bit b)
    for (;;) {
        // scan phase of newly arrived blocks (Alg. 3 l.5-18): the offset of
        // every element is formed, the buffer grows by the misplaced flag
        for (int side = 0; side < 2; side++) {
            if (!sm.fresh[side]) continue;   // uniform
            const uint32_t b = sm.slot[side];
            mbar_wait(&sm.bar[b], (phase >> b) & 1u);
            phase ^= 1u << b;
            const T *blk = sm.buf[b];
            uint32_t mis = 0, ne = 0;
            if constexpr (KT::is_record) {
#pragma unroll
                for (uint32_t j = 0; j < IPT; j++) {
                    const K k = KT::key(blk[j * NT + tid]);
                    const bool left = P.mode ? !(pk < k) : (k < pk);
                    ne += !(k < pk) && !(pk < k);
                    mis |= (uint32_t)(side == 0 ? !left : left) << j;
                }
            } else {
                const uint4 *v4 = reinterpret_cast<const uint4 *>(blk);
#pragma unroll
                for (uint32_t j = 0; j < IPT / VW; j++) {
                    const uint4 u = v4[j * NT + tid];
                    T x[VW];
                    memcpy(x, &u, 16);
#pragma unroll
                    for (uint32_t q = 0; q < VW; q++) {
                        const K k = KT::key(x[q]);
                        const bool left = P.mode ? !(pk < k) : (k < pk);
                        ne += !(k < pk) && !(pk < k);
                        mis |= (uint32_t)(side == 0 ? !left : left) << (j * VW + q);
                    }
                }
            }
            // one warp scan carries both counts: misplaced (low half, a
            // prefix) and equal to p (high half, only the warp total is used);
            // each is <= 32 * IPT <= 1024 per warp
            const uint32_t cnt = __popc(mis);
            uint32_t inc = cnt | (ne << 16);
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= (uint32_t)d) inc += o;
            }
            if (lane == 31) {
                const uint32_t we = inc >> 16;
                sm.wsum[warp] = inc & 0xffffu;
                sm.weq[warp] = we;
                if (we) atomicAdd(&st->n_equal, (unsigned long long)we);
            }
            inc &= 0xffffu;
            __syncthreads();
            uint32_t pre = 0, tot = 0;
#pragma unroll
            for (uint32_t w2 = 0; w2 < NW; w2++) {
                const uint32_t v = sm.wsum[w2];
                pre += w2 < warp ? v : 0;
                tot += v;
            }
            uint32_t r = pre + inc - cnt;
#pragma unroll
            for (uint32_t jj = 0; jj < IPT; jj++) {
                const uint32_t e = KT::is_record ? jj * NT + tid : ((jj / VW) * NT + tid) * VW + jj % VW;
                if ((mis >> jj) & 1) sm.off[side][r] = (uint16_t)e;
                r += (mis >> jj) & 1;
            }
            if (tid == 0) {
                sm.start[side] = 0;
                sm.num[side] = tot;
                sm.dirty[side] = 0;
                sm.fresh[side] = 0;
                uint32_t eq = 0;
                for (uint32_t w2 = 0; w2 < NW; w2++) eq += sm.weq[w2];
                sm.eqcnt[side] = eq;
            }
            __syncthreads();
        }
        const uint32_t bL = sm.slot[0], bR = sm.slot[1];
        if (bL == 3 || bR == 3) break;   // one side is exhausted (uniform)

        // rearrangement phase (l.19-21): swap num = min(num_L, num_R) pairs
        const uint32_t nL = sm.num[0], nR = sm.num[1], sL = sm.start[0], sR = sm.start[1];
        const uint32_t num = nL < nR ? nL : nR;
        const bool e0 = nL == num, e1 = nR == num;   // sides neutralized by this round
        const int pf = e0 ? 0 : 1;
        uint32_t pf_blk = IP_NONE;
        if (tid == 0) {
            // claim the next block of the side about to be neutralized and
            // stream it into the spare buffer while the swaps run
            pf_blk = ip_claim(st, pf);
            if (pf_blk != IP_NONE) {
                const uint32_t sp = sm.spare;
                bulk_wait_read0();   // the spare's last write-back has left shared memory
                sm.blk[sp] = pf_blk;
                mbar_arrive_expect_tx(&sm.bar[sp], BYTES);
                tma_load_1d(sm.buf[sp], base + (uint64_t)pf_blk * TILE, BYTES, &sm.bar[sp]);
            }
        }
        T *L = sm.buf[bL];
        T *R = sm.buf[bR];
        uint32_t eq_in = 0;   // keys equal to p moving into the right block (mode 0)
        for (uint32_t q = tid; q < num; q += NT) {
            const uint32_t a = sm.off[0][sL + q], c = sm.off[1][sR + q];
            const T t0 = L[a];
            L[a] = R[c];
            R[c] = t0;
            const K k0 = KT::key(t0);
            eq_in += !(k0 < pk) && !(pk < k0);
        }
        if (P.eqpos) {
            eq_in = __reduce_add_sync(0xffffffffu, eq_in);
            if (lane == 0 && eq_in) atomicAdd(&sm.eqcnt[1], eq_in);
        }
        fence_proxy_async_smem();   // the swaps become visible to the bulk stores
        __syncthreads();
        if (P.eqpos && e1 && sm.eqcnt[1]) {
            // the neutralized right block is final: record where its keys equal
            // to p sit, so the equal band needs no scan of the right part
            const uint32_t rb = sm.blk[bR];
            for (uint32_t j0 = 0; j0 < TILE; j0 += NT) {
                const uint32_t j = j0 + tid;
                const K kk = KT::key(R[j]);
                const bool eq = !(kk < pk) && !(pk < kk);
                const uint32_t m = __ballot_sync(0xffffffffu, eq);
                if (!m) continue;
                uint32_t b0 = 0;
                if (lane == 0) b0 = atomicAdd(&st->neqpos, (uint32_t)__popc(m));
                b0 = __shfl_sync(0xffffffffu, b0, 0) + __popc(m & lanemask_lt());
                if (eq && b0 < P.eqcap) P.eqpos[b0] = ((uint64_t)rb << 32) | j;
            }
            __syncthreads();   // R is refilled below only after these reads
        }
        if (tid == 0) {
            // l.24-27: a neutralized block is final — written back if a swap touched it
            const uint32_t d0 = sm.dirty[0] | (num > 0), d1 = sm.dirty[1] | (num > 0);
            if (e0 && d0) tma_store_1d(base + (uint64_t)sm.blk[bL] * TILE, L, BYTES);
            if (e1 && d1) tma_store_1d(base + (uint64_t)sm.blk[bR] * TILE, R, BYTES);
            bulk_commit();
            sm.dirty[0] = d0;
            sm.dirty[1] = d1;
            for (int side = 0; side < 2; side++) {
                sm.start[side] += num;
                sm.num[side] -= num;
            }
            const uint32_t old = sm.slot[pf];
            if (pf_blk != IP_NONE) {
                sm.slot[pf] = sm.spare;
                sm.fresh[pf] = 1;
            } else {
                sm.slot[pf] = 3;
            }
            sm.spare = old;
            if (pf == 0 && e1) {
                // both sides neutralized: the right one refills in place
                const uint32_t got = pf_blk != IP_NONE ? ip_claim(st, 1) : IP_NONE;
                if (got == IP_NONE) {
                    sm.slot[1] = 3;
                } else {
                    bulk_wait_read0();
                    sm.blk[bR] = got;
                    sm.fresh[1] = 1;
                    mbar_arrive_expect_tx(&sm.bar[bR], BYTES);
                    tma_load_1d(R, base + (uint64_t)got * TILE, BYTES, &sm.bar[bR]);
                }
            }
        }
        __syncthreads();
    }
    // the block still held (at most one) is the cleanup's: written back if
    // modified, its keys equal to p recounted there
    for (int side = 0; side < 2; side++) {
        const uint32_t b = sm.slot[side];
        if (b == 3) continue;
        const T *blk = sm.buf[b];
        uint32_t ne = 0;
#pragma unroll
        for (uint32_t j = 0; j < IPT; j++) {
            const K k = KT::key(blk[j * NT + tid]);
            ne += !(k < pk) && !(pk < k);
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) ne += __shfl_xor_sync(0xffffffffu, ne, d);
        if (lane == 0 && ne) atomicAdd(&st->n_equal_held, (unsigned long long)ne);
        if (tid == 0) {
            if (sm.dirty[side]) tma_store_1d(base + (uint64_t)sm.blk[b] * TILE, blk, BYTES);
            bulk_commit();
            const uint32_t k = atomicAdd(&st->nleftover, 1u);
            P.leftover[2 * k] = sm.blk[b];
            P.leftover[2 * k + 1] = side;
        }
    }
    if (tid == 0) bulk_wait0();
}

// ---- the pass's set-up and cleanup (Alg. 3 l.29), all on the device ----------

// the range of pass k: [0, n) for pass 0; for pass 1 (the equal band) the
// right part of pass 0, if pass 0 met keys equal to p
template <class KT>
__global__ void k_ip_setup(const typename KT::T *data, IpPass *ps, const IpPass *prev, uint64_t n,
                           uint64_t list_cap, uint32_t eqcap) {
    using T = typename KT::T;
    constexpr uint32_t TILE = ip_tile<KT>();
    IpPass q;
    memset(&q, 0, sizeof q);
    if (prev == nullptr) {
        q.off = 0;
        q.active = n > 0;
    } else {
        // the equal band: by compaction when its size fits the lists,
        // otherwise by a second block pass with mode 1 (left <=> key <= p)
        q.off = prev->n_left;
        const bool any = prev->active && prev->n_eq > 0;
        q.compact = any && prev->n_eq <= list_cap;
        q.active = any && !q.compact;
        q.n_eq = prev->n_eq;
        q.fast_eq = q.compact && prev->st.neqpos <= eqcap;
    }
    q.len = n - q.off;
    const uint64_t mis16 = (uintptr_t)(data + q.off) & 15;
    uint64_t h = mis16 ? (16 - mis16) / sizeof(T) : 0;
    q.h = h < q.len ? h : q.len;
    q.nb = (uint32_t)((q.len - q.h) / TILE);
    q.st.claim = ((unsigned long long)(IP_BIAS + q.nb) << 32) | IP_BIAS;
    q.n_left = q.compact ? q.off + q.n_eq : q.off;
    *ps = q;
}

// where the leftover blocks go: the left ones to [X - a, X), the right ones
// to [X, X + c), each swapping with a neutralized block found there
template <class KT, int NT>
__global__ void __launch_bounds__(NT) k_ip_plan(IpPass *ps, const uint32_t *leftover, uint32_t *pairs,
                                                 uint64_t *eqpos, uint32_t eqcap) {
    constexpr uint32_t TILE = ip_tile<KT>();
    __shared__ uint8_t win[IP_GMAX];
    __shared__ uint32_t cnt[2], nout[2], nin[2];
    const uint32_t tid = threadIdx.x;
    if (!ps->active) return;
    const uint32_t X = ps->st.left_ok, k = ps->st.nleftover;
    if (tid < 2) cnt[tid] = nout[tid] = nin[tid] = 0;
    for (uint32_t j = tid; j < IP_GMAX; j += NT) win[j] = 0;
    __syncthreads();
    for (uint32_t i = tid; i < k; i += NT) atomicAdd(&cnt[leftover[2 * i] < X ? 0 : 1], 1u);
    __syncthreads();
    const uint32_t a = cnt[0], c = cnt[1];
    uint32_t *pl = pairs, *pr = pairs + 2 * IP_GMAX;
    for (uint32_t i = tid; i < k; i += NT) {
        const uint32_t b = leftover[2 * i];
        if (b < X) {
            if (b >= X - a) win[b - (X - a)] = 1;
            else pl[2 * atomicAdd(&nout[0], 1u)] = b;
        } else {
            if (b < X + c) win[a + (b - X)] = 1;
            else pr[2 * atomicAdd(&nout[1], 1u)] = b;
        }
    }
    __syncthreads();
    for (uint32_t j = tid; j < a + c; j += NT) {
        if (win[j]) continue;
        if (j < a) pl[2 * atomicAdd(&nin[0], 1u) + 1] = X - a + j;
        else pr[2 * atomicAdd(&nin[1], 1u) + 1] = X + (j - a);
    }
    __syncthreads();
    const uint32_t mL = nout[0], mR = nout[1];
    if (eqpos) {
        // recorded positions of keys equal to p follow their block when it
        // moves out of the right window (it swaps with a leftover)
        __shared__ uint32_t newblk[IP_GMAX];
        for (uint32_t q = tid; q < mR; q += NT) newblk[pr[2 * q + 1] - X] = pr[2 * q];
        __syncthreads();
        const uint32_t ne = ps->st.neqpos < eqcap ? ps->st.neqpos : eqcap;
        for (uint32_t i = tid; i < ne; i += NT) {
            const uint64_t e = eqpos[i];
            const uint32_t b = (uint32_t)(e >> 32);
            if (b >= X && b < X + c) eqpos[i] = ((uint64_t)newblk[b - X] << 32) | (uint32_t)e;
        }
    }
    for (uint32_t i = tid; i < 2 * mR; i += NT) pairs[2 * mL + i] = pr[i];   // right pairs after the left ones
    if (tid == 0) {
        ps->npairs = mL + mR;
        ps->o1 = ps->h + (uint64_t)(X - a) * TILE;
        ps->n1 = (uint64_t)(a + c) * TILE;
        ps->o2 = ps->h + (uint64_t)ps->nb * TILE;
        ps->tail = ps->len - ps->o2;
        ps->v = ps->h + ps->n1 + ps->tail;
    }
}

// block pairs (a, b) swap their contents
template <class KT, int NT, int IPT>
__global__ void __launch_bounds__(NT) k_swap_blocks(typename KT::T *data, const IpPass *ps, const uint32_t *pairs) {
    using T = typename KT::T;
    constexpr uint32_t TILE = NT * IPT;
    if (!ps->active) return;
    T *base = data + ps->off + ps->h;
    for (uint32_t q = blockIdx.x; q < ps->npairs; q += gridDim.x) {
        T *a = base + (uint64_t)pairs[2 * q] * TILE;
        T *b = base + (uint64_t)pairs[2 * q + 1] * TILE;
        for (uint32_t j = threadIdx.x; j < TILE; j += NT) {
            const T x = a[j];
            a[j] = b[j];
            b[j] = x;
        }
    }
}

// the buffer back into the head, middle and tail positions (dir 1), or the reverse
template <class KT>
__global__ void k_gather3(typename KT::T *data, typename KT::T *buf, const IpPass *ps, int dir) {
    if (!ps->active) return;
    typename KT::T *base = data + ps->off;
    const uint64_t h = ps->h, n1 = ps->n1, o1 = ps->o1, o2 = ps->o2, v = ps->v;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < v; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t g = i < h ? i : i < h + n1 ? o1 + (i - h) : o2 + (i - h - n1);
        if (dir == 0) buf[i] = base[g];
        else base[g] = buf[i];
    }
}

// two-way split of the head, middle and tail into [left | right] in a buffer
// (their order is free): chunks of NT*IPT, one cursor claim per side and chunk
template <class KT, int NT, int IPT>
__global__ void __launch_bounds__(NT) k_vsplit(const typename KT::T *data, typename KT::T *dst, IpPass *ps,
                                                uint64_t pivot, int mode) {
    using T = typename KT::T;
    using K = typename KT::K;
    constexpr uint32_t CH = NT * IPT, NW = NT / 32;
    __shared__ uint32_t wl[NW], we[NW];
    __shared__ unsigned long long lb, rb;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (!ps->active) return;
    const uint64_t v = ps->v, h = ps->h, n1 = ps->n1, o1 = ps->o1, o2 = ps->o2;
    const T *src = data + ps->off;   // gathered on the fly: head, middle, tail
    const K pk = (K)pivot;
    for (uint64_t c0 = (uint64_t)blockIdx.x * CH; c0 < v; c0 += (uint64_t)gridDim.x * CH) {
        T x[IPT];
        uint32_t lf = 0, vm = 0, ne = 0;
#pragma unroll
        for (uint32_t j = 0; j < IPT; j++) {
            const uint64_t i = c0 + j * NT + tid;
            if (i < v) {
                x[j] = src[i < h ? i : i < h + n1 ? o1 + (i - h) : o2 + (i - h - n1)];
                const K k = KT::key(x[j]);
                const bool left = mode ? !(pk < k) : (k < pk);
                lf |= (uint32_t)left << j;
                vm |= 1u << j;
                ne += !(k < pk) && !(pk < k);
            }
        }
        // warp-contiguous runs (ballots), so that the writes coalesce: the
        // warp's left / right totals first, then the CTA's bases
        uint32_t nl = 0, nr = 0;
#pragma unroll
        for (uint32_t j = 0; j < IPT; j++) {
            const uint32_t bl = __ballot_sync(0xffffffffu, (lf >> j) & 1), bv = __ballot_sync(0xffffffffu, (vm >> j) & 1);
            nl += __popc(bl);
            nr += __popc(bv & ~bl);
        }
        ne = __reduce_add_sync(0xffffffffu, ne);
        if (lane == 0) { wl[warp] = nl; we[warp] = nr; }
        __syncthreads();
        uint32_t pl = 0, pr = 0, tl = 0, tr = 0;
#pragma unroll
        for (uint32_t w2 = 0; w2 < NW; w2++) {
            pl += w2 < warp ? wl[w2] : 0;
            pr += w2 < warp ? we[w2] : 0;
            tl += wl[w2];
            tr += we[w2];
        }
        if (lane == 0 && ne) atomicAdd(&ps->ev, (unsigned long long)ne);
        if (tid == 0) {
            lb = tl ? atomicAdd(&ps->lcur, (unsigned long long)tl) : 0;
            rb = tr ? atomicAdd(&ps->rcur, (unsigned long long)tr) : 0;
        }
        __syncthreads();
        uint64_t ol = lb + pl, orr = rb + pr;
        const uint32_t lt = lanemask_lt();
#pragma unroll
        for (uint32_t j = 0; j < IPT; j++) {
            const bool isl = (lf >> j) & 1, isv = (vm >> j) & 1;
            const uint32_t bl = __ballot_sync(0xffffffffu, isl), br = __ballot_sync(0xffffffffu, isv && !isl);
            if (isl) dst[ol + __popc(bl & lt)] = x[j];
            else if (isv) dst[v - 1 - (orr + __popc(br & lt))] = x[j];
            ol += __popc(bl);
            orr += __popc(br);
        }
        __syncthreads();   // wl/we/lb/rb are reused by the next chunk
    }
}

// the split lands in the head, middle and tail positions in that order; two
// cases leave right keys inside the left part, fixed by one range swap:
// the head ends in right keys while left blocks follow (lv < h), or the left
// part spills from the middle into the tail past right blocks.  Then the
// pass's results.
template <class KT, int NT>
__global__ void __launch_bounds__(NT) k_ip_fix(typename KT::T *data, IpPass *ps) {
    using T = typename KT::T;
    if (!ps->active) return;
    T *base = data + ps->off;
    const uint64_t lv = ps->lcur, h = ps->h, o1 = ps->o1, n1 = ps->n1, o2 = ps->o2;
    uint64_t a = 0, b = 0, e = 0;
    if (lv < h) {
        if (o1 > h) { e = h - lv; a = lv; b = o1 - e; }
    } else if (lv - h > n1 && o1 + n1 < o2) {
        e = lv - h - n1; a = o1 + n1; b = o2;
    }
    for (uint64_t i = threadIdx.x; i < e; i += NT) {
        const T x = base[a + i];
        base[a + i] = base[b + i];
        base[b + i] = x;
    }
    if (threadIdx.x == 0) {
        ps->n_left = ps->off + o1 - h + lv;
        ps->n_eq = ps->st.n_equal - ps->st.n_equal_held + ps->ev;
    }
}

// ---- the equal band by compaction ---------------------------------------------
// The right part R = data[off, off + len) of pass 0 holds only keys >= p, and
// n_eq of them equal p.  The band is R's first n_eq positions: every key > p
// there (list G) swaps with a key = p found past it (list E); |G| = |E|.
// One read of R, then 2|G| element moves.

// append this thread's hits (bit b of `mask` <-> position pos0(b)) to a list,
// one atomic per warp
template <class F>
__device__ __forceinline__ void warp_append(uint32_t mask, uint32_t lane, unsigned long long *ctr, uint32_t *list,
                                            F pos_of) {
    const uint32_t cnt = __popc(mask);
    uint32_t inc = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= (uint32_t)d) inc += o;
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
    if (tot == 0) return;
    unsigned long long b = 0;
    if (lane == 31) b = atomicAdd(ctr, (unsigned long long)tot);
    b = __shfl_sync(0xffffffffu, b, 31);
    uint64_t r = b + inc - cnt;
    while (mask) {
        const uint32_t bit = __ffs(mask) - 1;
        mask &= mask - 1;
        list[r++] = pos_of(bit);
    }
}

template <class KT, int NT>
__global__ void __launch_bounds__(NT) k_eq_scan(const typename KT::T *data, IpPass *ps, uint64_t pivot, uint32_t *E,
                                                 uint32_t *G) {
    using T = typename KT::T;
    using K = typename KT::K;
    if (!ps->compact || ps->fast_eq) return;
    const K pk = (K)pivot;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t off = ps->off, len = ps->len, band = ps->n_eq;
    const T *R = data + off;
    if constexpr (KT::is_record) {
        const uint64_t step = (uint64_t)gridDim.x * NT;
        for (uint64_t i0 = (uint64_t)blockIdx.x * NT; i0 < len; i0 += step) {
            const uint64_t i = i0 + threadIdx.x;
            uint32_t me = 0, mg = 0;
            if (i < len) {
                const K k = KT::key(R[i]);
                const bool eq = !(k < pk) && !(pk < k);
                mg = i < band && !eq;
                me = i >= band && eq;
            }
            if (__any_sync(0xffffffffu, me | mg)) {
                warp_append(me, lane, &ps->cnt_eq, E, [&](uint32_t) { return (uint32_t)i; });
                warp_append(mg, lane, &ps->cnt_gt, G, [&](uint32_t) { return (uint32_t)i; });
            }
        }
    } else {
        // 16-byte units from the aligned address at or below R; bit r*U+q of
        // a mask is key q of the thread's unit r
        constexpr uint32_t W = sizeof(T), U = 16 / W, UNR = 4, FULL = (1u << U) - 1;
        const uintptr_t a0 = (uintptr_t)R & ~(uintptr_t)15;
        const int64_t skew = (int64_t)(((uintptr_t)R - a0) / W);   // elements of the first unit before R
        const uint64_t units = (len + skew + U - 1) / U;
        const uint4 *V = reinterpret_cast<const uint4 *>(a0);
        const uint64_t step = (uint64_t)gridDim.x * NT * UNR;
        for (uint64_t u0 = (uint64_t)blockIdx.x * NT * UNR; u0 < units; u0 += step) {
            uint4 x[UNR];
#pragma unroll
            for (uint32_t r = 0; r < UNR; r++) {
                const uint64_t u = u0 + r * NT + threadIdx.x;
                x[r] = u < units ? __ldcs(V + u) : make_uint4(0, 0, 0, 0);
            }
            uint32_t me = 0, mg = 0;
#pragma unroll
            for (uint32_t r = 0; r < UNR; r++) {
                const uint64_t u = u0 + r * NT + threadIdx.x;
                if (u >= units) continue;
                T e[U];
                memcpy(e, &x[r], 16);
                uint32_t eqb = 0;
#pragma unroll
                for (uint32_t q = 0; q < U; q++) {
                    const K k = KT::key(e[q]);
                    eqb |= (uint32_t)(!(k < pk) && !(pk < k)) << q;
                }
                const int64_t i0 = (int64_t)(u * U) - skew;   // index of key 0 of the unit
                uint32_t valid = FULL, inband;
                if (i0 < 0 || i0 + U > len) {
                    valid = 0;
#pragma unroll
                    for (uint32_t q = 0; q < U; q++) valid |= (uint32_t)(i0 + q >= 0 && (uint64_t)(i0 + q) < len) << q;
                }
                if (i0 + (int64_t)U <= (int64_t)band) inband = FULL;
                else if (i0 >= (int64_t)band) inband = 0;
                else {
                    inband = 0;
#pragma unroll
                    for (uint32_t q = 0; q < U; q++) inband |= (uint32_t)(i0 + (int64_t)q < (int64_t)band) << q;
                }
                me |= (eqb & ~inband & valid) << (r * U);
                mg |= (~eqb & inband & valid & FULL) << (r * U);
            }
            if (__any_sync(0xffffffffu, me | mg)) {
                auto pos = [&](uint32_t bit) {
                    return (uint32_t)((int64_t)((u0 + (bit / U) * NT + threadIdx.x) * U + bit % U) - skew);
                };
                warp_append(me, lane, &ps->cnt_eq, E, pos);
                warp_append(mg, lane, &ps->cnt_gt, G, pos);
            }
        }
    }
}

// The equal band from pass 0's records (fast_eq): the right part's keys
// equal to p sit at recorded positions in the neutralized right blocks, or in
// the cleanup's ranges (the middle's right part with the fixed-up head, and
// the tail); only those, and the band itself, are read.
template <class KT, int NT>
__global__ void __launch_bounds__(NT) k_eq_scan2(const typename KT::T *data, IpPass *ps, const IpPass *p0,
                                                  uint64_t pivot, uint32_t *E, uint32_t *G, const uint64_t *eqpos,
                                                  uint32_t eqcap) {
    using K = typename KT::K;
    if (!ps->fast_eq) return;
    constexpr uint32_t TILE = ip_tile<KT>();
    const K pk = (K)pivot;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nl = ps->off, band_end = nl + ps->n_eq, n = p0->off + p0->len;
    const uint64_t h0 = p0->h, o1 = p0->o1, n1 = p0->n1, o2 = p0->o2, lv = p0->lcur;
    const uint64_t e_spill = (lv >= h0 && lv - h0 > n1 && o1 + n1 < o2) ? lv - h0 - n1 : 0;
    // element ranges, in pass 0's coordinates: S1 = [nl, o1+n1), S2 = [max(o2,
    // nl), n), S3 = the band's part between them
    const uint64_t s1b = nl, s1e = (o1 + n1 > nl) ? o1 + n1 : nl;
    const uint64_t s2b = o2 > nl ? o2 : nl, s2e = n;   // the tail's right part
    const uint64_t s3b = s1e, s3e = band_end < o2 ? (band_end > s1e ? band_end : s1e) : (o2 > s1e ? o2 : s1e);
    const uint64_t l1 = s1e - s1b, l2 = s2e - s2b, l3 = s3e - s3b;
    const uint32_t nrec = p0->st.neqpos < eqcap ? p0->st.neqpos : eqcap;
    const uint64_t total = l1 + l2 + l3 + nrec;
    const uint64_t step = (uint64_t)gridDim.x * NT;
    for (uint64_t i0 = (uint64_t)blockIdx.x * NT; i0 < total; i0 += step) {
        const uint64_t q = i0 + threadIdx.x;
        uint32_t me = 0, mg = 0;
        uint64_t idx = 0;
        if (q < l1 + l2 + l3) {
            idx = q < l1 ? s1b + q : q < l1 + l2 ? s2b + (q - l1) : s3b + (q - l1 - l2);
            const K kk = KT::key(data[idx]);
            const bool eq = !(kk < pk) && !(pk < kk);
            mg = idx < band_end && !eq;
            me = idx >= band_end && eq;
        } else if (q < total) {
            const uint64_t e = eqpos[q - l1 - l2 - l3];
            idx = h0 + (e >> 32) * TILE + (uint32_t)e;
            const bool moved = e_spill && idx >= o1 + n1 && idx < o1 + n1 + e_spill;
            me = idx >= band_end && !moved;
        }
        if (__any_sync(0xffffffffu, me | mg)) {
            warp_append(me, lane, &ps->cnt_eq, E, [&](uint32_t) { return (uint32_t)(idx - nl); });
            warp_append(mg, lane, &ps->cnt_gt, G, [&](uint32_t) { return (uint32_t)(idx - nl); });
        }
    }
}

template <class KT>
__global__ void k_eq_swap(typename KT::T *data, const IpPass *ps, const uint32_t *E, const uint32_t *G) {
    using T = typename KT::T;
    if (!ps->compact) return;
    T *R = data + ps->off;
    const uint64_t m = ps->cnt_eq < ps->cnt_gt ? ps->cnt_eq : ps->cnt_gt;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        T *a = R + E[i], *b = R + G[i];
        const T x = *a;
        *a = *b;
        *b = x;
    }
}

}  // namespace bq
