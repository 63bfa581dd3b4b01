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
// The host then (run_partition_inplace, driver.cuh) swaps the leftover
// blocks into the middle of the range, partitions the middle (<= #CTAs + 1
// blocks: "compare and rearrange remaining elements", l.29) out of place in
// a small buffer, and repeats on the right part for the equal band.
#pragma once

namespace bq {

// claim-word bias: lo and hi start at IP_BIAS and IP_BIAS + #blocks
constexpr uint32_t IP_BIAS = 1u << 30;

struct InplaceState {
    unsigned long long claim;        // lo: next left block, hi: end of the right blocks
    unsigned long long n_equal;      // keys equal to the pivot in the neutralized blocks
    uint32_t nleftover;              // blocks a CTA held when its partner side ran out
    uint32_t left_ok;                // blocks claimed from the left (= the meeting point)
    uint32_t pad[10];
};
static_assert(sizeof(InplaceState) == 64, "InplaceState layout");

template <class KT>
struct InplaceParams {
    using T = typename KT::T;
    T *base;                 // range start (any alignment of the element type)
    uint32_t nblk;           // full blocks in the range
    uint64_t pivot;          // pivot key (KT::K)
    int mode;                // 0: left <=> key < p; 1: left <=> key <= p
    InplaceState *st;
    uint32_t *leftover;      // [2 * k]: block index, side (0 left, 1 right)
};

template <class KT, int NT, int IPT>
struct InplaceSmem {
    using T = typename KT::T;
    static constexpr int TILE = NT * IPT;
    static constexpr int NW = NT / 32;
    T blk[2][TILE];                   // [0]: left block, [1]: right block
    uint16_t off[2][TILE];            // offsets buffers of their misplaced elements
    uint32_t wsum[NW];
    uint32_t idx[2], start[2], num[2], done[2];
};

template <class KT>
constexpr int inplace_smem_bytes() {
    return (int)sizeof(InplaceSmem<KT, Tune<KT>::PART_THREADS, Tune<KT>::PART_IPT>);
}

template <class KT, int NT, int IPT>
__global__ void __launch_bounds__(NT) k_inplace(InplaceParams<KT> P) {
    using T = typename KT::T;
    using K = typename KT::K;
    using SM = InplaceSmem<KT, NT, IPT>;
    constexpr uint32_t TILE = SM::TILE, NW = SM::NW;
    static_assert(TILE <= 65536, "16-bit offsets");
    extern __shared__ __align__(128) unsigned char smraw[];
    SM &sm = *reinterpret_cast<SM *>(smraw);
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const K pk = (K)P.pivot;
    if (tid == 0) {
        sm.idx[0] = sm.idx[1] = 0xffffffffu;
        sm.done[0] = sm.done[1] = 0;
        sm.num[0] = sm.num[1] = 0;
    }
    __syncthreads();

    for (;;) {
        // refill the empty side(s): claim, load, scan (Alg. 3 l.5-18)
        for (int side = 0; side < 2; side++) {
            if (sm.idx[side] != 0xffffffffu || sm.done[side]) continue;   // uniform
            __syncthreads();
            if (tid == 0) {
                // one fetch-and-add on the packed word decides the claim; a
                // failed claim moves lo past hi (or hi below lo), which keeps
                // failing — IP_BIAS keeps both halves clear of wrap-around
                // (at most one failure per CTA and side)
                uint32_t got = 0xffffffffu;
                const unsigned long long old =
                    atomicAdd(&P.st->claim, side == 0 ? 1ull : 0xffffffff00000000ull);   // lo += 1 | hi -= 1
                const uint32_t lo = (uint32_t)old, hi = (uint32_t)(old >> 32);
                if (lo < hi) {
                    got = (side == 0 ? lo : hi - 1) - IP_BIAS;
                    if (side == 0) atomicAdd(&P.st->left_ok, 1u);
                }
                if (got == 0xffffffffu) sm.done[side] = 1;
                sm.idx[side] = got;
            }
            __syncthreads();
            const uint32_t b = sm.idx[side];
            if (b == 0xffffffffu) continue;
            const T *g = P.base + (uint64_t)b * TILE;
            T x[IPT];
#pragma unroll
            for (uint32_t j = 0; j < IPT; j++) x[j] = g[j * NT + tid];   // coalesced
            // misplaced: on the left side elements that belong right, and vice versa
            uint32_t mis = 0;
#pragma unroll
            for (uint32_t j = 0; j < IPT; j++) {
                const K k = KT::key(x[j]);
                const bool left = P.mode ? !(pk < k) : (k < pk);
                mis |= (uint32_t)(side == 0 ? !left : left) << j;
                sm.blk[side][j * NT + tid] = x[j];
            }
            const uint32_t cnt = __popc(mis);
            uint32_t inc = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= (uint32_t)d) inc += o;
            }
            if (lane == 31) sm.wsum[warp] = inc;
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
            for (uint32_t j = 0; j < IPT; j++) {
                // the offset is formed for every element; the buffer grows by the flag
                if ((mis >> j) & 1) sm.off[side][r] = (uint16_t)(j * NT + tid);
                r += (mis >> j) & 1;
            }
            if (tid == 0) {
                sm.start[side] = 0;
                sm.num[side] = tot;
            }
            __syncthreads();
        }
        const bool hl = sm.idx[0] != 0xffffffffu, hr = sm.idx[1] != 0xffffffffu;
        if (!(hl && hr)) break;   // one side is exhausted (uniform)

        // rearrangement phase (l.19-21): swap num = min(num_L, num_R) pairs
        const uint32_t nL = sm.num[0], nR = sm.num[1], sL = sm.start[0], sR = sm.start[1];
        const uint32_t num = nL < nR ? nL : nR;
        for (uint32_t q = tid; q < num; q += NT) {
            const uint32_t a = sm.off[0][sL + q], c = sm.off[1][sR + q];
            const T t0 = sm.blk[0][a];
            sm.blk[0][a] = sm.blk[1][c];
            sm.blk[1][c] = t0;
        }
        __syncthreads();
        // l.24-27: advance; a side whose buffer ran empty is written back
        for (int side = 0; side < 2; side++) {
            const uint32_t left_now = (side == 0 ? nL : nR) - num;
            if (left_now == 0) {
                // neutralized: final in place; its keys equal to p are counted
                // here (the middle blocks are counted by the cleanup)
                T *g = P.base + (uint64_t)sm.idx[side] * TILE;
                uint32_t ne = 0;
#pragma unroll
                for (uint32_t j = 0; j < IPT; j++) {
                    const T x = sm.blk[side][j * NT + tid];
                    const K k = KT::key(x);
                    ne += !(k < pk) && !(pk < k);
                    g[j * NT + tid] = x;
                }
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) ne += __shfl_xor_sync(0xffffffffu, ne, d);
                if (lane == 0 && ne) atomicAdd(&P.st->n_equal, (unsigned long long)ne);
            }
        }
        __syncthreads();
        if (tid == 0) {
            for (int side = 0; side < 2; side++) {
                sm.num[side] -= num;
                sm.start[side] += num;
                if (sm.num[side] == 0) sm.idx[side] = 0xffffffffu;
            }
        }
        __syncthreads();
    }
    // the block still held (at most one) goes back as is and is listed
    for (int side = 0; side < 2; side++) {
        const uint32_t b = sm.idx[side];
        if (b == 0xffffffffu) continue;
        T *g = P.base + (uint64_t)b * TILE;
#pragma unroll
        for (uint32_t j = 0; j < IPT; j++) g[j * NT + tid] = sm.blk[side][j * NT + tid];
        if (tid == 0) {
            const uint32_t k = atomicAdd(&P.st->nleftover, 1u);
            P.leftover[2 * k] = b;
            P.leftover[2 * k + 1] = side;
        }
    }
}

// block pairs (a, b) of the range swap their contents (one CTA per pair)
template <class KT, int NT, int IPT>
__global__ void __launch_bounds__(NT) k_swap_blocks(typename KT::T *base, const uint32_t *pairs) {
    using T = typename KT::T;
    constexpr uint32_t TILE = NT * IPT;
    T *a = base + (uint64_t)pairs[2 * blockIdx.x] * TILE;
    T *b = base + (uint64_t)pairs[2 * blockIdx.x + 1] * TILE;
    for (uint32_t j = threadIdx.x; j < TILE; j += NT) {
        const T x = a[j];
        a[j] = b[j];
        b[j] = x;
    }
}

// copy two ranges of `base` into one contiguous buffer (dir 0) or back (dir 1)
template <class KT>
__global__ void k_gather2(typename KT::T *base, typename KT::T *buf, uint64_t o1, uint64_t n1, uint64_t o2,
                          uint64_t n2, int dir) {
    const uint64_t n = n1 + n2;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t g = i < n1 ? o1 + i : o2 + (i - n1);
        if (dir == 0) buf[i] = base[g];
        else base[g] = buf[i];
    }
}

// swap base[a + i] <-> base[b + i] for i < len (the spill of the middle's left part)
template <class KT>
__global__ void k_swap_ranges(typename KT::T *base, uint64_t a, uint64_t b, uint64_t len) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (uint64_t)gridDim.x * blockDim.x) {
        const typename KT::T x = base[a + i];
        base[a + i] = base[b + i];
        base[b + i] = x;
    }
}

}  // namespace bq
