// driver.cuh — host driver of the hot path (H8): workspace layout, the
// single-pass partition, and the breadth-first level loop that replaces the
// paper's recursion / explicit stack.
//
// Level loop (one iteration per recursion level, all segments of the level at
// once):
//   k_partition  a2-a5 for every tile of every segment of the level
//   k_post       one CTA per segment: a6 equal band, a7 children -> next level
//                (pivot a1, tile map, cursor) / leaves / fallback
//   one 64-byte counter read-back per level (host decides whether to go on)
//   k_fill       (only if a band was too long for k_post) tile-parallel bands
//   k_leaf       a8 for this level's leaves
// then a9 for depth-capped segments.  Every launch goes to the caller's stream.
#pragma once

#include <algorithm>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "fallback.cuh"
#include "leaf.cuh"
#include "partition.cuh"
#include "loop.cuh"

namespace bq {

constexpr uint32_t POST_GRID = 148 * 8;
constexpr int POST_THREADS = 256;
// the sort's per-level k_post: one small CTA (a warp per child) per segment,
// many resident per SM — deep levels have tens of thousands of segments
#ifndef BQ_POST_LEVEL_THREADS
#define BQ_POST_LEVEL_THREADS 128
#endif
constexpr int POST_LEVEL_THREADS = BQ_POST_LEVEL_THREADS;
constexpr uint32_t POST_LEVEL_GRID = 148 * (2048 / POST_LEVEL_THREADS < 32 ? 2048 / POST_LEVEL_THREADS : 32);

bq_status set_error(bq_status st, const char *fmt, ...);
bq_status check_device();

#define BQ_CK(call)                                                                     \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return ::bq::set_error(BQ_ERR_CUDA, "%s: %s (%s:%d)", #call,                \
                                   cudaGetErrorString(e_), __FILE__, __LINE__);         \
    } while (0)
#define BQ_CK_LAUNCH() BQ_CK(cudaGetLastError())
#define BQ_LAUNCHED(st) ((st).kernel_launches++)

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

template <class KT>
struct Layout {
    size_t scratch, status, tile_map[2], segs[2], cursor[2], ecursor[2], leaves[2], fallback, ctrl, misc, total;
    size_t msegs[2], mtile_map[2], mhist[2], mcursor[2];   // multiway segment lists (N4)
    size_t copies[2], max_copies;                           // records: finished equal runs to copy
    size_t tprefix, fbst;                                   // a9 over the depth-capped segments
    size_t mtab, mblk;                                      // 8-way tile counts and block prefixes
    size_t max_tiles, max_segs, max_leaves, max_fb;
};

// The largest segment a sort of n keys hands to the leaf sort: S for large
// inputs; smaller for small ones, whose few S-sized leaves would leave most
// SMs idle (c1: 64 leaves of ~16 K keys on 148 SMs) — one more 8-way level
// over an L2-resident input costs less than the long leaves it removes.
// A multiple of the leaf classes' sizes, a function of (kind, n) only, so
// bq_workspace_bytes stays one; BQ_LEAF_MAX overrides it (tools/leaf_sweep.py).
template <class KT>
inline uint32_t leaf_max_for(size_t n) {
    constexpr uint32_t S = Tune<KT>::LEAF, C1 = (uint32_t)LeafTraits<KT>::IPT * 64u;
    uint32_t lm = S;
    if (const char *e = std::getenv("BQ_LEAF_MAX")) {
        const long v = std::atol(e);
        if (v > 0) lm = (uint32_t)std::min<long>(std::max<long>(v, C1), S);
    }
    (void)n;
    return lm;
}
inline int batch_extra() {
    if (const char *e = std::getenv("BQ_BATCH_EXTRA")) return std::atoi(e);
    return 1;
}

template <class KT>
Layout<KT> make_layout(size_t n) {
    constexpr size_t TILE = tile_elems<KT>();
    constexpr size_t S0 = Tune<KT>::LEAF;
    const size_t S = leaf_max_for<KT>(n);   // segments of a level are longer than this
    Layout<KT> L;
    // segments of a level are disjoint and longer than S, or (the duplicate
    // check, keys) at least BQ_DC_MIN long
    const size_t seg_min = KT::is_record ? S + 1 : (S + 1 < (size_t)BQ_DC_MIN ? S + 1 : (size_t)BQ_DC_MIN);
    L.max_segs = n / seg_min + 2;
    L.max_tiles = n / TILE + 2 * L.max_segs + 2;
    L.max_fb = n / (S + 1) + 2;
    // the leaf lists of one level (set level & 1): at most kmax children per
    // segment; set 0's class-0 list also holds the fallback's chunks at the end
    const size_t per_level = (mw_capable<KT>() ? MW_K * (n / (S + 1) + 2) : 0) + 2 * L.max_segs;
    L.max_leaves = per_level;
    if (L.max_leaves < n / S0 + L.max_fb + 2) L.max_leaves = n / S0 + L.max_fb + 2;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
    L.scratch = take(n * sizeof(typename KT::T));
    L.status = take(L.max_tiles * sizeof(uint64_t));
    // per-level arrays ping-pong between consecutive levels (k_post writes the
    // next level's while k_fill may still read the current one)
    for (int p = 0; p < 2; p++) {
        L.tile_map[p] = take(L.max_tiles * sizeof(uint32_t));
        L.segs[p] = take(L.max_segs * sizeof(Seg));
        L.cursor[p] = take(L.max_segs * sizeof(unsigned long long));
        L.ecursor[p] = take(L.max_segs * sizeof(uint32_t));
        L.msegs[p] = take(L.max_segs * sizeof(MSeg<KT>));
        L.mtile_map[p] = take(L.max_tiles * sizeof(uint32_t));
        L.mhist[p] = take(MW_K * L.max_segs * sizeof(uint32_t));
        L.mcursor[p] = take(MW_K * L.max_segs * sizeof(uint32_t));
    }
    // per set, one list per leaf class (leaf.cuh), max_leaves each
    L.leaves[0] = take(leaf_nclass<KT>() * L.max_leaves * sizeof(Leaf));
    L.leaves[1] = take(leaf_nclass<KT>() * L.max_leaves * sizeof(Leaf));
    L.fallback = take(L.max_fb * sizeof(Leaf));
    L.max_copies = KT::is_record ? L.max_segs + 2 + n / 65536 + 2 : 1;
    L.copies[0] = take(L.max_copies * sizeof(Leaf));
    L.copies[1] = take(L.max_copies * sizeof(Leaf));
    const size_t mrows = L.max_tiles * mw8w_umin<KT>() + MW8W_ROWS_EXTRA;   // (units of small levels, multiway8w.cuh)
    L.mtab = take(mw_capable<KT>() ? mrows * MW8 * sizeof(uint32_t) : 0);
    L.mblk = take(mw_capable<KT>() ? (mrows / MWS_BR + 2) * MW8 * sizeof(uint32_t) : 0);
    L.tprefix = take((L.max_fb + 1) * sizeof(uint32_t));
    L.fbst = take(sizeof(FbState));
    L.ctrl = take((MAX_LEVELS + 1) * sizeof(LevelCtrl));   // [MAX_LEVELS]: the root's counts
    L.misc = take(256);   // LoopMisc (loop.cuh); bq_pivot_*: the pivot
    L.total = off;
    return L;
}

template <class KT>
struct Kernels {
    static constexpr int NT = Tune<KT>::PART_THREADS;
    static constexpr int IPT = Tune<KT>::PART_IPT;
    static constexpr int STAGES = Tune<KT>::PART_STAGES;
    static constexpr int MINB = Tune<KT>::PART_MINB;
};

// Persistent launch of the partition kernel: min(ntiles, resident CTAs).
template <class KT, bool ORDERED>
bq_status launch_partition_t(const PassParams<KT> &P, cudaStream_t s) {
    using Kn = Kernels<KT>;
    auto kern = k_partition<KT, Kn::NT, Kn::IPT, Kn::STAGES, Kn::MINB, ORDERED>;
    constexpr int smem = part_smem_bytes<KT>();
    constexpr int threads = Kn::NT + (ORDERED ? 96 : 64);
    static CapCache cc;
    int cap = 0;
    BQ_CK(resident_ctas(kern, threads, smem, cc, &cap));
    const uint32_t grid = P.ntiles < (uint32_t)cap ? P.ntiles : (uint32_t)cap;
    kern<<<grid, threads, smem, s>>>(P);
    BQ_CK_LAUNCH();
    return BQ_OK;
}

// The atomic-cursor pass (keys three-way, records two-way by Seg::pad0); the
// standalone pass API keeps records on the ordered (look-back) mode, whose
// equal elements are staged in already-consumed input tiles.
template <class KT>
bq_status launch_partition_fast(const PassParams<KT> &P, cudaStream_t s) {
    using Kn = Kernels<KT>;
    auto kern = k_part_fast<KT, Kn::NT, Kn::IPT, Kn::STAGES, Kn::MINB>;
    constexpr int smem = fast_smem_bytes<KT>();
    constexpr int threads = Kn::NT + 32;
    static CapCache cc;
    int cap = 0;
    BQ_CK(resident_ctas(kern, threads, smem, cc, &cap));
    const uint32_t grid = P.ntiles < (uint32_t)cap ? P.ntiles : (uint32_t)cap;
    kern<<<grid, threads, smem, s>>>(P);
    BQ_CK_LAUNCH();
    return BQ_OK;
}

// resident-CTA capacity of a persistent kernel (cached per kernel)
template <class F>
bq_status persistent_cap(F kern, int threads, int smem, CapCache &cc, int *cap) {
    BQ_CK(resident_ctas(kern, threads, (size_t)smem, cc, cap));
    return BQ_OK;
}

// one multiway level (N4): count, scan, scatter (children by k_post_mw)
template <class KT>
bq_status launch_multiway(MwParams<KT> MP, LevelCtrl *lc, cudaStream_t s, int ways, cudaEvent_t mid = nullptr) {
    using Kn = Kernels<KT>;
    constexpr int threads = Kn::NT + 32;
#if BQ_MW8W
    if (ways == MW8) {   // warp-private tiles, exact offsets (multiway8w.cuh)
        constexpr int IPTW = Mw8wTune<KT>::IPT, smemw = mw8w_smem_bytes<KT>(), tw = MW8W_WARPS * 32;
        auto kc = k_mw8w_count<KT, IPTW>;
        auto ks = k_mw8w_scatter<KT, IPTW>;
        static CapCache cc_c, cc_s;
        int cap_c = 0, cap_s = 0;
        bq_status st = persistent_cap(kc, tw, 0, cc_c, &cap_c);
        if (st != BQ_OK) return st;
        st = persistent_cap(ks, tw, smemw, cc_s, &cap_s);
        if (st != BQ_OK) return st;
        kc<<<cap_c, tw, 0, s>>>(MP);
        BQ_CK_LAUNCH();
        const uint32_t nb = (MP.max_tiles * mw8w_umin<KT>() + MW8W_ROWS_EXTRA + MWS_BR - 1) / MWS_BR;
        k_mw8w_scan<KT><<<nb < 592 ? nb : 592, 256, 0, s>>>(MP);
        BQ_CK_LAUNCH();
        if (mid) BQ_CK(cudaEventRecord(mid, s));   // timing: count + scan | scatter
#if BQ_MW8T
#ifndef BQ_MW8T_PAIR
#define BQ_MW8T_PAIR 1
#endif
        if (MP.aligned && (BQ_MW8T_PAIR || sizeof(typename KT::T) != 16)) {   // bucket runs staged per unit, bulk stores
            constexpr int smemt = mw8t_smem_bytes<KT>();
            auto kt = k_mw8t_scatter<KT, IPTW>;
            static CapCache cc_t;
            int cap_t = 0;
            st = persistent_cap(kt, tw, smemt, cc_t, &cap_t);
            if (st != BQ_OK) return st;
            kt<<<cap_t, tw, smemt, s>>>(MP);
            BQ_CK_LAUNCH();
            return BQ_OK;
        }
#endif
        ks<<<cap_s, tw, smemw, s>>>(MP);
        BQ_CK_LAUNCH();
        return BQ_OK;
    }
#endif
    if (ways == MW8) {
        constexpr int smem8 = mw8_smem_bytes<KT>();
        auto kc8 = k_mw8_count<KT, Kn::NT, Kn::IPT, MW_STAGES, Tune<KT>::MW8_MINB>;
        auto ks8 = k_mw8_scatter<KT, Kn::NT, Kn::IPT, MW_STAGES, Tune<KT>::MW8_MINB>;
        static CapCache cc_c8, cc_s8;
        int cap_c8 = 0, cap_s8 = 0;
        bq_status st = persistent_cap(kc8, threads, smem8, cc_c8, &cap_c8);
        if (st != BQ_OK) return st;
        st = persistent_cap(ks8, threads, smem8, cc_s8, &cap_s8);
        if (st != BQ_OK) return st;
        MP.ticket = lc ? &lc->mw_ticket_count : nullptr;
        MP.ticket_sel = 0;
        kc8<<<cap_c8, threads, smem8, s>>>(MP);
        BQ_CK_LAUNCH();
        k_mw_scan<KT><<<POST_GRID / 8, 256, 0, s>>>(MP);
        BQ_CK_LAUNCH();
        if (mid) BQ_CK(cudaEventRecord(mid, s));
        MP.ticket = lc ? &lc->mw_ticket_scatter : nullptr;
        MP.ticket_sel = 1;
        ks8<<<cap_s8, threads, smem8, s>>>(MP);
        BQ_CK_LAUNCH();
        return BQ_OK;
    }
    constexpr int smem = mw_smem_bytes<KT>();
    auto kc = k_mw_count<KT, Kn::NT, Kn::IPT, MW_STAGES, Kn::MINB>;
    auto ks = k_mw_scatter<KT, Kn::NT, Kn::IPT, MW_STAGES, Kn::MINB>;
    static CapCache cc_c, cc_s;
    int cap_c = 0, cap_s = 0;
    bq_status st = persistent_cap(kc, threads, smem, cc_c, &cap_c);
    if (st != BQ_OK) return st;
    st = persistent_cap(ks, threads, smem, cc_s, &cap_s);
    if (st != BQ_OK) return st;
    MP.ticket = lc ? &lc->mw_ticket_count : nullptr;
    MP.ticket_sel = 0;
    kc<<<cap_c, threads, smem, s>>>(MP);
    BQ_CK_LAUNCH();
    k_mw_scan<KT><<<POST_GRID / 8, 256, 0, s>>>(MP);
    BQ_CK_LAUNCH();
    if (mid) BQ_CK(cudaEventRecord(mid, s));
    MP.ticket = lc ? &lc->mw_ticket_scatter : nullptr;
    MP.ticket_sel = 1;
    ks<<<cap_s, threads, smem, s>>>(MP);
    BQ_CK_LAUNCH();
    return BQ_OK;
}

// ordered: decoupled look-back (deterministic layout; the staging of equal
// records needs it); otherwise the atomic-cursor kernel (keys three-way,
// records two-way)
template <class KT>
bq_status launch_partition(const PassParams<KT> &P, cudaStream_t s) {
    if (P.ordered) return launch_partition_t<KT, true>(P, s);
    return launch_partition_fast<KT>(P, s);
}

template <class KT>
bq_status launch_leaves(int cls, const LeafParams<KT> &LP, uint32_t count, cudaStream_t s) {
    if (count == 0 && LP.count_dev == nullptr && LP.set == nullptr) return BQ_OK;   // count 0 + a device count: persistent grid
    BQ_CK(launch_leaf_class<KT>(cls, LP, count, s));
    return BQ_OK;
}

inline bool aligned16(const void *p) { return ((uintptr_t)p & 15) == 0; }

template <class KT>
bq_status validate(const void *data, size_t n, void *ws, size_t ws_bytes) {
    if (n > 0x7fffffffull) return set_error(BQ_ERR_INVALID_ARGUMENT, "n = %zu exceeds 2^31-1", n);
    if (n > 0 && data == nullptr) return set_error(BQ_ERR_INVALID_ARGUMENT, "NULL data with n > 0");
    if (KT::is_record && !aligned16(data))
        return set_error(BQ_ERR_INVALID_ARGUMENT, "records must be 16-byte aligned");
    if (!KT::is_record && ((uintptr_t)data % sizeof(typename KT::T)) != 0)
        return set_error(BQ_ERR_INVALID_ARGUMENT, "keys not aligned to their size");
    const size_t need = make_layout<KT>(n).total;
    if (ws == nullptr || ws_bytes < need)
        return set_error(BQ_ERR_WORKSPACE, "workspace %zu B < required %zu B", ws ? ws_bytes : 0, need);
    if (((uintptr_t)ws & 255) != 0) return set_error(BQ_ERR_WORKSPACE, "workspace not 256-byte aligned");
    return check_device();
}

constexpr uint32_t FILL_GRID = 148 * 8;
// equal bands up to this many elements are filled by k_post's CTA for the
// segment; longer ones (duplicate-heavy inputs) tile-parallel by k_fill
#ifndef BQ_BAND_INLINE_MAX
#define BQ_BAND_INLINE_MAX (1u << 16)
#endif
constexpr uint32_t BAND_INLINE_MAX = BQ_BAND_INLINE_MAX;

// Equal bands left to k_fill (records: both phases).
template <class KT>
bq_status launch_fill(const PostParams<KT> &Q, cudaStream_t s) {
    const uint32_t grid = Q.pass.ntiles < FILL_GRID ? Q.pass.ntiles : FILL_GRID;
    if (grid == 0) return BQ_OK;
    k_fill<KT, POST_THREADS><<<grid, POST_THREADS, 0, s>>>(Q, 0);
    BQ_CK_LAUNCH();
    if (KT::is_record) {
        k_fill<KT, POST_THREADS><<<grid, POST_THREADS, 0, s>>>(Q, 1);
        BQ_CK_LAUNCH();
    }
    return BQ_OK;
}

// After a standalone pass (no children): per-segment counts, then every
// equal band tile-parallel.  Fully asynchronous.
template <class KT>
bq_status launch_pass_post(const PassParams<KT> &P, uint32_t nseg, uint64_t *d_counts, cudaStream_t s) {
    PostParams<KT> Q{};
    Q.pass = P;
    Q.d_counts = d_counts;
    Q.emit_children = 0;
    Q.band_inline_max = 0;
    Q.nseg = nseg;
    k_post<KT, POST_THREADS><<<nseg < POST_GRID ? nseg : POST_GRID, POST_THREADS, 0, s>>>(Q);
    BQ_CK_LAUNCH();
    return launch_fill<KT>(Q, s);
}

// One out-of-place three-way pass over a single segment [0, n).
template <class KT>
bq_status run_pass(const typename KT::T *src, typename KT::T *dst, typename KT::T *stage, size_t n,
                   typename KT::K pivot_key, uint64_t *d_counts, void *ws, cudaStream_t s, int ordered) {
    using T = typename KT::T;
    constexpr uint32_t TILE = tile_elems<KT>();
    const Layout<KT> L = make_layout<KT>(n);
    char *w = static_cast<char *>(ws);
    uint64_t *status = reinterpret_cast<uint64_t *>(w + L.status);
    unsigned long long *cursor = reinterpret_cast<unsigned long long *>(w + L.cursor[0]);
    uint32_t *ecursor = reinterpret_cast<uint32_t *>(w + L.ecursor[0]);
    LevelCtrl *ctrl = reinterpret_cast<LevelCtrl *>(w + L.ctrl);
    if (n == 0) {
        BQ_CK(cudaMemsetAsync(d_counts, 0, 3 * sizeof(uint64_t), s));
        return BQ_OK;
    }
    const uint32_t ntiles = seg_tiles<KT>(0, (uint32_t)n);
    if (ordered || KT::is_record) BQ_CK(cudaMemsetAsync(status, 0, ntiles * sizeof(uint64_t), s));
    BQ_CK(cudaMemsetAsync(ctrl, 0, sizeof(LevelCtrl), s));
    BQ_CK(cudaMemsetAsync(cursor, 0, sizeof(unsigned long long), s));
    BQ_CK(cudaMemsetAsync(ecursor, 0, sizeof(uint32_t), s));
    PassParams<KT> P{};
    P.bufs[0] = const_cast<T *>(src);
    P.bufs[1] = dst;
    P.stage[0] = P.stage[1] = stage;
    P.final_buf = dst;
    P.segs = nullptr;
    P.tile_map = nullptr;
    P.seg0 = Seg{(uint64_t)pivot_key, 0, (uint32_t)n, 0, ntiles, 0, 0, 0, 0};
    P.status = status;
    P.cursor = cursor;
    P.ecursor = ecursor;
    P.ctrl = ctrl;
    P.ntiles = ntiles;
    P.n_total = n;
    P.aligned = aligned16(src) && aligned16(dst);
    P.ordered = ordered || KT::is_record;   // the partition API is three-way for records too
    bq_status st = launch_partition<KT>(P, s);
    if (st != BQ_OK) return st;
    return launch_pass_post<KT>(P, 1, d_counts, s);
}

template <class KT>
bq_status run_pivot(const typename KT::T *data, size_t n, int rule, uint64_t *key_out, void *ws,
                    size_t ws_bytes, cudaStream_t s) {
    if (n == 0) return set_error(BQ_ERR_INVALID_ARGUMENT, "pivot of an empty array");
    if (rule != BQ_PIVOT_MO3 && rule != BQ_PIVOT_NINTHER && rule != BQ_PIVOT_SAMPLE64)
        return set_error(BQ_ERR_INVALID_ARGUMENT, "bad pivot rule %d", rule);
    bq_status st = validate<KT>(data, n, ws, ws_bytes);
    if (st != BQ_OK) return st;
    const Layout<KT> L = make_layout<KT>(n);
    uint64_t *misc = reinterpret_cast<uint64_t *>(static_cast<char *>(ws) + L.misc);
    k_pivot<KT><<<1, 32, 0, s>>>(data, (uint32_t)n, rule, misc);
    BQ_CK_LAUNCH();
    BQ_CK(cudaMemcpyAsync(key_out, misc, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    BQ_CK(cudaStreamSynchronize(s));
    return BQ_OK;
}

// bq_partition_*: the in-place block partition (N2, run_partition_inplace_ip
// below), after the checks every entry point makes.
template <class KT>
bq_status run_partition_inplace_ip(typename KT::T *data, size_t n, typename KT::K pk, size_t *split,
                                   size_t *n_equal, void *ws, size_t ws_bytes, cudaStream_t s);
template <class KT>
bq_status run_partition_inplace(typename KT::T *data, size_t n, typename KT::K pivot_key, size_t *split,
                                size_t *n_equal, void *ws, size_t ws_bytes, cudaStream_t s) {
    bq_status st = validate<KT>(data, n, ws, ws_bytes);
    if (st != BQ_OK) return st;
    return run_partition_inplace_ip<KT>(data, n, pivot_key, split, n_equal, ws, ws_bytes, s);
}

// ---- N2: in-place block partition (inplace.cuh) ------------------------------
template <class KT>
struct IpLayout {
    size_t passes, leftover, pairs, s1, s2, total, vmax;
};
template <class KT>
IpLayout<KT> make_ip_layout(size_t n) {
    constexpr size_t TILE = ip_tile<KT>();
    IpLayout<KT> L;
    L.vmax = (IP_GMAX + 1) * TILE + 16 < n ? (IP_GMAX + 1) * TILE + 16 : n;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
    L.passes = take(2 * sizeof(IpPass));
    L.leftover = take(2 * IP_GMAX * sizeof(uint32_t));
    L.pairs = take(4 * IP_GMAX * sizeof(uint32_t));
    L.s1 = take(L.vmax * sizeof(typename KT::T));
    L.s2 = take(L.vmax * sizeof(typename KT::T));
    L.total = off;
    return L;
}

// bq_partition_inplace: three-way in place with O(#CTAs * T) workspace —
// pass 0 splits [< p | >= p]; pass 1, if keys equal to p exist, splits the
// right part into [= p | > p].  Each pass: k_ip_setup, k_inplace (block
// neutralization from both ends), k_ip_plan + k_swap_blocks (leftover blocks
// into the middle), k_vsplit + k_gather3 + k_ip_fix (Alg. 3
// l.29's "remaining elements": head, middle and tail).  All sizes stay on the
// device; the host reads the two results once at the end.
template <class KT>
bq_status run_partition_inplace_ip(typename KT::T *data, size_t n, typename KT::K pk, size_t *split,
                                   size_t *n_equal, void *ws, size_t ws_bytes, cudaStream_t s) {
    using T = typename KT::T;
    using Kn = Kernels<KT>;
    constexpr uint32_t TILE = ip_tile<KT>();
    if (n > 0x7fffffffull) return set_error(BQ_ERR_INVALID_ARGUMENT, "n = %zu exceeds 2^31-1", n);
    if (n > 0 && data == nullptr) return set_error(BQ_ERR_INVALID_ARGUMENT, "NULL data with n > 0");
    if (KT::is_record && !aligned16(data)) return set_error(BQ_ERR_INVALID_ARGUMENT, "records must be 16-byte aligned");
    if ((uintptr_t)data % sizeof(typename KT::K) != 0)
        return set_error(BQ_ERR_INVALID_ARGUMENT, "data not aligned to its key size");
    const IpLayout<KT> L = make_ip_layout<KT>(n);
    if (ws == nullptr || ws_bytes < L.total)
        return set_error(BQ_ERR_WORKSPACE, "workspace %zu B < required %zu B", ws ? ws_bytes : 0, L.total);
    if (((uintptr_t)ws & 255) != 0) return set_error(BQ_ERR_WORKSPACE, "workspace not 256-byte aligned");
    bq_status st = check_device();
    if (st != BQ_OK) return st;
    if (n == 0) {
        if (split) *split = 0;
        if (n_equal) *n_equal = 0;
        return BQ_OK;
    }
    char *w = static_cast<char *>(ws);
    IpPass *ps = reinterpret_cast<IpPass *>(w + L.passes);
    uint32_t *leftover = reinterpret_cast<uint32_t *>(w + L.leftover);
    uint32_t *pairs = reinterpret_cast<uint32_t *>(w + L.pairs);
    T *s1 = reinterpret_cast<T *>(w + L.s1);
    T *s2 = reinterpret_cast<T *>(w + L.s2);

    auto kern = k_inplace<KT, Kn::NT, ip_ipt<KT>()>;
    constexpr int smem = inplace_smem_bytes<KT>();
    static CapCache cc;
    int cap = 0;
    st = persistent_cap(kern, Kn::NT, smem, cc, &cap);
    if (st != BQ_OK) return st;
    uint32_t grid = (uint32_t)cap < IP_GMAX ? (uint32_t)cap : IP_GMAX;
    const size_t nb_max = n / TILE;
    if (nb_max < grid) grid = nb_max ? (uint32_t)nb_max : 1;
    constexpr uint32_t VG = 148 * 4;   // cleanup kernels: grid-stride over <= vmax elements
    // pass 0 records the positions of keys equal to p in its final right
    // blocks in s1 (unused by the cleanup); the equal band's compaction lists
    // (E, G) take the two halves of s2 (used by pass 0's cleanup, not by pass 1's)
    const uint32_t eqcap = (uint32_t)(L.vmax * sizeof(T) / sizeof(uint64_t));
    uint64_t *eqpos = reinterpret_cast<uint64_t *>(s1);
    const uint64_t list_cap = L.vmax * sizeof(T) / (2 * sizeof(uint32_t));
    uint32_t *lists = reinterpret_cast<uint32_t *>(s2);
    for (int k = 0; k < 2; k++) {
        IpPass *q = ps + k;
        k_ip_setup<KT><<<1, 1, 0, s>>>(data, q, k ? ps : nullptr, n, list_cap, eqcap);
        BQ_CK_LAUNCH();
        if (k == 1) {
            k_eq_scan<KT, 256><<<148 * 8, 256, 0, s>>>(data, q, (uint64_t)pk, lists, lists + list_cap);
            BQ_CK_LAUNCH();
            k_eq_scan2<KT, 256><<<148 * 2, 256, 0, s>>>(data, q, ps, (uint64_t)pk, lists, lists + list_cap, eqpos,
                                                         eqcap);
            BQ_CK_LAUNCH();
            k_eq_swap<KT><<<VG, 256, 0, s>>>(data, q, lists, lists + list_cap);
            BQ_CK_LAUNCH();
        }
        kern<<<grid, Kn::NT, smem, s>>>(
            InplaceParams<KT>{data, q, (uint64_t)pk, k, leftover, k == 0 ? eqpos : nullptr, eqcap});
        BQ_CK_LAUNCH();
        k_ip_plan<KT, 1024><<<1, 1024, 0, s>>>(q, leftover, pairs, k == 0 ? eqpos : nullptr, eqcap);
        BQ_CK_LAUNCH();
        k_swap_blocks<KT, Kn::NT, ip_ipt<KT>()><<<grid, Kn::NT, 0, s>>>(data, q, pairs);
        BQ_CK_LAUNCH();
        k_vsplit<KT, Kn::NT, Kn::IPT><<<VG, Kn::NT, 0, s>>>(data, s2, q, (uint64_t)pk, k);
        BQ_CK_LAUNCH();
        k_gather3<KT><<<VG, 256, 0, s>>>(data, s2, q, 1);
        BQ_CK_LAUNCH();
        k_ip_fix<KT, 256><<<1, 256, 0, s>>>(data, q);
        BQ_CK_LAUNCH();
    }
    IpPass h[2];
    BQ_CK(cudaMemcpyAsync(h, ps, sizeof h, cudaMemcpyDeviceToHost, s));
    BQ_CK(cudaStreamSynchronize(s));
    if (h[1].compact && (h[1].cnt_eq != h[1].cnt_gt))
        return set_error(BQ_ERR_CUDA, "in-place partition: equal band lists %llu != %llu",
                         (unsigned long long)h[1].cnt_eq, (unsigned long long)h[1].cnt_gt);
    if (h[1].active && h[1].n_left - h[0].n_left != h[0].n_eq)
        return set_error(BQ_ERR_CUDA, "in-place partition: equal band %llu != %llu",
                         (unsigned long long)(h[1].n_left - h[0].n_left), (unsigned long long)h[0].n_eq);
    if (split) *split = (size_t)h[0].n_left;
    if (n_equal) *n_equal = (size_t)h[0].n_eq;
    return BQ_OK;
}

template <class KT>
bq_status run_partition_pass(const typename KT::T *src, typename KT::T *dst, size_t n,
                             typename KT::K pivot_key, uint64_t *d_counts, void *ws, size_t ws_bytes,
                             cudaStream_t s, int ordered) {
    using T = typename KT::T;
    bq_status st = validate<KT>(src, n, ws, ws_bytes);
    if (st != BQ_OK) return st;
    if (n > 0 && dst == nullptr) return set_error(BQ_ERR_INVALID_ARGUMENT, "NULL dst");
    if (d_counts == nullptr) return set_error(BQ_ERR_INVALID_ARGUMENT, "NULL d_counts");
    if (KT::is_record && !aligned16(dst)) return set_error(BQ_ERR_INVALID_ARGUMENT, "dst not 16-byte aligned");
    const size_t bytes = n * sizeof(T);
    const char *a = reinterpret_cast<const char *>(src), *c = reinterpret_cast<const char *>(dst);
    if (n && a < c + bytes && c < a + bytes) return set_error(BQ_ERR_INVALID_ARGUMENT, "src and dst overlap");
    const Layout<KT> L = make_layout<KT>(n);
    T *scratch = reinterpret_cast<T *>(static_cast<char *>(ws) + L.scratch);
    return run_pass<KT>(src, dst, scratch, n, pivot_key, d_counts, ws, s, ordered);
}

// Batched pass over caller-given disjoint segments (bq_partition_segments).
template <class KT>
bq_status run_partition_segments(const typename KT::T *src, typename KT::T *dst, size_t n, const uint32_t *begins,
                                 const uint32_t *lens, const typename KT::K *pivot_keys, size_t nseg,
                                 uint64_t *d_counts, void *ws, size_t ws_bytes, cudaStream_t s, int ordered) {
    using T = typename KT::T;
    constexpr uint32_t TILE = tile_elems<KT>();
    bq_status st = validate<KT>(src, n, ws, ws_bytes);
    if (st != BQ_OK) return st;
    if (nseg == 0) return BQ_OK;
    if (!dst || !begins || !lens || !pivot_keys || !d_counts)
        return set_error(BQ_ERR_INVALID_ARGUMENT, "NULL argument");
    if (KT::is_record && !aligned16(dst)) return set_error(BQ_ERR_INVALID_ARGUMENT, "dst not 16-byte aligned");
    const Layout<KT> L = make_layout<KT>(n);
    if (nseg > L.max_segs) return set_error(BQ_ERR_INVALID_ARGUMENT, "nseg %zu > %zu", nseg, L.max_segs);
    std::vector<Seg> hs(nseg);
    std::vector<std::pair<uint64_t, uint64_t>> iv(nseg);
    uint64_t tiles = 0;
    uint32_t maxtiles = 0;
    for (size_t i = 0; i < nseg; i++) {
        if (lens[i] == 0 || (uint64_t)begins[i] + lens[i] > n)
            return set_error(BQ_ERR_INVALID_ARGUMENT, "segment %zu out of range or empty", i);
        const uint32_t nt = seg_tiles<KT>(begins[i], lens[i]);
        hs[i] = Seg{(uint64_t)pivot_keys[i], begins[i], lens[i], (uint32_t)tiles, nt, 0, 0, 0, 0};
        tiles += nt;
        maxtiles = nt > maxtiles ? nt : maxtiles;
        iv[i] = {begins[i], (uint64_t)begins[i] + lens[i]};
    }
    if (tiles > L.max_tiles) return set_error(BQ_ERR_INVALID_ARGUMENT, "segments need too many tiles");
    std::sort(iv.begin(), iv.end());
    for (size_t i = 1; i < nseg; i++)
        if (iv[i].first < iv[i - 1].second) return set_error(BQ_ERR_INVALID_ARGUMENT, "segments overlap");
    const size_t bytes = n * sizeof(T);
    const char *a = reinterpret_cast<const char *>(src), *c = reinterpret_cast<const char *>(dst);
    if (a < c + bytes && c < a + bytes) return set_error(BQ_ERR_INVALID_ARGUMENT, "src and dst overlap");

    char *w = static_cast<char *>(ws);
    T *scratch = reinterpret_cast<T *>(w + L.scratch);
    uint64_t *status = reinterpret_cast<uint64_t *>(w + L.status);
    uint32_t *tile_map = reinterpret_cast<uint32_t *>(w + L.tile_map[0]);
    Seg *segs = reinterpret_cast<Seg *>(w + L.segs[0]);
    unsigned long long *cursor = reinterpret_cast<unsigned long long *>(w + L.cursor[0]);
    uint32_t *ecursor = reinterpret_cast<uint32_t *>(w + L.ecursor[0]);
    LevelCtrl *ctrl = reinterpret_cast<LevelCtrl *>(w + L.ctrl);
    BQ_CK(cudaMemcpyAsync(segs, hs.data(), nseg * sizeof(Seg), cudaMemcpyHostToDevice, s));
    BQ_CK(cudaMemsetAsync(ctrl, 0, sizeof(LevelCtrl), s));
    k_map<<<dim3((uint32_t)nseg, (maxtiles + 255) / 256), 256, 0, s>>>(segs, tile_map, status, cursor, ecursor);
    BQ_CK_LAUNCH();
    PassParams<KT> P{};
    P.bufs[0] = const_cast<T *>(src);
    P.bufs[1] = dst;
    P.stage[0] = P.stage[1] = scratch;
    P.final_buf = dst;
    P.segs = segs;
    P.tile_map = tile_map;
    P.status = status;
    P.cursor = cursor;
    P.ecursor = ecursor;
    P.ctrl = ctrl;
    P.ntiles = (uint32_t)tiles;
    P.n_total = n;
    P.aligned = aligned16(src) && aligned16(dst);
    P.ordered = ordered || KT::is_record;
    st = launch_partition<KT>(P, s);
    if (st != BQ_OK) return st;
    st = launch_pass_post<KT>(P, (uint32_t)nseg, d_counts, s);
    if (st != BQ_OK) return st;
    BQ_CK(cudaStreamSynchronize(s));
    return BQ_OK;
}

// ---- the sort (a1-a9) -----------------------------------------------------------
// Everything the launches of one sort need: workspace pointers, options, and
// the parameter templates of the level-loop kernels (their level-dependent
// fields are resolved on the device, LoopPtrs).
template <class KT>
struct SortPlan {
    using T = typename KT::T;
    Layout<KT> L;
    size_t n;
    T *user, *scratch;
    LoopPtrs<KT> lp;
    LoopMisc *misc;
    LevelCtrl *ctrl, *root;
    Leaf *leaves[2], *fallback, *copies[2];
    uint32_t *tprefix;
    FbState *fbst;
    int rule, depth_limit, ordered, ways, aligned;
    uint32_t leaf_max;    // leaf_max_for(n)
    uint32_t batch;       // levels per loop iteration
    PostParams<KT> Q;     // k_post / k_fill / k_post_mw of a level (dynamic)
    PassParams<KT> P;     // the binary partition of a level (dynamic)
    MwParams<KT> MP;      // the multiway kernels of a level (dynamic)
    LeafParams<KT> LP;    // leaf kernels (count_dev per class)
};

template <class KT>
bq_status make_plan(SortPlan<KT> &pl, typename KT::T *data, size_t n, void *ws, int rule, int depth_limit, int ordered,
                    int ways) {
    using T = typename KT::T;
    constexpr uint32_t S = Tune<KT>::LEAF;
    pl.L = make_layout<KT>(n);
    const Layout<KT> &L = pl.L;
    char *w = static_cast<char *>(ws);
    pl.n = n;
    pl.user = data;
    pl.scratch = reinterpret_cast<T *>(w + L.scratch);
    pl.rule = rule;
    pl.depth_limit = depth_limit;
    pl.ordered = ordered;
    pl.ways = ways;
    pl.aligned = aligned16(pl.user) && aligned16(pl.scratch);
    const uint32_t lm = leaf_max_for<KT>(n);
    pl.leaf_max = lm;
    pl.batch = n <= LOOP_SMALL_N ? LOOP_BATCH_SMALL : LOOP_BATCH;
    if (mw_capable<KT>() && ways > 2 && (n > LOOP_SMALL_N || lm < S)) {
        // the levels a multiway sort needs if every bucket gets its share —
        // a level splits m keys into min(ways, ceil(m / (S * fill))) buckets
        // (mw_splitters) — plus one for the buckets the sample makes larger:
        // one batch of that many levels leaves few empty level slots behind
        const uint64_t S = lm;
        uint64_t m = n;
        uint32_t lv = 0;
        while (m > S && lv < LOOP_BATCH_MAX) {
            const uint64_t k = std::min<uint64_t>((uint64_t)ways, (m * 100 + S * BQ_MW_FILL - 1) / (S * BQ_MW_FILL));
            m = (m + k - 1) / std::max<uint64_t>(k, 2);
            lv++;
        }
        pl.batch = std::min<uint32_t>(LOOP_BATCH_MAX, std::max<uint32_t>(2u, lv + (n > LOOP_SMALL_N ? 1 : batch_extra())));
    }
    pl.ctrl = reinterpret_cast<LevelCtrl *>(w + L.ctrl);
    pl.root = pl.ctrl + MAX_LEVELS;
    pl.misc = reinterpret_cast<LoopMisc *>(w + L.misc);
    pl.leaves[0] = reinterpret_cast<Leaf *>(w + L.leaves[0]);
    pl.leaves[1] = reinterpret_cast<Leaf *>(w + L.leaves[1]);
    pl.fallback = reinterpret_cast<Leaf *>(w + L.fallback);
    pl.copies[0] = reinterpret_cast<Leaf *>(w + L.copies[0]);
    pl.copies[1] = reinterpret_cast<Leaf *>(w + L.copies[1]);
    pl.tprefix = reinterpret_cast<uint32_t *>(w + L.tprefix);
    pl.fbst = reinterpret_cast<FbState *>(w + L.fbst);
    LoopPtrs<KT> &lp = pl.lp;
    lp.level = &pl.misc->level;
    lp.set = &pl.misc->set;
    for (int p = 0; p < 2; p++) {
        lp.segs[p] = reinterpret_cast<Seg *>(w + L.segs[p]);
        lp.tile_map[p] = reinterpret_cast<uint32_t *>(w + L.tile_map[p]);
        lp.cursor[p] = reinterpret_cast<unsigned long long *>(w + L.cursor[p]);
        lp.ecursor[p] = reinterpret_cast<uint32_t *>(w + L.ecursor[p]);
        lp.msegs[p] = w + L.msegs[p];
        lp.mtile_map[p] = reinterpret_cast<uint32_t *>(w + L.mtile_map[p]);
        lp.mhist[p] = reinterpret_cast<uint32_t *>(w + L.mhist[p]);
        lp.mcursor[p] = reinterpret_cast<uint32_t *>(w + L.mcursor[p]);
    }
    lp.ctrl = pl.ctrl;
    lp.root = pl.root;
    for (int p = 0; p < 2; p++) {
        lp.leaves[p] = pl.leaves[p];
        lp.leaf_counts[p] = pl.misc->leaf_counts[p];
        lp.copies[p] = pl.copies[p];
        lp.copy_count[p] = &pl.misc->copy_count[p];
    }

    // the binary partition pass of a level
    PassParams<KT> &P = pl.P;
    P = PassParams<KT>{};
    P.bufs[0] = pl.user;
    P.bufs[1] = pl.scratch;
    P.stage[0] = pl.user;
    P.stage[1] = pl.scratch;
    P.final_buf = pl.user;
    P.status = ordered ? reinterpret_cast<uint64_t *>(w + L.status) : nullptr;
    P.ordered = ordered;
    P.ntiles = 0xffffffffu;   // upper bound: the grid is the resident capacity
    P.n_total = n;
    P.aligned = pl.aligned;
    P.lp = lp;
    // the multiway kernels of a level
    MwParams<KT> &MP = pl.MP;
    MP = MwParams<KT>{};
    MP.bufs[0] = pl.user;
    MP.bufs[1] = pl.scratch;
    MP.hstride = (uint32_t)L.max_segs;
    MP.mtab = reinterpret_cast<uint32_t *>(w + L.mtab);
    MP.mblk = reinterpret_cast<uint32_t *>(w + L.mblk);
    MP.max_tiles = (uint32_t)L.max_tiles;
    MP.tabmode = (BQ_MW8W && pl.ways == MW8) ? 1 : 0;
    MP.n_total = n;
    MP.aligned = pl.aligned;
    MP.lp = lp;
    // bookkeeping of a level (children, bands, leaves, fallback)
    PostParams<KT> &Q = pl.Q;
    Q = PostParams<KT>{};
    Q.pass = P;
    Q.mw = MP;
    Q.mhstride = (uint32_t)L.max_segs;
    Q.status = P.status;
    Q.copies = pl.copies[0];
    Q.copy_count = &pl.misc->copy_count[0];
    Q.copy_cap = (uint32_t)L.max_copies;
    Q.leaves = pl.leaves[0];
    Q.leaf_counts = pl.misc->leaf_counts[0];
    Q.leaf_cap = (uint32_t)L.max_leaves;
    Q.fallback = pl.fallback;
    Q.fallback_count = &pl.misc->fb_count;
    Q.leaf_max = lm;
    Q.depth_limit = depth_limit;
    Q.pivot_rule = rule;
    Q.ways = ways;
    Q.emit_children = 1;
    Q.band_inline_max = BAND_INLINE_MAX;
    Q.overflow = &pl.misc->overflow;
    Q.nseg_cap = (uint32_t)L.max_segs;
    Q.ntile_cap = (uint32_t)L.max_tiles;
    // leaves
    LeafParams<KT> &LP = pl.LP;
    LP = LeafParams<KT>{};
    LP.bufs[0] = pl.user;
    LP.bufs[1] = pl.scratch;
    LP.out = pl.user;
    LP.n_total = n;
    LP.aligned = pl.aligned;
    LP.set = &pl.misc->set;
    for (int p = 0; p < 2; p++) {
        LP.lsets[p] = pl.leaves[p];
        LP.csets[p] = pl.misc->leaf_counts[p];
    }
    return BQ_OK;
}

// root: zero the control blocks, [0, n) becomes the first segment (level 0)
template <class KT>
bq_status enqueue_prefix(const SortPlan<KT> &pl, cudaStream_t s) {
    BQ_CK(cudaMemsetAsync(pl.ctrl, 0, (MAX_LEVELS + 1) * sizeof(LevelCtrl), s));
    BQ_CK(cudaMemsetAsync(pl.misc, 0, sizeof(LoopMisc), s));
    PostParams<KT> Q0 = pl.Q;
    Q0.pass.lp.level = nullptr;
    Q0.mw.lp.level = nullptr;
    Q0.next_segs = pl.lp.segs[0];
    Q0.next_tile_map = pl.lp.tile_map[0];
    Q0.next_cursor = pl.lp.cursor[0];
    Q0.next_ecursor = pl.lp.ecursor[0];
    Q0.next_msegs = static_cast<MSeg<KT> *>(pl.lp.msegs[0]);
    Q0.next_mtile_map = pl.lp.mtile_map[0];
    Q0.next_mhist = pl.lp.mhist[0];
    Q0.child_ctrl = pl.root;
    k_init_root<KT, POST_THREADS><<<1, POST_THREADS, 0, s>>>(Q0, (uint32_t)pl.n);
    BQ_CK_LAUNCH();
    return BQ_OK;
}

// one level of the recursion (every array resolved on the device); `ev`
// (optional) brackets the binary partition launch
template <class KT>
bq_status enqueue_level(const SortPlan<KT> &pl, cudaStream_t s, int use_cond, cudaGraphConditionalHandle h_loop,
                        cudaGraphConditionalHandle h_fb, cudaEvent_t ev0, cudaEvent_t ev1, cudaEvent_t mev0 = nullptr,
                        cudaEvent_t mev1 = nullptr, cudaEvent_t mmid = nullptr, cudaStream_t sb = nullptr,
                        cudaEvent_t *fj = nullptr) {
    // graph capture of a multiway sort of keys (sb, fj given): the binary
    // chain (pass, k_post, k_fill) is a branch beside the multiway chain —
    // the two work on disjoint segments and append children, leaves and
    // counts with atomics only, so a level's critical path is the longer
    // chain, not their sum (mostly empty launches on one side)
    cudaStream_t s2 = s;
    if constexpr (mw_capable<KT>()) if (pl.ways > 2) {
        if (sb && !KT::is_record && !std::getenv("BQ_CHAIN_SERIAL")) {
            s2 = sb;
            BQ_CK(cudaEventRecord(fj[0], s));
            BQ_CK(cudaStreamWaitEvent(s2, fj[0], 0));
        }
        MwParams<KT> MP = pl.MP;
        if (mev0) BQ_CK(cudaEventRecord(mev0, s));
        bq_status st = launch_multiway<KT>(MP, nullptr, s, pl.ways, mmid);
        if (st != BQ_OK) return st;
        if (mev1) BQ_CK(cudaEventRecord(mev1, s));
        k_post_mw<KT, POST_THREADS><<<POST_GRID, POST_THREADS, 0, s>>>(pl.Q);
        BQ_CK_LAUNCH();
    }
    if (ev0) BQ_CK(cudaEventRecord(ev0, s2));
    bq_status st = launch_partition<KT>(pl.P, s2);
    if (st != BQ_OK) return st;
    if (ev1) BQ_CK(cudaEventRecord(ev1, s2));
    k_post<KT, POST_LEVEL_THREADS><<<POST_LEVEL_GRID, POST_LEVEL_THREADS, 0, s2>>>(pl.Q);
    BQ_CK_LAUNCH();
    st = launch_fill<KT>(pl.Q, s2);   // exits at once unless a band was too long for k_post
    if (st != BQ_OK) return st;
    if (s2 != s) {
        BQ_CK(cudaEventRecord(fj[1], s2));
        BQ_CK(cudaStreamWaitEvent(s, fj[1], 0));
    }
    return BQ_OK;
}
template <class KT>
bq_status enqueue_level_end(const SortPlan<KT> &pl, cudaStream_t s, int use_cond, cudaGraphConditionalHandle h_loop,
                            cudaGraphConditionalHandle h_fb) {
    k_level_end<KT><<<1, 1, 0, s>>>(pl.lp, pl.misc, pl.batch, use_cond, h_loop, h_fb);
    BQ_CK_LAUNCH();
    return BQ_OK;
}

// sort the previous level's leaves (set (level + 1) & 1; one persistent
// launch per class), copy its finished equal-record runs, empty the set
template <class KT>
bq_status enqueue_flush(const SortPlan<KT> &pl, cudaStream_t s, cudaEvent_t l0 = nullptr, cudaEvent_t l1 = nullptr,
                        cudaStream_t *aux = nullptr, cudaEvent_t *aev = nullptr) {
    if (l0) BQ_CK(cudaEventRecord(l0, s));   // timing: around the leaf launches
    // graph capture (aux, aev given): class c > 0 on its own branch aux[c - 1]
    // (fork aev[0], joins aev[c]) — the classes' lists are disjoint, and a
    // small sort's few large leaves of two classes then run side by side
    // (keys only: the records' and pairs' classes measured 2 % slower side by
    // side, c5 8.73 -> 8.9 ms; BQ_LEAF_SERIAL is the A/B switch of tools/gpu_var.sh)
    if (KT::is_record || std::getenv("BQ_LEAF_SERIAL")) aux = nullptr;
    if (aux) BQ_CK(cudaEventRecord(aev[0], s));
    for (int c = 0; c < leaf_nclass<KT>(); c++) {
        LeafParams<KT> LP = pl.LP;
        LP.lcls = (size_t)c * pl.L.max_leaves;
        LP.cls = c;
        cudaStream_t sc = (aux && c > 0) ? aux[c - 1] : s;
        if (aux && c > 0) BQ_CK(cudaStreamWaitEvent(sc, aev[0], 0));
        bq_status st = launch_leaves<KT>(c, LP, 0, sc);
        if (st != BQ_OK) return st;
        if (aux && c > 0) {
            BQ_CK(cudaEventRecord(aev[c], sc));
            BQ_CK(cudaStreamWaitEvent(s, aev[c], 0));
        }
    }
    if (l1) BQ_CK(cudaEventRecord(l1, s));
    if (KT::is_record && !pl.ordered) {
        k_copy_runs<KT, POST_THREADS><<<POST_GRID, POST_THREADS, 0, s>>>(pl.lp, &pl.misc->level, pl.user, pl.scratch);   // (set: pl.lp.set)
        BQ_CK_LAUNCH();
    }
    k_flush_reset<<<1, 1, 0, s>>>(pl.misc);
    BQ_CK_LAUNCH();
    return BQ_OK;
}

constexpr uint32_t FB_GRID = 148 * 8;

// a9 over every depth-capped segment; npass < 0: merge passes under a
// conditional WHILE node (graph), else that many passes
template <class KT>
bq_status enqueue_fb_setup(const SortPlan<KT> &pl, cudaStream_t s, int use_cond, cudaGraphConditionalHandle h) {
    Leaf *chunks = pl.leaves[0];   // set 0, class 0: free after the last flush
    k_fb_setup<<<1, 1024, 0, s>>>(pl.fallback, &pl.misc->fb_count, chunks, pl.tprefix, pl.fbst, Tune<KT>::LEAF, use_cond,
                                  h);
    BQ_CK_LAUNCH();
    LeafParams<KT> LP = pl.LP;
    LP.set = nullptr;
    LP.leaves = chunks;
    LP.count_dev = &pl.fbst->nchunk;
    LP.out_other = 1;   // sorted chunks land in the other buffer
    return launch_leaves<KT>(leaf_nclass<KT>() - 1, LP, 0, s);
}
template <class KT>
bq_status enqueue_fb_pass(const SortPlan<KT> &pl, cudaStream_t s, int use_cond, cudaGraphConditionalHandle h) {
    k_fb_merge<KT><<<FB_GRID, MERGE_THREADS, 0, s>>>(pl.fallback, pl.tprefix, pl.fbst, pl.user, pl.scratch);
    BQ_CK_LAUNCH();
    k_fb_next<<<1, 1, 0, s>>>(pl.fbst, use_cond, h);
    BQ_CK_LAUNCH();
    return BQ_OK;
}
template <class KT>
bq_status enqueue_fb_finish(const SortPlan<KT> &pl, cudaStream_t s) {
    k_fb_finish<KT><<<FB_GRID, MERGE_THREADS, 0, s>>>(pl.fallback, pl.tprefix, pl.fbst, pl.user, pl.scratch);
    BQ_CK_LAUNCH();
    return BQ_OK;
}

// ---- the graph of a sort, cached per (device, kind, buffers, n, options) --------
struct GraphKey {
    int dev, kind, rule, depth_limit, ordered, ways;
    uint32_t leaf_max, batch;
    const void *data, *ws;
    size_t n, ws_bytes;
    bool operator==(const GraphKey &o) const {
        return dev == o.dev && kind == o.kind && rule == o.rule && depth_limit == o.depth_limit &&
               ordered == o.ordered && ways == o.ways && leaf_max == o.leaf_max && batch == o.batch && data == o.data && ws == o.ws && n == o.n &&
               ws_bytes == o.ws_bytes;
    }
};
bool graph_cache_get(const GraphKey &k, cudaGraphExec_t *ex);
void graph_cache_put(const GraphKey &k, cudaGraphExec_t ex);

// a conditional node at the capture point of stream s; returns its body graph
inline cudaError_t add_cond_node(cudaStream_t s, cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type,
                                 cudaGraph_t *body) {
    cudaStreamCaptureStatus cs;
    cudaGraph_t g;
    const cudaGraphNode_t *deps = nullptr;
    size_t nd = 0;
    cudaError_t e = cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, &deps, &nd);
    if (e != cudaSuccess) return e;
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = type;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    if ((e = cudaGraphAddNode(&node, g, deps, nd, &p)) != cudaSuccess) return e;
    *body = p.conditional.phGraph_out[0];
    return cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies);
}

// Builds the graph: prefix; WHILE(the last level had children) { fork: [sort
// the previous batch's leaves] || [partition LOOP_BATCH levels]; join };
// sort the last level's leaves; IF(capped segments) { setup; chunk leaves;
// WHILE(passes) merge; finish }.  Captured on private streams, instantiated once.
// Key sorts: a flush's leaf classes and a level's binary / multiway chains
// are parallel branches (enqueue_flush, enqueue_level).
template <class KT>
bq_status build_sort_graph(const SortPlan<KT> &pl, cudaGraphExec_t *ex) {
    constexpr int NC = leaf_nclass<KT>();
    cudaStream_t cs[6] = {};
    cudaEvent_t ev[2 + 2 * LOOP_BATCH_MAX] = {};   // [2 + 2k], [3 + 2k]: level slot k's chain fork and join
    cudaStream_t aux[2][MAX_LEAF_CLASSES] = {};   // leaf-class branches of the two flushes
    cudaEvent_t aev[2][MAX_LEAF_CLASSES + 1] = {};
    cudaGraph_t g = nullptr;
    auto fail = [&](bq_status e) {
        for (auto &x : cs) if (x) cudaStreamDestroy(x);
        for (auto &x : ev) if (x) cudaEventDestroy(x);
        for (auto &r : aux) for (auto &x : r) if (x) cudaStreamDestroy(x);
        for (auto &r : aev) for (auto &x : r) if (x) cudaEventDestroy(x);
        if (g) cudaGraphDestroy(g);
        return e;
    };
#define BQ_GK(call)                                                                                     \
    do {                                                                                                \
        cudaError_t e_ = (call);                                                                        \
        if (e_ != cudaSuccess)                                                                          \
            return fail(set_error(BQ_ERR_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                                  __LINE__));                                                           \
    } while (0)
#define BQ_GS(call)                       \
    do {                                  \
        bq_status s_ = (call);            \
        if (s_ != BQ_OK) return fail(s_); \
    } while (0)
    for (auto &x : cs) BQ_GK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    for (auto &x : ev) BQ_GK(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    for (auto &r : aux) for (int c = 0; c + 1 < NC; c++) BQ_GK(cudaStreamCreateWithFlags(&r[c], cudaStreamNonBlocking));
    for (auto &r : aev) for (int c = 0; c < NC; c++) BQ_GK(cudaEventCreateWithFlags(&r[c], cudaEventDisableTiming));
    BQ_GK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h_loop, h_fbany;
    BQ_GK(cudaGraphConditionalHandleCreate(&h_loop, g, 1, cudaGraphCondAssignDefault));
    BQ_GK(cudaGraphConditionalHandleCreate(&h_fbany, g, 0, cudaGraphCondAssignDefault));
    BQ_GK(cudaStreamBeginCaptureToGraph(cs[0], g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    BQ_GS(enqueue_prefix<KT>(pl, cs[0]));
    // the level loop
    cudaGraph_t body, fbbody, pbody, tmp;
    BQ_GK(add_cond_node(cs[0], h_loop, cudaGraphCondTypeWhile, &body));
    BQ_GK(cudaStreamBeginCaptureToGraph(cs[1], body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    BQ_GK(cudaEventRecord(ev[0], cs[1]));
    BQ_GK(cudaStreamWaitEvent(cs[2], ev[0], 0));          // fork
    BQ_GS(enqueue_flush<KT>(pl, cs[2], nullptr, nullptr, aux[0], aev[0]));   // the previous batch's leaves
    for (uint32_t k = 0; k < pl.batch; k++) {
        BQ_GS(enqueue_level<KT>(pl, cs[1], 1, h_loop, h_fbany, nullptr, nullptr, nullptr, nullptr, nullptr, cs[5],
                                &ev[2 + 2 * k]));
        if (k + 1 < pl.batch) BQ_GS(enqueue_level_end<KT>(pl, cs[1], 1, h_loop, h_fbany));
    }
    BQ_GK(cudaEventRecord(ev[1], cs[2]));
    BQ_GK(cudaStreamWaitEvent(cs[1], ev[1], 0));          // join
    BQ_GS(enqueue_level_end<KT>(pl, cs[1], 1, h_loop, h_fbany));
    BQ_GK(cudaStreamEndCapture(cs[1], &tmp));
    BQ_GS(enqueue_flush<KT>(pl, cs[0], nullptr, nullptr, aux[1], aev[1]));   // the last level's leaves
    // the depth-capped segments (a9)
    BQ_GK(add_cond_node(cs[0], h_fbany, cudaGraphCondTypeIf, &fbbody));
    BQ_GK(cudaStreamBeginCaptureToGraph(cs[3], fbbody, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    cudaGraphConditionalHandle h_pass;
    BQ_GK(cudaGraphConditionalHandleCreate(&h_pass, fbbody, 0, cudaGraphCondAssignDefault));
    BQ_GS(enqueue_fb_setup<KT>(pl, cs[3], 1, h_pass));
    BQ_GK(add_cond_node(cs[3], h_pass, cudaGraphCondTypeWhile, &pbody));
    BQ_GK(cudaStreamBeginCaptureToGraph(cs[4], pbody, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    BQ_GS(enqueue_fb_pass<KT>(pl, cs[4], 1, h_pass));
    BQ_GK(cudaStreamEndCapture(cs[4], &tmp));
    BQ_GS(enqueue_fb_finish<KT>(pl, cs[3]));
    BQ_GK(cudaStreamEndCapture(cs[3], &tmp));
    BQ_GK(cudaStreamEndCapture(cs[0], &g));
    BQ_GK(cudaGraphInstantiate(ex, g, 0));
    fail(BQ_OK);
#undef BQ_GK
#undef BQ_GS
    return BQ_OK;
}

template <class KT>
bq_status run_sort(typename KT::T *data, size_t n, const bq_sort_options *opt, bq_sort_stats *stats, void *ws,
                   size_t ws_bytes, cudaStream_t s) {
    using T = typename KT::T;
    constexpr uint32_t S = Tune<KT>::LEAF;
    constexpr int NCLS = leaf_nclass<KT>();
    bq_sort_stats local;
    std::memset(&local, 0, sizeof local);
    int rule = BQ_PIVOT_SAMPLE64, depth_limit = -1, timing = 0, ordered = 0, ways = 0;
    if (opt) {
        rule = opt->pivot_rule;
        depth_limit = opt->depth_limit;
        timing = opt->timing;
        ordered = opt->ordered;
        ways = opt->ways;
        if (ways != 0 && ways != 2 && ways != MW8 && ways != MW_K)
            return set_error(BQ_ERR_INVALID_ARGUMENT, "ways %d not in {0, 2, %d, %d}", ways, MW8, MW_K);
        if (rule != BQ_PIVOT_MO3 && rule != BQ_PIVOT_NINTHER && rule != BQ_PIVOT_SAMPLE64)
            return set_error(BQ_ERR_INVALID_ARGUMENT, "bad pivot rule %d", rule);
        if (depth_limit >= MAX_LEVELS - (int)LOOP_BATCH_MAX - 2)
            return set_error(BQ_ERR_INVALID_ARGUMENT, "depth_limit %d too large", depth_limit);
    }
    bq_status st = validate<KT>(data, n, ws, ws_bytes);
    if (st != BQ_OK) return st;
    if (n <= 1) {
        if (stats) *stats = local;
        return BQ_OK;
    }
    // default: 8-way passes (N4) for 64-bit keys and key+index pairs, and for
    // int32 keys above 2^17 (16-way for 2^21 < n <= 2^23; tools/ways_sweep.py,
    // profiles/r02/mw8t.md: an 8-way level of the TMA-staged scatter costs
    // less than the three binary levels it replaces); binary passes for
    // small int32 sorts; 32-byte records stay binary
    if (ways == 0) {
        if (sizeof(typename KT::K) == 8 && mw_capable<KT>()) ways = MW8;
        else if (!KT::is_record && n > (1u << 21) && n <= (1u << 23)) ways = MW_K;
        else if (!KT::is_record && n > (1u << 17)) ways = MW8;
        else ways = 2;
    }
    if (!mw_capable<KT>()) ways = 2;
    if (depth_limit < 0) {
        int lg = 0;
        for (size_t m = n; m > 1; m >>= 1) lg++;
        depth_limit = 2 * lg + 3;   // P:295, P:1224 (2*ilogb(n)+3)
    }

    SortPlan<KT> pl;
    st = make_plan<KT>(pl, data, n, ws, rule, depth_limit, ordered, ways);
    if (st != BQ_OK) return st;

    if (n <= S) {   // one leaf
        k_single_leaf<<<1, 1, 0, s>>>(pl.leaves[0], (uint32_t)n);
        BQ_CK_LAUNCH();
        LeafParams<KT> LP = pl.LP;
        LP.set = nullptr;
        LP.leaves = pl.leaves[0];
        st = launch_leaves<KT>((int)leaf_class<KT>((uint32_t)n), LP, 1, s);
        if (st != BQ_OK) return st;
        local.kernel_launches = 2;
        local.leaves = 1;
        if (stats) *stats = local;
        return BQ_OK;
    }

    // host-driven loop: with per-launch timing (CUDA events between the
    // launches of a level), or BQ_HOST_LOOP=1 (diagnostics)
    static const bool host_env = [] {
        const char *e = std::getenv("BQ_HOST_LOOP");
        return e && e[0] == '1';
    }();
    const bool host_loop = timing || host_env;
    std::vector<cudaEvent_t> evs;   // timing: one pair per level
    std::vector<cudaEvent_t> mevs;  // timing: one triple per level around the multiway step (count+scan | scatter)
    std::vector<cudaEvent_t> levs;  // timing: one pair per flush around the leaf launches
    auto mkev = [&](std::vector<cudaEvent_t> &v) -> cudaEvent_t {
        cudaEvent_t e = nullptr;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        v.push_back(e);
        return e;
    };
    cudaStream_t side = nullptr;    // host-driven loop: the leaves' stream
    cudaEvent_t efork = nullptr, ejoin = nullptr;
    auto cleanup = [&]() {
        for (auto e : evs) cudaEventDestroy(e);
        for (auto e : mevs) cudaEventDestroy(e);
        for (auto e : levs) cudaEventDestroy(e);
        if (side) cudaStreamDestroy(side);
        if (efork) cudaEventDestroy(efork);
        if (ejoin) cudaEventDestroy(ejoin);
    };
#define BQ_CKC(call)                                                         \
    do {                                                                     \
        bq_status st_ = [&]() -> bq_status { BQ_CK(call); return BQ_OK; }(); \
        if (st_ != BQ_OK) { cleanup(); return st_; }                          \
    } while (0)
#define BQ_SKC(call)                                 \
    do {                                             \
        bq_status st_ = (call);                      \
        if (st_ != BQ_OK) { cleanup(); return st_; } \
    } while (0)

    int host_levels = 0;
    if (!host_loop) {
        int dev = 0;
        BQ_CK(cudaGetDevice(&dev));
        const GraphKey key{dev, (int)KT::kind, rule, depth_limit, ordered, ways, pl.leaf_max, pl.batch, data, ws, n, ws_bytes};
        cudaGraphExec_t ex = nullptr;
        if (!graph_cache_get(key, &ex)) {
            st = build_sort_graph<KT>(pl, &ex);
            if (st != BQ_OK) return st;
            graph_cache_put(key, ex);
        }
        BQ_CK(cudaGraphLaunch(ex, s));
    } else {
        // the graph's structure with two streams: the previous level's leaves
        // on `side` while `s` partitions the level
        BQ_CKC(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
        BQ_CKC(cudaEventCreateWithFlags(&efork, cudaEventDisableTiming));
        BQ_CKC(cudaEventCreateWithFlags(&ejoin, cudaEventDisableTiming));
        BQ_SKC(enqueue_prefix<KT>(pl, s));
        std::vector<LevelCtrl> hc(1);
        for (int level = 0;; level++) {
            if (level + (int)LOOP_BATCH_MAX + 1 >= MAX_LEVELS) {
                cleanup();
                return set_error(BQ_ERR_CUDA, "level loop did not terminate");
            }
            cudaEvent_t e0 = nullptr, e1 = nullptr, m0 = nullptr, m1 = nullptr, mm = nullptr;
            if (timing) {
                if (!(e0 = mkev(evs)) || !(e1 = mkev(evs))) { cleanup(); return set_error(BQ_ERR_CUDA, "event"); }
                if (ways > 2 && (!(m0 = mkev(mevs)) || !(mm = mkev(mevs)) || !(m1 = mkev(mevs)))) {
                    cleanup();
                    return set_error(BQ_ERR_CUDA, "event");
                }
            }
            const int B = (int)pl.batch;
            if (level % B == 0) {   // fork
                cudaEvent_t l0 = nullptr, l1 = nullptr;
                if (timing && (!(l0 = mkev(levs)) || !(l1 = mkev(levs)))) { cleanup(); return set_error(BQ_ERR_CUDA, "event"); }
                BQ_CKC(cudaEventRecord(efork, s));
                BQ_CKC(cudaStreamWaitEvent(side, efork, 0));
                BQ_SKC(enqueue_flush<KT>(pl, side, l0, l1));
                BQ_CKC(cudaEventRecord(ejoin, side));
            }
            BQ_SKC(enqueue_level<KT>(pl, s, 0, 0, 0, e0, e1, m0, m1, mm));
            if (level % B == B - 1) BQ_CKC(cudaStreamWaitEvent(s, ejoin, 0));   // join
            BQ_SKC(enqueue_level_end<KT>(pl, s, 0, 0, 0));
            host_levels = level + 1;
            if ((level + 1) % B == 0) {
                BQ_CKC(cudaMemcpyAsync(hc.data(), pl.ctrl + level, sizeof(LevelCtrl), cudaMemcpyDeviceToHost, s));
                BQ_CKC(cudaStreamSynchronize(s));
                if (hc[0].nseg_next + hc[0].nmseg_next == 0) break;
            }
        }
        {
            cudaEvent_t l0 = nullptr, l1 = nullptr;
            if (timing && (!(l0 = mkev(levs)) || !(l1 = mkev(levs)))) { cleanup(); return set_error(BQ_ERR_CUDA, "event"); }
            BQ_SKC(enqueue_flush<KT>(pl, s, l0, l1));   // (the loop always ends on a batch boundary)
        }
        // a9: the depth-capped segments
        LoopMisc hm;
        BQ_CKC(cudaMemcpyAsync(&hm, pl.misc, sizeof hm, cudaMemcpyDeviceToHost, s));
        BQ_CKC(cudaStreamSynchronize(s));
        if (hm.fb_count) {
            BQ_SKC(enqueue_fb_setup<KT>(pl, s, 0, 0));
            FbState hf;
            BQ_CKC(cudaMemcpyAsync(&hf, pl.fbst, sizeof hf, cudaMemcpyDeviceToHost, s));
            BQ_CKC(cudaStreamSynchronize(s));
            for (uint32_t p = 0; p < hf.npass; p++) BQ_SKC(enqueue_fb_pass<KT>(pl, s, 0, 0));
            BQ_SKC(enqueue_fb_finish<KT>(pl, s));
        }
    }

    // statistics (and the overflow check) need the device counters: only with
    // stats != NULL or per-launch timing does the call wait for the stream
    if (stats || timing) {
        LoopMisc hm;
        BQ_CKC(cudaMemcpyAsync(&hm, pl.misc, sizeof hm, cudaMemcpyDeviceToHost, s));
        BQ_CKC(cudaStreamSynchronize(s));
        const int levels = (int)hm.level;
        std::vector<LevelCtrl> hctrl(levels > 0 ? levels : 1);
        if (levels > 0) BQ_CKC(cudaMemcpyAsync(hctrl.data(), pl.ctrl, levels * sizeof(LevelCtrl), cudaMemcpyDeviceToHost, s));
        LevelCtrl hroot;
        BQ_CKC(cudaMemcpyAsync(&hroot, pl.root, sizeof hroot, cudaMemcpyDeviceToHost, s));
        BQ_CKC(cudaStreamSynchronize(s));
        if (hm.overflow) {
            cleanup();
            return set_error(BQ_ERR_CUDA, "leaf list overflow");
        }
        const int per_level = 4 + (KT::is_record ? 1 : 0) + (ways > 2 ? 4 : 0);
        local.kernel_launches = 1 + levels * per_level + hm.nflush * (NCLS + 1 + (KT::is_record && !ordered ? 1 : 0)) +
                                (hm.fb_count ? 4 : 0);
        for (int l = 0; l < levels; l++) {
            const LevelCtrl &h = hctrl[l];
            const uint32_t nseg_l = l == 0 ? hroot.nseg_next + hroot.nmseg_next : hctrl[l - 1].nseg_next + hctrl[l - 1].nmseg_next;
            if (nseg_l == 0) break;
            local.levels++;
            local.partition_launches++;
            local.partitioned_segments += nseg_l;
            local.element_passes += h.element_passes + h.mw_element_passes;
            local.multiway_element_passes += h.mw_element_passes;
            local.band_elements += h.band_elems;
            local.leaves += h.nleaf;
        }
        local.leaves += hroot.nleaf;
        local.fallback_segments = hm.fb_count;
        local.partition_bytes = 2.0 * (double)sizeof(T) * (double)(local.element_passes - local.multiway_element_passes);
        if (timing) {
            double ms = 0;
            for (size_t i = 0; i + 1 < evs.size() && (int)(i / 2) < (int)local.levels; i += 2) {
                float f = 0;
                BQ_CKC(cudaEventElapsedTime(&f, evs[i], evs[i + 1]));
                ms += f;
            }
            local.partition_ms = ms;
            double mc = 0, msc = 0;
            for (size_t i = 0; i + 2 < mevs.size() && (int)(i / 3) < (int)local.levels; i += 3) {
                float f = 0, g = 0;
                BQ_CKC(cudaEventElapsedTime(&f, mevs[i], mevs[i + 1]));
                BQ_CKC(cudaEventElapsedTime(&g, mevs[i + 1], mevs[i + 2]));
                mc += f;
                msc += g;
            }
            local.multiway_ms = mc + msc;
            local.mw_count_ms = mc;
            local.mw_scatter_ms = msc;
            double lm = 0;
            for (size_t i = 0; i + 1 < levs.size(); i += 2) {
                float f = 0;
                BQ_CKC(cudaEventElapsedTime(&f, levs[i], levs[i + 1]));
                lm += f;
            }
            local.leaf_ms = lm;
        }
    }
#undef BQ_CKC
#undef BQ_SKC
    cleanup();
    if (stats) *stats = local;
    return BQ_OK;
}

}  // namespace bq
