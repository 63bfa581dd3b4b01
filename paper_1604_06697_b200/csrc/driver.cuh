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

namespace bq {

constexpr int MAX_LEVELS = 128;
// the level loop is enqueued LEVEL_BATCH levels at a time between host checks
#ifndef BQ_LEVEL_BATCH
#define BQ_LEVEL_BATCH 4
#endif
constexpr int LEVEL_BATCH = BQ_LEVEL_BATCH;
constexpr uint32_t POST_GRID = 148 * 8;
constexpr int POST_THREADS = 256;
// the sort's per-level k_post: one small CTA (a warp per child) per segment,
// many resident per SM — deep levels have tens of thousands of segments
#ifndef BQ_POST_LEVEL_THREADS
#define BQ_POST_LEVEL_THREADS 128
#endif
constexpr int POST_LEVEL_THREADS = BQ_POST_LEVEL_THREADS;
constexpr uint32_t POST_LEVEL_GRID = 148 * (2048 / POST_LEVEL_THREADS < 32 ? 2048 / POST_LEVEL_THREADS : 32);
constexpr int MERGE_THREADS = 256, MERGE_IPT = 8;

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
    size_t max_tiles, max_segs, max_leaves, max_fb;
};

template <class KT>
Layout<KT> make_layout(size_t n) {
    constexpr size_t TILE = tile_elems<KT>();
    constexpr size_t S = Tune<KT>::LEAF;
    Layout<KT> L;
    L.max_segs = n / (S + 1) + 2;                 // segments > S are disjoint
    L.max_tiles = n / TILE + 2 * L.max_segs + 2;
    // leaves of one batch of LEVEL_BATCH levels per class list; also fallback chunks
    L.max_leaves = LEVEL_BATCH * (2 * L.max_segs + 2) + (n / S + 2);
    L.max_fb = n / (S + 1) + 2;
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
    // one list per leaf network-size class (leaf.cuh), max_leaves each
    L.leaves[0] = take(leaf_nclass<KT>() * L.max_leaves * sizeof(Leaf));
    L.leaves[1] = take(leaf_nclass<KT>() * L.max_leaves * sizeof(Leaf));
    L.fallback = take(L.max_fb * sizeof(Leaf));
    L.max_copies = KT::is_record ? LEVEL_BATCH * (L.max_segs + 2) + n / 65536 + 2 : 1;
    L.copies[0] = take(L.max_copies * sizeof(Leaf));
    L.copies[1] = take(L.max_copies * sizeof(Leaf));
    L.ctrl = take((MAX_LEVELS + 1) * sizeof(LevelCtrl));   // [MAX_LEVELS]: the root's counts
    L.misc = take(256);   // fallback count, leaf-list counts (2 sets x 8 classes), copy counts, overflow flag; pass counts
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
bq_status launch_multiway(MwParams<KT> MP, LevelCtrl *lc, cudaStream_t s, int ways) {
    using Kn = Kernels<KT>;
    constexpr int threads = Kn::NT + 32;
    if (ways == MW8) {
        constexpr int smem8 = mw8_smem_bytes<KT>();
        auto kc8 = k_mw8_count<KT, Kn::NT, Kn::IPT, MW_STAGES, MW8_MINB>;
        auto ks8 = k_mw8_scatter<KT, Kn::NT, Kn::IPT, MW_STAGES, MW8_MINB>;
        static CapCache cc_c8, cc_s8;
        int cap_c8 = 0, cap_s8 = 0;
        bq_status st = persistent_cap(kc8, threads, smem8, cc_c8, &cap_c8);
        if (st != BQ_OK) return st;
        st = persistent_cap(ks8, threads, smem8, cc_s8, &cap_s8);
        if (st != BQ_OK) return st;
        MP.ticket = &lc->mw_ticket_count;
        kc8<<<cap_c8, threads, smem8, s>>>(MP);
        BQ_CK_LAUNCH();
        k_mw_scan<KT><<<POST_GRID / 8, 256, 0, s>>>(MP);
        BQ_CK_LAUNCH();
        MP.ticket = &lc->mw_ticket_scatter;
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
    MP.ticket = &lc->mw_ticket_count;
    kc<<<cap_c, threads, smem, s>>>(MP);
    BQ_CK_LAUNCH();
    k_mw_scan<KT><<<POST_GRID / 8, 256, 0, s>>>(MP);
    BQ_CK_LAUNCH();
    MP.ticket = &lc->mw_ticket_scatter;
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
    if (count == 0 && LP.count_dev == nullptr) return BQ_OK;   // count 0 + count_dev: persistent grid
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

// Depth-capped segment: chunk leaf sorts + merge passes, result in the user buffer.
template <class KT>
bq_status run_fallback(const Leaf &f, typename KT::T *user, typename KT::T *scratch, Leaf *chunk_list,
                       uint64_t n_total, cudaStream_t s) {
    using T = typename KT::T;
    constexpr uint32_t S = Tune<KT>::LEAF;
    T *bufs[2] = {user, scratch};
    const uint32_t nch = (f.len + S - 1) / S;
    k_chunk_leaves<<<(nch + 255) / 256, 256, 0, s>>>(chunk_list, f.begin, f.len, f.parity, S);
    BQ_CK_LAUNCH();
    LeafParams<KT> LP{};
    LP.leaves = chunk_list;
    LP.bufs[0] = user;
    LP.bufs[1] = scratch;
    LP.out = nullptr;
    LP.out_other = 1;   // sorted chunks land in the other buffer
    LP.n_total = n_total;
    LP.aligned = aligned16(user) && aligned16(scratch);
    bq_status st = launch_leaves<KT>(leaf_nclass<KT>() - 1, LP, nch, s);
    if (st != BQ_OK) return st;
    uint32_t cur = f.parity ^ 1;
    for (uint64_t w = S; w < f.len; w *= 2) {
        const uint64_t threads = (f.len + MERGE_IPT - 1) / MERGE_IPT;
        const uint32_t grid = (uint32_t)((threads + MERGE_THREADS - 1) / MERGE_THREADS);
        k_merge<KT, MERGE_THREADS, MERGE_IPT><<<grid, MERGE_THREADS, 0, s>>>(bufs[cur], bufs[cur ^ 1], f.begin,
                                                                          f.len, (uint32_t)w);
        BQ_CK_LAUNCH();
        cur ^= 1;
    }
    if (cur != 0)
        BQ_CK(cudaMemcpyAsync(user + f.begin, scratch + f.begin, (size_t)f.len * sizeof(T),
                              cudaMemcpyDeviceToDevice, s));
    return BQ_OK;
}

template <class KT>
bq_status run_sort(typename KT::T *data, size_t n, const bq_sort_options *opt, bq_sort_stats *stats, void *ws,
                   size_t ws_bytes, cudaStream_t s) {
    using T = typename KT::T;
    constexpr uint32_t TILE = tile_elems<KT>();
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
        if (depth_limit >= MAX_LEVELS - 2)
            return set_error(BQ_ERR_INVALID_ARGUMENT, "depth_limit %d too large", depth_limit);
    }
    bq_status st = validate<KT>(data, n, ws, ws_bytes);
    if (st != BQ_OK) return st;
    if (n <= 1) {
        if (stats) *stats = local;
        return BQ_OK;
    }
    // default: binary passes for int32 keys (the binary pass is already near
    // the HBM roofline and the cheapest in ALU work per key), 8-way passes
    // (N4) for 64-bit keys, whose binary passes leave ALU headroom (c3:
    // 11.2 -> 10.4 ms random, 12.9 -> 10.3 ms sorted); records stay binary
    // (int32: also multiway where a sort is only a few levels and each
    // level's fixed costs matter: 8-way for 2^17 < n <= 2^23, 16-way up to
    // 2^24 — c1 0.48 -> 0.39 ms, 2^24 0.99 -> 0.90 ms; profiles/r01/ways_sweep.jsonl)
    if (ways == 0) {
        if (sizeof(typename KT::K) == 8 && mw_capable<KT>()) ways = MW8;
        else if (!KT::is_record && n > (1u << 17) && n <= (1u << 23)) ways = MW8;
        else if (!KT::is_record && n > (1u << 23) && n <= (1u << 24)) ways = MW_K;
        else ways = 2;
    }
    if (!mw_capable<KT>()) ways = 2;
    if (depth_limit < 0) {
        int lg = 0;
        for (size_t m = n; m > 1; m >>= 1) lg++;
        depth_limit = 2 * lg + 3;   // P:295, P:1224 (2*ilogb(n)+3)
    }

    const Layout<KT> L = make_layout<KT>(n);
    char *w = static_cast<char *>(ws);
    T *user = data;
    T *scratch = reinterpret_cast<T *>(w + L.scratch);
    uint64_t *status = reinterpret_cast<uint64_t *>(w + L.status);
    uint32_t *tile_map[2];
    Seg *segs[2];
    unsigned long long *cursor[2];
    uint32_t *ecursor[2];
    MSeg<KT> *msegs[2];
    uint32_t *mtile_map[2], *mhist[2], *mcursor[2];
    for (int p = 0; p < 2; p++) {
        tile_map[p] = reinterpret_cast<uint32_t *>(w + L.tile_map[p]);
        segs[p] = reinterpret_cast<Seg *>(w + L.segs[p]);
        cursor[p] = reinterpret_cast<unsigned long long *>(w + L.cursor[p]);
        ecursor[p] = reinterpret_cast<uint32_t *>(w + L.ecursor[p]);
        msegs[p] = reinterpret_cast<MSeg<KT> *>(w + L.msegs[p]);
        mtile_map[p] = reinterpret_cast<uint32_t *>(w + L.mtile_map[p]);
        mhist[p] = reinterpret_cast<uint32_t *>(w + L.mhist[p]);
        mcursor[p] = reinterpret_cast<uint32_t *>(w + L.mcursor[p]);
    }
    // look-back words are only used by the ordered placement
    uint64_t *lb_status = ordered ? status : nullptr;
    Leaf *leaves[2] = {reinterpret_cast<Leaf *>(w + L.leaves[0]), reinterpret_cast<Leaf *>(w + L.leaves[1])};
    Leaf *fallback = reinterpret_cast<Leaf *>(w + L.fallback);
    LevelCtrl *ctrl = reinterpret_cast<LevelCtrl *>(w + L.ctrl);
    LevelCtrl *root = ctrl + MAX_LEVELS;
    uint32_t *fb_count = reinterpret_cast<uint32_t *>(w + L.misc);
    // misc words: [0] fallback count, [4, 12) / [12, 20) leaf counts of set 0 / 1
    // (by class), [20, 22) copy counts, [24] leaf-list overflow flag
    uint32_t *leaf_counts[2] = {fb_count + 4, fb_count + 12};   // [set][class]
    uint32_t *copy_counts[2] = {fb_count + 20, fb_count + 21};
    Leaf *copies[2] = {reinterpret_cast<Leaf *>(w + L.copies[0]), reinterpret_cast<Leaf *>(w + L.copies[1])};
    uint32_t *overflow = fb_count + 24;

    LeafParams<KT> LP{};
    LP.bufs[0] = user;
    LP.bufs[1] = scratch;
    LP.out = user;
    LP.out_other = 0;
    LP.n_total = n;
    LP.aligned = aligned16(user) && aligned16(scratch);

    if (n <= S) {
        k_single_leaf<<<1, 1, 0, s>>>(leaves[0], (uint32_t)n);
        BQ_CK_LAUNCH();
        local.kernel_launches++;
        LP.leaves = leaves[0];
        st = launch_leaves<KT>((int)leaf_class<KT>((uint32_t)n), LP, 1, s);
        if (st != BQ_OK) return st;
        local.kernel_launches++;
        local.leaves = 1;
        if (stats) *stats = local;
        return BQ_OK;
    }

    // Leaves are sorted on a side stream, concurrently with the deeper
    // partition levels: a batch's leaf lists (set batch & 1) are consumed
    // there while the main stream partitions the next batch into the other set.
    cudaStream_t side = nullptr;
    cudaEvent_t ev_levels[2] = {nullptr, nullptr}, ev_leaves[2] = {nullptr, nullptr};
    std::vector<cudaEvent_t> evs;
    std::vector<LevelCtrl> hvec(MAX_LEVELS + 1);   // host copy of the control blocks
    LevelCtrl *hctrl = hvec.data();
    auto cleanup = [&]() {
        for (auto e : evs) cudaEventDestroy(e);
        for (int i = 0; i < 2; i++) {
            if (ev_levels[i]) cudaEventDestroy(ev_levels[i]);
            if (ev_leaves[i]) cudaEventDestroy(ev_leaves[i]);
        }
        if (side) cudaStreamDestroy(side);
    };
#define BQ_CKC(call)                \
    do {                            \
        bq_status st_ = [&]() -> bq_status { BQ_CK(call); return BQ_OK; }(); \
        if (st_ != BQ_OK) { cleanup(); return st_; } \
    } while (0)
    BQ_CKC(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    for (int i = 0; i < 2; i++) {
        BQ_CKC(cudaEventCreateWithFlags(&ev_levels[i], cudaEventDisableTiming));
        BQ_CKC(cudaEventCreateWithFlags(&ev_leaves[i], cudaEventDisableTiming));
    }

    BQ_CKC(cudaMemsetAsync(ctrl, 0, (MAX_LEVELS + 1) * sizeof(LevelCtrl), s));
    BQ_CKC(cudaMemsetAsync(fb_count, 0, 25 * sizeof(uint32_t), s));
    const int aligned = aligned16(user) && aligned16(scratch);
    // children sink of level `lv` (its children form level lv+1; the root is
    // the only "child" of the virtual level -1, counted in `root`)
    auto sink = [&](int lv, int set) {
        PostParams<KT> Q{};
        const int np = (lv + 1) & 1;
        Q.pass.bufs[0] = user;
        Q.pass.bufs[1] = scratch;
        Q.pass.ordered = ordered;
        Q.copies = copies[set];
        Q.copy_count = copy_counts[set];
        Q.next_segs = segs[np];
        Q.next_tile_map = tile_map[np];
        Q.next_cursor = cursor[np];
        Q.next_ecursor = ecursor[np];
        Q.status = lb_status;
        Q.next_msegs = msegs[np];
        Q.next_mtile_map = mtile_map[np];
        Q.next_mhist = mhist[np];
        Q.mhstride = (uint32_t)L.max_segs;
        Q.child_ctrl = lv < 0 ? root : ctrl + lv;
        Q.leaves = leaves[set];
        Q.leaf_counts = leaf_counts[set];
        Q.leaf_cap = (uint32_t)L.max_leaves;
        Q.fallback = fallback;
        Q.fallback_count = fb_count;
        Q.leaf_max = S;
        Q.depth_limit = depth_limit;
        Q.pivot_rule = rule;
        Q.ways = ways;
        Q.emit_children = 1;
        Q.band_inline_max = BAND_INLINE_MAX;
        Q.overflow = overflow;
        return Q;
    };
    {
        PostParams<KT> Q0 = sink(-1, 0);
        k_init_root<KT, POST_THREADS><<<1, POST_THREADS, 0, s>>>(Q0, (uint32_t)n);
        BQ_CKC(cudaGetLastError());
        local.kernel_launches++;
    }

    int level = 0;
    bool done = false;
    for (int batch = 0; !done; batch++) {
        const int set = batch & 1;
        if (level + LEVEL_BATCH >= MAX_LEVELS) {
            cleanup();
            return set_error(BQ_ERR_CUDA, "level loop did not terminate");
        }
        // the side stream has finished the leaves of batch-2 (same set)
        if (batch >= 2) BQ_CKC(cudaStreamWaitEvent(s, ev_leaves[set], 0));
        BQ_CKC(cudaMemsetAsync(leaf_counts[set], 0, MAX_LEAF_CLASSES * sizeof(uint32_t), s));
        BQ_CKC(cudaMemsetAsync(copy_counts[set], 0, sizeof(uint32_t), s));
        for (int k = 0; k < LEVEL_BATCH; k++, level++) {
            const int cp = level & 1;
            const LevelCtrl *prev = level == 0 ? root : ctrl + level - 1;
            PostParams<KT> Q = sink(level, set);
            if (timing) {
                cudaEvent_t e0, e1;
                BQ_CKC(cudaEventCreate(&e0));
                evs.push_back(e0);
                BQ_CKC(cudaEventCreate(&e1));
                evs.push_back(e1);
                BQ_CKC(cudaEventRecord(e0, s));
            }
            if constexpr (mw_capable<KT>()) if (ways > 2) {
                // the level's multiway segments: count, scan, scatter, children
                MwParams<KT> MP{};
                MP.bufs[0] = user;
                MP.bufs[1] = scratch;
                MP.msegs = msegs[cp];
                MP.tile_map = mtile_map[cp];
                MP.hist = mhist[cp];
                MP.cursor = mcursor[cp];
                MP.hstride = (uint32_t)L.max_segs;
                MP.nseg_dev = &prev->nmseg_next;
                MP.ntiles_dev = &prev->nmtiles_next;
                MP.n_total = n;
                MP.aligned = aligned;
                MP.ctrl = ctrl + level;
                st = launch_multiway<KT>(MP, ctrl + level, s, ways);
                if (st != BQ_OK) { cleanup(); return st; }
                local.kernel_launches += 3;
                Q.mw = MP;
                k_post_mw<KT, POST_THREADS><<<POST_GRID, POST_THREADS, 0, s>>>(Q);
                BQ_CKC(cudaGetLastError());
                local.kernel_launches++;
            }
            // the level's binary segments
            PassParams<KT> P{};
            P.bufs[0] = user;
            P.bufs[1] = scratch;
            P.stage[0] = user;
            P.stage[1] = scratch;
            P.final_buf = user;
            P.segs = segs[cp];
            P.tile_map = tile_map[cp];
            P.status = lb_status;
            P.cursor = cursor[cp];
            P.ecursor = ecursor[cp];
            P.ordered = ordered;
            P.ctrl = ctrl + level;
            P.ntiles = 0xffffffffu;             // upper bound: the grid is the resident capacity
            P.ntiles_dev = &prev->ntiles_next;
            P.n_total = n;
            P.aligned = aligned;
            st = launch_partition<KT>(P, s);
            if (st != BQ_OK) { cleanup(); return st; }
            local.kernel_launches++;
            if (timing) BQ_CKC(cudaEventRecord(evs.back(), s));

            Q.pass = P;
            Q.d_counts = nullptr;
            Q.nseg_dev = &prev->nseg_next;
            k_post<KT, POST_LEVEL_THREADS><<<POST_LEVEL_GRID, POST_LEVEL_THREADS, 0, s>>>(Q);
            BQ_CKC(cudaGetLastError());
            local.kernel_launches++;
            st = launch_fill<KT>(Q, s);   // exits at once unless a band was too long for k_post
            if (st != BQ_OK) { cleanup(); return st; }
            local.kernel_launches += KT::is_record ? 2 : 1;
        }
        // leaves of this batch on the side stream
#ifndef BQ_LEAF_MAIN
        cudaStream_t ls = side;
#else
        cudaStream_t ls = s;
#endif
        BQ_CKC(cudaEventRecord(ev_levels[set], s));
        BQ_CKC(cudaStreamWaitEvent(ls, ev_levels[set], 0));
        for (int c = 0; c < NCLS; c++) {
            LP.leaves = leaves[set] + (size_t)c * L.max_leaves;
            LP.count_dev = leaf_counts[set] + c;
            st = launch_leaves<KT>(c, LP, 0, ls);
            if (st != BQ_OK) { cleanup(); return st; }
            local.kernel_launches++;
        }
        if (KT::is_record && !ordered) {
            k_copy_runs<KT, POST_THREADS><<<POST_GRID, POST_THREADS, 0, ls>>>(copies[set], copy_counts[set], user,
                                                                               scratch);
            BQ_CKC(cudaGetLastError());
            local.kernel_launches++;
        }
        BQ_CKC(cudaEventRecord(ev_leaves[set], ls));
        // is there a next level?
        BQ_CKC(cudaMemcpyAsync(hctrl + level - 1, ctrl + level - 1, sizeof(LevelCtrl), cudaMemcpyDeviceToHost, s));
        BQ_CKC(cudaStreamSynchronize(s));
        done = hctrl[level - 1].nseg_next == 0 && hctrl[level - 1].nmseg_next == 0;
    }
    LP.count_dev = nullptr;
    BQ_CKC(cudaStreamWaitEvent(s, ev_leaves[0], 0));
    BQ_CKC(cudaStreamWaitEvent(s, ev_leaves[1], 0));

    // statistics of every level, and the depth-capped segments
    BQ_CKC(cudaMemcpyAsync(hctrl, ctrl, level * sizeof(LevelCtrl), cudaMemcpyDeviceToHost, s));
    uint32_t misc_h[25];
    BQ_CKC(cudaMemcpyAsync(misc_h, fb_count, sizeof misc_h, cudaMemcpyDeviceToHost, s));
    BQ_CKC(cudaStreamSynchronize(s));
    const uint32_t nfb_total = misc_h[0];
    if (misc_h[24]) { cleanup(); return set_error(BQ_ERR_CUDA, "leaf list overflow"); }
    for (int l = 0; l < level; l++) {
        const LevelCtrl &hc = hctrl[l];
        const uint32_t nseg_l = l == 0 ? 1u : hctrl[l - 1].nseg_next + hctrl[l - 1].nmseg_next;
        if (nseg_l == 0) break;
        local.levels++;
        local.partition_launches++;
        local.partitioned_segments += nseg_l;
        local.element_passes += hc.element_passes;
        local.band_elements += hc.band_elems;
        local.leaves += hc.nleaf;
    }
    local.fallback_segments = nfb_total;

    if (nfb_total) {
        std::vector<Leaf> fl(nfb_total);
        BQ_CKC(cudaMemcpyAsync(fl.data(), fallback, nfb_total * sizeof(Leaf), cudaMemcpyDeviceToHost, s));
        BQ_CKC(cudaStreamSynchronize(s));
        for (const Leaf &f : fl) {
            st = run_fallback<KT>(f, user, scratch, leaves[0], n, s);
            if (st != BQ_OK) { cleanup(); return st; }
        }
    }
    local.partition_bytes = 2.0 * (double)sizeof(T) * (double)local.element_passes;
    if (timing) {
        BQ_CKC(cudaStreamSynchronize(s));
        double ms = 0;
        // only the launches of non-empty levels count
        for (size_t i = 0; i + 1 < evs.size() && (int)(i / 2) < (int)local.levels; i += 2) {
            float f = 0;
            BQ_CKC(cudaEventElapsedTime(&f, evs[i], evs[i + 1]));
            ms += f;
        }
        local.partition_ms = ms;
    }
#undef BQ_CKC
    cleanup();
    if (stats) *stats = local;
    return BQ_OK;
}

}  // namespace bq
