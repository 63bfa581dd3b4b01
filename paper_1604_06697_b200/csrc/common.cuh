// common.cuh — key traits, tile geometry, status words and PTX helpers shared
// by the sm_100a kernels of libbq.so.  (The CPU oracle in oracle/ shares
// nothing with this file.)
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstddef>
#include <type_traits>
#include <cuda_runtime.h>

#include "bq.h"

namespace bq {

// Bounds checks of the kernels' computed indices, compiled in only with
// -DBQ_CHECKS (a checking build of the library, tools/variants.py; the pool's
// compute-sanitizer is closed): a failed check prints where and traps, so the
// call fails with a CUDA error instead of corrupting memory silently.
#ifdef BQ_CHECKS
#define BQ_CHECK(cond)                                                                          \
    do {                                                                                        \
        if (!(cond)) {                                                                          \
            printf("BQ_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
                   (int)blockIdx.x, (int)threadIdx.x);                                          \
            __trap();                                                                           \
        }                                                                                       \
    } while (0)
#else
#define BQ_CHECK(cond) \
    do {               \
    } while (0)
#endif

// ---------------------------------------------------------------------------
// Resident-CTA capacity of a kernel, cached per device: the library's only
// mutable host state (include/bq.h: "an immutable per-device cache of launch
// limits").  Each slot is written once, with the same value by any racing
// caller, through atomic builtins; the shared-memory attribute is set on the
// first launch per device.
// ---------------------------------------------------------------------------
constexpr int MAX_DEVICES = 64;
struct CapCache {
    int v[MAX_DEVICES];
};
template <class F>
cudaError_t resident_ctas(F kern, int threads, size_t smem, CapCache &cc, int *cap, int per_sm_max = 0) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= MAX_DEVICES) return cudaErrorInvalidDevice;
    int c = __atomic_load_n(&cc.v[dev], __ATOMIC_ACQUIRE);
    if (c == 0) {
        if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
            return e;
        int nb = 0, sms = 0;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, smem)) != cudaSuccess) return e;
        if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
        if (nb < 1) return cudaErrorInvalidConfiguration;   // the kernel does not fit on an SM
        if (per_sm_max > 0 && nb > per_sm_max) nb = per_sm_max;
        c = nb * sms;
        __atomic_store_n(&cc.v[dev], c, __ATOMIC_RELEASE);
    }
    *cap = c;
    return cudaSuccess;
}

// ---------------------------------------------------------------------------
// Key traits.  `T` is the storage type moved by the passes, `K` the unsigned
// or signed type compared.  H0: float64 is compared through the
// order-preserving bijection  sign set -> ~bits, else bits | 2^63  (IEEE 754
// totalOrder on non-NaN values, R9); the stored bits are never
// changed, so decode(encode(x)) == x bit for bit.
// ---------------------------------------------------------------------------
struct alignas(16) Rec32 {
    uint64_t key;
    uint64_t p[3];
};

struct KI32 {
    using T = int32_t;
    using K = int32_t;
    static constexpr bq_kind kind = BQ_I32;
    static constexpr int W = 4;          // bytes per element
    static constexpr bool is_record = false;
    __host__ __device__ static K key(T v) { return v; }
    __host__ __device__ static T from_key(K k) { return k; }
    static constexpr K KMAX = 0x7fffffff;
};

struct KU64 {
    using T = uint64_t;
    using K = uint64_t;
    static constexpr bq_kind kind = BQ_U64;
    static constexpr int W = 8;
    static constexpr bool is_record = false;
    __host__ __device__ static K key(T v) { return v; }
    __host__ __device__ static T from_key(K k) { return k; }
    static constexpr K KMAX = ~0ull;
};

struct KF64 {
    using T = uint64_t;                  // the double's bit pattern
    using K = uint64_t;
    static constexpr bq_kind kind = BQ_F64;
    static constexpr int W = 8;
    static constexpr bool is_record = false;
    __host__ __device__ static K key(T b) {
        return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
    }
    __host__ __device__ static T from_key(K k) {
        return (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    }
    static constexpr K KMAX = ~0ull;
};

struct KRec {
    using T = Rec32;
    using K = uint64_t;
    static constexpr bq_kind kind = BQ_REC32;
    static constexpr int W = 32;
    static constexpr bool is_record = true;
    __host__ __device__ static K key(const T &r) { return r.key; }
    static constexpr K KMAX = ~0ull;
};

// key + index pair (bq_keyidx16): the key+index record path (SURVEY §8(f)
// N3) sorts these and gathers the records once; also a public kind
struct alignas(16) KeyIdx16 {
    uint64_t key;
    uint64_t idx;
};

struct KPair {
    using T = KeyIdx16;
    using K = uint64_t;
    static constexpr bq_kind kind = BQ_KEYIDX16;
    static constexpr int W = 16;
    static constexpr bool is_record = true;
    __host__ __device__ static K key(const T &r) { return r.key; }
    static constexpr K KMAX = ~0ull;
};

// Per-kind tuning constants.  TILE = elements per partition tile (one CTA),
// LEAF = largest segment finished by the shared-memory leaf sort (S) =
// LEAF_IPT keys per thread x LEAF_NT threads (leaf.cuh: a merge sort whose
// runs start as per-thread register networks of LEAF_IPT keys; LEAF_IPT is
// odd so that per-thread strided shared-memory accesses are conflict-free).
// PART_THREADS = consumer threads of the partition kernel (one more producer
// warp is added), PART_IPT = elements per consumer thread, PART_STAGES = TMA
// load pipeline depth, PART_MINB = CTAs per SM the register budget targets.
template <class KT> struct Tune;
#ifndef BQ_I32_IPT
#define BQ_I32_IPT 16
#endif
#ifndef BQ_I32_STAGES
#define BQ_I32_STAGES 4
#endif
#ifndef BQ_I32_MINB
#define BQ_I32_MINB 2
#endif
#ifndef BQ_LEAF_IPT32
#define BQ_LEAF_IPT32 31
#endif
#ifndef BQ_LEAF_NT32
#define BQ_LEAF_NT32 1024
#endif
#ifndef BQ_LEAF_IPT64
#define BQ_LEAF_IPT64 15
#endif
#ifndef BQ_LEAF_NT64
#define BQ_LEAF_NT64 1024
#endif
#ifndef BQ_LEAF_IPTREC
#define BQ_LEAF_IPTREC 9
#endif
#ifndef BQ_LEAF_NTREC
#define BQ_LEAF_NTREC 1024
#endif
#ifndef BQ_MW8_MINB
#define BQ_MW8_MINB 2
#endif
#ifndef BQ_MW8_MINB_PAIR
#define BQ_MW8_MINB_PAIR 3
#endif
// MW8_MINB: resident CTAs per SM the 8-way kernels are compiled for (pairs:
// 3, their 4-key threads fit 72 registers; 64-bit keys spill there)
template <> struct Tune<KI32> {
    static constexpr int PART_THREADS = 256, PART_IPT = BQ_I32_IPT, PART_STAGES = BQ_I32_STAGES,
                         PART_MINB = BQ_I32_MINB, MW8_MINB = BQ_MW8_MINB;
    static constexpr int LEAF_IPT = BQ_LEAF_IPT32, LEAF_NT = BQ_LEAF_NT32, LEAF = LEAF_IPT * LEAF_NT;
};
template <> struct Tune<KU64> {
    static constexpr int PART_THREADS = 256, PART_IPT = 8, PART_STAGES = 4, PART_MINB = 2,   // 16 KB tiles
                         MW8_MINB = BQ_MW8_MINB;
    static constexpr int LEAF_IPT = BQ_LEAF_IPT64, LEAF_NT = BQ_LEAF_NT64, LEAF = LEAF_IPT * LEAF_NT;
};
template <> struct Tune<KF64> : Tune<KU64> {};
#ifndef BQ_REC_STAGES
#define BQ_REC_STAGES 4
#endif
template <> struct Tune<KRec> {
    static constexpr int PART_THREADS = 256, PART_IPT = 2, PART_STAGES = BQ_REC_STAGES, PART_MINB = 2,   // 16 KB tiles
                         MW8_MINB = BQ_MW8_MINB;
    static constexpr int LEAF_IPT = BQ_LEAF_IPTREC, LEAF_NT = BQ_LEAF_NTREC, LEAF = LEAF_IPT * LEAF_NT;
};
template <> struct Tune<KPair> {
    static constexpr int PART_THREADS = 256, PART_IPT = 4, PART_STAGES = 4, PART_MINB = 2,   // 16 KB tiles
                         MW8_MINB = BQ_MW8_MINB_PAIR;
    static constexpr int LEAF_IPT = BQ_LEAF_IPTREC, LEAF_NT = BQ_LEAF_NTREC, LEAF = LEAF_IPT * LEAF_NT;
};

#ifndef BQ_MW8W
#define BQ_MW8W 1   // 8-way levels: warp-private tiles with exact offsets (multiway8w.cuh)
#endif
#ifndef BQ_PART_CHUNK
#define BQ_PART_CHUNK 4
#endif
constexpr uint32_t PART_CHUNK = BQ_PART_CHUNK;   // consecutive tiles per ticket of k_part_fast's loader

template <class KT> constexpr int tile_elems() { return Tune<KT>::PART_THREADS * Tune<KT>::PART_IPT; }

// Tiles are laid out from each segment's 16-byte-aligned begin: with
// ab = b rounded down to VW elements (VW = elements per 16 bytes), tile j of
// [b, e) covers [ab + j*T, ab + (j+1)*T) ∩ [b, e).  Every tile starts 16-byte
// aligned (a 1D TMA copy), interior tiles are full, and a
// segment has ceil((e - ab) / T) tiles — not the extra partial tile that
// anchoring at absolute multiples of T costs small segments.
template <class KT>
__host__ __device__ constexpr uint32_t tile_vw() { return sizeof(typename KT::T) >= 16 ? 1u : 16u / (uint32_t)sizeof(typename KT::T); }
template <class KT>
__host__ __device__ inline uint32_t seg_tiles(uint32_t b, uint32_t len) {
    constexpr uint32_t T = (uint32_t)tile_elems<KT>();
    return (uint32_t)(((uint64_t)len + b % tile_vw<KT>() + T - 1) / T);
}

// ---------------------------------------------------------------------------
// Segment descriptor (the GPU form of the paper's explicit stack frame,
// P:1225-1229, plus the pivot and the tile range of the current level).
// ---------------------------------------------------------------------------
struct alignas(16) Seg {
    uint64_t pivot;      // key (K) of the pivot; raw bits recovered via from_key
    uint32_t begin;
    uint32_t len;
    uint32_t tile_base;  // first tile id of this segment in the level
    uint32_t ntiles;
    uint16_t depth;      // recursion depth (Introsort counter)
    uint8_t parity;      // 0: data in the user buffer, 1: in scratch
    uint8_t pad0;
    uint32_t pad1;
};
static_assert(sizeof(Seg) == 32, "Seg layout");

struct alignas(16) Leaf {
    uint32_t begin;
    uint32_t len;
    uint32_t parity;
    uint32_t pad;
};

constexpr int MAX_LEVELS = 128;   // control blocks of a sort's level loop (depth limit < MAX_LEVELS - 3)
// levels per iteration of the level loop (driver.cuh): at most LOOP_BATCH;
// sorts of up to LOOP_SMALL_N keys use LOOP_BATCH_SMALL (fewer trailing empty
// levels).  Leaves of a batch go to list set (level / batch) & 1, kept in
// LoopMisc::set by k_level_end.
#ifndef BQ_LOOP_BATCH
#define BQ_LOOP_BATCH 4
#endif
constexpr uint32_t LOOP_BATCH = BQ_LOOP_BATCH;
constexpr uint32_t LOOP_BATCH_SMALL = 2;
// multiway sorts run their predicted number of levels as one batch (no
// trailing empty level slots), up to this many
constexpr uint32_t LOOP_BATCH_MAX = 6;
constexpr size_t LOOP_SMALL_N = (size_t)1 << 22;

// Per-level control block.  One per level, zeroed once per sort, so no
// counter is reused within a call.
struct alignas(64) LevelCtrl {
    uint32_t ticket;         // tile tickets of the binary partition kernel
    uint32_t nseg_next;      // binary children appended to the next level
    uint32_t ntiles_next;    // their tiles
    uint32_t maxtiles_next;  // largest child tile count
    uint32_t nleaf;          // leaves appended by this level
    uint32_t nfallback;      // depth-capped segments appended by this level
    uint32_t nbig;           // equal bands left to k_fill
    uint32_t mw_ticket_count;    // tile tickets of the multiway count kernel
    unsigned long long element_passes;  // sum of partitioned lengths this level
    unsigned long long band_elems;      // equal-band elements this level
    uint32_t nleaf_cls[8];              // leaves appended per network-size class
    uint32_t mw_ticket_scatter;  // tile tickets of the multiway scatter kernel
    uint32_t nmseg_next;         // multiway children appended to the next level
    uint32_t nmtiles_next;       // their tiles
    uint32_t mw_scan_done;       // 8-way: blocks of the tile-count scan done (multiway8w.cuh)
    unsigned long long mw_element_passes;   // sum of multiway-partitioned lengths this level
    uint32_t pad2[6];
};
static_assert(sizeof(LevelCtrl) == 128, "LevelCtrl layout");

// ---------------------------------------------------------------------------
// Decoupled look-back status word: flag:2 | lt:31 | gt:31.
// ---------------------------------------------------------------------------
constexpr uint64_t ST_AGG = 1ull << 62;
constexpr uint64_t ST_INC = 2ull << 62;
constexpr uint64_t M31 = 0x7fffffffull;
__host__ __device__ inline uint64_t st_pack(uint64_t flag, uint32_t lt, uint32_t gt) {
    return flag | ((uint64_t)lt << 31) | (uint64_t)gt;
}
__host__ __device__ inline uint32_t st_lt(uint64_t w) { return (uint32_t)((w >> 31) & M31); }
__host__ __device__ inline uint32_t st_gt(uint64_t w) { return (uint32_t)(w & M31); }
__host__ __device__ inline uint32_t st_flag(uint64_t w) { return (uint32_t)(w >> 62); }

// Status words carry self-contained counts, so publishing and polling need no
// acquire/release ordering: relaxed gpu-scope 64-bit accesses (single-copy
// atomic) avoid the L1 invalidation (CCTL.IVALL) an acquire load costs per poll.
// A tile's word is published twice by different threads (aggregate by the
// producer warp, inclusive by the consumers) and the two stores are not
// ordered in L2, so both are published with atom.max: ST_INC > ST_AGG in the
// flag bits, so the inclusive word wins whatever the arrival order.
__device__ __forceinline__ void st_publish_u64(uint64_t *p, uint64_t v) {
    atomicMax(reinterpret_cast<unsigned long long *>(p), (unsigned long long)v);
}
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// ---- optional per-tile phase trace (tools/trace_pass.py; build with -DBQ_TRACE) --
#ifdef BQ_TRACE
static __device__ unsigned long long g_trace[1 << 17][8];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define BQ_TR(t, k, v)                                   \
    do {                                                 \
        if ((t) < (1u << 17)) g_trace[(t)][(k)] = (v);   \
    } while (0)
#else
#define BQ_TR(t, k, v) \
    do {               \
    } while (0)
#endif

// Waiting warps must not steal issue slots from the working ones: try_wait
// suspends the thread for up to this many ns per attempt (it wakes as soon as
// the phase completes), and look-back polls back off with nanosleep.
#ifndef BQ_MBAR_SLEEP_NS
#define BQ_MBAR_SLEEP_NS 1000000
#endif
#ifndef BQ_POLL_SLEEP_NS
#define BQ_POLL_SLEEP_NS 64
#endif

// ---- mbarrier / bulk-copy (TMA) helpers (sm_90+ PTX, used on sm_100a) --------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(BQ_MBAR_SLEEP_NS)
        : "memory");
}
// 1D bulk copy global -> shared, completion counted on an mbarrier (UBLKCP).
__device__ __forceinline__ void tma_load_1d(void *smem_dst, const void *gsrc, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem_dst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// 1D bulk copy shared -> global (bulk-group completion).
__device__ __forceinline__ void tma_store_1d(void *gdst, const void *smem_src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
                 "r"(smem_u32(smem_src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// make generic-proxy shared-memory writes visible to the async (TMA) proxy
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Streaming 128-bit loads of read-once data (no L1 allocation).
__device__ __forceinline__ uint4 ldg_stream(const uint4 *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
// Plain (coherent) streaming load, for buffers written during the same kernel.
__device__ __forceinline__ uint4 ldg_cs(const uint4 *p) { return __ldcs(p); }

// Pivot sample selection (hot-path step a1; Appendix B sort_pair /
// median_of_3): a three-comparator network with selects.
template <class K>
__device__ __forceinline__ void sort_pair(K &a, K &b) {
    K lo = b < a ? b : a;
    K hi = b < a ? a : b;
    a = lo;
    b = hi;
}
template <class K>
__device__ __forceinline__ K median3(K a, K b, K c) {
    sort_pair(a, b);
    sort_pair(b, c);
    sort_pair(a, b);
    return b;
}

template <class KT>
__device__ __forceinline__ typename KT::K load_key(const typename KT::T *buf, uint64_t i) {
    return KT::key(buf[i]);
}

// SAMPLE64 (N1, R18/R19): one warp loads 64 keys, key j from the
// j-th of 64 equal strata of the segment at an offset drawn by SplitMix64
// from (segment begin, length, j) — the paper's suggestion of a fast
// pseudo-random generator for sample selection, which keeps
// periodic inputs from aliasing with the sample (lane l holds j = l and
// j = l + 32); sorts them with a bitonic network (register compare-exchange
// for index bit 5, shuffles for bits 0-4) and returns the 32nd smallest to
// every lane.
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t sample64_pos(uint32_t b, uint32_t len, uint32_t j) {
    const uint64_t s0 = ((uint64_t)j * len) >> 6, s1 = ((uint64_t)(j + 1) * len) >> 6;
    const uint64_t r = splitmix64((((uint64_t)b << 32) | len) + (uint64_t)(j + 1) * 0x9E3779B97F4A7C15ull) >> 32;
    uint64_t pos = s0 + ((r * (s1 - s0)) >> 32);
    return (uint64_t)b + (pos < len - 1 ? pos : len - 1);
}
template <class KT>
__device__ typename KT::K sample64_pivot_warp(const typename KT::T *buf, uint32_t b, uint32_t len, uint32_t lane,
                                              uint32_t q = 31) {
    using K = typename KT::K;
    K v[2];
#pragma unroll
    for (int r = 0; r < 2; r++) v[r] = load_key<KT>(buf, sample64_pos(b, len, lane + 32 * r));
#pragma unroll
    for (int m = 1; m <= 6; m++) {
#pragma unroll
        for (int bb = m - 1; bb >= 0; bb--) {
            if (bb == 5) {   // only in the last merge: ascending
                const K lo = v[1] < v[0] ? v[1] : v[0], hi = v[1] < v[0] ? v[0] : v[1];
                v[0] = lo;
                v[1] = hi;
                continue;
            }
#pragma unroll
            for (int r = 0; r < 2; r++) {
                const uint32_t i = lane + 32 * r;
                const K p = __shfl_xor_sync(0xffffffffu, v[r], 1 << bb);
                const bool lower = ((lane >> bb) & 1) == 0;
                const bool asc = m == 6 || ((i >> m) & 1) == 0;
                const bool take_min = lower == asc;
                v[r] = take_min ? (p < v[r] ? p : v[r]) : (v[r] < p ? p : v[r]);
            }
        }
    }
    // the (q+1)-th smallest sample key (q uniform; 31: the lower median)
    return __shfl_sync(0xffffffffu, q < 32 ? v[0] : v[1], q & 31);
}
// the same, plus whether the 31st or 33rd smallest sample key equals the pivot
template <class KT>
__device__ typename KT::K sample64_pivot_warp_dup(const typename KT::T *buf, uint32_t b, uint32_t len,
                                                  uint32_t lane, bool *dup) {
    using K = typename KT::K;
    K v[2];
#pragma unroll
    for (int r = 0; r < 2; r++) v[r] = load_key<KT>(buf, sample64_pos(b, len, lane + 32 * r));
#pragma unroll
    for (int m = 1; m <= 6; m++) {
#pragma unroll
        for (int bb = m - 1; bb >= 0; bb--) {
            if (bb == 5) {
                const K lo = v[1] < v[0] ? v[1] : v[0], hi = v[1] < v[0] ? v[0] : v[1];
                v[0] = lo;
                v[1] = hi;
                continue;
            }
#pragma unroll
            for (int r = 0; r < 2; r++) {
                const uint32_t i = lane + 32 * r;
                const K p = __shfl_xor_sync(0xffffffffu, v[r], 1 << bb);
                const bool lower = ((lane >> bb) & 1) == 0;
                const bool asc = m == 6 || ((i >> m) & 1) == 0;
                v[r] = (lower == asc) ? (p < v[r] ? p : v[r]) : (v[r] < p ? p : v[r]);
            }
        }
    }
    const K piv = __shfl_sync(0xffffffffu, v[0], 31);
    const K below = __shfl_sync(0xffffffffu, v[0], 30), above = __shfl_sync(0xffffffffu, v[1], 0);
    *dup = !(below < piv) || !(piv < above);
    return piv;
}

// The duplicate check "dc" at the leaf boundary: the lower median
// of the 64-key sample of a segment and the number of distinct keys in the
// sample (whole warp).
template <class KT>
__device__ typename KT::K sample64_median_distinct(const typename KT::T *buf, uint32_t b, uint32_t len, uint32_t lane,
                                                    uint32_t *distinct) {
    using K = typename KT::K;
    K v[2];
#pragma unroll
    for (int r = 0; r < 2; r++) v[r] = load_key<KT>(buf, sample64_pos(b, len, lane + 32 * r));
#pragma unroll
    for (int m = 1; m <= 6; m++) {
#pragma unroll
        for (int bb = m - 1; bb >= 0; bb--) {
            if (bb == 5) {
                const K lo = v[1] < v[0] ? v[1] : v[0], hi = v[1] < v[0] ? v[0] : v[1];
                v[0] = lo;
                v[1] = hi;
                continue;
            }
#pragma unroll
            for (int r = 0; r < 2; r++) {
                const uint32_t i = lane + 32 * r;
                const K p = __shfl_xor_sync(0xffffffffu, v[r], 1 << bb);
                const bool lower = ((lane >> bb) & 1) == 0;
                const bool asc = m == 6 || ((i >> m) & 1) == 0;
                v[r] = (lower == asc) ? (p < v[r] ? p : v[r]) : (v[r] < p ? p : v[r]);
            }
        }
    }
    // sorted: index i = lane + 32 r; a new value starts where it differs from i - 1
    const K prev0 = __shfl_up_sync(0xffffffffu, v[0], 1);
    const K last0 = __shfl_sync(0xffffffffu, v[0], 31);
    const K prev1 = __shfl_up_sync(0xffffffffu, v[1], 1);
    const bool n0 = lane == 0 || prev0 != v[0];
    const bool n1 = lane == 0 ? last0 != v[1] : prev1 != v[1];
    *distinct = __popc(__ballot_sync(0xffffffffu, n0)) + __popc(__ballot_sync(0xffffffffu, n1));
    return __shfl_sync(0xffffffffu, v[0], 31);
}

// Pivot of buf[b, b+len) by `rule`, computed by a whole warp (all 32 lanes
// must call it; every lane gets the result).  *dup (if non-null) tells whether
// another key of the rule's sample equals the pivot.
template <class KT>
__device__ typename KT::K select_pivot_warp(const typename KT::T *buf, uint32_t b, uint32_t len, int rule,
                                            uint32_t lane, bool *dup = nullptr, uint32_t q = 31);

// Mo3 over {b, b+len/2, e-1}; ninther over b + floor(k*(len-1)/8), k=0..8.
template <class KT>
__device__ typename KT::K select_pivot(const typename KT::T *buf, uint32_t b, uint32_t len, int rule) {
    using K = typename KT::K;
    if (rule == BQ_PIVOT_NINTHER && len >= 9) {
        K m[3];
#pragma unroll
        for (int g = 0; g < 3; g++) {
            K x[3];
#pragma unroll
            for (int k = 0; k < 3; k++)
                x[k] = load_key<KT>(buf, (uint64_t)b + ((uint64_t)(3 * g + k) * (len - 1)) / 8);
            m[g] = median3(x[0], x[1], x[2]);
        }
        return median3(m[0], m[1], m[2]);
    }
    return median3(load_key<KT>(buf, b), load_key<KT>(buf, (uint64_t)b + len / 2),
                   load_key<KT>(buf, (uint64_t)b + len - 1));
}

template <class KT>
__device__ typename KT::K select_pivot_warp(const typename KT::T *buf, uint32_t b, uint32_t len, int rule,
                                            uint32_t lane, bool *dup, uint32_t q) {
    using K = typename KT::K;
    if (rule == BQ_PIVOT_SAMPLE64) {
        if (dup) return sample64_pivot_warp_dup<KT>(buf, b, len, lane, dup);
        return sample64_pivot_warp<KT>(buf, b, len, lane, q);
    }
    K p = 0;
    uint32_t eq = 0;
    if (lane == 0) {
        p = select_pivot<KT>(buf, b, len, rule);
        if (dup) {
            // how many keys of the rule's sample equal the pivot
            if (rule == BQ_PIVOT_NINTHER && len >= 9) {
                for (int k = 0; k < 9; k++) eq += load_key<KT>(buf, (uint64_t)b + ((uint64_t)k * (len - 1)) / 8) == p;
            } else {
                eq = (load_key<KT>(buf, b) == p) + (load_key<KT>(buf, (uint64_t)b + len / 2) == p) +
                     (load_key<KT>(buf, (uint64_t)b + len - 1) == p);
            }
        }
    }
    if (dup) *dup = __shfl_sync(0xffffffffu, eq, 0) >= 2;
    return __shfl_sync(0xffffffffu, p, 0);
}

}  // namespace bq
