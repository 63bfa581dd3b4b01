/*
 * bq.h — C-ABI of libbq.so, the B200-native (sm_100a) BlockQuicksort hot path.
 *
 * Paper: S. Edelkamp, A. Weiß, "BlockQuicksort: How Branch Mispredictions
 * don't affect Quicksort", arXiv 1604.06697 (PAPER.md; P:n = line n).
 *
 * The operations follow the paper's problem statements:
 *   - partition: "returns a pointer p ... all elements left of p are smaller
 *     or equal the pivot and all elements on the right are greater or equal"
 *     (§2); realised three-way (< | == | >), so the returned split
 *     is #{k < pivot} and the equal band is reported separately (the paper's
 *     duplicate check "dc", always on);
 *   - sort: Quicksort/Introsort driven by that partitioner (Alg. 1 P:272-284;
 *     §2 "Quicksort and improvements" P:286-330; Appendix B).
 *
 * Conventions for every entry point
 *   - Data pointers (keys, recs, src, dst) are DEVICE pointers owned by the
 *     caller (e.g. torch tensors); the library keeps none of them after the
 *     call returns.  Host pointers appear only where stated (bq_sort_host,
 *     split/n_equal/pivot/stats out-params).
 *   - `ws` is caller-allocated DEVICE workspace of at least
 *     bq_workspace_bytes(kind, n) bytes, 256-byte aligned, not aliasing the
 *     data.  It may be reused across calls on the same stream.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream).  All device work is enqueued on it.
 *   - n must satisfy n <= 2^31 - 1 (BQ_ERR_INVALID_ARGUMENT otherwise);
 *     n = 0 and n = 1 are valid no-ops.
 *   - Errors are returned as bq_status; no exception crosses the ABI.  On
 *     BQ_ERR_CUDA the CUDA error text is available from bq_last_error()
 *     (thread-local).  A device that is not sm_100 gives BQ_ERR_UNSUPPORTED.
 *   - The library's only mutable host state is a per-device cache of launch
 *     limits and a mutex-protected cache of instantiated sort graphs (see
 *     bq_sort_*); concurrent calls on disjoint data and distinct workspaces are
 *     safe.
 *
 * Orders
 *   - int32, uint64: natural order (signed / unsigned).
 *   - float64: IEEE 754 totalOrder restricted to non-NaN values (-0.0 < +0.0)
 *     (reading R9; the paper sorts ints).  NaN inputs are
 *     outside the contract (they are ordered deterministically by bit pattern).
 *   - records: by `key` only ("Only the first component is compared",
 *     P:671-672); the order among equal keys is unspecified, as in Quicksort.
 */
#ifndef BQ_H
#define BQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define BQ_API __attribute__((visibility("default")))
#else
#define BQ_API
#endif

typedef enum {
    BQ_OK = 0,
    BQ_ERR_INVALID_ARGUMENT = 1, /* NULL with n > 0, n >= 2^31, bad alignment, bad enum */
    BQ_ERR_WORKSPACE = 2,        /* ws NULL or ws_bytes < bq_workspace_bytes(kind, n) */
    BQ_ERR_CUDA = 3,             /* a CUDA runtime call failed; see bq_last_error() */
    BQ_ERR_UNSUPPORTED = 4       /* no CUDA device, or the device is not sm_100 */
} bq_status;

typedef enum { BQ_I32 = 0, BQ_U64 = 1, BQ_F64 = 2, BQ_REC32 = 3, BQ_KEYIDX16 = 4 } bq_kind;

/* Pivot sample rules (§2; §4 "pivot selection" P:719-753):
 *   MO3     median of the keys at segment positions {b, b+floor(len/2), e-1}
 *           (Appendix B median_of_3, P:1069-1075, P:1215 read with e-1);
 *   NINTHER pseudomedian of 9 = median of the medians of three triples, at
 *           positions b + floor(k*(len-1)/8), k = 0..8;
 *   SAMPLE64 lower median (the 32nd smallest) of 64 keys, key j drawn from
 *           the j-th of 64 equal strata of the segment at an offset given by
 *           SplitMix64 of (segment begin, length, j): the paper's "larger
 *           sample" idea (median of sqrt(n)) at a fixed
 *           sample size, with the pseudo-random sample selection it suggests
 *            (R18, R19); computed by one warp with a
 *           shuffle network.  For bq_pivot_* the segment is [0, n). */
typedef enum { BQ_PIVOT_MO3 = 0, BQ_PIVOT_NINTHER = 1, BQ_PIVOT_SAMPLE64 = 2 } bq_pivot_rule;

/* 32-byte record: key + 24-byte payload, 16-byte aligned in device memory
 * (BASELINE.json config 5; the paper's "Record" element). */
typedef struct {
    uint64_t key;
    uint64_t payload[3];
} bq_record32;

/* 16-byte key + index pair, 16-byte aligned (the key+index
 * record variant).  Ordered by `key` only, like records; `idx` travels with
 * its key.  bq_sort_records sorts (key, position) pairs of this type and
 * then gathers every 32-byte record once (bq_sort_options.records). */
typedef struct {
    uint64_t key;
    uint64_t idx;
} bq_keyidx16;

typedef struct {
    int32_t pivot_rule;   /* bq_pivot_rule for segments > leaf size; default SAMPLE64 */
    int32_t depth_limit;  /* < 0: Introsort limit 2*floor(log2 n)+3 */
    int32_t timing;       /* != 0: host-driven level loop, CUDA events around every binary
                             partition launch, each multiway level's count + scan and
                             scatter, and the leaf launches (bq_sort_stats.partition_ms,
                             mw_count_ms, mw_scatter_ms, leaf_ms); the call waits */
    int32_t ordered;      /* != 0: ticket-ordered tile placement (decoupled look-back),
                             deterministic layout; 0: one atomicAdd per tile (faster; tiles
                             of a segment placed in completion order; records then move
                             by two-way passes).  Sorted keys are identical. */
    int32_t ways;         /* 0 (default): 8-way passes for int32 keys above 2^17 (16-way for
                             2^21 < n <= 2^23; binary up to 2^17), for uint64/float64 keys
                             and key+index pairs (so also for bq_sort_records' default
                             path); binary for 32-byte records; 2: binary; 8 or 16:
                             multi-pivot block partition (segments whose
                             sample has duplicate splitters use the binary pass).  32-byte
                             records always use the binary pass. */
    int32_t records;      /* records only: 0 (default) or 2: key+index path — the passes move
                             16-byte (key, position) pairs (bq_keyidx16) instead of 32-byte
                             records and every record is gathered once at the end (P:867-870:
                             the cost of moving large elements); 1: the passes move the
                             records themselves.  Sorted keys are identical. */
    int32_t subtree;      /* ignored (kept for ABI layout): the on-chip subtree pass it
                             selected was superseded by leaves of S >= 9 Ki elements
                              */
    int32_t reserved[1];  /* must be 0 */
} bq_sort_options;

typedef struct {
    uint32_t levels;               /* breadth-first partition levels executed */
    uint32_t partition_launches;   /* launches of the tile-partition kernel */
    uint32_t kernel_launches;      /* all libbq kernel launches of the call */
    uint32_t reserved0;
    uint64_t element_passes;       /* sum of segment lengths over all partition passes (binary + multiway) */
    uint64_t partitioned_segments; /* segments partitioned (calls of the partitioner) */
    uint64_t leaves;               /* segments finished by the shared-memory leaf sort */
    uint64_t fallback_segments;    /* segments that hit the depth limit (fallback sort) */
    uint64_t band_elements;        /* keys placed by the equal-band fill */
    double partition_ms;           /* sum of binary partition-kernel times (timing != 0) */
    double partition_bytes;        /* algorithmic bytes of those launches: 2*w*(element_passes -
                                      multiway_element_passes) */
    double multiway_ms;            /* sum of multiway level times: count + scan + scatter (timing != 0) */
    uint64_t multiway_element_passes;  /* elements through multiway levels (also in element_passes) */
    double mw_count_ms;            /* timing != 0: the multiway levels' count + scan launches */
    double mw_scatter_ms;          /* timing != 0: the multiway levels' scatter launches */
    double leaf_ms;                /* timing != 0: the leaf-sort launches (a8; on the leaves' own
                                      stream, concurrent with partition levels where the loop
                                      overlaps them) */
} bq_sort_stats;

/* Workspace bytes every call below needs for `n` elements of `kind`:
 * an n*w scratch buffer for the out-of-place partition passes plus O(n/T)
 * bytes of tile status words, segment descriptors and leaf lists (and at
 * least bq_inplace_workspace_bytes(kind, n)).  For
 * BQ_REC32 it also covers the key+index sort path: 16n bytes of pairs, the
 * pair sort's own workspace (16n scratch + O(n/T)) and a 32n-byte copy of the
 * records that the final gather reads (about 65n).  A pure function of
 * (kind, n) — unless the tuning override BQ_LEAF_MAX (environment; a smaller
 * leaf bound than bq_leaf_elems(kind), used by tools/leaf_sweep.py and the
 * tests) is set, which must then hold the same value for this call and the
 * sort that uses the workspace (a sort checks ws_bytes against it). */
BQ_API size_t bq_workspace_bytes(bq_kind kind, size_t n);

/* ---- pivot selection (hot-path step a1) -------------------------------------
 * Computes the pivot value of keys[0, n) with `rule` on the device and
 * returns it in *pivot (host).  Synchronises `stream`.  n >= 1.
 * (For records the "pivot" is a key.) */
BQ_API bq_status bq_pivot_i32(const int32_t *keys, size_t n, bq_pivot_rule rule, int32_t *pivot,
                              void *ws, size_t ws_bytes, void *stream);
BQ_API bq_status bq_pivot_u64(const uint64_t *keys, size_t n, bq_pivot_rule rule, uint64_t *pivot,
                              void *ws, size_t ws_bytes, void *stream);
BQ_API bq_status bq_pivot_f64(const double *keys, size_t n, bq_pivot_rule rule, double *pivot,
                              void *ws, size_t ws_bytes, void *stream);
BQ_API bq_status bq_pivot_records(const bq_record32 *recs, size_t n, bq_pivot_rule rule,
                                  uint64_t *pivot_key, void *ws, size_t ws_bytes, void *stream);

/* ---- partition (hot-path steps a2-a6; Alg. 3) ---------------------
 * Permutes keys[0, n) in place so that
 *     [0, split)                  < pivot
 *     [split, split + n_equal)   == pivot
 *     [split + n_equal, n)        > pivot
 * with split = #{k < pivot}, and preserves the multiset (records move whole).
 * This is the in-place block partition (the same algorithm as
 * bq_partition_inplace): blocks are neutralized from both ends by swapping
 * misplaced keys, so the order inside each band is unspecified (for a
 * deterministic layout use bq_partition_pass with ordered = 1).  Returns split
 * and n_equal to the host (synchronises `stream`).  A NaN f64 pivot is
 * BQ_ERR_INVALID_ARGUMENT. */
BQ_API bq_status bq_partition_i32(int32_t *keys, size_t n, int32_t pivot, size_t *split,
                                  size_t *n_equal, void *ws, size_t ws_bytes, void *stream);
BQ_API bq_status bq_partition_u64(uint64_t *keys, size_t n, uint64_t pivot, size_t *split,
                                  size_t *n_equal, void *ws, size_t ws_bytes, void *stream);
BQ_API bq_status bq_partition_f64(double *keys, size_t n, double pivot, size_t *split,
                                  size_t *n_equal, void *ws, size_t ws_bytes, void *stream);
BQ_API bq_status bq_partition_records(bq_record32 *recs, size_t n, uint64_t pivot_key,
                                      size_t *split, size_t *n_equal, void *ws, size_t ws_bytes,
                                      void *stream);

/* One out-of-place partition pass, fully asynchronous (no host sync): reads
 * src[0, n), writes the three-way partitioned permutation to dst[0, n) and
 * writes {split, n_equal, n_greater} as three uint64 to the DEVICE pointer
 * d_counts.  `pivot` points to a HOST value of the kind's storage type (int32
 * / uint64 / double; a uint64 key for records).  src and dst must not
 * overlap.  ordered != 0 gives the bq_partition_* layout (< keys in input
 * order, > keys reversed, tiles in ticket order, via decoupled look-back);
 * ordered == 0 places each tile's runs with one atomicAdd per tile (runs in
 * input order within a tile, tiles in completion order) — the sort's default.
 * Records (32-byte, and key+index pairs) always use the ordered placement in
 * this standalone pass (three-way, their equal elements staged in consumed
 * input).  This is the timed unit of the
 * partition-pass roofline. */
BQ_API bq_status bq_partition_pass(bq_kind kind, const void *src, void *dst, size_t n,
                                   const void *pivot, uint64_t *d_counts, int ordered, void *ws,
                                   size_t ws_bytes, void *stream);

/* ---- in-place partition (Alg. 3 at CTA granularity) ---------
 * Permutes data[0, n) in place into [< pivot | == pivot | > pivot], split =
 * #{k < pivot}, with no n-element scratch: every CTA runs the paper's block
 * main loop on blocks claimed from both ends — offsets buffers of
 * the misplaced elements, min(num_L, num_R) swaps, a neutralized block
 * written back and the next one claimed — and the few blocks left when the
 * two sides meet are rearranged in a small buffer ("compare and rearrange
 * remaining elements", l.29).  The order inside each band is unspecified.
 * `pivot` points to a HOST value of the kind's storage type (a uint64 key for
 * records); `ws` needs bq_inplace_workspace_bytes(kind, n) bytes (about
 * 1200 tiles, independent of n for large n).  Synchronises `stream`.  A NaN
 * f64 pivot is BQ_ERR_INVALID_ARGUMENT. */
BQ_API size_t bq_inplace_workspace_bytes(bq_kind kind, size_t n);
BQ_API bq_status bq_partition_inplace(bq_kind kind, void *data, size_t n, const void *pivot, size_t *split,
                                      size_t *n_equal, void *ws, size_t ws_bytes, void *stream);

/* Batched pass over `nseg` disjoint segments of src (one breadth-first level
 * of the Quicksort recursion, executed at once): segment i is
 * [begins[i], begins[i] + lens[i]) with pivot pivots[i] (HOST arrays; pivots
 * of the kind's storage type, uint64 keys for records).  Each segment's
 * three-way partition (layout as bq_partition_*) is written to the same range
 * of dst (`ordered` as in bq_partition_pass); {split, n_equal, n_greater} of
 * segment i go to d_counts[3i..3i+2] (DEVICE).  Positions of dst outside every segment are left untouched.
 * Requires lens[i] >= 1, segments inside [0, n) and pairwise disjoint, and
 * nseg <= n / (leaf size + 1) + 2 for the workspace of (kind, n)
 * (BQ_ERR_INVALID_ARGUMENT otherwise).  Synchronises `stream` before
 * returning (the host arrays are read during the call). */
BQ_API bq_status bq_partition_segments(bq_kind kind, const void *src, void *dst, size_t n,
                                       const uint32_t *begins, const uint32_t *lens,
                                       const void *pivots, size_t nseg, uint64_t *d_counts,
                                       int ordered, void *ws, size_t ws_bytes, void *stream);

/* ---- sort (hot-path steps a1-a9) ---------------------------------------------
 * Sorts data[0, n) ascending in place (orders above).  Fully asynchronous:
 * the whole sort is enqueued on `stream` and the call returns without waiting
 * for it (the sorted data is valid once the stream reaches that point; `ws`
 * must stay allocated until then).  The breadth-first level loop that replaces
 * the paper's explicit stack runs on the device: a CUDA graph
 * whose WHILE node repeats a batch of partition levels while the last level
 * produced children, sorting the previous batch's leaves concurrently, then
 * finishes depth-capped segments (a9) under an IF node.  The instantiated
 * graph is cached per (device, kind, data, n, ws, ws_bytes, options); the
 * cache holds at most 32 graphs (least recently used evicted) and is the
 * library's only mutable host state besides the launch-limit cache. */
BQ_API bq_status bq_sort_i32(int32_t *keys, size_t n, void *ws, size_t ws_bytes, void *stream);
BQ_API bq_status bq_sort_u64(uint64_t *keys, size_t n, void *ws, size_t ws_bytes, void *stream);
BQ_API bq_status bq_sort_f64(double *keys, size_t n, void *ws, size_t ws_bytes, void *stream);
BQ_API bq_status bq_sort_records(bq_record32 *recs, size_t n, void *ws, size_t ws_bytes,
                                 void *stream);

/* Kind-generic sort with options (NULL = defaults) and statistics (NULL =
 * none).  Asynchronous like bq_sort_*, except that stats != NULL or
 * opt->timing != 0 makes the call wait for the stream (the statistics are
 * device counters; timing runs the level loop from the host with CUDA events
 * around the partition, multiway and leaf launches).  A leaf-list overflow (never expected: the
 * lists are sized for every child of a level) is reported as BQ_ERR_CUDA only
 * when the call waits. */
BQ_API bq_status bq_sort_ex(bq_kind kind, void *data, size_t n, const bq_sort_options *opt,
                            bq_sort_stats *stats, void *ws, size_t ws_bytes, void *stream);

/* End-to-end sort of a HOST array: copies host_data[0,n) to dev_data (a
 * caller-owned device buffer of n elements), sorts it there, copies the
 * result back into host_data and synchronises `stream`.  host_data should be
 * pinned for full PCIe bandwidth. */
BQ_API bq_status bq_sort_host(bq_kind kind, void *host_data, size_t n, void *dev_data,
                              const bq_sort_options *opt, void *ws, size_t ws_bytes,
                              void *stream);

/* Tuning constants of `kind` (0 for a bad kind): the partition tile T (elements
 * per tile of a pass) and the leaf size S (segments of at most S elements are
 * finished by the shared-memory leaf sort, hot-path step a8). */
BQ_API size_t bq_tile_elems(bq_kind kind);
BQ_API size_t bq_leaf_elems(bq_kind kind);

BQ_API const char *bq_status_string(bq_status s);
BQ_API const char *bq_last_error(void);
/* Library version as 10000*major + 100*minor + patch. */
BQ_API int bq_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BQ_H */
