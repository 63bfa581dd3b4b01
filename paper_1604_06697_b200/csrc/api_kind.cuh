// api_kind.cuh — per-kind entry points; included once per kind by
// api_i32.cu / api_u64.cu / api_f64.cu / api_rec.cu so the kernel families
// compile in parallel translation units.
#pragma once

#include <cmath>

#include "driver.cuh"

#define BQ_DETAIL_DECLS(SUF)                                                                        \
    namespace bq {                                                                                  \
    namespace detail {                                                                              \
    size_t ws_##SUF(size_t n);                                                                      \
    bq_status sort_##SUF(void *data, size_t n, const bq_sort_options *opt, bq_sort_stats *st,       \
                         void *ws, size_t wsb, cudaStream_t s);                                     \
    bq_status pass_##SUF(const void *src, void *dst, size_t n, const void *pivot, uint64_t *dc,     \
                         void *ws, size_t wsb, cudaStream_t s, int ordered);                        \
    bq_status segs_##SUF(const void *src, void *dst, size_t n, const uint32_t *begins,              \
                         const uint32_t *lens, const void *pivots, size_t nseg, uint64_t *dc,       \
                         void *ws, size_t wsb, cudaStream_t s, int ordered);                        \
    }                                                                                               \
    }

BQ_DETAIL_DECLS(i32)
BQ_DETAIL_DECLS(u64)
BQ_DETAIL_DECLS(f64)
BQ_DETAIL_DECLS(rec)

#define BQ_DETAIL_DEFS(SUF, KT)                                                                     \
    namespace bq {                                                                                  \
    namespace detail {                                                                              \
    size_t ws_##SUF(size_t n) { return make_layout<KT>(n).total; }                                  \
    bq_status sort_##SUF(void *data, size_t n, const bq_sort_options *opt, bq_sort_stats *st,       \
                         void *ws, size_t wsb, cudaStream_t s) {                                    \
        return run_sort<KT>(static_cast<KT::T *>(data), n, opt, st, ws, wsb, s);                    \
    }                                                                                               \
    bq_status pass_##SUF(const void *src, void *dst, size_t n, const void *pivot, uint64_t *dc,     \
                         void *ws, size_t wsb, cudaStream_t s, int ordered) {                       \
        KT::T pv;                                                                                   \
        std::memcpy(&pv, pivot, sizeof pv);                                                         \
        return run_partition_pass<KT>(static_cast<const KT::T *>(src), static_cast<KT::T *>(dst),  \
                                      n, KT::key(pv), dc, ws, wsb, s, ordered);                     \
    }                                                                                               \
    bq_status segs_##SUF(const void *src, void *dst, size_t n, const uint32_t *begins,              \
                         const uint32_t *lens, const void *pivots, size_t nseg, uint64_t *dc,       \
                         void *ws, size_t wsb, cudaStream_t s, int ordered) {                       \
        std::vector<KT::K> keys(nseg);                                                             \
        for (size_t i = 0; i < nseg; i++) {                                                         \
            KT::T pv;                                                                               \
            std::memcpy(&pv, static_cast<const char *>(pivots) + i * sizeof(KT::T), sizeof pv);    \
            keys[i] = KT::key(pv);                                                                  \
        }                                                                                           \
        return run_partition_segments<KT>(static_cast<const KT::T *>(src), static_cast<KT::T *>(dst), \
                                          n, begins, lens, keys.data(), nseg, dc, ws, wsb, s, ordered); \
    }                                                                                               \
    }                                                                                               \
    }
