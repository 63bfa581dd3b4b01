// api_kind.cuh — per-kind entry points; included once per kind by
// api_i32.cu / api_u64.cu / api_f64.cu / api_rec.cu so the kernel families
// compile in parallel translation units.
#pragma once

#include <cmath>

#include "driver.cuh"

namespace bq {
namespace detail {
// a host pivot of the kind's storage type (a uint64 key for records)
template <class KT>
inline typename KT::K pivot_key_from(const void *p) {
    if constexpr (KT::is_record) {
        typename KT::K k;
        std::memcpy(&k, p, sizeof k);
        return k;
    } else {
        typename KT::T v;
        std::memcpy(&v, p, sizeof v);
        return KT::key(v);
    }
}
}  // namespace detail
}  // namespace bq

#define BQ_DETAIL_DECLS(SUF)                                                                        \
    namespace bq {                                                                                  \
    namespace detail {                                                                              \
    size_t ws_##SUF(size_t n);                                                                      \
    size_t ipws_##SUF(size_t n);                                                                    \
    bq_status inplace_##SUF(void *data, size_t n, const void *pivot, size_t *split, size_t *neq,     \
                            void *ws, size_t wsb, cudaStream_t s);                                  \
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
BQ_DETAIL_DECLS(pair)

#define BQ_DETAIL_DEFS(SUF, KT)                                                                     \
    namespace bq {                                                                                  \
    namespace detail {                                                                              \
    size_t ws_##SUF(size_t n) {                                                                     \
        const size_t a = make_layout<KT>(n).total, b = make_ip_layout<KT>(n).total;                 \
        return a > b ? a : b;                                                                       \
    }                                                                                               \
    size_t ipws_##SUF(size_t n) { return make_ip_layout<KT>(n).total; }                             \
    bq_status inplace_##SUF(void *data, size_t n, const void *pivot, size_t *split, size_t *neq,     \
                            void *ws, size_t wsb, cudaStream_t s) {                                 \
        return run_partition_inplace_ip<KT>(static_cast<KT::T *>(data), n, pivot_key_from<KT>(pivot), \
                                            split, neq, ws, wsb, s);                                \
    }                                                                                               \
    bq_status sort_##SUF(void *data, size_t n, const bq_sort_options *opt, bq_sort_stats *st,       \
                         void *ws, size_t wsb, cudaStream_t s) {                                    \
        return run_sort<KT>(static_cast<KT::T *>(data), n, opt, st, ws, wsb, s);                    \
    }                                                                                               \
    bq_status pass_##SUF(const void *src, void *dst, size_t n, const void *pivot, uint64_t *dc,     \
                         void *ws, size_t wsb, cudaStream_t s, int ordered) {                       \
        return run_partition_pass<KT>(static_cast<const KT::T *>(src), static_cast<KT::T *>(dst),  \
                                      n, pivot_key_from<KT>(pivot), dc, ws, wsb, s, ordered);       \
    }                                                                                               \
    bq_status segs_##SUF(const void *src, void *dst, size_t n, const uint32_t *begins,              \
                         const uint32_t *lens, const void *pivots, size_t nseg, uint64_t *dc,       \
                         void *ws, size_t wsb, cudaStream_t s, int ordered) {                       \
        std::vector<KT::K> keys(nseg);                                                             \
        constexpr size_t PW = KT::is_record ? sizeof(KT::K) : sizeof(KT::T);                        \
        for (size_t i = 0; i < nseg; i++)                                                           \
            keys[i] = pivot_key_from<KT>(static_cast<const char *>(pivots) + i * PW);               \
        return run_partition_segments<KT>(static_cast<const KT::T *>(src), static_cast<KT::T *>(dst), \
                                          n, begins, lens, keys.data(), nseg, dc, ws, wsb, s, ordered); \
    }                                                                                               \
    }                                                                                               \
    }
