// api_rec.cu — 32-byte record entry points of libbq.so (see include/bq.h).
// Records compare by key only.
#include "api_kind.cuh"

namespace bq {
namespace detail {
size_t ws_rec(size_t n) { return make_layout<KRec>(n).total; }
size_t ipws_rec(size_t n) { return make_ip_layout<KRec>(n).total; }
bq_status inplace_rec(void *data, size_t n, const void *pivot, size_t *split, size_t *neq, void *ws, size_t wsb,
                      cudaStream_t s) {
    return run_partition_inplace_ip<KRec>(static_cast<Rec32 *>(data), n, pivot_key_from<KRec>(pivot), split, neq,
                                          ws, wsb, s);
}
bq_status sort_rec(void *data, size_t n, const bq_sort_options *opt, bq_sort_stats *st, void *ws, size_t wsb,
                   cudaStream_t s) {
    return run_sort<KRec>(static_cast<Rec32 *>(data), n, opt, st, ws, wsb, s);
}
bq_status pass_rec(const void *src, void *dst, size_t n, const void *pivot, uint64_t *dc, void *ws, size_t wsb,
                   cudaStream_t s, int ordered) {
    uint64_t pk;
    std::memcpy(&pk, pivot, sizeof pk);
    return run_partition_pass<KRec>(static_cast<const Rec32 *>(src), static_cast<Rec32 *>(dst), n, pk, dc, ws,
                                    wsb, s, ordered);
}
bq_status segs_rec(const void *src, void *dst, size_t n, const uint32_t *begins, const uint32_t *lens,
                   const void *pivots, size_t nseg, uint64_t *dc, void *ws, size_t wsb, cudaStream_t s, int ordered) {
    return run_partition_segments<KRec>(static_cast<const Rec32 *>(src), static_cast<Rec32 *>(dst), n, begins, lens,
                                        static_cast<const uint64_t *>(pivots), nseg, dc, ws, wsb, s, ordered);
}
}  // namespace detail
}  // namespace bq

extern "C" {

BQ_API bq_status bq_pivot_records(const bq_record32 *recs, size_t n, bq_pivot_rule rule, uint64_t *pivot_key,
                                  void *ws, size_t ws_bytes, void *stream) {
    return bq::run_pivot<bq::KRec>(reinterpret_cast<const bq::Rec32 *>(recs), n, rule, pivot_key, ws, ws_bytes,
                                   (cudaStream_t)stream);
}

BQ_API bq_status bq_partition_records(bq_record32 *recs, size_t n, uint64_t pivot_key, size_t *split,
                                      size_t *n_equal, void *ws, size_t ws_bytes, void *stream) {
    return bq::run_partition_inplace<bq::KRec>(reinterpret_cast<bq::Rec32 *>(recs), n, pivot_key, split, n_equal,
                                               ws, ws_bytes, (cudaStream_t)stream);
}

BQ_API bq_status bq_sort_records(bq_record32 *recs, size_t n, void *ws, size_t ws_bytes, void *stream) {
    return bq::run_sort<bq::KRec>(reinterpret_cast<bq::Rec32 *>(recs), n, nullptr, nullptr, ws, ws_bytes,
                                  (cudaStream_t)stream);
}

}
