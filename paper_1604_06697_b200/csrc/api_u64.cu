// api_u64.cu — uint64 entry points of libbq.so (see include/bq.h).
#include "api_kind.cuh"

BQ_DETAIL_DEFS(u64, bq::KU64)

extern "C" {

BQ_API bq_status bq_pivot_u64(const uint64_t *keys, size_t n, bq_pivot_rule rule, uint64_t *pivot, void *ws,
                              size_t ws_bytes, void *stream) {
    uint64_t k = 0;
    bq_status st = bq::run_pivot<bq::KU64>(keys, n, rule, &k, ws, ws_bytes, (cudaStream_t)stream);
    if (st == BQ_OK && pivot) *pivot = bq::KU64::from_key(k);
    return st;
}

BQ_API bq_status bq_partition_u64(uint64_t *keys, size_t n, uint64_t pivot, size_t *split, size_t *n_equal,
                                  void *ws, size_t ws_bytes, void *stream) {
    return bq::run_partition_inplace<bq::KU64>(keys, n, bq::KU64::key(pivot), split, n_equal, ws, ws_bytes,
                                               (cudaStream_t)stream);
}

BQ_API bq_status bq_sort_u64(uint64_t *keys, size_t n, void *ws, size_t ws_bytes, void *stream) {
    return bq::run_sort<bq::KU64>(keys, n, nullptr, nullptr, ws, ws_bytes, (cudaStream_t)stream);
}

}
