// api_i32.cu — int32 entry points of libbq.so (see include/bq.h).
#include "api_kind.cuh"

BQ_DETAIL_DEFS(i32, bq::KI32)

extern "C" {

BQ_API bq_status bq_pivot_i32(const int32_t *keys, size_t n, bq_pivot_rule rule, int32_t *pivot, void *ws,
                              size_t ws_bytes, void *stream) {
    uint64_t k = 0;
    bq_status st = bq::run_pivot<bq::KI32>(keys, n, rule, &k, ws, ws_bytes, (cudaStream_t)stream);
    if (st == BQ_OK && pivot) *pivot = bq::KI32::from_key((int32_t)k);
    return st;
}

BQ_API bq_status bq_partition_i32(int32_t *keys, size_t n, int32_t pivot, size_t *split, size_t *n_equal,
                                  void *ws, size_t ws_bytes, void *stream) {
    return bq::run_partition_inplace<bq::KI32>(keys, n, bq::KI32::key(pivot), split, n_equal, ws, ws_bytes,
                                               (cudaStream_t)stream);
}

#ifdef BQ_TRACE
// debug-only (not in bq.h): copy the per-tile phase trace of the int32 kernels
BQ_API int bq_debug_trace(void *host, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host, bq::g_trace, bytes);
}
#endif

BQ_API bq_status bq_sort_i32(int32_t *keys, size_t n, void *ws, size_t ws_bytes, void *stream) {
    return bq::run_sort<bq::KI32>(keys, n, nullptr, nullptr, ws, ws_bytes, (cudaStream_t)stream);
}

}
