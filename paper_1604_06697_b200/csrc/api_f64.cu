// api_f64.cu — float64 entry points of libbq.so (see include/bq.h).  Keys are
// compared through the order-preserving H0 codec (common.cuh KF64).
#include "api_kind.cuh"

BQ_DETAIL_DEFS(f64, bq::KF64)

namespace {
inline uint64_t bits_of(double d) { uint64_t b; std::memcpy(&b, &d, 8); return b; }
inline double double_of(uint64_t b) { double d; std::memcpy(&d, &b, 8); return d; }
}

extern "C" {

BQ_API bq_status bq_pivot_f64(const double *keys, size_t n, bq_pivot_rule rule, double *pivot, void *ws,
                              size_t ws_bytes, void *stream) {
    uint64_t k = 0;
    bq_status st = bq::run_pivot<bq::KF64>(reinterpret_cast<const uint64_t *>(keys), n, rule, &k, ws, ws_bytes,
                                           (cudaStream_t)stream);
    if (st == BQ_OK && pivot) *pivot = double_of(bq::KF64::from_key(k));
    return st;
}

BQ_API bq_status bq_partition_f64(double *keys, size_t n, double pivot, size_t *split, size_t *n_equal,
                                  void *ws, size_t ws_bytes, void *stream) {
    if (std::isnan(pivot)) return bq::set_error(BQ_ERR_INVALID_ARGUMENT, "NaN pivot");
    return bq::run_partition_inplace<bq::KF64>(reinterpret_cast<uint64_t *>(keys), n,
                                               bq::KF64::key(bits_of(pivot)), split, n_equal, ws, ws_bytes,
                                               (cudaStream_t)stream);
}

BQ_API bq_status bq_sort_f64(double *keys, size_t n, void *ws, size_t ws_bytes, void *stream) {
    return bq::run_sort<bq::KF64>(reinterpret_cast<uint64_t *>(keys), n, nullptr, nullptr, ws, ws_bytes,
                                  (cudaStream_t)stream);
}

}
