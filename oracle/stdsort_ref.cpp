/*
 * std::sort reference — TEST / BENCH INFRASTRUCTURE ONLY.
 *
 * libstdc++'s std::sort (introsort) with the natural orders the C-ABI
 * defines.  Two uses:
 *   1. an independent library routine that pins the oracle in tests (the
 *      sorted sequence of keys is unique, so any correct sort must agree);
 *   2. the "std::sort timed on the GPU box's host cores" context number the
 *      north_star asks bench.py to report next to the oracle (P:755-780 name
 *      GCC std::sort as the paper's main comparison system).
 * It shares nothing with the oracle or the CUDA path.
 */
#include <algorithm>
#include <cmath>
#include <cstdint>

namespace {
struct Rec32 { uint64_t key; uint64_t payload[3]; };
}

extern "C" {

void bq_std_sort_i32(int32_t *a, long long n) { std::sort(a, a + n); }
void bq_std_sort_u64(uint64_t *a, long long n) { std::sort(a, a + n); }

/* totalOrder on non-NaN doubles: numeric order, -0.0 before +0.0. */
void bq_std_sort_f64(double *a, long long n) {
    std::sort(a, a + n, [](double x, double y) {
        if (x != y) return x < y;
        return std::signbit(x) && !std::signbit(y);
    });
}

/* Records by key, equal keys in unspecified order (std::sort is unstable). */
void bq_std_sort_rec32(Rec32 *a, long long n) {
    std::sort(a, a + n, [](const Rec32 &x, const Rec32 &y) { return x.key < y.key; });
}

}
