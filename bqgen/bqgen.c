/*
 * bqgen — seeded synthetic input generators shared by the oracle tests, the
 * GPU parity tests and bench.py.
 *
 * This module holds NO arithmetic of the sorting method: it only produces
 * inputs shaped like the paper's workloads (§4, "random
 * permutations"/"random ints", Figs. 5-11) and like BASELINE.json's five
 * configs.  Neither oracle/ nor the CUDA path is imported here, and neither of
 * them imports this file; both consume its output arrays.
 *
 * PRNG: SplitMix64 (Steele, Lea & Flood 2014), written from its published
 * definition, used counter-based:
 *     u(seed, i) = mix64(mix64(seed) + (i + 1) * 0x9E3779B97F4A7C15)
 * so element i of every stream can be drawn independently and in any order.
 * Stream identity with the paper's mt19937 is not required.
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>

#define GAMMA 0x9E3779B97F4A7C15ULL

static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* The i-th (0-based) output of the stream `seed`. */
uint64_t bqgen_u64_at(uint64_t seed, uint64_t i) {
    return mix64(mix64(seed) + (i + 1) * GAMMA);
}

/* Sequential cursor over a stream, for algorithms that draw a data-dependent
 * number of values (bounded draws with rejection). */
typedef struct { uint64_t base; uint64_t ctr; } stream_t;
static inline stream_t stream_make(uint64_t seed) { stream_t s = {mix64(seed), 0}; return s; }
static inline uint64_t stream_next(stream_t *s) { s->ctr++; return mix64(s->base + s->ctr * GAMMA); }

/* Unbiased draw from [0, bound), bound >= 1: Lemire's multiply-shift with
 * rejection (2019), on the 64-bit stream. */
static uint64_t bounded(stream_t *s, uint64_t bound) {
    uint64_t x = stream_next(s);
    __uint128_t m = (__uint128_t)x * bound;
    uint64_t l = (uint64_t)m;
    if (l < bound) {
        uint64_t t = (0 - bound) % bound;
        while (l < t) {
            x = stream_next(s);
            m = (__uint128_t)x * bound;
            l = (uint64_t)m;
        }
    }
    return (uint64_t)(m >> 64);
}

void bqgen_u64(uint64_t seed, size_t n, uint64_t *out) {
    uint64_t b = mix64(seed);
    for (size_t i = 0; i < n; i++) out[i] = mix64(b + (uint64_t)(i + 1) * GAMMA);
}

/* Config 2: int32 i.i.d. uniform over the full int32 range (top 32 bits). */
void bqgen_i32_full(uint64_t seed, size_t n, int32_t *out) {
    uint64_t b = mix64(seed);
    for (size_t i = 0; i < n; i++)
        out[i] = (int32_t)(uint32_t)(mix64(b + (uint64_t)(i + 1) * GAMMA) >> 32);
}

/* Config 4a: int32 uniform over {0 .. m-1} (multiply-high of the top 32 bits;
 * for m a power of two this is exactly the top log2(m) bits). */
void bqgen_i32_range(uint64_t seed, size_t n, uint32_t m, int32_t *out) {
    uint64_t b = mix64(seed);
    for (size_t i = 0; i < n; i++) {
        uint64_t hi = mix64(b + (uint64_t)(i + 1) * GAMMA) >> 32;
        out[i] = (int32_t)((hi * (uint64_t)m) >> 32);
    }
}

/* Config 4b: all keys equal. */
void bqgen_i32_const(size_t n, int32_t value, int32_t *out) {
    for (size_t i = 0; i < n; i++) out[i] = value;
}

/* Config 1: uniformly random permutation of 0..n-1 by Fisher-Yates with
 * unbiased bounded draws. */
void bqgen_i32_perm(uint64_t seed, size_t n, int32_t *out) {
    for (size_t i = 0; i < n; i++) out[i] = (int32_t)i;
    stream_t s = stream_make(seed);
    for (size_t i = n; i > 1; i--) {
        size_t j = (size_t)bounded(&s, (uint64_t)i);
        int32_t t = out[i - 1]; out[i - 1] = out[j]; out[j] = t;
    }
}

/* Config 3 "random": doubles i.i.d. uniform in [0,1) as (u >> 11) * 2^-53
 * (no NaN, no -0.0). */
void bqgen_f64_unit(uint64_t seed, size_t n, double *out) {
    uint64_t b = mix64(seed);
    const double scale = 1.0 / 9007199254740992.0; /* 2^-53 */
    for (size_t i = 0; i < n; i++)
        out[i] = (double)(mix64(b + (uint64_t)(i + 1) * GAMMA) >> 11) * scale;
}

/* Config 3 "ascending": a strictly increasing sequence in [0,1) drawn without
 * sorting: element i is uniform within its stratum
 * [floor(i*2^53/n), floor((i+1)*2^53/n)) * 2^-53.  Requires n <= 2^53. */
void bqgen_f64_ascending(uint64_t seed, size_t n, double *out) {
    uint64_t b = mix64(seed);
    const double scale = 1.0 / 9007199254740992.0;
    const __uint128_t full = (__uint128_t)1 << 53;
    for (size_t i = 0; i < n; i++) {
        uint64_t lo = (uint64_t)((full * i) / n);
        uint64_t hi = (uint64_t)((full * (i + 1)) / n);
        uint64_t w = hi - lo; /* >= 1 */
        uint64_t u = mix64(b + (uint64_t)(i + 1) * GAMMA);
        out[i] = (double)(lo + u % w) * scale;
    }
}

/* Config 3 "descending": the ascending sequence reversed. */
void bqgen_f64_descending(uint64_t seed, size_t n, double *out) {
    bqgen_f64_ascending(seed, n, out);
    for (size_t i = 0, j = n ? n - 1 : 0; i < j; i++, j--) {
        double t = out[i]; out[i] = out[j]; out[j] = t;
    }
}

/* Config 3 "1% swapped": the ascending sequence followed by floor(n/200)
 * sequential transpositions of uniformly random index pairs (i, j) drawn from
 * stream seed+1 (SURVEY §8(c) ambiguity 11): ~1% of positions displaced. */
void bqgen_f64_swapped(uint64_t seed, size_t n, double *out) {
    bqgen_f64_ascending(seed, n, out);
    if (n < 2) return;
    stream_t s = stream_make(seed + 1);
    size_t k = n / 200;
    for (size_t t = 0; t < k; t++) {
        size_t i = (size_t)bounded(&s, n), j = (size_t)bounded(&s, n);
        double x = out[i]; out[i] = out[j]; out[j] = x;
    }
}

/* Config 5: 32-byte records {key, payload[3]}: key i.i.d. uniform u64,
 * payload = {i, i, i} (the record's original index). out has 4*n words. */
void bqgen_rec32(uint64_t seed, size_t n, uint64_t *out) {
    uint64_t b = mix64(seed);
    for (size_t i = 0; i < n; i++) {
        out[4 * i + 0] = mix64(b + (uint64_t)(i + 1) * GAMMA);
        out[4 * i + 1] = i;
        out[4 * i + 2] = i;
        out[4 * i + 3] = i;
    }
}

/* Records with forced duplicate keys (tie tests): key drawn from {0..m-1}. */
void bqgen_rec32_dupkeys(uint64_t seed, size_t n, uint64_t m, uint64_t *out) {
    uint64_t b = mix64(seed);
    for (size_t i = 0; i < n; i++) {
        uint64_t u = mix64(b + (uint64_t)(i + 1) * GAMMA);
        out[4 * i + 0] = (uint64_t)(((__uint128_t)u * m) >> 64);
        out[4 * i + 1] = i;
        out[4 * i + 2] = i;
        out[4 * i + 3] = i;
    }
}

/* ---- the paper's structured workloads -------------------
 * int32 patterns of Figs. 7, 9, 10, 11, selected by
 * `which`:
 *   0 IModSqrtN      A[i] = i mod floor(sqrt(n))                 (Fig. 7 left)
 *   1 SquarePattern  A[i] = (i^2 + n/2) mod n                    (Fig. 7 middle, R15)
 *   2 Pow8Pattern    A[i] = (i^8 + n/2) mod n, i^8 by modular squaring (Fig. 7 right)
 *   3 Sorted         A[i] = i                                    (Fig. 9 left)
 *   4 Reversed       A[i] = n-1-i                                (Fig. 9 middle)
 *   5 Rotation       A[i] = (i + n/2) mod n                      (Fig. 9 right)
 *   6,7,8 NeighborSwaps: the sorted array after k swaps of uniformly random
 *                    neighbours (A[j], A[j+1]), k = floor(sqrt n), n, n*floor(log2 n)
 *                    (Fig. 10), j drawn from stream `seed`
 *   9 HalfHalf       A[i] = 0 for i < n/2, else 1                (Fig. 11 middle)
 *  10 RandomZeroOne  A[i] = top bit of u(seed, i)                (Fig. 11 right)
 * Returns 0, or -1 for an unknown pattern. */
static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t m) {
    return (uint64_t)(((__uint128_t)a * b) % m);
}

static uint64_t isqrt_floor(uint64_t n) {
    uint64_t r = 0;
    while ((r + 1) * (r + 1) <= n) r++;
    return r;
}

int bqgen_i32_pattern(int which, uint64_t seed, size_t n, int32_t *out) {
    if (n == 0) return (which >= 0 && which <= 10) ? 0 : -1;
    const uint64_t N = n, half = N / 2;
    switch (which) {
    case 0: {
        uint64_t r = isqrt_floor(N);
        if (r == 0) r = 1;
        for (uint64_t i = 0; i < N; i++) out[i] = (int32_t)(i % r);
        return 0;
    }
    case 1:
        for (uint64_t i = 0; i < N; i++) out[i] = (int32_t)((mulmod(i, i, N) + half) % N);
        return 0;
    case 2:
        for (uint64_t i = 0; i < N; i++) {
            uint64_t x = i % N;
            x = mulmod(x, x, N);   /* i^2 */
            x = mulmod(x, x, N);   /* i^4 */
            x = mulmod(x, x, N);   /* i^8 */
            out[i] = (int32_t)((x + half) % N);
        }
        return 0;
    case 3:
        for (uint64_t i = 0; i < N; i++) out[i] = (int32_t)i;
        return 0;
    case 4:
        for (uint64_t i = 0; i < N; i++) out[i] = (int32_t)(N - 1 - i);
        return 0;
    case 5:
        for (uint64_t i = 0; i < N; i++) out[i] = (int32_t)((i + half) % N);
        return 0;
    case 6: case 7: case 8: {
        for (uint64_t i = 0; i < N; i++) out[i] = (int32_t)i;
        uint64_t lg = 0;
        while ((2ull << lg) <= N) lg++;
        const uint64_t k = which == 6 ? isqrt_floor(N) : which == 7 ? N : N * lg;
        if (N < 2) return 0;
        stream_t s = stream_make(seed);
        for (uint64_t t = 0; t < k; t++) {
            const uint64_t j = bounded(&s, N - 1);
            int32_t x = out[j]; out[j] = out[j + 1]; out[j + 1] = x;
        }
        return 0;
    }
    case 9:
        for (uint64_t i = 0; i < N; i++) out[i] = i < half ? 0 : 1;
        return 0;
    case 10: {
        uint64_t b = mix64(seed);
        for (uint64_t i = 0; i < N; i++) out[i] = (int32_t)(mix64(b + (i + 1) * GAMMA) >> 63);
        return 0;
    }
    }
    return -1;
}
