/*
 * bq_oracle — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU BlockQuicksort written from the paper
 * (Edelkamp & Weiß, "BlockQuicksort: How Branch Mispredictions don't affect
 * Quicksort", arXiv 1604.06697; PAPER.md).  It is the parity reference for the
 * CUDA path in paper_1604_06697_b200/ and shares no code with it (no headers,
 * no helpers, no constants).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library; the
 * product path never does.
 *
 * Citations: P:n = PAPER.md line n (the Appendix B listing line k is P:1059+k).
 *
 * What is implemented (the paper's *basic* variant, block_partition_simple,
 * P:615-618, Appendix B):
 *   - sort_pair / median_of_3: branch-free compare-exchange.
 *   - hoare_block_partition_simple = Alg. 3 with
 *     the block-style final iteration and the Lomuto-like move of the
 *     remaining buffered elements, pivot parked at the end and fetched.
 *   - the explicit-stack Quicksort main loop with the Introsort depth limit
 *     2*ilogb(n)+3 and Heapsort fallback, Insertionsort for arrays of <= 16
 *     elements during the recursion, larger side pushed (P:286-330,
 *     P:1221-1268).
 *   - the value-pivot partition the C-ABI's bq_partition defines
 *     (SURVEY §8(c) "O-partition"): Alg. 3 run with a pivot *value* on the
 *     whole array, then the duplicate check of §3.2 applied to
 *     both sides without its "every fourth" stop rule, so the result is
 *     [ < p | == p | > p ] with split = #{<p}.
 *
 * Readings of the paper:
 *   R1  Alg. 3 lines 9/16 print the scan predicates swapped;
 *       the prose and the code count A >= p on
 *       the left and A <= p on the right.  The code's predicates are used.
 *   R2  P:1215 passes `end` to median_of_3 (one past the end); the third
 *       sample is end-1, the only in-bounds reading consistent with
 *       partitioning [begin+1, end-1).
 *   R3  BLOCKSIZE = 128, IS_THRESH = 16 (insertion sort
 *       iff e-b <= 16).  Both are test-tunable here.
 *   R4  depth limit = 2*floor(log2 n)+3 from the top-level n (P:295, P:1224
 *       `ilogb`).
 *   R5  std::partial_sort(begin,end,end) = a textbook heapsort.
 *   R9  float64 order: IEEE 754 totalOrder restricted to non-NaN values
 *       (-0.0 < +0.0), written below from its definition.  NaN inputs are
 *       outside the contract.
 *   R10 records compare by key only ("Only the first component is
 *       compared").
 */
#include <cmath>
#include <cstdint>
#include <cstring>
#include <utility>

namespace {

struct Rec32 {
    uint64_t key;
    uint64_t payload[3];
};

/* ---- comparators ("less") --------------------------------- */
struct LessI32 { bool operator()(int32_t a, int32_t b) const { return a < b; } };
struct LessU64 { bool operator()(uint64_t a, uint64_t b) const { return a < b; } };
/* IEEE 754-2008 §5.10 totalOrder for non-NaN operands: x < y numerically, or
 * x == y and x is -0 while y is +0. */
struct LessF64 {
    bool operator()(double a, double b) const {
        if (a < b) return true;
        if (a > b) return false;
        return std::signbit(a) && !std::signbit(b);
    }
};
struct LessRec { bool operator()(const Rec32 &a, const Rec32 &b) const { return a.key < b.key; } };

/* A comparator wrapper that counts calls (SPEC instrumentation). */
template <class T, class L>
struct Counting {
    L less;
    uint64_t *count;
    bool operator()(const T &a, const T &b) const { ++*count; return less(a, b); }
};

struct Stats {
    uint64_t comparisons;
    uint64_t partitions;
    uint64_t heapsort_calls;
    uint64_t insertion_calls;
    uint64_t max_stack;       /* high-water mark of pending frames */
};

template <class T>
inline void swap_elems(T *a, T *b) { T t = *a; *a = *b; *b = t; }

/* sort_pair: after the call *i1 <= *i2; the exchange is done
 * with selects on the comparison result, no data-dependent jump. */
template <class T, class C>
inline void sort_pair(T *i1, T *i2, C &less) {
    bool smaller = less(*i2, *i1);
    T temp = smaller ? *i1 : *i2;
    *i1 = smaller ? *i2 : *i1;
    *i2 = smaller ? temp : *i2;
}

/* median_of_3: sorts the three positions, returns the middle. */
template <class T, class C>
inline T *median_of_3(T *i1, T *i2, T *i3, C &less) {
    sort_pair(i1, i2, less);
    sort_pair(i2, i3, less);
    sort_pair(i1, i2, less);
    return i2;
}

/*
 * Alg. 3 main loop + final iteration + remaining-buffer moves, on the working
 * range [begin, last] (inclusive), with the pivot *value* `pivot`.
 * Returns the cut: [orig_begin, cut) <= pivot, [cut, orig_last] >= pivot.
 * This is hoare_block_partition_simple with the pivot parking
 * and fetching factored out so that the
 * same routine serves the element-pivot form (paper) and the value-pivot form
 * (C-ABI).  Offsets buffers: P:362-368.
 */
template <class T, class C>
long long block_partition_range(T *begin, T *last, const T &pivot, long long B, C &less) {
    long long *indexL = new long long[B];
    long long *indexR = new long long[B];
    long long num_left = 0, num_right = 0, start_left = 0, start_right = 0, num;
    T *const orig_begin = begin;

    /* main loop (Alg. 3 lines 4-27) */
    while (last - begin + 1 > 2 * B) {
        if (num_left == 0) {              /* refill left buffer (Alg. 3 l.5-11) */
            start_left = 0;
            for (long long j = 0; j < B; j++) {
                indexL[num_left] = j;                       /* store always   */
                num_left += (!(less(begin[j], pivot)));     /* advance by cmp */
            }
        }
        if (num_right == 0) {             /* refill right buffer (l.12-18) */
            start_right = 0;
            for (long long j = 0; j < B; j++) {
                indexR[num_right] = j;
                num_right += !(less(pivot, *(last - j)));
            }
        }
        /* rearrangement phase (l.19-22) */
        num = num_left < num_right ? num_left : num_right;
        for (long long j = 0; j < num; j++)
            swap_elems(begin + indexL[start_left + j], last - indexR[start_right + j]);
        num_left -= num;
        num_right -= num;
        start_left += num;
        start_right += num;
        begin += (num_left == 0) ? B : 0;   /* l.24 */
        last -= (num_right == 0) ? B : 0;   /* l.25 */
    }

    /* final iteration: scan the < 2B remaining elements as one or two
     * smaller blocks */
    long long shiftR = 0, shiftL = 0;
    if (num_right == 0 && num_left == 0) {
        shiftL = ((last - begin) + 1) / 2;
        shiftR = (last - begin) + 1 - shiftL;
        start_left = 0; start_right = 0;
        for (long long j = 0; j < shiftL; j++) {
            indexL[num_left] = j;
            num_left += (!less(begin[j], pivot));
            indexR[num_right] = j;
            num_right += !less(pivot, *(last - j));
        }
        if (shiftL < shiftR) {
            indexR[num_right] = shiftR - 1;
            num_right += !less(pivot, *(last - shiftR + 1));
        }
    } else if (num_right != 0) {
        shiftL = (last - begin) - B + 1;
        shiftR = B;
        start_left = 0;
        for (long long j = 0; j < shiftL; j++) {
            indexL[num_left] = j;
            num_left += (!less(begin[j], pivot));
        }
    } else {
        shiftL = B;
        shiftR = (last - begin) - B + 1;
        start_right = 0;
        for (long long j = 0; j < shiftR; j++) {
            indexR[num_right] = j;
            num_right += !(less(pivot, *(last - j)));
        }
    }
    num = num_left < num_right ? num_left : num_right;
    for (long long j = 0; j < num; j++)
        swap_elems(begin + indexL[start_left + j], last - indexR[start_right + j]);
    num_left -= num;
    num_right -= num;
    start_left += num;
    start_right += num;
    begin += (num_left == 0) ? shiftL : 0;
    last -= (num_right == 0) ? shiftR : 0;

    /* move the elements remaining in one buffer to the inner end of their
     * side, Lomuto-style without comparisons */
    long long cut;
    if (num_left != 0) {
        long long lowerI = start_left + num_left - 1;
        long long upper = last - begin;
        while (lowerI >= start_left && indexL[lowerI] == upper) { upper--; lowerI--; }
        while (lowerI >= start_left) swap_elems(begin + upper--, begin + indexL[lowerI--]);
        cut = (begin + upper + 1) - orig_begin;
    } else if (num_right != 0) {
        long long lowerI = start_right + num_right - 1;
        long long upper = last - begin;
        while (lowerI >= start_right && indexR[lowerI] == upper) { upper--; lowerI--; }
        while (lowerI >= start_right) swap_elems(last - upper--, last - indexR[lowerI--]);
        cut = (last - upper) - orig_begin;
    } else {
        cut = begin - orig_begin;
    }
    delete[] indexL;
    delete[] indexR;
    return cut;
}

/* hoare_block_partition_simple(begin, end, pivot_position):
 * park the pivot in the last slot, partition [begin, end-2],
 * fetch the pivot into the cut (P:1188/1202/1206).  Returns the pivot's final
 * index relative to begin. */
template <class T, class C>
long long hoare_block_partition_simple(T *begin, T *end, T *pivot_position, long long B, C &less) {
    T *last = end - 1;
    swap_elems(pivot_position, last);
    const T pivot = *last;               /* the pivot value lives in *last */
    pivot_position = last;
    last--;
    long long cut = block_partition_range(begin, last, pivot, B, less);
    swap_elems(pivot_position, begin + cut);   /* fetch the pivot */
    return cut;
}

/* Hoare_block_partition_simple::partition: median-of-3 of
 * (begin, middle, end-1) [reading R2], then block-partition [begin+1, end-1)
 * around it.  Returns the pivot position relative to begin. */
template <class T, class C>
long long partition_mo3(T *begin, T *end, long long B, C &less) {
    T *mid = median_of_3(begin, begin + (end - begin) / 2, end - 1, less);
    return 1 + hoare_block_partition_simple(begin + 1, end - 1, mid, B, less);
}

/* Insertionsort (R3): textbook straight insertion. */
template <class T, class C>
void insertion_sort(T *begin, T *end, C &less) {
    for (T *i = begin + 1; i < end; ++i) {
        T v = *i;
        T *j = i;
        while (j > begin && less(v, *(j - 1))) { *j = *(j - 1); --j; }
        *j = v;
    }
}

/* Heapsort (Williams 1964 / Floyd 1964, R5): textbook max-heap. */
template <class T, class C>
void sift_down(T *a, long long root, long long n, C &less) {
    for (;;) {
        long long child = 2 * root + 1;
        if (child >= n) return;
        if (child + 1 < n && less(a[child], a[child + 1])) child++;
        if (!less(a[root], a[child])) return;
        swap_elems(a + root, a + child);
        root = child;
    }
}
template <class T, class C>
void heap_sort(T *begin, T *end, C &less) {
    long long n = end - begin;
    for (long long i = n / 2 - 1; i >= 0; --i) sift_down(begin, i, n, less);
    for (long long k = n - 1; k > 0; --k) {
        swap_elems(begin, begin + k);
        sift_down(begin, 0, k, less);
    }
}

/* floor(log2 n) for n >= 1 (`ilogb((double)n)`). */
inline int ilog2(long long n) { int r = -1; while (n) { n >>= 1; r++; } return r; }

/* Quicksort main loop: explicit stack, push the larger side,
 * continue on the smaller one; Introsort depth limit; Insertionsort for
 * sub-arrays of <= cutoff elements during the recursion. */
template <class T, class C>
void qsort_block(T *first, T *last_excl, long long B, long long cutoff, int depth_limit_override,
                 C &less, Stats *st) {
    long long n = last_excl - first;
    if (n <= 1) return;
    const int depth_limit = depth_limit_override >= 0 ? depth_limit_override : 2 * ilog2(n) + 3;
    /* stack sizes: the listing uses stack[80]/depth_stack[40] for 64-bit n;
     * frames <= log2(n)+2 because the smaller side is processed first. */
    T *stack[200];
    int depth_stack[100];
    T **s = stack;
    int *d_s_top = depth_stack;
    T *begin = first, *end = last_excl;
    int depth = 0;
    *s = begin; *(s + 1) = end; s += 2;
    *d_s_top = 0; ++d_s_top;
    do {
        if (depth < depth_limit && end - begin > cutoff) {
            long long p = partition_mo3(begin, end, B, less);
            st->partitions++;
            T *pivot = begin + p;
            if (pivot - begin > end - pivot) {    /* push the large side */
                *s = begin; *(s + 1) = pivot;
                begin = pivot + 1;
            } else {
                *s = pivot + 1; *(s + 1) = end;
                end = pivot;
            }
            s += 2;
            depth++;
            *d_s_top = depth;
            ++d_s_top;
            uint64_t frames = (uint64_t)((s - stack) / 2 - 1);
            if (frames > st->max_stack) st->max_stack = frames;
        } else {
            if (end - begin > cutoff) {           /* depth limit exceeded */
                heap_sort(begin, end, less);
                st->heapsort_calls++;
            } else {
                insertion_sort(begin, end, less);
                st->insertion_calls++;
            }
            s -= 2;                              /* pop */
            begin = *s; end = *(s + 1);
            --d_s_top;
            depth = *d_s_top;
        }
    } while (s != stack);
}

/* Value-pivot partition + two-sided equal gather (SURVEY §8(c) O-partition).
 * Step 1: Alg. 3 on [0, n-1] with the pivot value (no parking, no fetch):
 *         [0,s2) <= p, [s2,n) >= p.
 * Step 2: the duplicate check of §3.2 on both sides, without the
 *         "every fourth" stop: keys of [0,s2) that are not < p move to its
 *         right end; keys of [s2,n) that are not > p move to its left end.
 * Result: [ <p | ==p | >p ], split = #{<p}, n_equal = #{==p}. */
template <class T, class C>
void partition_value(T *A, long long n, const T &pivot, long long B, C &less,
                     long long *split, long long *n_equal) {
    long long s2 = (n > 0) ? block_partition_range(A, A + n - 1, pivot, B, less) : 0;
    /* left side: scan down from s2-1, gather the equal keys at its right end */
    long long eqL = s2;                   /* [eqL, s2) holds keys == p */
    for (long long i = s2 - 1; i >= 0; --i) {
        if (!less(A[i], pivot)) {         /* A[i] <= p known, so == p */
            --eqL;
            swap_elems(A + i, A + eqL);
        }
    }
    /* right side: scan up from s2, gather the equal keys at its left end */
    long long eqR = s2;                   /* [s2, eqR) holds keys == p */
    for (long long i = s2; i < n; ++i) {
        if (!less(pivot, A[i])) {         /* A[i] >= p known, so == p */
            swap_elems(A + i, A + eqR);
            ++eqR;
        }
    }
    *split = eqL;
    *n_equal = eqR - eqL;
}

/* SplitMix64's output function (Steele, Lea & Flood 2014), from its
 * published definition: the counter-based generator of R19. */
static inline uint64_t splitmix64_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* Pivot sample rules, used to pin the GPU pivot kernel (SURVEY §8(a) a1 and
 * §8(f) N1).
 * Mo3 over positions {0, floor(n/2), n-1} (P:313-317, P:1215 + R2);
 * pseudomedian of 9 ("median of three medians of three") over
 * positions floor(k*(n-1)/8), k=0..8, grouped as consecutive triples
 * (SURVEY §8(c) ambiguity 13).  Values are copied; the array is untouched. */
template <class T, class C>
T pivot_value(const T *A, long long n, int rule, C &less) {
    if (rule == 2) {
        /* median of a 64-key sample (R18/R19: the paper's "median of
         * a larger sample" idea, with the sample size
         * fixed at 64, and its suggestion to pick the sample with a fast
         * pseudo-random generator): key j is drawn from the j-th
         * of 64 equal strata of [0, n), at an offset given by SplitMix64 of
         * (segment begin = 0, n, j); the 64 keys are sorted by insertion sort
         * and the lower median (index 31) is the pivot. */
        T smp[64];
        const uint64_t un = (uint64_t)n;
        for (int j = 0; j < 64; j++) {
            const uint64_t s0 = ((uint64_t)j * un) >> 6, s1 = ((uint64_t)(j + 1) * un) >> 6;
            const uint64_t r = splitmix64_mix(un + (uint64_t)(j + 1) * 0x9E3779B97F4A7C15ull) >> 32;
            uint64_t pos = s0 + ((r * (s1 - s0)) >> 32);
            if (pos > un - 1) pos = un - 1;
            smp[j] = A[pos];
        }
        for (int j = 1; j < 64; j++)
            for (int k = j; k > 0 && less(smp[k], smp[k - 1]); k--) swap_elems(&smp[k], &smp[k - 1]);
        return smp[31];
    }
    if (rule == 0 || n < 9) {
        T a = A[0], b = A[n / 2], c = A[n - 1];
        return *median_of_3(&a, &b, &c, less);
    }
    T m[3];
    for (int g = 0; g < 3; g++) {
        T x[3];
        for (int k = 0; k < 3; k++) x[k] = A[((long long)(3 * g + k) * (n - 1)) / 8];
        m[g] = *median_of_3(&x[0], &x[1], &x[2], less);
    }
    return *median_of_3(&m[0], &m[1], &m[2], less);
}

} // namespace

extern "C" {

typedef struct {
    long long block;            /* B; paper: 128 */
    long long cutoff;           /* Insertionsort iff len <= cutoff; paper: 16 */
    int depth_limit;            /* < 0: paper rule 2*floor(log2 n)+3 */
} bq_oracle_opts;

typedef Stats bq_oracle_stats;

static const bq_oracle_opts kPaperOpts = {128, 16, -1};

#define BQ_ORACLE_DEFINE(SUF, T, LESS)                                                        \
    void bq_oracle_sort_##SUF(T *A, long long n, const bq_oracle_opts *o, bq_oracle_stats *st) { \
        const bq_oracle_opts *op = o ? o : &kPaperOpts;                                      \
        bq_oracle_stats local;                                                               \
        std::memset(&local, 0, sizeof local);                                                \
        Counting<T, LESS> less{LESS{}, &local.comparisons};                                  \
        qsort_block(A, A + n, op->block, op->cutoff, op->depth_limit, less, &local);         \
        if (st) *st = local;                                                                 \
    }                                                                                        \
    long long bq_oracle_block_partition_##SUF(T *A, long long n, long long pivot_index,      \
                                              long long B, unsigned long long *cmp) {        \
        uint64_t c = 0;                                                                      \
        Counting<T, LESS> less{LESS{}, &c};                                                  \
        long long cut = hoare_block_partition_simple(A, A + n, A + pivot_index, B, less);    \
        if (cmp) *cmp = c;                                                                   \
        return cut;                                                                          \
    }                                                                                        \
    void bq_oracle_partition_##SUF(T *A, long long n, T pivot, long long B,                  \
                                   long long *split, long long *n_equal) {                   \
        LESS less;                                                                           \
        partition_value(A, n, pivot, B, less, split, n_equal);                               \
    }                                                                                        \
    T bq_oracle_pivot_##SUF(const T *A, long long n, int rule) {                             \
        LESS less;                                                                           \
        return pivot_value(A, n, rule, less);                                                \
    }                                                                                        \
    void bq_oracle_heapsort_##SUF(T *A, long long n) {                                       \
        LESS less;                                                                           \
        heap_sort(A, A + n, less);                                                           \
    }                                                                                        \
    void bq_oracle_insertion_sort_##SUF(T *A, long long n) {                                 \
        LESS less;                                                                           \
        insertion_sort(A, A + n, less);                                                      \
    }

BQ_ORACLE_DEFINE(i32, int32_t, LessI32)
BQ_ORACLE_DEFINE(u64, uint64_t, LessU64)
BQ_ORACLE_DEFINE(f64, double, LessF64)

/* Records: pivot passed as a key (records compare by key only, R10). */
void bq_oracle_sort_rec32(Rec32 *A, long long n, const bq_oracle_opts *o, bq_oracle_stats *st) {
    const bq_oracle_opts *op = o ? o : &kPaperOpts;
    bq_oracle_stats local;
    std::memset(&local, 0, sizeof local);
    Counting<Rec32, LessRec> less{LessRec{}, &local.comparisons};
    qsort_block(A, A + n, op->block, op->cutoff, op->depth_limit, less, &local);
    if (st) *st = local;
}
long long bq_oracle_block_partition_rec32(Rec32 *A, long long n, long long pivot_index,
                                          long long B, unsigned long long *cmp) {
    uint64_t c = 0;
    Counting<Rec32, LessRec> less{LessRec{}, &c};
    long long cut = hoare_block_partition_simple(A, A + n, A + pivot_index, B, less);
    if (cmp) *cmp = c;
    return cut;
}
void bq_oracle_partition_rec32(Rec32 *A, long long n, uint64_t pivot_key, long long B,
                               long long *split, long long *n_equal) {
    LessRec less;
    Rec32 p;
    std::memset(&p, 0, sizeof p);
    p.key = pivot_key;
    partition_value(A, n, p, B, less, split, n_equal);
}
uint64_t bq_oracle_pivot_rec32(const Rec32 *A, long long n, int rule) {
    LessRec less;
    return pivot_value(A, n, rule, less).key;
}

/* Default depth limit of the paper for n (R4), exported for tests. */
int bq_oracle_depth_limit(long long n) { return n >= 1 ? 2 * ilog2(n) + 3 : 0; }

/* the SplitMix64 output function used by SAMPLE64 (R19), exported for its
 * known-answer test (tests/test_oracle.py) */
uint64_t bq_oracle_splitmix64_mix(uint64_t z) { return splitmix64_mix(z); }

} // extern "C"
