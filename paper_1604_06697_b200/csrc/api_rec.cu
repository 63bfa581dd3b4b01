// api_rec.cu — 32-byte record entry points of libbq.so (see include/bq.h).
// Records compare by key only.
#include "api_kind.cuh"

namespace bq {

// ---- the key+index path -------------------------------------
// Records are large elements with cheap comparisons: every
// partition pass of the direct path moves 32 bytes per record.  Here the
// passes move 16-byte (key, position) pairs, and each record moves once, in a
// final gather.  Workspace: [pairs 16n | pair-sort workspace | records 32n]:
// the extraction reads every record once and also copies it aside, so the
// gather reads the copy and writes the user buffer directly.
__global__ void k_ki_extract(const Rec32 *r, KeyIdx16 *p, Rec32 *copy, uint64_t n) {
    const uint4 *r4 = reinterpret_cast<const uint4 *>(r);
    uint4 *c4 = reinterpret_cast<uint4 *>(copy);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 v0 = __ldcs(r4 + 2 * i), v1 = __ldcs(r4 + 2 * i + 1);
        p[i] = KeyIdx16{(uint64_t)v0.x | ((uint64_t)v0.y << 32), i};
        c4[2 * i] = v0;
        c4[2 * i + 1] = v1;
    }
}
// the records in sorted order: pair i names the record of rank i; random
// 32-byte reads of the copy, so each thread keeps U of them in flight (their
// positions first, then the independent loads)
__global__ void k_ki_gather(const Rec32 *copy, const KeyIdx16 *p, Rec32 *out, uint64_t n) {
    constexpr int U = 8;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint4 *r4 = reinterpret_cast<const uint4 *>(copy);
    uint4 *g4 = reinterpret_cast<uint4 *>(out);
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += stride * U) {
        uint64_t k[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint64_t j = i0 + u * stride;
            k[u] = j < n ? __ldcs(&p[j].idx) : 0u;
        }
        uint4 v[U][2];
#pragma unroll
        for (int u = 0; u < U; u++) {
            if (i0 + u * stride < n) {
                // one 32-byte load per record (sm_100's 256-bit LDG) with a 64-byte
                // DRAM fetch hint: 2.1 B fetched per byte used instead of 4.2
                asm volatile("ld.global.nc.L2::64B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=r"(v[u][0].x), "=r"(v[u][0].y), "=r"(v[u][0].z), "=r"(v[u][0].w),
                               "=r"(v[u][1].x), "=r"(v[u][1].y), "=r"(v[u][1].z), "=r"(v[u][1].w)
                             : "l"(r4 + 2 * k[u]));
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint64_t j = i0 + u * stride;
            if (j < n) {
                __stcs(g4 + 2 * j, v[u][0]);
                __stcs(g4 + 2 * j + 1, v[u][1]);
            }
        }
    }
}

namespace detail {
struct KiLayout {
    size_t pairs, pws, pws_bytes, copy, total;
};
static KiLayout ki_layout(size_t n) {
    KiLayout L;
    L.pairs = 0;
    L.pws = align_up(n * sizeof(KeyIdx16), 256);
    L.pws_bytes = make_layout<KPair>(n).total;   // the pair sort's own layout (not the in-place partition's)
    L.copy = align_up(L.pws + L.pws_bytes, 256);
    L.total = align_up(L.copy + n * sizeof(Rec32), 256);
    return L;
}
// records below this size are one leaf (or a few): the direct path
constexpr size_t KI_MIN = 2 * (size_t)Tune<KRec>::LEAF;

static bq_status sort_rec_ki(Rec32 *data, size_t n, const bq_sort_options *opt, bq_sort_stats *st, void *ws,
                             size_t wsb, cudaStream_t s) {
    const KiLayout L = ki_layout(n);
    if (wsb < L.total) return set_error(BQ_ERR_WORKSPACE, "workspace %zu B < required %zu B", wsb, L.total);
    char *w = static_cast<char *>(ws);
    KeyIdx16 *pairs = reinterpret_cast<KeyIdx16 *>(w + L.pairs);
    Rec32 *copy = reinterpret_cast<Rec32 *>(w + L.copy);
    const uint32_t grid = 148 * 8;
    k_ki_extract<<<grid, 256, 0, s>>>(data, pairs, copy, n);
    BQ_CK_LAUNCH();
    bq_status r = sort_pair(pairs, n, opt, st, w + L.pws, L.pws_bytes, s);
    if (r != BQ_OK) return r;
    k_ki_gather<<<grid, 256, 0, s>>>(copy, pairs, data, n);
    BQ_CK_LAUNCH();
    if (st) st->kernel_launches += 2;
    return BQ_OK;
}

size_t ws_rec(size_t n) {
    const size_t a = make_layout<KRec>(n).total, b = ki_layout(n).total, c = make_ip_layout<KRec>(n).total;
    return a > b ? (a > c ? a : c) : (b > c ? b : c);
}
size_t ipws_rec(size_t n) { return make_ip_layout<KRec>(n).total; }
bq_status inplace_rec(void *data, size_t n, const void *pivot, size_t *split, size_t *neq, void *ws, size_t wsb,
                      cudaStream_t s) {
    return run_partition_inplace_ip<KRec>(static_cast<Rec32 *>(data), n, pivot_key_from<KRec>(pivot), split, neq,
                                          ws, wsb, s);
}
bq_status sort_rec(void *data, size_t n, const bq_sort_options *opt, bq_sort_stats *st, void *ws, size_t wsb,
                   cudaStream_t s) {
    const int path = opt ? opt->records : 0;
    if (path < 0 || path > 2) return set_error(BQ_ERR_INVALID_ARGUMENT, "records path %d", path);
    Rec32 *r = static_cast<Rec32 *>(data);
    if (path == 1 || n < KI_MIN) return run_sort<KRec>(r, n, opt, st, ws, wsb, s);
    bq_status v = validate<KRec>(data, n, ws, wsb);
    if (v != BQ_OK) return v;
    return sort_rec_ki(r, n, opt, st, ws, wsb, s);
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
    return bq::detail::sort_rec(recs, n, nullptr, nullptr, ws, ws_bytes, (cudaStream_t)stream);
}

}
