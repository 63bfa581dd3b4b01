// api.cu — kind-independent entry points of libbq.so: errors, device check,
// workspace sizing and the kind-generic calls (see include/bq.h).
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "api_kind.cuh"

namespace bq {

static thread_local char g_last_error[512] = "";

bq_status set_error(bq_status st, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(g_last_error, sizeof g_last_error, fmt, ap);
    va_end(ap);
    return st;
}

// Immutable per-device cache: 1 = sm_100, -1 = unsupported, 0 = unknown.
static int g_dev_ok[64];

bq_status check_device() {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return set_error(BQ_ERR_UNSUPPORTED, "no CUDA device: %s", cudaGetErrorString(e));
    if (dev < 0 || dev >= 64) return set_error(BQ_ERR_UNSUPPORTED, "device ordinal %d", dev);
    int ok = __atomic_load_n(&g_dev_ok[dev], __ATOMIC_RELAXED);
    if (ok == 0) {
        int major = 0, minor = 0;
        if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess)
            return set_error(BQ_ERR_UNSUPPORTED, "cannot query device %d", dev);
        ok = (major == 10 && minor == 0) ? 1 : -1;
        __atomic_store_n(&g_dev_ok[dev], ok, __ATOMIC_RELAXED);
    }
    if (ok < 0) return set_error(BQ_ERR_UNSUPPORTED, "libbq.so is built for sm_100a only");
    return BQ_OK;
}

// Instantiated sort graphs (driver.cuh build_sort_graph), keyed by device,
// kind, buffers, n and options: a small LRU list under a mutex.  The graphs
// are never destroyed at exit (the CUDA context may already be gone).
namespace {
struct GraphSlot {
    GraphKey key;
    cudaGraphExec_t exec;
    uint64_t used;
};
std::mutex g_graph_mu;
std::vector<GraphSlot> *g_graphs = new std::vector<GraphSlot>();
uint64_t g_graph_clock = 0;
constexpr size_t GRAPH_SLOTS = 32;
}  // namespace

bool graph_cache_get(const GraphKey &k, cudaGraphExec_t *ex) {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    for (auto &g : *g_graphs)
        if (g.key == k) {
            g.used = ++g_graph_clock;
            *ex = g.exec;
            return true;
        }
    return false;
}

void graph_cache_put(const GraphKey &k, cudaGraphExec_t ex) {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    if (g_graphs->size() >= GRAPH_SLOTS) {
        size_t lru = 0;
        for (size_t i = 1; i < g_graphs->size(); i++)
            if ((*g_graphs)[i].used < (*g_graphs)[lru].used) lru = i;
        cudaGraphExecDestroy((*g_graphs)[lru].exec);
        g_graphs->erase(g_graphs->begin() + lru);
    }
    g_graphs->push_back(GraphSlot{k, ex, ++g_graph_clock});
}

}  // namespace bq

using namespace bq::detail;

extern "C" {

BQ_API size_t bq_workspace_bytes(bq_kind kind, size_t n) {
    switch (kind) {
        case BQ_I32: return ws_i32(n);
        case BQ_U64: return ws_u64(n);
        case BQ_F64: return ws_f64(n);
        case BQ_REC32: return ws_rec(n);
        case BQ_KEYIDX16: return ws_pair(n);
    }
    return 0;
}

BQ_API bq_status bq_partition_pass(bq_kind kind, const void *src, void *dst, size_t n, const void *pivot,
                                   uint64_t *d_counts, int ordered, void *ws, size_t ws_bytes, void *stream) {
    if (pivot == nullptr) return bq::set_error(BQ_ERR_INVALID_ARGUMENT, "NULL pivot");
    cudaStream_t s = (cudaStream_t)stream;
    switch (kind) {
        case BQ_I32: return pass_i32(src, dst, n, pivot, d_counts, ws, ws_bytes, s, ordered);
        case BQ_U64: return pass_u64(src, dst, n, pivot, d_counts, ws, ws_bytes, s, ordered);
        case BQ_F64: {
            double d;
            std::memcpy(&d, pivot, 8);
            if (d != d) return bq::set_error(BQ_ERR_INVALID_ARGUMENT, "NaN pivot");
            return pass_f64(src, dst, n, pivot, d_counts, ws, ws_bytes, s, ordered);
        }
        case BQ_REC32: return pass_rec(src, dst, n, pivot, d_counts, ws, ws_bytes, s, ordered);
        case BQ_KEYIDX16: return pass_pair(src, dst, n, pivot, d_counts, ws, ws_bytes, s, ordered);
    }
    return bq::set_error(BQ_ERR_INVALID_ARGUMENT, "bad kind %d", (int)kind);
}

BQ_API size_t bq_inplace_workspace_bytes(bq_kind kind, size_t n) {
    switch (kind) {
        case BQ_I32: return ipws_i32(n);
        case BQ_U64: return ipws_u64(n);
        case BQ_F64: return ipws_f64(n);
        case BQ_REC32: return ipws_rec(n);
        case BQ_KEYIDX16: return ipws_pair(n);
    }
    return 0;
}

BQ_API bq_status bq_partition_inplace(bq_kind kind, void *data, size_t n, const void *pivot, size_t *split,
                                      size_t *n_equal, void *ws, size_t ws_bytes, void *stream) {
    if (pivot == nullptr) return bq::set_error(BQ_ERR_INVALID_ARGUMENT, "NULL pivot");
    cudaStream_t s = (cudaStream_t)stream;
    switch (kind) {
        case BQ_I32: return inplace_i32(data, n, pivot, split, n_equal, ws, ws_bytes, s);
        case BQ_U64: return inplace_u64(data, n, pivot, split, n_equal, ws, ws_bytes, s);
        case BQ_F64: {
            double d;
            std::memcpy(&d, pivot, 8);
            if (d != d) return bq::set_error(BQ_ERR_INVALID_ARGUMENT, "NaN pivot");
            return inplace_f64(data, n, pivot, split, n_equal, ws, ws_bytes, s);
        }
        case BQ_REC32: return inplace_rec(data, n, pivot, split, n_equal, ws, ws_bytes, s);
        case BQ_KEYIDX16: return inplace_pair(data, n, pivot, split, n_equal, ws, ws_bytes, s);
    }
    return bq::set_error(BQ_ERR_INVALID_ARGUMENT, "bad kind %d", (int)kind);
}

BQ_API bq_status bq_partition_segments(bq_kind kind, const void *src, void *dst, size_t n, const uint32_t *begins,
                                       const uint32_t *lens, const void *pivots, size_t nseg, uint64_t *d_counts,
                                       int ordered, void *ws, size_t ws_bytes, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (nseg && pivots == nullptr) return bq::set_error(BQ_ERR_INVALID_ARGUMENT, "NULL pivots");
    if (kind == BQ_F64)
        for (size_t i = 0; i < nseg; i++) {
            double d;
            std::memcpy(&d, static_cast<const char *>(pivots) + 8 * i, 8);
            if (d != d) return bq::set_error(BQ_ERR_INVALID_ARGUMENT, "NaN pivot");
        }
    switch (kind) {
        case BQ_I32: return segs_i32(src, dst, n, begins, lens, pivots, nseg, d_counts, ws, ws_bytes, s, ordered);
        case BQ_U64: return segs_u64(src, dst, n, begins, lens, pivots, nseg, d_counts, ws, ws_bytes, s, ordered);
        case BQ_F64: return segs_f64(src, dst, n, begins, lens, pivots, nseg, d_counts, ws, ws_bytes, s, ordered);
        case BQ_REC32: return segs_rec(src, dst, n, begins, lens, pivots, nseg, d_counts, ws, ws_bytes, s, ordered);
        case BQ_KEYIDX16:
            return segs_pair(src, dst, n, begins, lens, pivots, nseg, d_counts, ws, ws_bytes, s, ordered);
    }
    return bq::set_error(BQ_ERR_INVALID_ARGUMENT, "bad kind %d", (int)kind);
}

BQ_API bq_status bq_sort_ex(bq_kind kind, void *data, size_t n, const bq_sort_options *opt, bq_sort_stats *stats,
                            void *ws, size_t ws_bytes, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    switch (kind) {
        case BQ_I32: return sort_i32(data, n, opt, stats, ws, ws_bytes, s);
        case BQ_U64: return sort_u64(data, n, opt, stats, ws, ws_bytes, s);
        case BQ_F64: return sort_f64(data, n, opt, stats, ws, ws_bytes, s);
        case BQ_REC32: return sort_rec(data, n, opt, stats, ws, ws_bytes, s);
        case BQ_KEYIDX16: return sort_pair(data, n, opt, stats, ws, ws_bytes, s);
    }
    return bq::set_error(BQ_ERR_INVALID_ARGUMENT, "bad kind %d", (int)kind);
}

BQ_API bq_status bq_sort_host(bq_kind kind, void *host_data, size_t n, void *dev_data, const bq_sort_options *opt,
                              void *ws, size_t ws_bytes, void *stream) {
    static const size_t W[5] = {4, 8, 8, 32, 16};
    if ((int)kind < 0 || (int)kind > 4) return bq::set_error(BQ_ERR_INVALID_ARGUMENT, "bad kind %d", (int)kind);
    if (n > 0 && (host_data == nullptr || dev_data == nullptr))
        return bq::set_error(BQ_ERR_INVALID_ARGUMENT, "NULL buffer with n > 0");
    cudaStream_t s = (cudaStream_t)stream;
    const size_t bytes = n * W[kind];
    if (bytes) BQ_CK(cudaMemcpyAsync(dev_data, host_data, bytes, cudaMemcpyHostToDevice, s));
    bq_status st = bq_sort_ex(kind, dev_data, n, opt, nullptr, ws, ws_bytes, stream);
    if (st != BQ_OK) return st;
    if (bytes) BQ_CK(cudaMemcpyAsync(host_data, dev_data, bytes, cudaMemcpyDeviceToHost, s));
    BQ_CK(cudaStreamSynchronize(s));
    return BQ_OK;
}

BQ_API const char *bq_status_string(bq_status s) {
    switch (s) {
        case BQ_OK: return "BQ_OK";
        case BQ_ERR_INVALID_ARGUMENT: return "BQ_ERR_INVALID_ARGUMENT";
        case BQ_ERR_WORKSPACE: return "BQ_ERR_WORKSPACE";
        case BQ_ERR_CUDA: return "BQ_ERR_CUDA";
        case BQ_ERR_UNSUPPORTED: return "BQ_ERR_UNSUPPORTED";
    }
    return "BQ_ERR_UNKNOWN";
}

BQ_API const char *bq_last_error(void) { return bq::g_last_error; }

BQ_API int bq_version(void) { return 200; }

BQ_API size_t bq_tile_elems(bq_kind kind) {
    switch (kind) {
        case BQ_I32: return bq::tile_elems<bq::KI32>();
        case BQ_U64: return bq::tile_elems<bq::KU64>();
        case BQ_F64: return bq::tile_elems<bq::KF64>();
        case BQ_REC32: return bq::tile_elems<bq::KRec>();
        case BQ_KEYIDX16: return bq::tile_elems<bq::KPair>();
    }
    return 0;
}

BQ_API size_t bq_leaf_elems(bq_kind kind) {
    switch (kind) {
        case BQ_I32: return bq::Tune<bq::KI32>::LEAF;
        case BQ_U64: return bq::Tune<bq::KU64>::LEAF;
        case BQ_F64: return bq::Tune<bq::KF64>::LEAF;
        case BQ_REC32: return bq::Tune<bq::KRec>::LEAF;
        case BQ_KEYIDX16: return bq::Tune<bq::KPair>::LEAF;
    }
    return 0;
}

}
