// microbench_copy.cu — ceilings for the partition kernel's memory structure
// (tools only, not part of libbq): plain 128-bit copy vs a persistent
// TMA-ring copy (1D bulk loads into a STAGES-deep ring, bulk stores out),
// the same load/store shape k_partition uses, without the partition work.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench_copy.cu && ./mb
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void copy128(const uint4 *__restrict__ a, uint4 *__restrict__ b, size_t n4) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    size_t stride = (size_t)gridDim.x * blockDim.x;
    for (; i + 3 * stride < n4; i += 4 * stride) {
        uint4 x0 = __ldcs(a + i), x1 = __ldcs(a + i + stride), x2 = __ldcs(a + i + 2 * stride), x3 = __ldcs(a + i + 3 * stride);
        __stcs(b + i, x0); __stcs(b + i + stride, x1); __stcs(b + i + 2 * stride, x2); __stcs(b + i + 3 * stride, x3);
    }
    for (; i < n4; i += stride) __stcs(b + i, __ldcs(a + i));
}

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int STAGES, int TILEB>
__global__ void __launch_bounds__(128) tma_ring_copy(const char *a, char *b, uint32_t ntiles, uint32_t *ticket) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + STAGES * TILEB);
    uint32_t *tl = reinterpret_cast<uint32_t *>(full + STAGES);
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < STAGES; s++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (tid != 0) return;   // one thread drives the whole ring
    uint32_t issued = 0, done = 0;
    auto issue = [&](uint32_t slot) {
        uint32_t t = atomicAdd(ticket, 1u);
        tl[slot] = t;
        if (t < ntiles) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[slot])), "r"(TILEB));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             su32(sm + slot * TILEB)),
                         "l"(a + (size_t)t * TILEB), "r"(TILEB), "r"(su32(&full[slot])));
        }
    };
    for (int s = 0; s < STAGES; s++) issue(s);
    issued = STAGES;
    while (true) {
        const uint32_t slot = done % STAGES, ph = (done / STAGES) & 1;
        const uint32_t t = tl[slot];
        if (t >= ntiles) break;
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(
                         su32(&full[slot])),
                     "r"(ph));
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(b + (size_t)t * TILEB),
                     "r"(su32(sm + slot * TILEB)), "r"(TILEB));
        asm volatile("cp.async.bulk.commit_group;");
        asm volatile("cp.async.bulk.wait_group.read 0;");   // slot free again
        done++;
        issue(slot);
    }
    asm volatile("cp.async.bulk.wait_group 0;");
}

template <int STAGES, int TILEB>
int run_ring(const char *a, char *b, size_t bytes, uint32_t *ticket, int ctas_per_sm, int sms) {
    const uint32_t ntiles = (uint32_t)(bytes / TILEB);
    const int smem = STAGES * TILEB + STAGES * 8 + STAGES * 4 + 64;
    CK(cudaFuncSetAttribute(tma_ring_copy<STAGES, TILEB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9;
    for (int r = 0; r < 6; r++) {
        cudaMemset(ticket, 0, 4);
        cudaEventRecord(e0);
        tma_ring_copy<STAGES, TILEB><<<sms * ctas_per_sm, 128, smem>>>(a, b, ntiles, ticket);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    printf("tma_ring STAGES=%d TILE=%dKB ctas/SM=%d: %.3f ms  %.0f GB/s\n", STAGES, TILEB / 1024, ctas_per_sm, best,
           2.0 * bytes / best / 1e6);
    return 0;
}

int main() {
    const size_t bytes = 1ull << 30;
    char *a, *b;
    uint32_t *ticket;
    CK(cudaMalloc(&a, bytes));
    CK(cudaMalloc(&b, bytes));
    CK(cudaMalloc(&ticket, 4));
    CK(cudaMemset(a, 1, bytes));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int bpsm : {2, 4, 8}) {
        float best = 1e9;
        for (int r = 0; r < 6; r++) {
            cudaEventRecord(e0);
            copy128<<<sms * bpsm, 512>>>((const uint4 *)a, (uint4 *)b, bytes / 16);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r > 0 && ms < best) best = ms;
        }
        printf("copy128 blocks/SM=%d: %.3f ms  %.0f GB/s\n", bpsm, best, 2.0 * bytes / best / 1e6);
    }
    run_ring<2, 16384>(a, b, bytes, ticket, 3, sms);
    run_ring<3, 16384>(a, b, bytes, ticket, 3, sms);
    run_ring<4, 16384>(a, b, bytes, ticket, 2, sms);
    run_ring<4, 16384>(a, b, bytes, ticket, 3, sms);
    run_ring<6, 16384>(a, b, bytes, ticket, 2, sms);
    run_ring<8, 16384>(a, b, bytes, ticket, 1, sms);
    run_ring<4, 32768>(a, b, bytes, ticket, 1, sms);
    run_ring<6, 32768>(a, b, bytes, ticket, 1, sms);
    run_ring<3, 32768>(a, b, bytes, ticket, 2, sms);
    run_ring<8, 8192>(a, b, bytes, ticket, 2, sms);
    run_ring<12, 8192>(a, b, bytes, ticket, 2, sms);
    return 0;
}
