// Probe: semantics of fmin/fmax on doubles (DMNMX) for signed zeros, and
// throughput of DMNMX vs the 64-bit integer compare-exchange on B200.
#include <cstdio>
#include <cstdint>
#include <cstring>
__global__ void k_sem(const double *in, unsigned long long *out) {
    const double a = in[threadIdx.x * 2], b = in[threadIdx.x * 2 + 1];
    const double lo = fmin(a, b), hi = fmax(a, b);
    out[threadIdx.x * 2] = __double_as_longlong(lo);
    out[threadIdx.x * 2 + 1] = __double_as_longlong(hi);
}
template <int MODE>
__global__ void k_tput(double *d, int iters) {
    double x[16];
    for (int i = 0; i < 16; i++) x[i] = d[threadIdx.x * 16 + i];
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            if (MODE == 0) {
                const double lo = fmin(x[i], x[i + 8]), hi = fmax(x[i], x[i + 8]);
                x[i] = hi; x[i + 8] = lo;
            } else {
                unsigned long long a = __double_as_longlong(x[i]), b = __double_as_longlong(x[i + 8]);
                const bool s = b < a;
                const unsigned long long lo = s ? b : a, hi = s ? a : b;
                x[i] = __longlong_as_double(hi); x[i + 8] = __longlong_as_double(lo);
            }
        }
    }
    for (int i = 0; i < 16; i++) d[threadIdx.x * 16 + i] = x[i];
}
int main() {
    double h[8] = {-0.0, 0.0, 0.0, -0.0, -1e-320, -0.0, 1.0, -0.0};
    double *d; unsigned long long *o, ho[8];
    cudaMalloc(&d, 64); cudaMalloc(&o, 64);
    cudaMemcpy(d, h, 64, cudaMemcpyHostToDevice);
    k_sem<<<1, 4>>>(d, o);
    cudaMemcpy(ho, o, 64, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 4; i++) printf("min/max(%g,%g): %016llx %016llx\n", h[2*i], h[2*i+1], ho[2*i], ho[2*i+1]);
    double *big; cudaMalloc(&big, 148 * 8 * 256 * 16 * 8);
    cudaMemset(big, 0, 148 * 8 * 256 * 16 * 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int mode = 0; mode < 2; mode++) {
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(e0);
            if (mode == 0) k_tput<0><<<148 * 8, 256>>>(big, 4096); else k_tput<1><<<148 * 8, 256>>>(big, 4096);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            const double ces = 148.0 * 8 * 256 * 4096 * 8;
            if (rep) printf("mode %d (%s): %.3f ms, %.1f G CE/s\n", mode, mode ? "int64 ISETP+SEL" : "DMNMX", ms, ces / ms / 1e6);
        }
    }
    return 0;
}
