// Do the FP64 pipe (DFMA) and the integer multiply (IMAD.WIDE) overlap on one SM?
// A: all warps DFMA chains; B: all warps IMAD.WIDE chains; C: even warps DFMA, odd warps
// IMAD.WIDE (same work per warp as A/B, half the warps each).  C ~ max(A, B)/2-ish means
// the pipes overlap; C ~ (A + B)/2 means they share issue/pipe resources.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void dfma_chain(double* x, int iters) {
    for (int it = 0; it < iters; it++)
#pragma unroll
        for (int k = 0; k < 8; k++) x[k] = __fma_rn(x[k], 1.0000001, 1e-9);
}
__device__ __forceinline__ void imadw_chain(uint64_t* x, int iters) {
    for (int it = 0; it < iters; it++)
#pragma unroll
        for (int k = 0; k < 8; k++) {
            uint64_t r;
            asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"((uint32_t)x[k]), "r"(0x9E3779B9u), "l"(x[k]));
            x[k] = r;
        }
}
__global__ void k(int mode, int iters, uint64_t* sink) {
    const int warp = threadIdx.x >> 5;
    bool fp = mode == 0 || (mode == 2 && (warp & 1) == 0);
    double xd[8];
    uint64_t xi[8];
    for (int k = 0; k < 8; k++) { xd[k] = threadIdx.x + k; xi[k] = threadIdx.x + k; }
    if (fp) dfma_chain(xd, iters); else imadw_chain(xi, iters);
    double a = 0; uint64_t b = 0;
    for (int k = 0; k < 8; k++) { a += xd[k]; b ^= xi[k]; }
    if (a == 1.5 || b == 0x1234567ull) sink[0] = b;
}
int main() {
    uint64_t* sink; cudaMalloc(&sink, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 4096;
    for (int mode = 0; mode < 3; mode++) {
        k<<<sms * 8, 256>>>(mode, 64, sink);
        cudaEventRecord(a);
        k<<<sms * 8, 256>>>(mode, iters, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double ops = (double)sms * 8 * 256 * 8 * iters;
        printf("mode %d (%s): %.3f ms  %.2f T lane-ops/s\n", mode, mode == 0 ? "all DFMA" : mode == 1 ? "all IMAD.WIDE" : "half/half", ms, ops / ms / 1e9);
    }
    return 0;
}
