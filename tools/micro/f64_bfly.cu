// Microbenchmark: register-only NTT butterflies, integer (Shoup / FP64-quotient, the
// library's ct_bfly) vs a pure-FP64 butterfly (residues held as doubles, error-free
// product via FMA).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I paper_2110_13638_b200/csrc tools/micro/f64_bfly.cu -o /tmp/f64_bfly
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ double mulmod_f64(double b, double w, double wq, double q) {
    const double M = 6755399441055744.0;   // 1.5 * 2^52: round to nearest integer
    const double hi = b * w;
    const double lo = fma(b, w, -hi);
    const double qt = fma(b, wq, M) - M;
    const double r = fma(-qt, q, hi);
    return r + lo;
}
__device__ __forceinline__ double mulmod_f64_rint(double b, double w, double wq, double q) {
    const double hi = b * w;
    const double lo = fma(b, w, -hi);
    const double qt = rint(b * wq);
    const double r = fma(-qt, q, hi);
    return r + lo;
}

template <int V>
__global__ void __launch_bounds__(256) k_f64(double q, const double2* __restrict__ tw, int iters, double* sink) {
    double x[16];
    double2 w[8];
#pragma unroll
    for (int k = 0; k < 16; k++) x[k] = (double)((threadIdx.x * 16 + k + 1) % 1000);
#pragma unroll
    for (int k = 0; k < 8; k++) w[k] = tw[k];
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const double t = V == 0 ? mulmod_f64(x[k + 8], w[k].x, w[k].y, q) : mulmod_f64_rint(x[k + 8], w[k].x, w[k].y, q);
            const double a = x[k];
            x[k] = a + t;
            x[k + 8] = a - t;
        }
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const double tmp = x[k];
            x[k] = x[(k + 3) & 15];
            x[(k + 3) & 15] = tmp;
        }
        if ((it & 7) == 7) {   // keep magnitudes bounded (reduce, 3 ops per value, amortised)
#pragma unroll
            for (int k = 0; k < 16; k++) x[k] = fma(-rint(x[k] * w[0].y), q, x[k]);
        }
    }
    double acc = 0;
#pragma unroll
    for (int k = 0; k < 16; k++) acc += x[k];
    if (acc == 1.2345) sink[0] = acc;
}

__device__ __forceinline__ uint64_t mulhi(uint64_t a, uint64_t b) { return __umul64hi(a, b); }
__global__ void __launch_bounds__(256) k_shoup(uint64_t q, const ulonglong2* __restrict__ tw, int iters, uint64_t* sink) {
    uint64_t x[16];
    ulonglong2 w[8];
#pragma unroll
    for (int k = 0; k < 16; k++) x[k] = (threadIdx.x * 16 + k + 1) % q;
#pragma unroll
    for (int k = 0; k < 8; k++) w[k] = tw[k];
    const uint64_t two_q = 2 * q;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 8; k++) {
            uint64_t X = x[k], Y = x[k + 8];
            X = X >= two_q ? X - two_q : X;
            const uint64_t t = Y * w[k].x - mulhi(Y, w[k].y) * q;
            x[k] = X + t;
            x[k + 8] = X - t + two_q;
        }
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const uint64_t tmp = x[k];
            x[k] = x[(k + 3) & 15];
            x[(k + 3) & 15] = tmp;
        }
    }
    uint64_t acc = 0;
#pragma unroll
    for (int k = 0; k < 16; k++) acc ^= x[k];
    if (acc == 0x123456789ull) sink[0] = acc;
}

// half the CTAs run the integer butterfly, half the FP64 one (pipe overlap test)
__global__ void __launch_bounds__(256) k_mixed(double q, const double2* __restrict__ tw, uint64_t qi,
                                               const ulonglong2* __restrict__ itw, int iters, double* sink) {
    if (blockIdx.x & 1) {
        double x[16];
        double2 w[8];
#pragma unroll
        for (int k = 0; k < 16; k++) x[k] = (double)((threadIdx.x * 16 + k + 1) % 1000);
#pragma unroll
        for (int k = 0; k < 8; k++) w[k] = tw[k];
        for (int it = 0; it < iters; it++) {
#pragma unroll
            for (int k = 0; k < 8; k++) {
                const double t = mulmod_f64(x[k + 8], w[k].x, w[k].y, q);
                const double a = x[k];
                x[k] = a + t;
                x[k + 8] = a - t;
            }
#pragma unroll
            for (int k = 0; k < 8; k++) {
                const double tmp = x[k];
                x[k] = x[(k + 3) & 15];
                x[(k + 3) & 15] = tmp;
            }
            if ((it & 7) == 7) {
#pragma unroll
                for (int k = 0; k < 16; k++) x[k] = fma(-rint(x[k] * w[0].y), q, x[k]);
            }
        }
        double acc = 0;
#pragma unroll
        for (int k = 0; k < 16; k++) acc += x[k];
        if (acc == 1.2345) sink[0] = acc;
    } else {
        uint64_t x[16];
        ulonglong2 w[8];
#pragma unroll
        for (int k = 0; k < 16; k++) x[k] = (threadIdx.x * 16 + k + 1) % qi;
#pragma unroll
        for (int k = 0; k < 8; k++) w[k] = itw[k];
        const uint64_t two_q = 2 * qi;
        for (int it = 0; it < iters / 2; it++) {   // integer butterflies are ~2.7x slower: balance the CTA times
#pragma unroll
            for (int k = 0; k < 8; k++) {
                uint64_t X = x[k], Y = x[k + 8];
                X = X >= two_q ? X - two_q : X;
                const uint64_t t = Y * w[k].x - mulhi(Y, w[k].y) * qi;
                x[k] = X + t;
                x[k + 8] = X - t + two_q;
            }
#pragma unroll
            for (int k = 0; k < 8; k++) {
                const uint64_t tmp = x[k];
                x[k] = x[(k + 3) & 15];
                x[(k + 3) & 15] = tmp;
            }
        }
        uint64_t acc = 0;
#pragma unroll
        for (int k = 0; k < 16; k++) acc ^= x[k];
        if (acc == 0x123456789ull) sink[1] = (double)acc;
    }
}

int main() {
    const double q = 1099511922689.0;   // ~2^40 prime-ish (value irrelevant for timing)
    double2 htw[8];
    for (int k = 0; k < 8; k++) { htw[k].x = 123456789.0 * (k + 3); htw[k].y = htw[k].x / q; }
    double2* dtw; cudaMalloc(&dtw, sizeof(htw)); cudaMemcpy(dtw, htw, sizeof(htw), cudaMemcpyHostToDevice);
    ulonglong2 itw[8];
    for (int k = 0; k < 8; k++) { itw[k].x = 123456789ull * (k + 3); itw[k].y = (uint64_t)(((unsigned __int128)itw[k].x << 64) / 1099511922689ull); }
    ulonglong2* ditw; cudaMalloc(&ditw, sizeof(itw)); cudaMemcpy(ditw, itw, sizeof(itw), cudaMemcpyHostToDevice);
    void* sink; cudaMalloc(&sink, 64);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, iters = 4096;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int v = 0; v < 3; v++) {
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(a);
            if (v == 0) k_f64<0><<<blocks, 256>>>(q, dtw, iters, (double*)sink);
            if (v == 1) k_f64<1><<<blocks, 256>>>(q, dtw, iters, (double*)sink);
            if (v == 2) k_shoup<<<blocks, 256>>>(1099511922689ull, ditw, iters, (uint64_t*)sink);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            const double bf = (double)blocks * 256 * iters * 8;
            if (rep) printf("variant %d (%s): %.1f Gbfly/s\n", v, v == 0 ? "f64 magic" : v == 1 ? "f64 rint" : "int shoup", bf / ms / 1e6);
        }
    }
    for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(a);
        k_mixed<<<blocks, 256>>>(q, dtw, 1099511922689ull, ditw, iters, (double*)sink);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        const double bf = (double)blocks / 2 * 256 * 8 * (iters + iters / 2);
        if (rep) printf("mixed (half f64 x iters, half int x iters/2): %.1f Gbfly/s total, %.3f ms\n", bf / ms / 1e6, ms);
    }
    // predicted with no overlap: time(f64 part) + time(int part) from the single-path rates
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
