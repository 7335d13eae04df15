// peak.cu -- integer-pipe ceiling for the "alu" roofline ("Integer peak
// must be measured").  Every thread runs 8 independent chains of lazy Shoup modular
// multiplications (the NTT butterfly's multiply, arith.cuh) entirely in registers, so
// the kernel measures how many 64-bit modmuls/s the SMs can issue with no memory
// traffic.  Reported in the same unit as the hot kernels' algorithmic work.
#include "kernels.cuh"

namespace edl {

__global__ void __launch_bounds__(256) k_modmul_peak(uint64_t q, uint64_t w, uint64_t ws, int iters, uint64_t* sink) {
    uint64_t x[8];
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = (threadIdx.x * 8 + k + 1) % q;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 8; k++) x[k] = shoup_lazy2(x[k], w, ws, q);
    }
    uint64_t acc = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) acc ^= x[k];
    if (acc == 0x123456789ull) sink[0] = acc;   // keep the chains alive
}

void launch_modmul_peak(const Dev& d, uint64_t q, uint64_t w, uint64_t ws, int iters, int blocks, uint64_t* sink) {
    EDL_LAUNCH(d, "k_modmul_peak", k_modmul_peak<<<blocks, 256, 0, d.st>>>(q, w, ws, iters, sink));
}

}  // namespace edl
