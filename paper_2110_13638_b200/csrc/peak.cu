// peak.cu -- integer-pipe ceiling for the "alu" roofline ("Integer peak
// must be measured").  Every thread runs 8 independent chains of lazy Shoup modular
// multiplications (the NTT butterfly's multiply, arith.cuh) entirely in registers, so
// the kernel measures how many 64-bit modmuls/s the SMs can issue with no memory
// traffic.  Reported in the same unit as the hot kernels' algorithmic work.
#include "kernels.cuh"
#include "ntt_core.cuh"

namespace edl {

__global__ void __launch_bounds__(256) k_modmul_peak(uint64_t q, uint64_t w, uint64_t ws, int iters, uint64_t* sink) {
    EDL_PDL_ENTRY();
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

// Register-only CT butterflies (ntt_core.cuh ct_bfly, the NTT's inner operation) on 16
// residues per thread: 8 independent butterflies per round, twiddles held in registers, so
// the kernel measures the butterfly issue ceiling of one arithmetic path (FP64 pipe for
// q < 2^44, Shoup otherwise) with no memory traffic.  The "alu" roofline of the NTT
// kernels (bench.py) is this rate for their mix of primes.
template <bool FP>
__global__ void __launch_bounds__(256) k_bfly_peak(uint64_t q, const ulonglong2* __restrict__ tw, int iters,
                                                   uint64_t* sink) {
    EDL_PDL_ENTRY();
    uint64_t x[16];
    ulonglong2 w[8];
#pragma unroll
    for (int k = 0; k < 16; k++) {
        x[k] = (threadIdx.x * 16 + k + 1) % q;
        if constexpr (FP) x[k] = f64_from_u(x[k]);
    }
#pragma unroll
    for (int k = 0; k < 8; k++)   // F64 primes: compact binary64 table (8-byte entries)
        w[k] = FP ? make_ulonglong2(reinterpret_cast<const uint64_t*>(tw)[k], 0) : tw[k];
    const uint64_t two_q = 2 * q;
    const double qd = u52_to_double(q);
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 8; k++) ct_bfly<FP>(x[k], x[k + 8], w[k], q, two_q, qd, 1.0 / qd);   // the NTT's own butterfly
#pragma unroll
        for (int k = 0; k < 8; k++) {   // pair different lanes next round
            const uint64_t tmp = x[k];
            x[k] = x[(k + 3) & 15];
            x[(k + 3) & 15] = tmp;
        }
        if constexpr (FP) {   // the F64 values grow by <= 0.625 q per round: reduce every 16 rounds
            if ((it & 15) == 15) {
#pragma unroll
                for (int k = 0; k < 16; k++) x[k] = bits_of(f64_reduce(f64_of(x[k]), qd, 1.0 / qd));
            }
        }
    }
    uint64_t acc = 0;
#pragma unroll
    for (int k = 0; k < 16; k++) acc ^= x[k];
    if (acc == 0x123456789ull) sink[0] = acc;
}

void launch_bfly_peak(const Dev& d, uint64_t q, bool fp, const ulonglong2* tw, int iters, int blocks, uint64_t* sink) {
    if (fp) EDL_LAUNCH(d, "k_bfly_peak", k_bfly_peak<true><<<blocks, 256, 0, d.st>>>(q, tw, iters, sink));
    else EDL_LAUNCH(d, "k_bfly_peak", k_bfly_peak<false><<<blocks, 256, 0, d.st>>>(q, tw, iters, sink));
}

// Raw pipe probes anchoring the butterfly ceilings: 8 independent chains per
// thread of (a) DFMA (FP64 pipe) or (b) 32x32->64 IMAD.WIDE.U32 (the fmaheavy integer
// multiply the Shoup path is built from), 256 threads x 8 CTAs per SM, register-only.
// Reports lane-operations per second (one DFMA or one IMAD.WIDE per lane).
__global__ void __launch_bounds__(256) k_pipe_dfma(double a, double b, int iters, uint64_t* sink) {
    EDL_PDL_ENTRY();
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = (double)(threadIdx.x + k);
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 8; k++) x[k] = __fma_rn(x[k], a, b);
    }
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 8; k++) acc += x[k];
    if (acc == 1.2345) sink[0] = 1;
}
__global__ void __launch_bounds__(256) k_pipe_imadw(uint32_t a, int iters, uint64_t* sink) {
    EDL_PDL_ENTRY();
    uint64_t x[8];
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = threadIdx.x + k;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 8; k++) {   // IMAD.WIDE.U32: x = lo32(x) * a + x (64-bit addend)
            uint64_t r;
            asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"((uint32_t)x[k]), "r"(a), "l"(x[k]));
            x[k] = r;
        }
    }
    uint64_t acc = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) acc ^= x[k];
    if (acc == 0x123456789ull) sink[0] = acc;
}

// Modular multiply-accumulate ceilings of the MAC layers (register-only, 8 independent
// accumulators per thread): (2) the F64 path acc += f64_mulc(x, w, RD(w/q), q) for a 40-bit
// prime, (3) the 60-bit path's lazy 128-bit acc += x w (mac128).  One MAC per lane-op.
__global__ void __launch_bounds__(256) k_pipe_fmac(double q, double w, double wq, int iters, uint64_t* sink) {
    EDL_PDL_ENTRY();
    double acc[8], x[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
        acc[k] = 0.0;
        x[k] = (double)(threadIdx.x * 8 + k + 1);
    }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 8; k++) acc[k] = __dadd_rn(acc[k], f64_mulc(x[k], w, wq, q));
#pragma unroll
        for (int k = 0; k < 8; k++) x[k] = __dadd_rn(x[k], 1.0);   // fresh operands (exact, small)
        if ((it & 255) == 255) {
#pragma unroll
            for (int k = 0; k < 8; k++) acc[k] = f64_reduce(acc[k], q, 1.0 / q);
        }
    }
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < 8; k++) a += acc[k];
    if (a == 1.5) sink[0] = 1;
}
__global__ void __launch_bounds__(256) k_pipe_imac(uint64_t w, int iters, uint64_t* sink) {
    EDL_PDL_ENTRY();
    U128 acc[8];
    uint64_t x[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
        acc[k].lo = acc[k].hi = 0;
        x[k] = threadIdx.x * 8 + k + 1;
    }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 8; k++) mac128(acc[k], x[k], w);
#pragma unroll
        for (int k = 0; k < 8; k++) x[k] += 0x9E3779B97F4A7C15ull;
    }
    uint64_t a = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) a ^= acc[k].lo ^ acc[k].hi;
    if (a == 0x123456789ull) sink[0] = a;
}

void launch_pipe_probe(const Dev& d, int which, int iters, int blocks, uint64_t* sink) {
    if (which == 0) EDL_LAUNCH(d, "k_pipe_dfma", k_pipe_dfma<<<blocks, 256, 0, d.st>>>(1.0000001, 1e-9, iters, sink));
    else if (which == 1) EDL_LAUNCH(d, "k_pipe_imadw", k_pipe_imadw<<<blocks, 256, 0, d.st>>>(0x9E3779B9u, iters, sink));
    else if (which == 2) {
        const double q = 1099511627689.0, w = 777777777777.0;   // a 40-bit odd modulus, w < q
        EDL_LAUNCH(d, "k_pipe_fmac", k_pipe_fmac<<<blocks, 256, 0, d.st>>>(q, w, __builtin_floor(w / q * 1e15) / 1e15, iters,
                                                                           sink));
    } else {
        EDL_LAUNCH(d, "k_pipe_imac", k_pipe_imac<<<blocks, 256, 0, d.st>>>(0xFEDCBA987654321ull, iters, sink));
    }
}

void launch_modmul_peak(const Dev& d, uint64_t q, uint64_t w, uint64_t ws, int iters, int blocks, uint64_t* sink) {
    EDL_LAUNCH(d, "k_modmul_peak", k_modmul_peak<<<blocks, 256, 0, d.st>>>(q, w, ws, iters, sink));
}

}  // namespace edl
