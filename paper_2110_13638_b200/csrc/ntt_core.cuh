// ntt_core.cuh -- one-CTA negacyclic NTT / INTT of a whole limb (N <= 2^14) on sm_100a.
//
// Definition (background to PAPER.md:470 "encoded into a single
// polynomial"): A[k] = sum_j a_j psi^{(2 brv(k) + 1) j} mod q, i.e. Cooley-Tukey
// decimation in time with stage twiddle psi^{brv(m+i)} (natural in, bit-reversed out);
// the inverse is Gentleman-Sande with psi^{-brv(m+i)} and N^{-1} folded into its last
// stage.
//
// B200 design: T threads (T = N/E) each hold E = 2^LOGE residues in registers; the
// log N stages run as ceil(log N / LOGE) register-resident radix-2^LOGE passes with a
// padded shared-memory exchange between passes.  Global traffic is exactly one
// coalesced read and one coalesced write of the limb: the forward's first pass and the
// inverse's last pass already hold the strided pattern idx = tid + T*r, and the other
// end goes through shared memory.  Butterflies are Harvey-lazy (forward values in
// [0,4q), inverse in [0,2q)) with Shoup twiddles, so q < 2^62.  Caller-supplied
// load/store functors fuse prologues (pointwise products, centered lifts, modulus
// raise) and epilogues (rescale, key-switch MAC, bias) into the same pass over HBM.
#pragma once
#include "arith.cuh"

namespace edl {

// Residues per thread: the plain transform keeps 32 per thread (fewer exchanges); the
// fused kernels, whose prologue/epilogue need registers and more warps to hide their
// extra global traffic, keep 16 (N = 2^14: 1024 threads).  Measured in round 1.
__host__ __device__ constexpr int loge_plain(int logn) { return logn >= 14 ? 5 : (logn >= 12 ? 4 : 3); }
__host__ __device__ constexpr int loge_fused(int logn) { return logn >= 14 ? 4 : 3; }

template <int LOGN, int LOGE_ = loge_fused(LOGN)>
struct NttShape {
    static constexpr int N = 1 << LOGN;
    static constexpr int LOGE = LOGE_;
    static constexpr int E = 1 << LOGE;
    static constexpr int T = N / E;
    static constexpr int NPASS = (LOGN + LOGE - 1) / LOGE;
    static constexpr int SMEM_WORDS = N + N / 16;
    static constexpr int SMEM_BYTES = SMEM_WORDS * 8;
};

__device__ __forceinline__ int spad(int idx) { return idx + (idx >> 4); }

// ---- forward CT butterfly (Harvey): X, Y in [0,4q) -> [0,4q)
__device__ __forceinline__ void ct_bfly(uint64_t& X, uint64_t& Y, ulonglong2 w, uint64_t q, uint64_t two_q) {
    uint64_t x = csub(X, two_q);
    uint64_t t = shoup_lazy2(Y, w.x, w.y, q);
    X = x + t;
    Y = x - t + two_q;
}

// ---- inverse GS butterfly (Harvey): X, Y in [0,2q) -> [0,2q)
__device__ __forceinline__ void gs_bfly(uint64_t& X, uint64_t& Y, uint64_t w, uint64_t ws, uint64_t q, uint64_t two_q) {
    uint64_t x = X, y = Y;
    X = csub(x + y, two_q);
    Y = shoup_lazy2(x - y + two_q, w, ws, q);
}

// One forward pass over stages [S0, S0+NS) for `v`-th virtual thread's group held in x[].
// Element r of the group sits at index  (high << (BTOP+1)) | (r << BLOW) | low.
template <int LOGN, int S0, int NS>
__device__ __forceinline__ void fwd_pass_regs(uint64_t* x, int high, const ulonglong2* __restrict__ tw,
                                              uint64_t q, uint64_t two_q) {
#pragma unroll
    for (int k = 0; k < NS; k++) {
        const int half = 1 << (NS - 1 - k);
#pragma unroll
        for (int r = 0; r < (1 << NS); r++) {
            if (r & half) continue;
            const int tidx = (1 << (S0 + k)) + (high << k) + (r >> (NS - k));
            ulonglong2 w = __ldg(tw + tidx);
            ct_bfly(x[r], x[r + half], w, q, two_q);
        }
    }
}

template <int LOGN, int S0, int NS, bool LAST>
__device__ __forceinline__ void inv_pass_regs(uint64_t* x, int high, const ModInfo& m, uint64_t two_q) {
#pragma unroll
    for (int k = NS - 1; k >= 0; k--) {
        const int half = 1 << (NS - 1 - k);
#pragma unroll
        for (int r = 0; r < (1 << NS); r++) {
            if (r & half) continue;
            if (LAST && S0 + k == 0) {
                // stage 0 (m = 1): fold N^-1 into both outputs
                uint64_t a = x[r], b = x[r + half];
                x[r] = shoup_lazy2(a + b, m.ninv, m.ninv_s, m.q);
                x[r + half] = shoup_lazy2(a - b + two_q, m.w1ninv, m.w1ninv_s, m.q);
            } else {
                const int tidx = (1 << (S0 + k)) + (high << k) + (r >> (NS - k));
                ulonglong2 w = __ldg(m.tw_inv + tidx);
                gs_bfly(x[r], x[r + half], w.x, w.y, m.q, two_q);
            }
        }
    }
}

// Compile-time pass descriptor: pass P covers stages [P*LOGE, min((P+1)*LOGE, LOGN)).
template <int LOGN, int LOGE, int P>
struct PassInfo {
    using S = NttShape<LOGN, LOGE>;
    static constexpr int S0 = P * S::LOGE;
    static constexpr int NS = (S0 + S::LOGE <= LOGN) ? S::LOGE : (LOGN - S0);
    static constexpr int BTOP = LOGN - 1 - S0;
    static constexpr int BLOW = BTOP - NS + 1;
    static constexpr int G = S::E >> NS;     // groups per thread
};

// Forward middle/last pass: read from smem, compute, write back to smem (natural index).
template <int LOGN, int LOGE, int P>
__device__ __forceinline__ void fwd_pass_smem(uint64_t* sm, const ulonglong2* __restrict__ tw, uint64_t q,
                                              uint64_t two_q) {
    using PI = PassInfo<LOGN, LOGE, P>;
    using S = NttShape<LOGN, LOGE>;
    uint64_t x[S::E];
#pragma unroll
    for (int g = 0; g < PI::G; g++) {
        const int v = threadIdx.x + g * S::T;
        const int low = v & ((1 << PI::BLOW) - 1);
        const int high = v >> PI::BLOW;
        const int base = (high << (PI::BTOP + 1)) | low;
#pragma unroll
        for (int r = 0; r < (1 << PI::NS); r++) x[g * (1 << PI::NS) + r] = sm[spad(base | (r << PI::BLOW))];
    }
    __syncthreads();
#pragma unroll
    for (int g = 0; g < PI::G; g++) {
        const int v = threadIdx.x + g * S::T;
        const int high = v >> PI::BLOW;
        fwd_pass_regs<LOGN, PI::S0, PI::NS>(x + g * (1 << PI::NS), high, tw, q, two_q);
    }
#pragma unroll
    for (int g = 0; g < PI::G; g++) {
        const int v = threadIdx.x + g * S::T;
        const int low = v & ((1 << PI::BLOW) - 1);
        const int high = v >> PI::BLOW;
        const int base = (high << (PI::BTOP + 1)) | low;
#pragma unroll
        for (int r = 0; r < (1 << PI::NS); r++) sm[spad(base | (r << PI::BLOW))] = x[g * (1 << PI::NS) + r];
    }
    __syncthreads();
}

template <int LOGN, int LOGE, int P>
__device__ __forceinline__ void inv_pass_smem(uint64_t* sm, const ModInfo& m, uint64_t two_q) {
    using PI = PassInfo<LOGN, LOGE, P>;
    using S = NttShape<LOGN, LOGE>;
    uint64_t x[S::E];
#pragma unroll
    for (int g = 0; g < PI::G; g++) {
        const int v = threadIdx.x + g * S::T;
        const int low = v & ((1 << PI::BLOW) - 1);
        const int high = v >> PI::BLOW;
        const int base = (high << (PI::BTOP + 1)) | low;
#pragma unroll
        for (int r = 0; r < (1 << PI::NS); r++) x[g * (1 << PI::NS) + r] = sm[spad(base | (r << PI::BLOW))];
    }
    __syncthreads();
#pragma unroll
    for (int g = 0; g < PI::G; g++) {
        const int v = threadIdx.x + g * S::T;
        const int high = v >> PI::BLOW;
        inv_pass_regs<LOGN, PI::S0, PI::NS, false>(x + g * (1 << PI::NS), high, m, two_q);
    }
#pragma unroll
    for (int g = 0; g < PI::G; g++) {
        const int v = threadIdx.x + g * S::T;
        const int low = v & ((1 << PI::BLOW) - 1);
        const int high = v >> PI::BLOW;
        const int base = (high << (PI::BTOP + 1)) | low;
#pragma unroll
        for (int r = 0; r < (1 << PI::NS); r++) sm[spad(base | (r << PI::BLOW))] = x[g * (1 << PI::NS) + r];
    }
    __syncthreads();
}

template <int LOGN, int LOGE, int P>
__device__ __forceinline__ void fwd_middle(uint64_t* sm, const ulonglong2* tw, uint64_t q, uint64_t two_q) {
    if constexpr (P < NttShape<LOGN, LOGE>::NPASS) {
        fwd_pass_smem<LOGN, LOGE, P>(sm, tw, q, two_q);
        fwd_middle<LOGN, LOGE, P + 1>(sm, tw, q, two_q);
    }
}

// Inverse passes run from the last pass down to pass 1 (pass 0 is register-resident).
template <int LOGN, int LOGE, int P>
__device__ __forceinline__ void inv_middle(uint64_t* sm, const ModInfo& m, uint64_t two_q) {
    if constexpr (P > 0) {
        inv_pass_smem<LOGN, LOGE, P>(sm, m, two_q);
        inv_middle<LOGN, LOGE, P - 1>(sm, m, two_q);
    }
}

// Forward NTT of one limb.  load(idx) -> residue in [0, 4q) (called with idx = tid + T*r);
// store(idx, value) receives canonical [0, q) values, idx = tid + T*r (coalesced).
template <int LOGN, int LOGE = loge_fused(LOGN), class Load, class Store>
__device__ __forceinline__ void ntt_fwd_block(uint64_t* sm, const ModInfo& m, Load load, Store store) {
    using S = NttShape<LOGN, LOGE>;
    using P0 = PassInfo<LOGN, LOGE, 0>;
    static_assert(P0::G == 1 && P0::BLOW == LOGN - S::LOGE, "pass 0 layout");
    const uint64_t q = m.q, two_q = 2 * q;
    const ulonglong2* tw = m.tw_fwd;
    uint64_t x[S::E];
#pragma unroll
    for (int r = 0; r < S::E; r++) x[r] = load(threadIdx.x + r * S::T);
    fwd_pass_regs<LOGN, 0, S::LOGE>(x, 0, tw, q, two_q);
#pragma unroll
    for (int r = 0; r < S::E; r++) sm[spad(threadIdx.x + r * S::T)] = x[r];
    __syncthreads();
    fwd_middle<LOGN, LOGE, 1>(sm, tw, q, two_q);
#pragma unroll
    for (int r = 0; r < S::E; r++) {
        const int idx = threadIdx.x + r * S::T;
        uint64_t v = sm[spad(idx)];
        v = csub(csub(v, two_q), q);
        store(idx, v);
    }
    __syncthreads();   // smem reusable by the caller's next transform
}

// Inverse NTT of one limb.  load(idx) -> residue in [0, 2q); store(idx, canonical value).
template <int LOGN, int LOGE = loge_fused(LOGN), class Load, class Store>
__device__ __forceinline__ void ntt_inv_block(uint64_t* sm, const ModInfo& m, Load load, Store store) {
    using S = NttShape<LOGN, LOGE>;
    const uint64_t q = m.q, two_q = 2 * q;
#pragma unroll
    for (int r = 0; r < S::E; r++) {
        const int idx = threadIdx.x + r * S::T;
        sm[spad(idx)] = load(idx);
    }
    __syncthreads();
    inv_middle<LOGN, LOGE, S::NPASS - 1>(sm, m, two_q);
    uint64_t x[S::E];
#pragma unroll
    for (int r = 0; r < S::E; r++) x[r] = sm[spad(threadIdx.x + r * S::T)];
    inv_pass_regs<LOGN, 0, S::LOGE, true>(x, 0, m, two_q);
#pragma unroll
    for (int r = 0; r < S::E; r++) store(threadIdx.x + r * S::T, csub(x[r], q));
    __syncthreads();   // smem reusable by the caller's next transform
}

}  // namespace edl
