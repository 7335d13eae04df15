// ntt_persist.cuh -- persistent NTT / INTT for N = K * M with thread-block clusters
// (N = 2^14 on the C1 hot path), twiddles resident in shared memory.
//
// Why (round-2 ncu of the round-1 kernels, profiles/round2/): the per-stage twiddle loads
// of the transforms read ~130 KB per CTA (the limb itself is 64 KB in + out) and missed
// L1 68 % of the time, because the 4 CTAs an SM holds belong to different cluster ranks
// (disjoint twiddle subsets, 4 x 64 KB against ~90 KB of L1); the arithmetic then stalls
// on L2 latency (long_scoreboard was the top stall of every NTT kernel).  Every limb
// transform needs all N-1 distinct twiddles of its prime, so the only way to cut that
// traffic is reuse ACROSS limbs: here a CTA stays resident (persistent grid, one loop
// over work items ordered prime-major), keeps the M-1 twiddles its cluster rank uses in
// shared memory and reloads them only when the prime changes (a few times per launch).
// The next item's input residues are fetched into registers before the current item's
// butterflies (software pipelining across items), and the CTA runs 128 registers per
// thread (2 CTAs per SM), so nothing spills.
//
// Shared-memory twiddle table of cluster rank r (local stage t = 0..log M - 1):
//   T_r[2^t + u] = tw[2^(t + log K) + r 2^t + u],  u < 2^t
// which is exactly the global stage-twiddle formula of ntt_core.cuh with the rank bits
// removed, so the pass code is unchanged (SA = local stage, high = local group index).
#pragma once
#include "ntt_core.cuh"

namespace edl {

// CTA-cooperative copy of rank crank's twiddle subset into shared memory: 16-byte
// {w, Shoup w'} entries, or (F64 primes, f64_mult butterflies) 8-byte w only.
template <class C>
__device__ __forceinline__ void load_tw_smem(ulonglong2* tws, const ulonglong2* __restrict__ g, bool f64) {
    uint64_t* tw8 = reinterpret_cast<uint64_t*>(tws);
    for (int u = threadIdx.x; u < C::M; u += C::T) {
        if (u == 0) continue;
        const int t = 31 - __clz(u);
        const int gi = (1 << (t + C::LOGK)) + (C::crank() << t) + (u - (1 << t));
        if (f64) tw8[u] = __ldg(reinterpret_cast<const uint64_t*>(g) + gi);   // compact table
        else tws[u] = __ldg(g + gi);
    }
}
struct SmemTw8 {   // compact F64 table: the companion slot is never read on that path
    const uint64_t* t;
    __device__ __forceinline__ ulonglong2 operator()(int i) const { return make_ulonglong2(t[i], 0); }
};
template <bool FP>
struct SmemTwOf {
    using type = SmemTw;
    __device__ static type make(const ulonglong2* t) { return SmemTw{t}; }
};
template <>
struct SmemTwOf<true> {
    using type = SmemTw8;
    __device__ static type make(const ulonglong2* t) { return SmemTw8{reinterpret_cast<const uint64_t*>(t)}; }
};

// In-CTA pass P on the local twiddle table.
template <class C, int P, bool INV, bool FP, class TW>
__device__ __forceinline__ void pass_smem_p(uint64_t* sm, const ModInfo& m, uint64_t two_q, TW tw) {
    using PI = PassInfo<C, P>;
    uint64_t x[C::E];
#pragma unroll
    for (int g = 0; g < PI::G; g++) {
        const int v = threadIdx.x + g * C::T;
        const int low = v & ((1 << PI::BLOW) - 1);
        const int high = v >> PI::BLOW;
        const int base = (high << (PI::BTOP + 1)) | low;
#pragma unroll
        for (int r = 0; r < (1 << PI::NS); r++) x[g * (1 << PI::NS) + r] = sm[spad(base | (r << PI::BLOW))];
    }
    __syncthreads();
#pragma unroll
    for (int g = 0; g < PI::G; g++) {
        const int v = threadIdx.x + g * C::T;
        const int high = v >> PI::BLOW;
        if constexpr (INV) inv_pass_regs_t<PI::SL, PI::NS, false, FP>(x + g * (1 << PI::NS), high, m, two_q, tw);
        else fwd_pass_regs_t<PI::SL, PI::NS, FP>(x + g * (1 << PI::NS), high, tw, m.q, two_q, u52_to_double(m.q), m.qinv_d);
    }
#pragma unroll
    for (int g = 0; g < PI::G; g++) {
        const int v = threadIdx.x + g * C::T;
        const int low = v & ((1 << PI::BLOW) - 1);
        const int high = v >> PI::BLOW;
        const int base = (high << (PI::BTOP + 1)) | low;
#pragma unroll
        for (int r = 0; r < (1 << PI::NS); r++) sm[spad(base | (r << PI::BLOW))] = x[g * (1 << PI::NS) + r];
    }
    __syncthreads();
}

template <class C, int P, bool INV, bool FP, class TW>
__device__ __forceinline__ void middle_p(uint64_t* sm, const ModInfo& m, uint64_t two_q, TW tw) {
    if constexpr (INV) {
        if constexpr (P > 0) {
            pass_smem_p<C, P, true, FP>(sm, m, two_q, tw);
            middle_p<C, P - 1, true, FP>(sm, m, two_q, tw);
        }
    } else {
        if constexpr (P < C::NPASS) {
            pass_smem_p<C, P, false, FP>(sm, m, two_q, tw);
            middle_p<C, P + 1, false, FP>(sm, m, two_q, tw);
        }
    }
}

// Per-item cluster handshake (same protocol as ntt_core.cuh): the item's exchange mbarrier
// is initialised and fenced, then the CTA arrives (relaxed) on the cluster barrier: its
// shared memory is free for its peers' remote stores.
__device__ __forceinline__ void item_open(uint32_t mb) {
    if (threadIdx.x == 0) mbar_init_cluster(mb);
    cluster_arrive_relaxed();
}

// Forward transform of one limb from residues already in registers in the phase-A layout
// (x[g K + t] = a[crank M/K + tid + g T + t M], as exact binary64 bits on the F64 path),
// after item_open().  store(idx, v) receives canonical residues at idx = C::idx(r).
template <class C, bool FP, class Store>
__device__ __forceinline__ void pfwd(uint64_t* sm, const ModInfo& m, const ulonglong2* tws, uint64_t* x, uint32_t mb,
                                     Store store) {
    const auto tw = SmemTwOf<FP>::make(tws);
    static_assert(C::K > 1, "persistent transforms are cluster transforms");
    const uint64_t q = m.q, two_q = 2 * q;
    const double qd = FP ? u52_to_double(q) : 0.0;
    const int tid = threadIdx.x;
    const int j0 = C::crank() * (C::M / C::K) + tid;
#pragma unroll
    for (int g = 0; g < C::E / C::K; g++) fwd_pass_regs<0, C::LOGK, FP>(x + g * C::K, 0, m.tw_fwd, q, two_q, qd, m.qinv_d);
    cluster_wait();
    if (tid == 0) mbar_expect(mb, (uint32_t)((C::K - 1) * (C::M / C::K) * 8));
#pragma unroll
    for (int t = 0; t < C::K; t++) {
        if (t == C::crank()) {
#pragma unroll
            for (int g = 0; g < C::E / C::K; g++) sm[spad(j0 + g * C::T)] = x[g * C::K + t];
        } else {
            const uint32_t rb = mapa_u32(mb, t);
            const uint32_t rs = mapa_u32(smem_u32(sm), t);
#pragma unroll
            for (int g = 0; g < C::E / C::K; g++) st_async_b64(rs + 8u * spad(j0 + g * C::T), x[g * C::K + t], rb);
        }
    }
    __syncthreads();
    mbar_wait0(mb);
#pragma unroll
    for (int r = 0; r < C::E; r++) x[r] = sm[spad(tid + r * C::T)];
    fwd_pass_regs_t<0, C::LOGE, FP>(x, 0, tw, q, two_q, qd, m.qinv_d);
#pragma unroll
    for (int r = 0; r < C::E; r++) sm[spad(tid + r * C::T)] = x[r];
    __syncthreads();
    middle_p<C, 1, false, FP>(sm, m, two_q, tw);
#pragma unroll
    for (int r = 0; r < C::E; r++) {
        uint64_t v = sm[spad(tid + r * C::T)];
        if constexpr (FP) v = f64_to_canon(f64_reduce(f64_of(v), qd, m.qinv_d), qd);
        else v = canon_fwd(v, q);
        store(C::idx(r), v);
    }
    __syncthreads();
    if (tid == 0) mbar_inval(mb);
}

// Inverse transform of one limb from residues in registers at idx = C::idx(r) (exact
// binary64 bits on the F64 path; item_open() is called inside, after the local passes,
// because the CTA's own shared memory is in use until then); store(idx, canonical value) at the
// phase-A' indices crank M/K + tid + g T + t M.
template <class C, bool FP, class Store>
__device__ __forceinline__ void pinv(uint64_t* sm, const ModInfo& m, const ulonglong2* tws, uint64_t* x, uint32_t mb,
                                     Store store) {
    const auto tw = SmemTwOf<FP>::make(tws);
    static_assert(C::K > 1, "persistent transforms are cluster transforms");
    const uint64_t q = m.q, two_q = 2 * q;
    const double qd = FP ? u52_to_double(q) : 0.0;
    const int tid = threadIdx.x;
#pragma unroll
    for (int r = 0; r < C::E; r++) sm[spad(tid + r * C::T)] = x[r];
    __syncthreads();
    middle_p<C, C::NPASS - 1, true, FP>(sm, m, two_q, tw);
#pragma unroll
    for (int r = 0; r < C::E; r++) x[r] = sm[spad(tid + r * C::T)];
    inv_pass_regs_t<0, C::LOGE, false, FP>(x, 0, m, two_q, tw);
    constexpr int MK = C::M / C::K;
    __syncthreads();   // this CTA's reads of its sub-block are performed ...
    item_open(mb);
    cluster_wait();    // ... and every peer's
    if (tid == 0) mbar_expect(mb, (uint32_t)((C::K - 1) * MK * 8));
    const uint32_t rs0 = smem_u32(sm);
#pragma unroll
    for (int r = 0; r < C::E; r++) {
        const int j = tid + r * C::T;
        const int t = r / (C::E / C::K);
        const int w = spad(C::crank() * MK + (j & (MK - 1)));
        if (t == C::crank()) sm[w] = x[r];
        else st_async_b64(mapa_u32(rs0, t) + 8u * w, x[r], mapa_u32(mb, t));
    }
    __syncthreads();
    mbar_wait0(mb);
    const int j0 = C::crank() * MK + tid;
#pragma unroll
    for (int g = 0; g < C::E / C::K; g++) {
#pragma unroll
        for (int t = 0; t < C::K; t++) x[g * C::K + t] = sm[spad(t * MK + tid + g * C::T)];
        inv_pass_regs<0, C::LOGK, true, FP>(x + g * C::K, 0, m, two_q);
#pragma unroll
        for (int t = 0; t < C::K; t++) {
            uint64_t v = x[g * C::K + t];
            if constexpr (FP) v = f64_to_canon(f64_of(v), qd);
            else v = canon_inv(v, q);
            store(j0 + g * C::T + t * C::M, v);
        }
    }
    __syncthreads();
    if (tid == 0) mbar_inval(mb);
}

}  // namespace edl
