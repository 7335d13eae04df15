// ntt_core.cuh -- negacyclic NTT / INTT of one limb on sm_100a, by one CTA (N <= 2^13)
// or by a thread-block cluster of K CTAs exchanging through distributed shared memory
// (N = 2^14 .. 2^16).
//
// Definition (background to PAPER.md:470 "encoded into a single
// polynomial"): A[k] = sum_j a_j psi^{(2 brv(k) + 1) j} mod q, i.e. Cooley-Tukey
// decimation in time with stage twiddle psi^{brv(m+i)} (natural in, bit-reversed out);
// the inverse is Gentleman-Sande with psi^{-brv(m+i)} and N^{-1} folded into its last
// stage.
//
// B200 design.  N = K * M with M <= 2^13 residues (64 KiB) per CTA, so two or three CTAs
// share an SM and one CTA's global loads overlap another's butterflies.
//   Forward: CTA r of the cluster loads, for its M/K low indices j, all K residues
//   j + t M (t < K) and runs the first log K stages in registers (they only mix the top
//   log K index bits); the residues of sub-block t are then stored into CTA t's shared
//   memory (DSMEM all-to-all), and every CTA finishes the remaining log M stages of its
//   own contiguous sub-block.  The inverse mirrors this (sub-block stages first, exchange,
//   last log K stages with N^-1 folded in).  K = 1 is the plain one-CTA transform.
//   Inside a CTA, T = M/E threads hold E = 2^LOGE residues in registers; the log M stages
//   run as ceil(log M / LOGE) register-resident radix-2^LOGE passes with a padded
//   shared-memory exchange between passes (pad 1 word per 16: conflict-free 64-bit
//   accesses in every pass).  Global traffic is one coalesced read and one coalesced
//   write of the limb.  Butterflies are Harvey-lazy (forward values in [0,4q), inverse in
//   [0,2q)) with Shoup twiddles {w, floor(w 2^64/q)}, so q < 2^61.  Caller-supplied
//   load(idx)/store(idx, v) functors (global coefficient index idx) fuse prologues and
//   epilogues (pointwise products, centered lifts, modulus raise, rescale, key-switch
//   MAC, bias) into the same pass over HBM.
#pragma once
#include <cooperative_groups.h>
#include <type_traits>

#include "arith.cuh"

namespace edl {

template <int LOGN_, int LOGK_, int LOGE_, int MINB_, bool STAGE_ = false, bool TWPF_ = false>
struct NttCfg {
    static constexpr bool STAGE_EPI = STAGE_;   // epilogue operand staged in smem by cp.async (epi_pre)
    static constexpr bool TW_PF_FWD = TWPF_;    // F64 forward: next-pass twiddles prefetched across barriers
    static constexpr int LOGN = LOGN_;
    static constexpr int LOGK = LOGK_;
    static constexpr int LOGM = LOGN_ - LOGK_;
    static constexpr int LOGE = LOGE_;
    static constexpr int N = 1 << LOGN;
    static constexpr int K = 1 << LOGK;
    static constexpr int M = 1 << LOGM;
    static constexpr int E = 1 << LOGE;
    static constexpr int T = M / E;                   // threads per CTA
    static constexpr int NPASS = (LOGM + LOGE - 1) / LOGE;
    static constexpr int MINB = MINB_;               // __launch_bounds__ min blocks / SM
    static constexpr int SMEM_WORDS = M + M / 16;
    static constexpr int SMEM_BYTES = SMEM_WORDS * 8;
    static_assert(E >= K, "phase A needs every thread to hold all K residues of a column");
    static_assert(LOGE <= LOGM && T >= 32, "at least one warp per CTA");
    // cluster rank (which sub-block this CTA owns) and the limb/grid index above it
    __device__ static __forceinline__ int crank() { return K == 1 ? 0 : (int)(blockIdx.x & (K - 1)); }
    __device__ static __forceinline__ int bx() { return (int)(blockIdx.x >> LOGK); }
    // The coefficient indices a thread stores after ntt_fwd and loads before ntt_inv,
    // r < E: idx(r) = crank*M + tid + T*r (coalesced).
    __device__ static __forceinline__ int idx(int r) { return (crank() << LOGM) + (int)threadIdx.x + r * T; }
};

__device__ __forceinline__ constexpr int spad(int idx) { return idx + (idx >> 4); }
// spad(a | b) = spad(a) + spad(b) for bit-disjoint a, b (the shift distributes over a
// disjoint OR): every shared-memory index below is a per-thread base plus spad() of a
// compile-time part, i.e. one register plus an immediate offset (round 2: ptxas does not
// know tid < T and recomputed idx + (idx >> 4) for every access, ~13 % of the transform's
// instructions).

// ---- L2 prefetch pipelining ---------------------------------------------------------
// One CTA per SM holds a whole 2^14 limb, so its global load phase and its butterflies do
// not overlap.  Bulk L2 prefetches (cp.async.bulk.prefetch.L2: one instruction per
// operand range, no registers, no completion tracking) issued at CTA start bring (a) the
// CTA's own epilogue operands and (b) the prologue inputs of the CTA that will occupy this
// slot one wave later into L2 while this CTA computes, so both load phases hit L2.
// Measured on B200 (round 1): +3 to +26 % kernel time (the prefetched limbs evict lines
// the running CTAs still need), so it is compiled out unless EDL_L2_PREFETCH is defined.
__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes) {
#ifdef EDL_L2_PREFETCH
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
#else
    (void)p;
    (void)bytes;
#endif
}

// Prefetch the CTA's own sub-block [crank*M, crank*M + M) of a limb starting at `limb`.
template <class C>
__device__ __forceinline__ void pf_own(const uint64_t* limb) {
#ifdef EDL_L2_PREFETCH_OWN
    if (limb)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(limb + ((size_t)C::crank() << C::LOGM)),
                     "r"((uint32_t)C::M * 8u)
                     : "memory");
#else
    if (limb) l2_prefetch(limb + ((size_t)C::crank() << C::LOGM), (uint32_t)C::M * 8u);
#endif
}

// Calls f(bx, crank, y, z) for the block that starts one wave (SMs x MINB CTAs) after this
// one in launch order, if it exists.  Thread 0 only.
template <class C, class F>
__device__ __forceinline__ void pf_next_wave(F f) {
    uint32_t nsm;
    asm("mov.u32 %0, %%nsmid;" : "=r"(nsm));
    const uint64_t lin = blockIdx.x + (uint64_t)gridDim.x * (blockIdx.y + (uint64_t)gridDim.y * blockIdx.z);
    const uint64_t nxt = lin + (uint64_t)nsm * C::MINB;
    const uint64_t total = (uint64_t)gridDim.x * gridDim.y * gridDim.z;
    if (nxt >= total) return;
    const uint32_t x = (uint32_t)(nxt % gridDim.x);
    const uint64_t yz = nxt / gridDim.x;
    f((int64_t)(x >> C::LOGK), (int)(x & (C::K - 1)), (int)(yz % gridDim.y), (int)(yz / gridDim.y));
}

// The sub-block of `limb` that CTA rank cr of a cluster loads (forward phase A loads K
// strided chunks; prefetch the whole limb then) or owns (inverse input, forward output).
template <class C>
__device__ __forceinline__ void pf_sub(const uint64_t* limb, int cr, bool whole) {
    if (whole || C::K == 1) l2_prefetch(limb, (uint32_t)C::N * 8u);
    else l2_prefetch(limb + ((size_t)cr << C::LOGM), (uint32_t)C::M * 8u);
}

__device__ __forceinline__ void cluster_sync_all() { cooperative_groups::this_cluster().sync(); }
// Split cluster barrier without the release fence: arrive once this CTA's shared memory may
// be overwritten by its peers (no pending reads: program start or after a __syncthreads),
// wait (acquire) right before writing into a peer's shared memory.
__device__ __forceinline__ void cluster_arrive_relaxed() { asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }

// ---- DSMEM exchange with asynchronous remote stores (K > 1) ---------------------------
// Each CTA's residues for peer t leave as st.async (shared::cluster, 8 bytes) that count
// their bytes against t's mbarrier; a CTA then waits on its own mbarrier for the (K-1)M/K
// words its peers owe it instead of a second full cluster barrier with a release fence.
// The mbarrier lives for one transform: initialised (and fenced for the cluster) before
// the transform's relaxed cluster arrive, which every peer waits on before its first
// remote store, and invalidated after the transform's closing __syncthreads.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async_b64(uint32_t raddr, uint64_t v, uint32_t rmbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr), "l"(v), "r"(rmbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_init_cluster(uint32_t mbar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n\tfence.mbarrier_init.release.cluster;" ::"r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}
// Phase 0 of a fresh mbarrier.  The bytes it counts arrive by st.async into this CTA's own
// shared memory, which the mbarrier's complete-tx makes visible at CTA scope: no
// cluster-scope acquire, so ptxas emits no L1 invalidation (CCTL.IVALL) here -- the
// round-2 ncu showed that invalidation at 2-4 % of stall samples, and it evicted the
// L1-cached twiddles after every exchange.  (EDL_MBAR_CLUSTER_ACQUIRE restores it.)
__device__ __forceinline__ void mbar_wait0(uint32_t mbar) {
    uint32_t done;
    do {
#ifdef EDL_MBAR_CLUSTER_ACQUIRE
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], 0;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done)
                     : "r"(mbar)
                     : "memory");
#else
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], 0;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done)
                     : "r"(mbar)
                     : "memory");
#endif
    } while (!done);
}
__device__ __forceinline__ void mbar_inval(uint32_t mbar) { asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(mbar) : "memory"); }
#ifndef EDL_XCHG_SYNC
#define EDL_XCHG_ASYNC 1
#endif

template <class C>
__device__ __forceinline__ uint64_t* cluster_smem(uint64_t* sm, int rank) {
    if constexpr (C::K == 1) return sm;
    else return cooperative_groups::this_cluster().map_shared_rank(sm, rank);
}

// ---- forward CT butterfly, Shoup path (Harvey): X, Y in [0,4q) -> [0,4q).
// ---- F64 path (ModInfo::fp == 2, q < 2^44): residues are held as exact binary64
// integers (bit patterns in the same 64-bit registers / shared-memory words) and every
// butterfly runs on the FP64 pipe, which the integer (fmaheavy) path leaves idle:
//   t = Y w mod q:  hi = RN(Y w), lo = Y w - hi (exact, one FMA), qt = nearest integer to
//   Y RD(w/q) (one FMA against 1.5 2^52, the product inside it exact), t = RN(hi - qt q) + lo.
//   |Y (w/q - RD(w/q))| < |Y| 2^-53 <= 1/8 for |Y| < 2^50, so |t| <= 0.625 q, hi - qt q is an
//   integer below 2^47 (exact), and t is exact.  Forward values stay signed and unreduced:
//   |x| <= 4q + 0.625 q per stage < 15 q through 16 stages, far below 2^50.
// 8 FP64 instructions per butterfly (B200: 64 FP64 lanes/clk/SM, measured 2.0 T
// butterflies/s register-only vs 1.26 T for the integer FP64-quotient path).
template <bool FP>
__device__ __forceinline__ void ct_bfly(uint64_t& X, uint64_t& Y, ulonglong2 w, uint64_t q, uint64_t two_q,
                                        double qd = 0.0, double qinv = 0.0) {
    if constexpr (FP) {   // twiddle = w only (f64_mult: no companion)
        const double x = f64_of(X);
        const double t = f64_mult(f64_of(Y), f64_of(w.x), qd, qinv);
        X = bits_of(__dadd_rn(x, t));
        Y = bits_of(__dsub_rn(x, t));
    } else {
#ifdef EDL_SHOUP3   // X, Y in [0, 8q): x in [0, 4q), t in [0, 3q) -> [0, 7q), (q, 8q)
        const uint64_t four_q = 2 * two_q;
        uint64_t x = csub(X, four_q);
        uint64_t t = shoup_lazy3(Y, w.x, w.y, q);
        X = x + t;
        Y = x - t + four_q;
#else
        uint64_t x = csub(X, two_q);
        uint64_t t = shoup_lazy2(Y, w.x, w.y, q);
        X = x + t;
        Y = x - t + two_q;
#endif
    }
}

// ---- inverse GS butterfly (Harvey): X, Y in [0,2q) -> [0,2q)
__device__ __forceinline__ void gs_bfly(uint64_t& X, uint64_t& Y, uint64_t w, uint64_t ws, uint64_t q, uint64_t two_q) {
    uint64_t x = X, y = Y;
#ifdef EDL_SHOUP3   // X, Y in [0, 4q) -> [0, 4q), [0, 3q)
    X = csub(x + y, 2 * two_q);
    Y = shoup_lazy3(x - y + 2 * two_q, w, ws, q);
#else
    X = csub(x + y, two_q);
    Y = shoup_lazy2(x - y + two_q, w, ws, q);
#endif
}
// Lazy bound added before a difference in the inverse (x - y + LB >= 0): 4q or 2q.
__device__ __forceinline__ uint64_t inv_lb(uint64_t two_q) {
#ifdef EDL_SHOUP3
    return 2 * two_q;
#else
    return two_q;
#endif
}
// Canonical residue of the integer path's outputs: forward [0, 8q) (or [0, 4q)), inverse
// [0, 3q) (or [0, 2q)).
__device__ __forceinline__ uint64_t canon_fwd(uint64_t v, uint64_t q) {
#ifdef EDL_SHOUP3
    v = csub(v, 4 * q);
#endif
    return csub(csub(v, 2 * q), q);
}
__device__ __forceinline__ uint64_t canon_inv(uint64_t v, uint64_t q) {
#ifdef EDL_SHOUP3
    v = csub(v, 2 * q);
#endif
    return csub(v, q);
}

// Twiddle accessors: the global table (read-only path), or a CTA's shared-memory copy of
// the entries its stages use (persistent kernels, ntt_persist.cuh).
struct GlobTw {
    const ulonglong2* __restrict__ t;
    __device__ __forceinline__ ulonglong2 operator()(int i) const { return __ldg(t + i); }
};
struct SmemTw {
    const ulonglong2* t;
    __device__ __forceinline__ ulonglong2 operator()(int i) const { return t[i]; }
};
// F64-pipe primes (ModInfo::fp == 2) keep compact tables of 8-byte twiddles (binary64 w;
// the f64_mult butterflies need no companion): half the twiddle bytes and L1 footprint.
struct GlobTw8 {
    const uint64_t* __restrict__ t;
    __device__ __forceinline__ ulonglong2 operator()(int i) const { return make_ulonglong2(__ldg(t + i), 0); }
};
template <bool FP>
__device__ __forceinline__ auto glob_tw(const ulonglong2* t) {
    if constexpr (FP) return GlobTw8{reinterpret_cast<const uint64_t*>(t)};
    else return GlobTw{t};
}

// NS forward stages on a group x[0..2^NS) held in registers; absolute stage SA + k uses
// twiddle index 2^(SA+k) + (high << k) + (r >> (NS-k)), `high` = the group's index bits
// above the stage window (SURVEY O3 stage twiddle psi^brv(m+i)).
template <int SA, int NS, bool FP, class TW>
__device__ __forceinline__ void fwd_pass_regs_t(uint64_t* x, int high, TW tw, uint64_t q, uint64_t two_q, double qd,
                                                double qinv) {
#pragma unroll
    for (int k = 0; k < NS; k++) {
        const int half = 1 << (NS - 1 - k);
#pragma unroll
        for (int r = 0; r < (1 << NS); r++) {
            if (r & half) continue;
            const int tidx = (1 << (SA + k)) + (high << k) + (r >> (NS - k));
            ulonglong2 w = tw(tidx);
            ct_bfly<FP>(x[r], x[r + half], w, q, two_q, qd, qinv);
        }
#ifdef EDL_STAGE_FENCE
        asm volatile("" ::: "memory");
#endif
    }
}
template <int SA, int NS, bool FP>
__device__ __forceinline__ void fwd_pass_regs(uint64_t* x, int high, const ulonglong2* __restrict__ tw, uint64_t q,
                                              uint64_t two_q, double qd, double qinv) {
    fwd_pass_regs_t<SA, NS, FP>(x, high, glob_tw<FP>(tw), q, two_q, qd, qinv);
}

// NS inverse stages, last to first; with LAST the absolute stage 0 folds N^-1 into both
// outputs (psi^-brv(1) N^-1 for the odd one).  F64 path: the differences leave through
// f64_mulc (|.| <= 0.625 q) and the sums of the pass's last stage are reduced, so every
// pass starts from |x| < 2q (first pass: loads in [0, 2q)) and grows to at most
// 2q 2^NS <= 64 q < 2^50 inside it.
template <int SA, int NS, bool LAST, bool FP, class TW>
__device__ __forceinline__ void inv_pass_regs_t(uint64_t* x, int high, const ModInfo& m, uint64_t two_q, TW tw) {
    double qd = 0.0;
    if constexpr (FP) qd = u52_to_double(m.q);
#pragma unroll
    for (int k = NS - 1; k >= 0; k--) {
        const int half = 1 << (NS - 1 - k);
#pragma unroll
        for (int r = 0; r < (1 << NS); r++) {
            if (r & half) continue;
            if constexpr (FP) {
                const double a = f64_of(x[r]), b = f64_of(x[r + half]);
                if (LAST && SA + k == 0) {
                    x[r] = bits_of(f64_mulc(__dadd_rn(a, b), u52_to_double(m.ninv), f64_of(m.ninv_s), qd));
                    x[r + half] = bits_of(f64_mulc(__dsub_rn(a, b), u52_to_double(m.w1ninv), f64_of(m.w1ninv_s), qd));
                } else {
                    const int tidx = (1 << (SA + k)) + (high << k) + (r >> (NS - k));
                    const ulonglong2 w = tw(tidx);
                    double s = __dadd_rn(a, b);
                    if (k == 0) s = f64_reduce(s, qd, m.qinv_d);
                    x[r] = bits_of(s);
                    x[r + half] = bits_of(f64_mult(__dsub_rn(a, b), f64_of(w.x), qd, m.qinv_d));
                }
            } else if (LAST && SA + k == 0) {
                uint64_t a = x[r], b = x[r + half];
                // fp == 1 primes (2^44 <= q < 2^46) take this path with RD(w/q) companions
                x[r] = m.fp ? tw_mul_fp(a + b, m.ninv, m.ninv_s, m.q) : shoup_lazy2(a + b, m.ninv, m.ninv_s, m.q);
                x[r + half] = m.fp ? tw_mul_fp(a - b + inv_lb(two_q), m.w1ninv, m.w1ninv_s, m.q)
                                   : shoup_lazy2(a - b + inv_lb(two_q), m.w1ninv, m.w1ninv_s, m.q);
            } else {
                const int tidx = (1 << (SA + k)) + (high << k) + (r >> (NS - k));
                ulonglong2 w = tw(tidx);
                gs_bfly(x[r], x[r + half], w.x, w.y, m.q, two_q);
            }
        }
#ifdef EDL_STAGE_FENCE
        asm volatile("" ::: "memory");
#endif
    }
}
template <int SA, int NS, bool LAST, bool FP>
__device__ __forceinline__ void inv_pass_regs(uint64_t* x, int high, const ModInfo& m, uint64_t two_q) {
    inv_pass_regs_t<SA, NS, LAST, FP>(x, high, m, two_q, glob_tw<FP>(m.tw_inv));
}

// A forward-transform epilogue may take the F64 path's outputs before canonicalisation:
// a Store with a member f64(idx, x, operand) receives x as the exact binary64 integer
// (|x| < 15 q, any residue class representative) and does its arithmetic on the FP64 pipe.
template <class L, class = void>
struct HasF64Load : std::false_type {};
template <class L>
struct HasF64Load<L, std::void_t<decltype(&L::f64)>> : std::true_type {};
template <class S, class = void>
struct HasF64Store : std::false_type {};
template <class S>
struct HasF64Store<S, std::void_t<decltype(&S::f64)>> : std::true_type {};

// In-CTA pass P over local stages [SL, SL+NS) of the M-point sub-block.
template <class C, int P>
struct PassInfo {
    static constexpr int SL = P * C::LOGE;
    static constexpr int NS = (SL + C::LOGE <= C::LOGM) ? C::LOGE : (C::LOGM - SL);
    static constexpr int SA = SL + C::LOGK;            // absolute stage (twiddle index)
    static constexpr int BTOP = C::LOGM - 1 - SL;
    static constexpr int BLOW = BTOP - NS + 1;
    static constexpr int G = C::E >> NS;              // groups per thread
};

// ---- barriers between in-CTA passes (round 2b) ------------------------------------------
// A pass reads and writes back exactly the same shared-memory words in every thread (each
// word belongs to one thread's group), so no barrier is needed between a pass's loads and
// its stores; only the next pass (or the epilogue / pass 0 layout, index tid + r T) reading
// words another thread wrote needs one -- and when every word a warp reads next was written
// by that same warp, __syncwarp suffices.  pass_warp_local<C, P, Q>() checks this for
// pass P followed by pass Q (Q = 0: the tid + r T layout) over all M words at compile time.
template <class C, int P>
__host__ __device__ constexpr int pass_word(int tid, int g, int r) {
    using PI = PassInfo<C, P>;
    const int v = tid + g * C::T;
    const int low = v & ((1 << PI::BLOW) - 1);
    const int high = v >> PI::BLOW;
    return ((high << (PI::BTOP + 1)) | low) + (r << PI::BLOW);
}
template <class C, int P, int Q>
__host__ __device__ constexpr bool pass_warp_local() {
    using PP = PassInfo<C, P>;
    using PQ = PassInfo<C, Q>;
    short owner[C::M] = {};
    for (int tid = 0; tid < C::T; tid++)
        for (int g = 0; g < PP::G; g++)
            for (int r = 0; r < (1 << PP::NS); r++) owner[pass_word<C, P>(tid, g, r)] = (short)(tid >> 5);
    for (int tid = 0; tid < C::T; tid++)
        for (int g = 0; g < PQ::G; g++)
            for (int r = 0; r < (1 << PQ::NS); r++)
                if (owner[pass_word<C, Q>(tid, g, r)] != (short)(tid >> 5)) return false;
    return true;
}
#ifndef EDL_PASS_SYNC_FULL
#define EDL_PASS_SYNC_LEAN 1
#endif
// barrier after pass P's stores, before pass Q's loads
template <class C, int P, int Q>
__device__ __forceinline__ void pass_barrier() {
#ifdef EDL_PASS_SYNC_LEAN
    if constexpr (pass_warp_local<C, P, Q>()) __syncwarp();
    else __syncthreads();
#else
    __syncthreads();
#endif
}
// barrier between a pass's loads and its stores (same words per thread: not needed)
__device__ __forceinline__ void pass_inner_barrier() {
#ifndef EDL_PASS_SYNC_LEAN
    __syncthreads();
#endif
}

template <class C, int P, bool INV, bool FP>
__device__ __forceinline__ void pass_smem(uint64_t* sm, const ModInfo& m, uint64_t two_q) {
    using PI = PassInfo<C, P>;
    constexpr int QN = INV ? (P > 1 ? P - 1 : 0) : (P + 1 < C::NPASS ? P + 1 : 0);   // next reader layout
    uint64_t x[C::E];
#pragma unroll
    for (int g = 0; g < PI::G; g++) {
        const int v = threadIdx.x + g * C::T;
        const int low = v & ((1 << PI::BLOW) - 1);
        const int high = v >> PI::BLOW;
        const int base = (high << (PI::BTOP + 1)) | low;
#pragma unroll
        for (int r = 0; r < (1 << PI::NS); r++) x[g * (1 << PI::NS) + r] = sm[spad(base) + spad(r << PI::BLOW)];
    }
    pass_inner_barrier();
    const int hc = C::crank() << PI::SL;
#pragma unroll
    for (int g = 0; g < PI::G; g++) {
        const int v = threadIdx.x + g * C::T;
        const int high = hc | (v >> PI::BLOW);
        if constexpr (INV) inv_pass_regs<PI::SA, PI::NS, false, FP>(x + g * (1 << PI::NS), high, m, two_q);
        else fwd_pass_regs<PI::SA, PI::NS, FP>(x + g * (1 << PI::NS), high, m.tw_fwd, m.q, two_q, u52_to_double(m.q), m.qinv_d);
    }
#pragma unroll
    for (int g = 0; g < PI::G; g++) {
        const int v = threadIdx.x + g * C::T;
        const int low = v & ((1 << PI::BLOW) - 1);
        const int high = v >> PI::BLOW;
        const int base = (high << (PI::BTOP + 1)) | low;
#pragma unroll
        for (int r = 0; r < (1 << PI::NS); r++) sm[spad(base) + spad(r << PI::BLOW)] = x[g * (1 << PI::NS) + r];
    }
    pass_barrier<C, P, QN>();
}

// ---- F64 path: twiddles of the next pass prefetched across the barrier ------------------
// ncu (round 2, plain 2^14 NTT on 40-bit primes): the DMUL of a butterfly waiting on its
// twiddle's global load (L2: the twiddle tables do not stay in L1) was the largest single
// stall (11-14 % of samples).  A pass with one group per thread (G == 1) uses 2^NS - 1
// distinct twiddles per thread -- stage k, group position r -> entry (2^k - 1) + (r >> (NS-k))
// -- and they do not depend on the data, so they are loaded right after the previous pass's
// shared-memory stores (its residues are dead then: the registers are free) and arrive
// while the CTA waits at the barrier.
// Measured (B200, round 2): inverse 40-bit transforms +9 %; forward: plain transforms and the
// modulus raise -1..4 %, the kernels with an epilogue operand (rescale, mod-down: CfgEpi) gain
// (mod-down NTT 0.565 -> 0.538 ms per C1 step; ptxas: its spills 224 -> 28 bytes), so the
// forward prefetch is a per-configuration choice (NttCfg::TW_PF_FWD).
#ifndef EDL_NO_TW_PREFETCH
#define EDL_TW_PREFETCH_INV 1
#endif
// Round 2c: with the prefetch's loads vectorised (EDL_TW_VEC: stage k's 2^k twiddles are consecutive
// and 2^k-aligned in the table, so 8 loads of <= 16 bytes replace 15 of 8) the forward prefetch
// wins everywhere: 40-bit plain NTT 1197 -> 1258 Gbfly/s forward, 1092 -> 1174 inverse; modulus
// raise 0.894 -> 0.888 ms; C1 3.970 -> 3.945 ms.  EDL_TW_VEC=0 / EDL_TW_PREFETCH_FWD=0 restore.
#ifndef EDL_TW_PREFETCH_FWD
#define EDL_TW_PREFETCH_FWD 1   // 1: every forward transform; 0: per configuration (NttCfg::TW_PF_FWD)
#endif
#ifndef EDL_TW_VEC
#define EDL_TW_VEC 1
#endif
template <class C, int P>
struct TwPre {
    static constexpr bool OK = (P >= 1 && P < C::NPASS && PassInfo<C, P>::G == 1);
    static constexpr int NW = (1 << C::LOGE) - 1;   // any pass's count (one buffer serves every pass)
};
template <class C, int P, bool INV>
__device__ __forceinline__ void tw_prefetch(double* w, const ModInfo& m) {
    using PI = PassInfo<C, P>;
    const int high = (C::crank() << PI::SL) | ((int)threadIdx.x >> PI::BLOW);
    const uint64_t* __restrict__ t = reinterpret_cast<const uint64_t*>(INV ? m.tw_inv : m.tw_fwd);
#if EDL_TW_VEC   // stage k's 2^k twiddles are consecutive and 2^k-aligned: 16-byte loads for k >= 1
    w[0] = f64_of(__ldg(t + (1 << PI::SA) + high));
#pragma unroll
    for (int k = 1; k < PI::NS; k++)
#pragma unroll
        for (int j = 0; j < (1 << k); j += 2) {
            const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(t + (1 << (PI::SA + k)) + (high << k) + j));
            w[(1 << k) - 1 + j] = f64_of(v.x);
            w[(1 << k) + j] = f64_of(v.y);
        }
#else
#pragma unroll
    for (int k = 0; k < PI::NS; k++)
#pragma unroll
        for (int j = 0; j < (1 << k); j++) w[(1 << k) - 1 + j] = f64_of(__ldg(t + (1 << (PI::SA + k)) + (high << k) + j));
#endif
}
// One G == 1 pass on the F64 path with its twiddles in w; on return w holds pass PN's
// twiddles when TwPre<C, PN>::OK (prefetched between the stores and the closing barrier).
template <class C, int P, bool INV, int PN>
__device__ __forceinline__ void pass_smem_pre(uint64_t* sm, const ModInfo& m, double* w) {
    using PI = PassInfo<C, P>;
    static_assert(PI::G == 1, "one group per thread");
    constexpr int NS = PI::NS;
    const double qd = u52_to_double(m.q), qinv = m.qinv_d;
    uint64_t x[1 << NS];
    const int base = ((threadIdx.x >> PI::BLOW) << (PI::BTOP + 1)) | (threadIdx.x & ((1 << PI::BLOW) - 1));
#pragma unroll
    for (int r = 0; r < (1 << NS); r++) x[r] = sm[spad(base) + spad(r << PI::BLOW)];
    pass_inner_barrier();
    if constexpr (!INV) {
#pragma unroll
        for (int k = 0; k < NS; k++) {
            const int half = 1 << (NS - 1 - k);
#pragma unroll
            for (int r = 0; r < (1 << NS); r++) {
                if (r & half) continue;
                const double wv = w[(1 << k) - 1 + (r >> (NS - k))];
                const double a = f64_of(x[r]);
                const double t = f64_mult(f64_of(x[r + half]), wv, qd, qinv);
                x[r] = bits_of(__dadd_rn(a, t));
                x[r + half] = bits_of(__dsub_rn(a, t));
            }
        }
    } else {
#pragma unroll
        for (int k = NS - 1; k >= 0; k--) {
            const int half = 1 << (NS - 1 - k);
#pragma unroll
            for (int r = 0; r < (1 << NS); r++) {
                if (r & half) continue;
                const double wv = w[(1 << k) - 1 + (r >> (NS - k))];
                const double a = f64_of(x[r]), b = f64_of(x[r + half]);
                double sum = __dadd_rn(a, b);
                if (k == 0) sum = f64_reduce(sum, qd, qinv);
                x[r] = bits_of(sum);
                x[r + half] = bits_of(f64_mult(__dsub_rn(a, b), wv, qd, qinv));
            }
        }
    }
#pragma unroll
    for (int r = 0; r < (1 << NS); r++) sm[spad(base) + spad(r << PI::BLOW)] = x[r];
    if constexpr (TwPre<C, PN>::OK) tw_prefetch<C, PN, INV>(w, m);
    constexpr int QN = (PN >= 1 && PN < C::NPASS) ? PN : 0;   // next reader layout (0: tid + r T)
    pass_barrier<C, P, QN>();
}
// F64 forward passes P.. with prefetched twiddles (w holds pass P's when HAVE).
template <class C, int P, bool HAVE>
__device__ __forceinline__ void fwd_middle_pre(uint64_t* sm, const ModInfo& m, double* w) {
    if constexpr (P < C::NPASS) {
        if constexpr (TwPre<C, P>::OK) {
            if constexpr (!HAVE) tw_prefetch<C, P, false>(w, m);
            pass_smem_pre<C, P, false, P + 1>(sm, m, w);
            fwd_middle_pre<C, P + 1, TwPre<C, P + 1>::OK>(sm, m, w);
        } else {
            pass_smem<C, P, false, true>(sm, m, 2 * m.q);
            fwd_middle_pre<C, P + 1, false>(sm, m, w);
        }
    }
}
template <class C, int P, bool HAVE>
__device__ __forceinline__ void inv_middle_pre(uint64_t* sm, const ModInfo& m, double* w) {
    if constexpr (P > 0) {
        if constexpr (TwPre<C, P>::OK) {
            if constexpr (!HAVE) tw_prefetch<C, P, true>(w, m);
            pass_smem_pre<C, P, true, P - 1>(sm, m, w);
            inv_middle_pre<C, P - 1, TwPre<C, P - 1>::OK>(sm, m, w);
        } else {
            pass_smem<C, P, true, true>(sm, m, 2 * m.q);
            inv_middle_pre<C, P - 1, false>(sm, m, w);
        }
    }
}

template <class C, int P, bool FP>
__device__ __forceinline__ void fwd_middle(uint64_t* sm, const ModInfo& m, uint64_t two_q) {
    if constexpr (P < C::NPASS) {
        pass_smem<C, P, false, FP>(sm, m, two_q);
        fwd_middle<C, P + 1, FP>(sm, m, two_q);
    }
}

template <class C, int P, bool FP>
__device__ __forceinline__ void inv_middle(uint64_t* sm, const ModInfo& m, uint64_t two_q) {
    if constexpr (P > 0) {
        pass_smem<C, P, true, FP>(sm, m, two_q);
        inv_middle<C, P - 1, FP>(sm, m, two_q);
    }
}

// Epilogue operand base[idx] loaded for all E outputs before the first store ...
struct PreLoad {
    const uint64_t* base;
    __device__ __forceinline__ uint64_t operator()(int idx) const { return base[idx]; }
};
// ... or copied into shared memory (stage[r T + tid] for output C::idx(r)) by cp.async at
// the transform's start, so the copy overlaps every butterfly and holds no registers.
struct PreStaged {
    const uint64_t* base;
    uint64_t* stage;
    __device__ __forceinline__ uint64_t operator()(int) const { return 0; }
};

// Forward NTT of one limb.  load(idx) -> residue in [0, 4q); store(idx, v) receives
// canonical values at idx = C::idx(r).
template <class C, bool FP, class Load, class Pre, class Store>
__device__ __forceinline__ void ntt_fwd_impl(uint64_t* sm, const ModInfo& m, Load load, Pre pre, Store store) {
    using P0 = PassInfo<C, 0>;
    static_assert(P0::G == 1 && P0::BLOW == C::LOGM - C::LOGE, "pass 0 layout");
    const uint64_t q = m.q, two_q = 2 * q;
    const double qd = FP ? u52_to_double(q) : 0.0;
    const int tid = threadIdx.x;
    constexpr bool STAGED = std::is_same<Pre, PreStaged>::value;
    if constexpr (STAGED) {   // epilogue operands -> shared memory, in flight during the transform
#pragma unroll
        for (int r = 0; r < C::E; r++)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(pre.stage + r * C::T + tid)),
                         "l"(pre.base + C::idx(r))
                         : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    __shared__ alignas(8) uint64_t xchg_mbar;
    const uint32_t mb = smem_u32(&xchg_mbar);
    (void)mb;
    // F64 path: the loaded residues (< 4q) become exact binary64 integers
    // (a Load with a member f64(idx) hands the F64 path its prologue's result directly as
    //  an exact binary64 integer of magnitude < 4q, any residue class representative)
    auto ld = [&](int idx) {
        if constexpr (FP && HasF64Load<Load>::value) {
            return bits_of(load.f64(idx));
        } else {
            const uint64_t v = load(idx);
            if constexpr (FP) return f64_from_u(v);
            else return v;
        }
    };
    uint64_t x[C::E];
    if constexpr (C::K == 1) {
#pragma unroll
        for (int r = 0; r < C::E; r++) x[r] = ld(tid + r * C::T);
    } else {
#ifdef EDL_XCHG_ASYNC
        if (tid == 0) mbar_init_cluster(mb);
#endif
#ifndef EDL_FULL_CLUSTER_SYNC
        cluster_arrive_relaxed();   // shared memory free: kernel start or past the caller's last __syncthreads
#endif
        // phase A: columns j (this CTA's M/K of them) x all K sub-blocks, stages 0..logK-1
        const int j0 = C::crank() * (C::M / C::K) + tid;
#pragma unroll
        for (int g = 0; g < C::E / C::K; g++) {
#pragma unroll
            for (int t = 0; t < C::K; t++) x[g * C::K + t] = ld(j0 + g * C::T + t * C::M);
            fwd_pass_regs<0, C::LOGK, FP>(x + g * C::K, 0, m.tw_fwd, q, two_q, qd, m.qinv_d);
        }
#ifndef EDL_FULL_CLUSTER_SYNC
        cluster_wait();       // every CTA is running and done with its shared memory
#else
        cluster_sync_all();
#endif
#ifdef EDL_XCHG_ASYNC
#ifdef EDL_XCHG_SELF
        // the CTA's own chunk also travels by st.async, so the mbarrier counts every word of
        // the sub-block and no CTA barrier is needed before reading it
        if (tid == 0) mbar_expect(mb, (uint32_t)(C::M * 8));
#pragma unroll
        for (int t = 0; t < C::K; t++) {
            const uint32_t rb = mapa_u32(mb, t);
            const uint32_t rs = mapa_u32(smem_u32(sm), t);
#pragma unroll
            for (int g = 0; g < C::E / C::K; g++) st_async_b64(rs + 8u * (spad(j0) + spad(g * C::T)), x[g * C::K + t], rb);
        }
#else
        if (tid == 0) mbar_expect(mb, (uint32_t)((C::K - 1) * (C::M / C::K) * 8));
#pragma unroll
        for (int t = 0; t < C::K; t++) {
            if (t == C::crank()) {
#pragma unroll
                for (int g = 0; g < C::E / C::K; g++) sm[spad(j0) + spad(g * C::T)] = x[g * C::K + t];
            } else {
                const uint32_t rb = mapa_u32(mb, t);
                const uint32_t rs = mapa_u32(smem_u32(sm), t);
#pragma unroll
                for (int g = 0; g < C::E / C::K; g++) st_async_b64(rs + 8u * (spad(j0) + spad(g * C::T)), x[g * C::K + t], rb);
            }
        }
        __syncthreads();
#endif
        mbar_wait0(mb);
#else
#pragma unroll
        for (int t = 0; t < C::K; t++) {
            uint64_t* dst = cluster_smem<C>(sm, t);
#pragma unroll
            for (int g = 0; g < C::E / C::K; g++) dst[spad(j0) + spad(g * C::T)] = x[g * C::K + t];
        }
        cluster_sync_all();
#endif
#pragma unroll
        for (int r = 0; r < C::E; r++) x[r] = sm[spad(tid) + spad(r * C::T)];
    }
    fwd_pass_regs<C::LOGK, C::LOGE, FP>(x, C::crank(), m.tw_fwd, q, two_q, qd, m.qinv_d);
#pragma unroll
    for (int r = 0; r < C::E; r++) sm[spad(tid) + spad(r * C::T)] = x[r];
#ifdef EDL_TW_PREFETCH_INV
    if constexpr (FP && (C::TW_PF_FWD || EDL_TW_PREFETCH_FWD)) {
        double w[TwPre<C, 1>::NW];
        if constexpr (TwPre<C, 1>::OK) tw_prefetch<C, 1, false>(w, m);
        __syncthreads();
        fwd_middle_pre<C, 1, TwPre<C, 1>::OK>(sm, m, w);
    } else
#endif
    {
        __syncthreads();
        fwd_middle<C, 1, FP>(sm, m, two_q);
    }
    // epilogue operands first (all E loads in flight, or the staged copies), then the outputs
    using PT = decltype(pre(0));
    PT pv[C::E];
    if constexpr (STAGED) {
        asm volatile("cp.async.wait_all;" ::: "memory");   // this thread's own copies
    } else {
#pragma unroll
        for (int r = 0; r < C::E; r++) pv[r] = pre(C::idx(r));
    }
#pragma unroll
    for (int r = 0; r < C::E; r++) {
        if constexpr (STAGED) pv[r] = pre.stage[r * C::T + tid];
        uint64_t v = sm[spad(tid) + spad(r * C::T)];
        if constexpr (FP && HasF64Store<Store>::value) {
            store.f64(C::idx(r), f64_of(v), pv[r]);
        } else {
            if constexpr (FP) v = f64_to_canon(f64_reduce(f64_of(v), qd, m.qinv_d), qd);
            else v = canon_fwd(v, q);
            store(C::idx(r), v, pv[r]);
        }
    }
    __syncthreads();   // smem reusable by the caller's next transform
#ifdef EDL_XCHG_ASYNC
    if (C::K > 1 && tid == 0) mbar_inval(mb);
#endif
}

// Inverse NTT of one limb.  load(idx) at idx = C::idx(r) -> residue in [0, 2q);
// store(idx, canonical value).
template <class C, bool FP, class Load, class Pre, class Store>
__device__ __forceinline__ void ntt_inv_impl(uint64_t* sm, const ModInfo& m, Load load, Pre pre, Store store) {
    const uint64_t q = m.q, two_q = 2 * q;
    const double qd = FP ? u52_to_double(q) : 0.0;
    const int tid = threadIdx.x;
    __shared__ alignas(8) uint64_t xchg_mbar;
    const uint32_t mb = smem_u32(&xchg_mbar);
    (void)mb;
    // F64 path: residues (< 2q) in as exact binary64 integers, canonical uint64 out
    auto canon = [&](uint64_t v) {
        if constexpr (FP) return f64_to_canon(f64_of(v), qd);
        else return canon_inv(v, q);
    };
    // outputs: canonical uint64, or (F64 path, Store with f64()) the binary64 value, |.| <= 0.625 q
    auto put = [&](int idx, uint64_t v, auto pvv) {
        if constexpr (FP && HasF64Store<Store>::value) store.f64(idx, f64_of(v), pvv);
        else store(idx, canon(v), pvv);
    };
    {
        // every load of the thread first, then the shared-memory stores: interleaved, a store
        // (generic pointer: possible alias of the load's source) would pin each next load
        // behind the previous one's full latency
        uint64_t t[C::E];
#pragma unroll
        for (int r = 0; r < C::E; r++) {
            if constexpr (FP && HasF64Load<Load>::value) t[r] = bits_of(load.f64(C::idx(r)));   // |.| < 2q
            else t[r] = load(C::idx(r));
        }
#pragma unroll
        for (int r = 0; r < C::E; r++) {
            if constexpr (FP && !HasF64Load<Load>::value) sm[spad(tid) + spad(r * C::T)] = f64_from_u(t[r]);
            else sm[spad(tid) + spad(r * C::T)] = t[r];
        }
    }
#ifdef EDL_TW_PREFETCH_INV
    if constexpr (FP) {
        constexpr int P1 = C::NPASS - 1;
        double w[TwPre<C, P1>::NW];
        if constexpr (TwPre<C, P1>::OK) tw_prefetch<C, P1, true>(w, m);
        __syncthreads();
        inv_middle_pre<C, P1, TwPre<C, P1>::OK>(sm, m, w);
    } else
#endif
    {
        __syncthreads();
        inv_middle<C, C::NPASS - 1, FP>(sm, m, two_q);
    }
    uint64_t x[C::E];
#pragma unroll
    for (int r = 0; r < C::E; r++) x[r] = sm[spad(tid) + spad(r * C::T)];
    inv_pass_regs<C::LOGK, C::LOGE, C::K == 1, FP>(x, C::crank(), m, two_q);
    using PT = decltype(pre(0));
    PT pv[C::E];
    if constexpr (C::K == 1) {
#pragma unroll
        for (int r = 0; r < C::E; r++) pv[r] = pre(tid + r * C::T);
#pragma unroll
        for (int r = 0; r < C::E; r++) put(tid + r * C::T, x[r], pv[r]);
        __syncthreads();
    } else {
        constexpr int MK = C::M / C::K;
#if defined(EDL_INV_RELAXED) || defined(EDL_XCHG_ASYNC)
#ifndef EDL_INV_NOSYNC_ARRIVE
        __syncthreads();      // this CTA's reads of its sub-block are performed
#endif
        // (EDL_INV_NOSYNC_ARRIVE: every thread arrives after its own reads -- the cluster
        //  barrier completes only when all threads of all CTAs have arrived; EDL_XCHG_SELF: the
        //  own chunk by st.async too, no CTA barrier before reading: both measured slower on
        //  B200, round 2b: 40-bit INTT 1085 -> 950 Gbfly/s together)
#ifdef EDL_XCHG_ASYNC
        if (tid == 0) mbar_init_cluster(mb);
#endif
        cluster_arrive_relaxed();
        cluster_wait();       // ... and every peer's
#else
        cluster_sync_all();   // every CTA has read its sub-block out of shared memory
#endif
#ifdef EDL_XCHG_ASYNC
#ifdef EDL_XCHG_SELF
        if (tid == 0) mbar_expect(mb, (uint32_t)(C::K * MK * 8));   // own chunk by st.async too
#else
        if (tid == 0) mbar_expect(mb, (uint32_t)((C::K - 1) * MK * 8));
#endif
        const uint32_t rs0 = smem_u32(sm);
#pragma unroll
        for (int r = 0; r < C::E; r++) {
            const int j = tid + r * C::T;
            const int t = r / (C::E / C::K);   // == j / MK (T divides MK)
            const int w = spad(C::crank() * MK) + spad(tid) + spad((r * C::T) & (MK - 1));   // disjoint parts of crank MK + (j mod MK)
#ifdef EDL_XCHG_SELF
            st_async_b64(mapa_u32(rs0, t) + 8u * w, x[r], mapa_u32(mb, t));
#else
            if (t == C::crank()) sm[w] = x[r];
            else st_async_b64(mapa_u32(rs0, t) + 8u * w, x[r], mapa_u32(mb, t));
#endif
        }
#ifndef EDL_XCHG_SELF
        __syncthreads();
#endif
        mbar_wait0(mb);
#else
#pragma unroll
        for (int r = 0; r < C::E; r++) {
            const int j = tid + r * C::T;
            cluster_smem<C>(sm, j / MK)[spad(C::crank() * MK + (j & (MK - 1)))] = x[r];
        }
        cluster_sync_all();
#endif
        // phase A': columns j x all K sub-blocks, stages logK-1..0 (N^-1 folded in)
        const int j0 = C::crank() * MK + tid;
#pragma unroll
        for (int g = 0; g < C::E / C::K; g++)
#pragma unroll
            for (int t = 0; t < C::K; t++) pv[g * C::K + t] = pre(j0 + g * C::T + t * C::M);
#pragma unroll
        for (int g = 0; g < C::E / C::K; g++) {
#pragma unroll
            for (int t = 0; t < C::K; t++) x[g * C::K + t] = sm[spad(t * MK) + spad(tid) + spad(g * C::T)];
            inv_pass_regs<0, C::LOGK, true, FP>(x + g * C::K, 0, m, two_q);
#pragma unroll
            for (int t = 0; t < C::K; t++) put(j0 + g * C::T + t * C::M, x[g * C::K + t], pv[g * C::K + t]);
        }
        __syncthreads();
#ifdef EDL_XCHG_ASYNC
        if (tid == 0) mbar_inval(mb);
#endif
    }
}

// Public entry points: the butterfly path is uniform per limb (ModInfo::fp == 2: F64,
// else Shoup), so the branch is uniform across the CTA.
// Epilogues come in two flavours: store(idx, v) or, with an operand fetcher,
// pre(idx) -> operand (issued for all E outputs of a thread before the first store, so
// the operand loads overlap) and store(idx, v, operand).
struct NoPre {
    __device__ __forceinline__ int operator()(int) const { return 0; }
};

template <class C, class Load, class Pre, class Store>
__device__ __forceinline__ void ntt_fwd(uint64_t* sm, const ModInfo& m, Load load, Pre pre, Store store) {
#ifndef EDL_NO_FP_QUOTIENT
    if (m.fp == 2) ntt_fwd_impl<C, true>(sm, m, load, pre, store);
    else
#endif
        ntt_fwd_impl<C, false>(sm, m, load, pre, store);
}

template <class C, class Load, class Store>
__device__ __forceinline__ void ntt_fwd(uint64_t* sm, const ModInfo& m, Load load, Store store) {
    auto st3 = [&](int idx, uint64_t v, int) { store(idx, v); };
    ntt_fwd<C>(sm, m, load, NoPre(), st3);
}

template <class C, class Load, class Pre, class Store>
__device__ __forceinline__ void ntt_inv(uint64_t* sm, const ModInfo& m, Load load, Pre pre, Store store) {
#ifndef EDL_NO_FP_QUOTIENT
    if (m.fp == 2) ntt_inv_impl<C, true>(sm, m, load, pre, store);
    else
#endif
        ntt_inv_impl<C, false>(sm, m, load, pre, store);
}

template <class C, class Load, class Store>
__device__ __forceinline__ void ntt_inv(uint64_t* sm, const ModInfo& m, Load load, Store store) {
    auto st3 = [&](int idx, uint64_t v, int) { store(idx, v); };
    ntt_inv<C>(sm, m, load, NoPre(), st3);
}

// ---- per-N configurations -------------------------------------------------------------
// M = N/K <= 2^13 per CTA.  Plain transforms keep E = 32 residues per thread (fewer
// exchanges); fused kernels, whose prologue/epilogue need registers, pick their own E.
// Measured on B200 (tools/ntt_bench.py, C1 step): the plain transform at N = 2^14 is
// fastest as one 1024-thread CTA x 16 residues (5.42 M limbs/s; 5.3 as a 2-CTA cluster of
// 256 x 32, 4.7 as one 512 x 32 CTA); the fused kernels are fastest as
// 2-CTA clusters of 512 threads x 16 residues with two CTAs per SM (64 registers, 32 warps
// per SM): 6.76 ms/step vs 6.92 (one 1024-thread CTA per limb), 7.50 (128 registers, one
// CTA per SM) and 8.87 (512 threads x 32 residues).  Latency hiding needs the warps more
// than the spill-free register budget.
#ifndef EDL_K14_PLAIN
#define EDL_K14_PLAIN 1
#endif
#ifndef EDL_K14_FUSED
#define EDL_K14_FUSED 4   // fused kernels at 2^14: 4-CTA clusters x 256 threads x 16 residues, 4 CTAs/SM
#endif
#ifndef EDL_LOGE_P14
#define EDL_LOGE_P14 4
#endif
#ifndef EDL_LOGE_F14
#define EDL_LOGE_F14 4
#endif
#ifndef EDL_LOGE_F13
#define EDL_LOGE_F13 4
#endif

__host__ __device__ constexpr int cfg_logk(int logn, bool plain) {
    return logn <= 13 ? 0
                      : (logn == 14 ? ((plain ? EDL_K14_PLAIN : EDL_K14_FUSED) == 4 ? 2 : ((plain ? EDL_K14_PLAIN : EDL_K14_FUSED) == 2 ? 1 : 0))
                                    : logn - 13);
}
__host__ __device__ constexpr int cfg_logm(int logn, bool plain) { return logn - cfg_logk(logn, plain); }
__host__ __device__ constexpr int cfg_loge(int logn, bool plain) {
    return cfg_logm(logn, plain) == 14 ? (plain ? EDL_LOGE_P14 : EDL_LOGE_F14)
                                       : (cfg_logm(logn, plain) >= 12 ? (plain ? 5 : EDL_LOGE_F13)
                                                                      : (cfg_logm(logn, plain) >= 10 ? 4 : 3));
}
// blocks per SM for __launch_bounds__.  Plain transforms: as many CTAs as leave 128
// registers per thread.  Fused kernels: 1024 threads per SM (64 registers), at most 4 CTAs.
// A whole 2^14 limb per CTA (136 KiB of shared memory) always runs one CTA.
__host__ __device__ constexpr int cfg_minb(int logm, int loge) {
    return logm == 14 ? 1
                      : ((65536 >> (logm - loge + 7)) < 1 ? 1 : ((65536 >> (logm - loge + 7)) > 3 ? 3 : (65536 >> (logm - loge + 7))));
}
// (8-CTA clusters, N = 2^16, keep 128 registers and one CTA per SM: with 64 registers the
// keygen kernels died with illegal-instruction / illegal-address errors on B200.)
__host__ __device__ constexpr int cfg_minb_fused(int logm, int loge, int logk = 0) {
    return (logm == 14 || logk >= 3) ? 1
                                     : ((1024 >> (logm - loge)) < 1 ? 1 : ((1024 >> (logm - loge)) > 4 ? 4 : (1024 >> (logm - loge))));
}

#ifndef EDL_MINB_F
#define EDL_MINB_F 0
#endif
template <int LOGN, bool PLAIN>
using CfgOf = NttCfg<LOGN, cfg_logk(LOGN, PLAIN), cfg_loge(LOGN, PLAIN),
                     PLAIN ? cfg_minb(cfg_logm(LOGN, PLAIN), cfg_loge(LOGN, PLAIN))
                           : (EDL_MINB_F > 0 ? EDL_MINB_F
                                             : cfg_minb_fused(cfg_logm(LOGN, PLAIN), cfg_loge(LOGN, PLAIN), cfg_logk(LOGN, PLAIN)))>;
template <int LOGN, int LOGE>   // fused config with an explicit residues-per-thread
using CfgFusedE = NttCfg<LOGN, cfg_logk(LOGN, false), LOGE, cfg_minb_fused(cfg_logm(LOGN, false), LOGE, cfg_logk(LOGN, false))>;
#ifndef EDL_LOGE_KS14
#define EDL_LOGE_KS14 EDL_LOGE_F14
#endif
template <int LOGN>   // key-switch MAC kernel (largest epilogue)
using CfgKs = CfgFusedE<LOGN, cfg_logm(LOGN, false) == 14 ? EDL_LOGE_KS14 : cfg_loge(LOGN, false)>;
template <int LOGN>
using CfgPlain = CfgOf<LOGN, true>;
// Batched plain transforms (k_ntt_limbs): at 2^14 the fused kernels' 4-CTA clusters of
// 256 threads x 16 residues, 4 CTAs/SM (round 2, after the st.async exchange and the inverse
// twiddle prefetch: 8.65 / 8.18 M limb-transforms/s forward / inverse on the C1 chain against
// 8.50 / 7.50 for round 1's 2-CTA clusters of 512 x 16; 48 registers and 5 CTAs/SM: equal
// forward, slower integer inverse); below 2^14 the fused config.
#ifndef EDL_PLAIN14_MINB
#define EDL_PLAIN14_MINB 4
#endif
template <int LOGN>
using CfgNttLimbs = typename std::conditional<
    (LOGN == 14), NttCfg<14, 2, 4, EDL_PLAIN14_MINB>,
    typename std::conditional<(LOGN < 14), CfgOf<LOGN, false>, CfgOf<LOGN, true>>::type>::type;
template <int LOGN>
using CfgFused = CfgOf<LOGN, false>;
// Forward transforms with an epilogue operand: optionally (EDL_STAGE_EPI) at 2^14 the fused
// configuration with the operand staged in shared memory (34 + 32 KB per CTA: 3 CTAs per
// SM, 80 registers, no spills) -- measured 12 % slower than 4 CTAs per SM with the operand
// in registers, so off by default.
#ifdef EDL_STAGE_EPI   // measured slower (C1: rescale_ntt 0.93 vs 0.83 ms): occupancy beats latency here
template <int LOGN>
using CfgEpi = typename std::conditional<(LOGN == 14 && cfg_logk(14, false) == 2), NttCfg<14, 2, 4, 3, true>,
                                         CfgFused<LOGN>>::type;
#else
template <class C>
using WithTwPf = NttCfg<C::LOGN, C::LOGK, C::LOGE, C::MINB, C::STAGE_EPI, true>;
template <int LOGN>
using CfgEpi = WithTwPf<CfgFused<LOGN>>;
#endif

}  // namespace edl
