// ntt_kernels.cu -- NTT-based kernels of the hot path (
// K1/K2/K5/K6).  Each CTA transforms whole limbs with ntt_core.cuh and fuses the
// surrounding pointwise work into the transform's prologue/epilogue, so every rescale
// and key-switch touches HBM once per input and once per output limb.
#pragma once
#include <type_traits>
#include "kernels.cuh"
#include "ntt_core.cuh"
#include "ntt_persist.cuh"

namespace edl {


// Grid order of the per-(ciphertext, polynomial, output limb) forward transforms whose
// prologue reads a per-(ciphertext, polynomial) limb once per output limb (rescale's r,
// mod-down's r and s): launch order walks groups of EDL_L2_GROUP ciphertexts, and inside a
// group output limb -> polynomial -> ciphertext, so a group's r / s limbs (G x 2 x 128 KB
// at 2^14) are re-read from L2 for every output limb instead of from HBM; co-resident
// clusters still share one output limb (one prime) at a time.  EDL_L2_GROUP = 0 restores
// the plain (ct fastest, limb slowest) order.
// Measured (C1, B200): the mod-down's two re-read limbs gain (0.62 -> 0.58 ms at G = 32),
// rescale's single one loses (0.84 -> 0.86), so only k_relin_moddown_ntt uses it.
#ifndef EDL_L2_GROUP
#define EDL_L2_GROUP 32
#endif
template <class C, int G = EDL_L2_GROUP>
__device__ __forceinline__ void grid_ct_p_i(int64_t& c, int& p, int& i) {
    const int64_t cnt = gridDim.x >> C::LOGK;
    if (G <= 0 || cnt <= G) {
        c = C::bx();
        p = blockIdx.y;
        i = blockIdx.z;
        return;
    }
    const int P2 = gridDim.y, NL = gridDim.z;
    const int64_t lin = (int64_t)C::bx() + cnt * (blockIdx.y + (int64_t)P2 * blockIdx.z);
    const int64_t per = (int64_t)G * P2 * NL;
    const int64_t g = lin / per;
    const int64_t rem = lin - g * per;
    const int64_t gg = (cnt - g * G) < G ? (cnt - g * G) : G;
    i = (int)(rem / (gg * P2));
    const int64_t r2 = rem - (int64_t)i * gg * P2;
    p = (int)(r2 / gg);
    c = g * G + (r2 - (int64_t)p * gg);
}

// Epilogue operand of a forward transform at the output indices (a limb laid out like the
// output): at N = 2^14 it is copied into shared memory by cp.async at the kernel's start
// (PreStaged, ntt_core.cuh: overlapped with the whole transform, no registers held), which
// needs M extra words of shared memory per CTA and runs 3 CTAs per SM (CfgEpi); elsewhere
// it is loaded for all E outputs before the first store (the round-1 form).
template <class C>
__device__ __forceinline__ auto epi_pre(const uint64_t* base, uint64_t* sm) {
    if constexpr (C::STAGE_EPI) return PreStaged{base, sm + C::SMEM_WORDS};
    else return PreLoad{base};
}

// ------------------------------------------------------------------------------------
// K1/K2: plain batched NTT / INTT, in place, data [batch][nl][N], limb j uses pm.idx[j].
template <class C, bool INV>
__global__ void __launch_bounds__(C::T, C::MINB)
k_ntt_limbs(uint64_t* __restrict__ data, int nl, const __grid_constant__ PrimeMap pm, const __grid_constant__ ModTable mods) {
    EDL_PDL_ENTRY();
    extern __shared__ uint64_t sm[];
    const int limb = blockIdx.y;    // limb-major grid: co-resident CTAs share a prime (code path, twiddles)
    uint64_t* p = data + (((size_t)C::bx() * nl + limb) << C::LOGN);
    if (threadIdx.x == 0)
        pf_next_wave<C>([&](int64_t bx, int cr, int y, int) { pf_sub<C>(data + (((size_t)bx * nl + y) << C::LOGN), cr, !INV); });
    const ModInfo& m = mods[pm.idx[limb]];
    auto ld = [&](int idx) { return p[idx]; };
    auto st = [&](int idx, uint64_t v) { p[idx] = v; };
    if constexpr (INV) ntt_inv<C>(sm, m, ld, st);
    else ntt_fwd<C>(sm, m, ld, st);
}

// Persistent variant (ntt_persist.cuh): items = (limb j, batch b), prime-major, item
// cl + k * nclusters for cluster cl; the next item's residues are fetched into registers
// before the current item's butterflies.
template <class C, bool INV>
__global__ void __launch_bounds__(C::T, C::MINB)
k_ntt_limbs_p(uint64_t* __restrict__ data, int64_t batch, int nl, const __grid_constant__ PrimeMap pm,
              const __grid_constant__ ModTable mods) {
    EDL_PDL_ENTRY();
    extern __shared__ __align__(16) uint64_t sm[];
    ulonglong2* tws = reinterpret_cast<ulonglong2*>(sm + C::SMEM_WORDS);
    __shared__ alignas(8) uint64_t mbar;
    const uint32_t mb = smem_u32(&mbar);
    const int64_t nitems = batch * nl;
    const int64_t ncl = gridDim.x >> C::LOGK;
    const int tid = threadIdx.x;
    auto fetch = [&](int64_t item, uint64_t* dst) {
        const int limb = (int)(item / batch);
        const int64_t b = item - (int64_t)limb * batch;
        const uint64_t* p = data + (((size_t)b * nl + limb) << C::LOGN);
        if constexpr (!INV) {
            const int j0 = C::crank() * (C::M / C::K) + tid;
#pragma unroll
            for (int g = 0; g < C::E / C::K; g++)
#pragma unroll
                for (int t = 0; t < C::K; t++) dst[g * C::K + t] = p[j0 + g * C::T + t * C::M];
        } else {
#pragma unroll
            for (int r = 0; r < C::E; r++) dst[r] = p[C::idx(r)];
        }
    };
    uint64_t xn[C::E];
    int cur = -1;
    int64_t item = C::bx();
    if (item < nitems) fetch(item, xn);
    for (; item < nitems; item += ncl) {
        const int limb = (int)(item / batch);
        const int64_t b = item - (int64_t)limb * batch;
        const int pi = pm.idx[limb];
        const ModInfo& m = mods[pi];
        uint64_t x[C::E];
#pragma unroll
        for (int r = 0; r < C::E; r++) x[r] = xn[r];
        if (item + ncl < nitems) fetch(item + ncl, xn);
        if (pi != cur) {   // uniform: the whole cluster works on one item
            __syncthreads();
            load_tw_smem<C>(tws, INV ? m.tw_inv : m.tw_fwd, m.fp == 2);
            __syncthreads();
            cur = pi;
        }
        uint64_t* p = data + (((size_t)b * nl + limb) << C::LOGN);
        auto st = [&](int idx, uint64_t v) { p[idx] = v; };
        if constexpr (!INV) item_open(mb);
#ifndef EDL_P_ONLY_INT
        if (m.fp == 2) {
#else
        if (false) {
#endif
#pragma unroll
            for (int r = 0; r < C::E; r++) x[r] = f64_from_u(x[r]);
            if constexpr (INV) pinv<C, true>(sm, m, tws, x, mb, st);
            else pfwd<C, true>(sm, m, tws, x, mb, st);
        } else {
#ifndef EDL_P_ONLY_FP
            if constexpr (INV) pinv<C, false>(sm, m, tws, x, mb, st);
            else pfwd<C, false>(sm, m, tws, x, mb, st);
#endif
        }
    }
}

// ------------------------------------------------------------------------------------
// K6 rescale, step 1 (O12): r = INTT_{q_l}(c[l] * w_l) for both polys of every ct.  With a
// second constant w2 the same INTT also yields r2 = INTT(c[l] * w2_l) (INTT is linear),
// which the sigma schedule uses for its two scalar products of y (O13 steps 2 and 4).
template <class C>
__global__ void __launch_bounds__(C::T, C::MINB)
k_rescale_intt(const uint64_t* __restrict__ in, int l, const ulonglong2* __restrict__ w,
               uint64_t* __restrict__ r_out, const ulonglong2* __restrict__ w2, uint64_t* __restrict__ r_out2,
               const __grid_constant__ ModTable mods) {
    EDL_PDL_ENTRY();
    extern __shared__ uint64_t sm[];
    const int p = blockIdx.y;
    const int64_t c = C::bx();
    const uint64_t* src = in + limb_off(c, p, l, l + 1, C::LOGN);
    uint64_t* dst = r_out + (((size_t)c * 2 + p) << C::LOGN);
    uint64_t* dst2 = r_out2 ? r_out2 + (((size_t)c * 2 + p) << C::LOGN) : nullptr;
    const ModInfo& m = mods[l];
    if (threadIdx.x == 0)
        pf_next_wave<C>([&](int64_t bx, int cr, int y, int) { pf_sub<C>(in + limb_off(bx, y, l, l + 1, C::LOGN), cr, false); });
    if (w2 == nullptr) {
        const bool has_w = (w != nullptr);
        ulonglong2 wl = has_w ? w[c * (l + 1) + l] : make_ulonglong2(1, 0);
        auto ld = [&](int idx) { return has_w ? mulc_lazy(src[idx], wl, m) : src[idx]; };
        auto st = [&](int idx, uint64_t v) { dst[idx] = v; };
        ntt_inv<C>(sm, m, ld, st);
    } else {
        const ulonglong2 wa = w[c * (l + 1) + l], wb = w2[c * (l + 1) + l];
        auto ld = [&](int idx) { return src[idx]; };
        struct Store {   // two scalar products of the INTT; F64 limbs on the FP64 pipe
            uint64_t *dst, *dst2;
            ulonglong2 wa, wb;
            const ModInfo& m;
            __device__ __forceinline__ void operator()(int idx, uint64_t v, int) const {
                dst[idx] = mulc(v, wa, m);
                dst2[idx] = mulc(v, wb, m);
            }
            __device__ __forceinline__ void f64(int idx, double v, int) const {
                const double qd = u52_to_double(m.q);
                dst[idx] = f64_to_canon(f64_mulc(v, u52_to_double(wa.x), f64_of(wa.y), qd), qd);
                dst2[idx] = f64_to_canon(f64_mulc(v, u52_to_double(wb.x), f64_of(wb.y), qd), qd);
            }
        };
        ntt_inv<C>(sm, m, ld, NoPre(), Store{dst, dst2, wa, wb, m});
    }
}

// K6 rescale, step 2: out_i = (c_i w_i - NTT_i([r]_{q_l} mod q_i)) q_l^{-1} (+ bias_i).
template <class C>
__global__ void __launch_bounds__(C::T, C::MINB)
k_rescale_ntt(const uint64_t* __restrict__ in, int l, const ulonglong2* __restrict__ w,
              const uint64_t* __restrict__ r, const uint64_t* __restrict__ bias, uint64_t* __restrict__ out, int nlo,
              const __grid_constant__ ModTable mods, const ChainConsts* __restrict__ cc) {
    EDL_PDL_ENTRY();
    extern __shared__ uint64_t sm[];
    int64_t c;
    int p, i;
    grid_ct_p_i<C, 0>(c, p, i);
    const ModInfo& m = mods[i];
    const uint64_t ql = mods[l].q;
    const uint64_t ql_mod = cc->qmod[l][i];
    const ulonglong2 qlinv = cc->qinv[l][i];
    const uint64_t* rr = r + (((size_t)c * 2 + p) << C::LOGN);
    const uint64_t* src = in + limb_off(c, p, i, l + 1, C::LOGN);
    uint64_t* dst = out + limb_off(c, p, i, nlo, C::LOGN);
    const bool has_w = (w != nullptr);
    const ulonglong2 wi = has_w ? w[c * (l + 1) + i] : make_ulonglong2(1, 0);
    const uint64_t b = (bias != nullptr && p == 0) ? bias[c * l + i] : 0;
    if (threadIdx.x == 0) {
        pf_own<C>(src);
        pf_next_wave<C>([&](int64_t bx, int cr, int y, int) { pf_sub<C>(r + (((size_t)bx * 2 + y) << C::LOGN), cr, true); });
    }
    auto ld = [&](int idx) { return center_mod(rr[idx], ql, ql_mod, m); };
    const auto pre = epi_pre<C>(src, sm);
    // out = (a w_i - x) q_l^-1 + b: integer path on canonical x, or (F64 limbs) on the
    // transform's unreduced binary64 output with exact FP64-pipe products
    struct Store {
        uint64_t* dst;
        const ModInfo& m;
        bool has_w;
        ulonglong2 wi, qlinv;
        uint64_t b;
        __device__ __forceinline__ void operator()(int idx, uint64_t x, uint64_t a) const {
            if (has_w) a = mulc(a, wi, m);
            uint64_t v = mulc(submod(a, x, m.q), qlinv, m);
            dst[idx] = addmod(v, b, m.q);
        }
        __device__ __forceinline__ void f64(int idx, double x, uint64_t a) const {
            const double qd = u52_to_double(m.q);
            double ad = u52_to_double(a);
            if (has_w) ad = f64_mulc(ad, u52_to_double(wi.x), f64_of(wi.y), qd);
            const double v = f64_mulc(__dsub_rn(ad, x), u52_to_double(qlinv.x), f64_of(qlinv.y), qd);
            dst[idx] = f64_to_canon(f64_reduce(__dadd_rn(v, u52_to_double(b)), qd, m.qinv_d), qd);
        }
    };
    ntt_fwd<C>(sm, m, ld, pre, Store{dst, m, has_w, wi, qlinv, b});
}

// ------------------------------------------------------------------------------------
// K5 relinearisation (O11) of the tensor product d = a (x) b at level l, in 4 launches:
//   M1 acoef_j = INTT_{q_j}(a1_j b1_j)                                   [cnt][l+1]
//   M2a xh_{j,t} = NTT_t(acoef_j mod t), t != q_j                        [cnt][l+1][l+2]
//   M2b acc_{c,t} = sum_j xh_{j,t} * rlk_j[c][t]  (t = q_0..q_l, P; the t == q_j term
//      uses d2_j = a1_j b1_j directly); for data limbs the same pass stores
//      v_{c,i} = d_{c,i} + acc_{c,i} P^-1 (the tensor's d0, d1 folded in)  [cnt][2][l+2]
//   M3 r_c = INTT_P(acc_{c,P}); if rescaling also
//      s_c = INTT_{q_l}(v_{c,l}) - [r_c]_{q_l} P^-1  (= INTT of the relinearised limb l,
//      by linearity)                                                       [cnt][2]
//   M4 out_{c,i} = v_{c,i} - NTT_i([r_c]_{q_i} P^-1)                         (no rescale)
//      out_{c,i} = (v_{c,i} - NTT_i([r_c]_{q_i} P^-1 + [s_c]_{q_i})) q_l^-1
//      which is bit-identical to mod-down followed by O12 rescale (all steps are exact
//      Z_q-linear maps of the same centered lifts).
template <class C>
__global__ void __launch_bounds__(C::T, C::MINB)
k_relin_intt_d2(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b, int l,
                uint64_t* __restrict__ acoef, const __grid_constant__ ModTable mods) {
    EDL_PDL_ENTRY();
    extern __shared__ uint64_t sm[];
    const int j = blockIdx.y;
    const int64_t c = C::bx();
    const ModInfo& m = mods[j];
    const uint64_t* a1 = a + limb_off(c, 1, j, l + 1, C::LOGN);
    // b == null: key switch of the single polynomial a1 (Galois rotation, NEXT f1)
    const uint64_t* b1 = b ? b + limb_off(c, 1, j, l + 1, C::LOGN) : a1;
    const bool single = (b == nullptr);
    uint64_t* dst = acoef + (((size_t)c * (l + 1) + j) << C::LOGN);
    struct Load {   // d2 = a1 b1 (or a1); F64 limbs: the exact product on the FP64 pipe, |.| <= 0.51 q
        const uint64_t *a1, *b1;
        bool single;
        const ModInfo& m;
        __device__ __forceinline__ uint64_t operator()(int idx) const {
            return single ? a1[idx] : mulmod(a1[idx], b1[idx], m);
        }
        __device__ __forceinline__ double f64(int idx) const {
            const double x = u52_to_double(a1[idx]);
            if (single) return x;
            const double y = u52_to_double(b1[idx]), qd = u52_to_double(m.q);
            const double hi = __dmul_rn(x, y);
            const double lo = __fma_rn(x, y, -hi);
            const double qt = __dsub_rn(__fma_rn(hi, m.qinv_d, F64_RND), F64_RND);
            return __dadd_rn(__fma_rn(-qt, qd, hi), lo);
        }
    };
    if (threadIdx.x == 0)
        pf_next_wave<C>([&](int64_t bx, int cr, int y, int) {
            pf_sub<C>(a + limb_off(bx, 1, y, l + 1, C::LOGN), cr, false);
            if (b && b != a) pf_sub<C>(b + limb_off(bx, 1, y, l + 1, C::LOGN), cr, false);
        });
    auto st = [&](int idx, uint64_t v) { dst[idx] = v; };
    ntt_inv<C>(sm, m, Load{a1, b1, single, m}, st);
}

// M2a modulus raise: xh_{j,t} = NTT_t(acoef_j mod t) for every digit j and target t != j
// (t = q_0..q_l, P), one limb transform per CTA with no epilogue work, so it runs at the
// plain transform's rate; the key products are a separate streaming pass (M2b).
template <class C>
__global__ void __launch_bounds__(C::T, C::MINB)
k_relin_modup(const uint64_t* __restrict__ acoef, int l, int L, uint64_t* __restrict__ xh,
              const __grid_constant__ ModTable mods) {
    EDL_PDL_ENTRY();
    extern __shared__ uint64_t sm[];
    // y enumerates (target, digit) target-major: data targets ti = 0..l with the l digits
    // j != ti, then P (ti = l+1) with all l+1 digits, so co-resident CTAs (limb-major
    // grid) share one prime: one arithmetic path in the I-cache, one twiddle table
    int ti, j;
#ifndef EDL_MODUP_TARGET_MAJOR
    // digit-major: the l+1 targets of one digit are consecutive rows, so the digit limb is
    // re-read from L2
    j = blockIdx.y / (l + 1);
    {
        const int tt = blockIdx.y % (l + 1);
        ti = tt < j ? tt : tt + 1;
    }
#else
    if ((int)blockIdx.y < (l + 1) * l) {
        ti = blockIdx.y / l;
        const int jj = blockIdx.y % l;
        j = jj < ti ? jj : jj + 1;
    } else {
        ti = l + 1;
        j = blockIdx.y - (l + 1) * l;
    }
#endif
    const int t = (ti == l + 1) ? (L + 1) : ti;
    const int64_t c = C::bx();
    const ModInfo& m = mods[t];
    const uint64_t* src = acoef + (((size_t)c * (l + 1) + j) << C::LOGN);
    uint64_t* dst = xh + ((((size_t)c * (l + 1) + j) * (l + 2) + ti) << C::LOGN);
    const bool need_red = mods[j].q > 4 * m.q;   // the forward NTT accepts [0, 4q)
    if (threadIdx.x == 0)
        pf_next_wave<C>([&](int64_t bx, int cr, int y, int) {
            const int jn = y < (l + 1) * l ? ((y % l) < (y / l) ? (y % l) : (y % l) + 1) : y - (l + 1) * l;
            pf_sub<C>(acoef + (((size_t)bx * (l + 1) + jn) << C::LOGN), cr, true);
        });
    auto ld = [&](int idx) {
        uint64_t v = src[idx];
        return need_red ? reduce64(v, m) : v;
    };
    auto st = [&](int idx, uint64_t v) { dst[idx] = v; };
    ntt_fwd<C>(sm, m, ld, st);
}

// M2 fused (round 2): modulus raise and key products in ONE pass, target-major.  CTA
// (cluster) = (ciphertext c, target ti); for every digit j != ti it runs
// x_{j,t} = NTT_t(acoef_j mod t) and accumulates x_{j,t} rlk_j[cc][t] (cc = 0, 1) in its
// epilogue into accumulators the thread keeps in shared memory (its own E slots per
// component, no synchronisation); the raised digits never reach HBM.  After the digits,
// for data targets the t == j term d2_t rlk_t[cc][t] (d2 = a1 b1, NTT domain), the
// tensor's d0 = a0 b0, d1 = a0 b1 + a1 b0 and the P^-1 fold give v_cc = d_cc + acc_cc P^-1;
// for P the accumulators themselves are stored -- exactly k_relin_mac's output layout
// [cnt][2][l+2][N], so the mod-down kernels are unchanged.
// Arithmetic: F64 targets (q < 2^44) f64_mult products (no key companion) of the
// transform's unreduced binary64 outputs, summed exactly in binary64 (<= l+2 terms of
// |.| <= 0.63 q); other targets Shoup products with the key companion in [0, 2q) summed
// lazily in uint64 ((l + 2) 2 q < 2^64 for q < 2^60, l <= 5) and reduced once.
template <class C>
__global__ void __launch_bounds__(C::T, C::MINB)
k_relin_ks(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b, int l, int L,
           const uint64_t* __restrict__ acoef, const uint64_t* __restrict__ rlk, const uint64_t* __restrict__ rlk_c,
           uint64_t* __restrict__ acc_out, const __grid_constant__ ModTable mods, const ChainConsts* __restrict__ cc) {
    EDL_PDL_ENTRY();
    extern __shared__ __align__(16) uint64_t sm[];
    uint64_t* accs = sm + C::SMEM_WORDS;   // [2][E][T]: slot of output C::idx(r) = r T + tid
    const int ti = blockIdx.y;              // 0..l data targets, l+1 = P
    const int t = (ti == l + 1) ? (L + 1) : ti;
    const int64_t c = C::bx();
    const ModInfo& m = mods[t];
    const bool f64 = m.fp == 2;            // uniform per CTA
    const int tid = threadIdx.x;
    const size_t limb_n = (size_t)1 << C::LOGN;
#pragma unroll
    for (int r = 0; r < C::E; r++) {
        accs[r * C::T + tid] = 0;   // binary64 +0 and integer 0 share the bit pattern
        accs[(C::E + r) * C::T + tid] = 0;
    }
    const uint64_t qd_bits = bits_of(u52_to_double(m.q));
    for (int j = 0; j <= l; j++) {
        if (j == ti) continue;
        const uint64_t* src = acoef + (((size_t)c * (l + 1) + j) << C::LOGN);
        const uint64_t* k0 = rlk + ((((size_t)j * 2 + 0) * (L + 2) + t) << C::LOGN);
        const uint64_t* k1 = rlk + ((((size_t)j * 2 + 1) * (L + 2) + t) << C::LOGN);
        const uint64_t* k0c = rlk_c + ((((size_t)j * 2 + 0) * (L + 2) + t) << C::LOGN);
        const uint64_t* k1c = rlk_c + ((((size_t)j * 2 + 1) * (L + 2) + t) << C::LOGN);
        const bool need_red = mods[j].q > 4 * m.q;   // the forward NTT accepts [0, 4q)
        auto ld = [&](int idx) {
            uint64_t v = src[idx];
            return need_red ? reduce64(v, m) : v;
        };
        struct Store {
            uint64_t* accs;
            const uint64_t *k0, *k1, *k0c, *k1c;
            const ModInfo& m;
            uint64_t qd_bits;
            int base;
            __device__ __forceinline__ int slot(int idx) const { return idx - base; }   // r T + tid
            __device__ __forceinline__ void operator()(int idx, uint64_t x, int) const {   // Shoup targets
                const int s = slot(idx);
                const uint64_t p0 = shoup_lazy2(x, __ldg(k0 + idx), __ldg(k0c + idx), m.q);
                const uint64_t p1 = shoup_lazy2(x, __ldg(k1 + idx), __ldg(k1c + idx), m.q);
                accs[s] += p0;
                accs[C::E * C::T + s] += p1;
            }
            __device__ __forceinline__ void f64(int idx, double x, int) const {   // F64 targets
                const int s = slot(idx);
                const double qd = f64_of(qd_bits);
                const double p0 = f64_mult(x, u52_to_double(__ldg(k0 + idx)), qd, m.qinv_d);
                const double p1 = f64_mult(x, u52_to_double(__ldg(k1 + idx)), qd, m.qinv_d);
                accs[s] = bits_of(__dadd_rn(f64_of(accs[s]), p0));
                accs[C::E * C::T + s] = bits_of(__dadd_rn(f64_of(accs[C::E * C::T + s]), p1));
            }
        };
        ntt_fwd<C>(sm, m, ld, NoPre(), Store{accs, k0, k1, k0c, k1c, m, qd_bits, C::crank() * C::M});
    }
    // final: data targets add d2_t rlk_t (the j == t digit needs no transform) and fold the
    // tensor's d0, d1 with P^-1; P stores the reduced accumulators
    const double qd = u52_to_double(m.q);
    const ulonglong2 pinv = (ti <= l) ? cc->qinv[L + 1][t] : make_ulonglong2(0, 0);
    const bool single = (b == nullptr);
    uint64_t* o0 = acc_out + ((((size_t)c * 2 + 0) * (l + 2) + ti) << C::LOGN);
    uint64_t* o1 = acc_out + ((((size_t)c * 2 + 1) * (l + 2) + ti) << C::LOGN);
    const uint64_t* a0 = a + limb_off(c, 0, ti <= l ? ti : 0, l + 1, C::LOGN);
    const uint64_t* a1 = a + limb_off(c, 1, ti <= l ? ti : 0, l + 1, C::LOGN);
    const uint64_t* b0 = single ? a0 : b + limb_off(c, 0, ti <= l ? ti : 0, l + 1, C::LOGN);
    const uint64_t* b1 = single ? a1 : b + limb_off(c, 1, ti <= l ? ti : 0, l + 1, C::LOGN);
    const uint64_t* kt0 = rlk + ((((size_t)(ti <= l ? ti : 0) * 2 + 0) * (L + 2) + t) << C::LOGN);
    const uint64_t* kt1 = rlk + ((((size_t)(ti <= l ? ti : 0) * 2 + 1) * (L + 2) + t) << C::LOGN);
    const uint64_t* kt0c = rlk_c + ((((size_t)(ti <= l ? ti : 0) * 2 + 0) * (L + 2) + t) << C::LOGN);
    const uint64_t* kt1c = rlk_c + ((((size_t)(ti <= l ? ti : 0) * 2 + 1) * (L + 2) + t) << C::LOGN);
    (void)limb_n;
#pragma unroll 4
    for (int r = 0; r < C::E; r++) {
        const int idx = C::idx(r);
        const uint64_t s0 = accs[r * C::T + tid], s1 = accs[(C::E + r) * C::T + tid];
        uint64_t v0, v1;
        if (ti > l) {   // P: reduced accumulators
            if (f64) {
                v0 = f64_to_canon(f64_reduce(f64_of(s0), qd, m.qinv_d), qd);
                v1 = f64_to_canon(f64_reduce(f64_of(s1), qd, m.qinv_d), qd);
            } else {
                v0 = reduce64(s0, m);
                v1 = reduce64(s1, m);
            }
        } else {
            const uint64_t x0 = __ldg(a0 + idx), x1 = __ldg(a1 + idx);
            const uint64_t y0 = single ? x0 : __ldg(b0 + idx), y1 = single ? x1 : __ldg(b1 + idx);
            const uint64_t d2 = single ? x1 : mulmod(x1, y1, m);
            uint64_t d0 = x0, d1 = 0;
            if (!single) {
                d0 = mulmod(x0, y0, m);
                d1 = addmod(mulmod(x0, y1, m), mulmod(x1, y0, m), m.q);
            }
            uint64_t e0, e1;
            if (f64) {
                const double dd = u52_to_double(d2);
                const double t0 = __dadd_rn(f64_of(s0), f64_mult(dd, u52_to_double(__ldg(kt0 + idx)), qd, m.qinv_d));
                const double t1 = __dadd_rn(f64_of(s1), f64_mult(dd, u52_to_double(__ldg(kt1 + idx)), qd, m.qinv_d));
                e0 = f64_to_canon(f64_reduce(t0, qd, m.qinv_d), qd);
                e1 = f64_to_canon(f64_reduce(t1, qd, m.qinv_d), qd);
            } else {
                e0 = reduce64(s0 + shoup_lazy2(d2, __ldg(kt0 + idx), __ldg(kt0c + idx), m.q), m);
                e1 = reduce64(s1 + shoup_lazy2(d2, __ldg(kt1 + idx), __ldg(kt1c + idx), m.q), m);
            }
            v0 = addmod(d0, mulc(e0, pinv, m), m.q);
            v1 = addmod(d1, mulc(e1, pinv, m), m.q);
        }
        o0[idx] = v0;
        o1[idx] = v1;
    }
}

// M1 + M2a fused (round 2, EDL_RAISE_FUSED=1): CTA (cluster) = (ciphertext c, digit j).
// a_j = INTT_{q_j}(a1_j b1_j), kept in a shared-memory copy (thread-private slots: the
// inverse's output indices of a thread are exactly the forward transform's phase-A input
// indices of the same thread), then x_{j,t} = NTT_t(a_j mod t) for every target t != j
// (t = q_0..q_l, P): the digit never round-trips through HBM and no transform waits on a
// global load of it.
template <class C>
__device__ __forceinline__ int raise_slot(int idx) {   // register slot (g K + t) of coefficient idx
    const int t = idx >> C::LOGM;
    const int g = ((idx & (C::M - 1)) - (C::crank() * (C::M / C::K) + (int)threadIdx.x)) / C::T;
    return g * C::K + t;
}

template <class C>
__global__ void __launch_bounds__(C::T, C::MINB)
k_relin_raise(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b, int l, int L, uint64_t* __restrict__ xh,
              const __grid_constant__ ModTable mods) {
    EDL_PDL_ENTRY();
    static_assert(C::K > 1, "cluster configuration");
    extern __shared__ __align__(16) uint64_t sm[];
    uint64_t* dig = sm + C::SMEM_WORDS;   // [E][T]
    const int j = blockIdx.y;
    const int64_t c = C::bx();
    const int tid = threadIdx.x;
    {
        const ModInfo& m = mods[j];
        const uint64_t* a1 = a + limb_off(c, 1, j, l + 1, C::LOGN);
        const uint64_t* b1 = b ? b + limb_off(c, 1, j, l + 1, C::LOGN) : a1;
        const bool single = (b == nullptr);
        struct Load {   // d2 = a1 b1 (or a1); F64 limbs: the exact product on the FP64 pipe
            const uint64_t *a1, *b1;
            bool single;
            const ModInfo& m;
            __device__ __forceinline__ uint64_t operator()(int idx) const {
                return single ? a1[idx] : mulmod(a1[idx], b1[idx], m);
            }
            __device__ __forceinline__ double f64(int idx) const {
                const double x = u52_to_double(a1[idx]);
                if (single) return x;
                const double y = u52_to_double(b1[idx]), qd = u52_to_double(m.q);
                const double hi = __dmul_rn(x, y);
                const double lo = __fma_rn(x, y, -hi);
                const double qt = __dsub_rn(__fma_rn(hi, m.qinv_d, F64_RND), F64_RND);
                return __dadd_rn(__fma_rn(-qt, qd, hi), lo);
            }
        };
        auto st = [&](int idx, uint64_t v) { dig[raise_slot<C>(idx) * C::T + tid] = v; };
        ntt_inv<C>(sm, m, Load{a1, b1, single, m}, st);
    }
    const uint64_t qj = mods[j].q;
    for (int ti = 0; ti <= l + 1; ti++) {
        if (ti == j) continue;
        const int t = (ti == l + 1) ? (L + 1) : ti;
        const ModInfo& m = mods[t];
        const bool need_red = qj > 4 * m.q;   // the forward NTT accepts [0, 4q)
        uint64_t* dst = xh + ((((size_t)c * (l + 1) + j) * (l + 2) + ti) << C::LOGN);
        auto ld = [&](int idx) {
            const uint64_t v = dig[raise_slot<C>(idx) * C::T + tid];
            return need_red ? reduce64(v, m) : v;
        };
        auto st = [&](int idx, uint64_t v) { dst[idx] = v; };
        ntt_fwd<C>(sm, m, ld, st);
    }
}

// RESCALE is a template parameter (round 2): each instantiation compiles only its own
// transforms and epilogues, which halves the mod-down kernels' spills at 64 registers.
template <class C, bool RESCALE>
__global__ void __launch_bounds__(C::T, C::MINB)
k_relin_moddown_intt(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b, int l,
                     const uint64_t* __restrict__ acc, int L, int rescale_unused, uint64_t* __restrict__ r_out,
                     uint64_t* __restrict__ s_out, const __grid_constant__ ModTable mods,
                     const ChainConsts* __restrict__ cc) {
    EDL_PDL_ENTRY();
    extern __shared__ uint64_t sm[];
    const int cp = blockIdx.y;
    const int64_t c = C::bx();
    const ModInfo& mp = mods[L + 1];
    const uint64_t* accP = acc + ((((size_t)c * 2 + cp) * (l + 2) + (l + 1)) << C::LOGN);
    uint64_t* rdst = r_out + (((size_t)c * 2 + cp) << C::LOGN);
    constexpr bool rescale = RESCALE;
    (void)rescale_unused;
    if (threadIdx.x == 0) {
        if (rescale) pf_own<C>(acc + ((((size_t)c * 2 + cp) * (l + 2) + l) << C::LOGN));
        pf_next_wave<C>([&](int64_t bx, int cr, int y, int) {
            pf_sub<C>(acc + ((((size_t)bx * 2 + y) * (l + 2) + (l + 1)) << C::LOGN), cr, false);
        });
    }
    {
        auto ld = [&](int idx) { return accP[idx]; };
        auto st = [&](int idx, uint64_t v) { rdst[idx] = v; };
        ntt_inv<C>(sm, mp, ld, st);
    }
    if constexpr (!RESCALE) return;
    const ModInfo& ml = mods[l];
    const ulonglong2 pinv = cc->qinv[L + 1][l];
    const uint64_t pmod = cc->qmod[L + 1][l];
    const uint64_t* vl = acc + ((((size_t)c * 2 + cp) * (l + 2) + l) << C::LOGN);   // d_l + acc_l P^-1 (M2b)
    uint64_t* sdst = s_out + (((size_t)c * 2 + cp) << C::LOGN);
    auto ld = [&](int idx) { return vl[idx]; };
    auto pre = [&](int idx) { return rdst[idx]; };
    struct Store {   // s = y - [r] P^-1; F64 limbs: y unreduced (|y| <= 0.625 q), product on the FP64 pipe
        uint64_t* sdst;
        uint64_t Pq, pmod;
        ulonglong2 pinv;
        const ModInfo& ml;
        __device__ __forceinline__ void operator()(int idx, uint64_t y, uint64_t rv) const {
            uint64_t z = mulc(center_mod(rv, Pq, pmod, ml), pinv, ml);
            sdst[idx] = submod(y, z, ml.q);
        }
        __device__ __forceinline__ void f64(int idx, double y, uint64_t rv) const {
            const double qd = u52_to_double(ml.q);
            const double z = f64_mulc(u52_to_double(center_mod(rv, Pq, pmod, ml)), u52_to_double(pinv.x), f64_of(pinv.y), qd);
            sdst[idx] = f64_to_canon(f64_reduce(__dsub_rn(y, z), qd, ml.qinv_d), qd);
        }
    };
    ntt_inv<C>(sm, ml, ld, pre, Store{sdst, mp.q, pmod, pinv, ml});
}

template <class C, bool RESCALE>
__global__ void __launch_bounds__(C::T, C::MINB)
k_relin_moddown_ntt(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b, int l,
                    const uint64_t* __restrict__ acc, const uint64_t* __restrict__ r,
                    const uint64_t* __restrict__ s, int L, int rescale_unused, uint64_t* __restrict__ out,
                    const uint64_t* __restrict__ add_w, const uint64_t* __restrict__ add_k,
                    const __grid_constant__ ModTable mods, const ChainConsts* __restrict__ cc) {
    EDL_PDL_ENTRY();
    extern __shared__ uint64_t sm[];
    int64_t c;
    int cp, i;
    grid_ct_p_i<C>(c, cp, i);
    const ModInfo& m = mods[i];
    const uint64_t P = mods[L + 1].q;
    const uint64_t pmod = cc->qmod[L + 1][i];
    const ulonglong2 pinv = cc->qinv[L + 1][i];
    const uint64_t* rr = r + (((size_t)c * 2 + cp) << C::LOGN);
    const uint64_t* ss = s + (((size_t)c * 2 + cp) << C::LOGN);
    const uint64_t* vi = acc + ((((size_t)c * 2 + cp) * (l + 2) + i) << C::LOGN);   // d_i + acc_i P^-1 (M2b)
    constexpr bool rescale = RESCALE;
    (void)rescale_unused;
    const int nlo = rescale ? l : l + 1;
    uint64_t* dst = out + limb_off(c, cp, i, nlo, C::LOGN);
    if (threadIdx.x == 0) {   // epilogue operand of this CTA, prologue inputs of the next wave
        pf_own<C>(vi);
        pf_next_wave<C>([&](int64_t bx, int cr, int y, int) {
            pf_sub<C>(r + (((size_t)bx * 2 + y) << C::LOGN), cr, true);
            if (rescale) pf_sub<C>(s + (((size_t)bx * 2 + y) << C::LOGN), cr, true);
        });
    }
    if constexpr (RESCALE) {
        const uint64_t ql = mods[l].q;
        const uint64_t qlmod = cc->qmod[l][i];
        const ulonglong2 qlinv = cc->qinv[l][i];
        struct Load {   // [r] P^-1 + [s]; F64 limbs: the product on the FP64 pipe, |.| < 1.7 q
            const uint64_t *rr, *ss;
            uint64_t P, pmod, ql, qlmod;
            ulonglong2 pinv;
            const ModInfo& m;
            __device__ __forceinline__ uint64_t operator()(int idx) const {
                uint64_t u = mulc(center_mod(rr[idx], P, pmod, m), pinv, m);
                return addmod(u, center_mod(ss[idx], ql, qlmod, m), m.q);
            }
            __device__ __forceinline__ double f64(int idx) const {
                const double qd = u52_to_double(m.q);
                const double u = f64_mulc(u52_to_double(center_mod(rr[idx], P, pmod, m)), u52_to_double(pinv.x),
                                          f64_of(pinv.y), qd);
                return __dadd_rn(u, u52_to_double(center_mod(ss[idx], ql, qlmod, m)));
            }
        };
        const Load ld{rr, ss, P, pmod, ql, qlmod, pinv, m};
        // (v - x) q_l^-1 (+ w + k: a fused ciphertext + constant addend, e.g. sigma's output
        // assembly); F64 limbs: on the unreduced binary64 transform output.  Both epilogue
        // operands (v and w) are fetched for all E outputs before the first store (pre).
        const uint64_t* wl = add_w ? add_w + limb_off(c, cp, i, nlo, C::LOGN) : nullptr;
        const uint64_t kk = (add_k && cp == 0) ? add_k[c * nlo + i] : 0;
        struct Store {
            uint64_t* dst;
            const uint64_t* wl;
            uint64_t kk;
            const ModInfo& m;
            ulonglong2 qlinv;
            __device__ __forceinline__ void operator()(int idx, uint64_t x, uint64_t v) const {
                uint64_t y = mulc(submod(v, x, m.q), qlinv, m);
                if (wl) y = addmod(addmod(y, wl[idx], m.q), kk, m.q);
                dst[idx] = y;
            }
            __device__ __forceinline__ void f64(int idx, double x, uint64_t v) const {
                const double qd = u52_to_double(m.q);
                double t = f64_mulc(__dsub_rn(u52_to_double(v), x), u52_to_double(qlinv.x), f64_of(qlinv.y), qd);
                if (wl) {
                    t = __dadd_rn(t, u52_to_double(wl[idx]) + u52_to_double(kk));   // < 2.7 q: exact
                    t = f64_reduce(t, qd, m.qinv_d);
                }
                dst[idx] = f64_to_canon(t, qd);
            }
        };
        ntt_fwd<C>(sm, m, ld, epi_pre<C>(vi, sm), Store{dst, wl, kk, m, qlinv});
    } else {
        // out = d + (acc - NTT([r])) P^-1 = v - NTT([r] P^-1)  (Z_q-linear, exact)
        struct Load {   // [r] P^-1; F64 limbs: on the FP64 pipe, |.| <= 0.625 q
            const uint64_t* rr;
            uint64_t P, pmod;
            ulonglong2 pinv;
            const ModInfo& m;
            __device__ __forceinline__ uint64_t operator()(int idx) const {
                return mulc(center_mod(rr[idx], P, pmod, m), pinv, m);
            }
            __device__ __forceinline__ double f64(int idx) const {
                return f64_mulc(u52_to_double(center_mod(rr[idx], P, pmod, m)), u52_to_double(pinv.x), f64_of(pinv.y),
                                u52_to_double(m.q));
            }
        };
        const Load ld{rr, P, pmod, pinv, m};
        auto st = [&](int idx, uint64_t x, uint64_t v) { dst[idx] = submod(v, x, m.q); };
        ntt_fwd<C>(sm, m, ld, epi_pre<C>(vi, sm), st);
    }
}

template <int LOGN>
void launch_ntt_limbs_n(const Dev& d, uint64_t* data, int64_t batch, int nl, const PrimeMap& pm, bool inverse) {
#ifdef EDL_NTT_PERSIST
    if constexpr (LOGN == 14) {
        using CP = NttCfg<14, 2, 4, 2>;
        if (inverse) launch_persist<CP>(d, "k_ntt_limbs", k_ntt_limbs_p<CP, true>, batch * nl, data, batch, nl, pm, *d.mt);
        else launch_persist<CP>(d, "k_ntt_limbs", k_ntt_limbs_p<CP, false>, batch * nl, data, batch, nl, pm, *d.mt);
        return;
    }
#endif
    using C = CfgNttLimbs<LOGN>;   // (ntt_core.cuh: measured per degree)
    const dim3 grid((unsigned)batch, nl);
    if (inverse) launch_cfg<C>(d, "k_ntt_limbs", k_ntt_limbs<C, true>, grid, data, nl, pm, *d.mt);
    else launch_cfg<C>(d, "k_ntt_limbs", k_ntt_limbs<C, false>, grid, data, nl, pm, *d.mt);
}

template <int LOGN>
void launch_rescale_intt_n(const Dev& d, const uint64_t* in, int64_t cnt, int l, const ulonglong2* w, uint64_t* r_out,
                           const ulonglong2* w2, uint64_t* r_out2) {
    using C = CfgFused<LOGN>;
    launch_cfg<C>(d, "k_rescale_intt", k_rescale_intt<C>, dim3((unsigned)cnt, 2), in, l, w, r_out, w2, r_out2, *d.mt);
}

template <int LOGN>
void launch_rescale_ntt_n(const Dev& d, const uint64_t* in, int64_t cnt, int l, const ulonglong2* w, const uint64_t* r,
                          const uint64_t* bias, uint64_t* out, int nlo) {
    using C = CfgEpi<LOGN>;
    launch_cfg_x<C>(d, "k_rescale_ntt", k_rescale_ntt<C>, dim3((unsigned)cnt, 2, nlo), C::STAGE_EPI ? C::M * 8 : 0, in, l,
                    w, r, bias, out, nlo, *d.mt, d.cc);
}

template <int LOGN>
void launch_relin_n(const Dev& d, const uint64_t* a, const uint64_t* b, int64_t cnt, int l, bool rescale,
                    const uint64_t* rlk, const uint64_t* rlk_c, uint64_t* acoef, uint64_t* xh, uint64_t* acc, uint64_t* r,
                    uint64_t* s, uint64_t* out, const uint64_t* add_w, const uint64_t* add_k) {
    using C = CfgFused<LOGN>;
    // the modulus raise is a plain transform but runs fastest in the fused configuration
    // (2-CTA clusters of 512 threads, 2 CTAs/SM at 2^14): 1.22 vs 1.32 ms per C1 step
    using CP = CfgFused<LOGN>;
    const int rs = rescale ? 1 : 0;
    if (LOGN == 14 && d.raise_fused && !d.ks_fused) {
        using CR = NttCfg<14, 2, 4, 3>;   // 3 CTAs per SM: transform buffer + digit copy
        launch_cfg_x<CR>(d, "k_relin_raise", k_relin_raise<CR>, dim3((unsigned)cnt, l + 1), CR::M * 8, a, b, l, d.L, xh,
                         *d.mt);
        launch_relin_mac(d, a, b, cnt, l, xh, rlk, rlk_c, acc);
        launch_cfg<C>(d, "k_relin_moddown_intt", (rescale ? k_relin_moddown_intt<C, true> : k_relin_moddown_intt<C, false>), dim3((unsigned)cnt, 2), a, b, l,
                      (const uint64_t*)acc, d.L, rs, r, s, *d.mt, d.cc);
        launch_cfg<C>(d, "k_relin_moddown_ntt", (rescale ? k_relin_moddown_ntt<C, true> : k_relin_moddown_ntt<C, false>), dim3((unsigned)cnt, 2, rescale ? l : l + 1), a, b,
                      l, (const uint64_t*)acc, (const uint64_t*)r, (const uint64_t*)s, d.L, rs, out, add_w, add_k, *d.mt,
                      d.cc);
        (void)acoef;
        return;
    }
    launch_cfg<C>(d, "k_relin_intt_d2", k_relin_intt_d2<C>, dim3((unsigned)cnt, l + 1), a, b, l, acoef, *d.mt);
#ifndef EDL_NO_KS_FUSED
    if (LOGN == 14 && d.ks_fused) {
        // fused modulus raise + key products (k_relin_ks): 2 CTAs per SM, accumulators in smem
#ifndef EDL_KS_LOGE
#define EDL_KS_LOGE 3
#endif
        using CK = NttCfg<14, 2, EDL_KS_LOGE, 2>;   // 4-CTA clusters, 2 CTAs/SM (smem accumulators)
        launch_cfg_x<CK>(d, "k_relin_ks", k_relin_ks<CK>, dim3((unsigned)cnt, l + 2), 2 * CK::M * 8, a, b, l, d.L,
                         (const uint64_t*)acoef, rlk, rlk_c, acc, *d.mt, d.cc);
        (void)xh;
    } else
#endif
    {
        launch_cfg<CP>(d, "k_relin_modup", k_relin_modup<CP>, dim3((unsigned)cnt, (l + 1) * (l + 1)),
                       (const uint64_t*)acoef, l, d.L, xh, *d.mt);
        launch_relin_mac(d, a, b, cnt, l, xh, rlk, rlk_c, acc);   // acc slots 0..l hold v
    }
    launch_cfg<C>(d, "k_relin_moddown_intt", (rescale ? k_relin_moddown_intt<C, true> : k_relin_moddown_intt<C, false>),
                  dim3((unsigned)cnt, 2), a, b, l, (const uint64_t*)acc, d.L, rs, r, s, *d.mt, d.cc);
    using CE = CfgEpi<LOGN>;
    launch_cfg_x<CE>(d, "k_relin_moddown_ntt", (rescale ? k_relin_moddown_ntt<CE, true> : k_relin_moddown_ntt<CE, false>),
                     dim3((unsigned)cnt, 2, rescale ? l : l + 1),
                     CE::STAGE_EPI ? CE::M * 8 : 0, a, b, l, (const uint64_t*)acc, (const uint64_t*)r, (const uint64_t*)s,
                     d.L, rs, out, add_w, add_k, *d.mt, d.cc);
}

// Hoisted rotations (several Galois elements of the same ciphertexts): the modulus raise of
// c1 once (single-polynomial d2 INTT + modup) ...
template <int LOGN>
void launch_relin_raise_n(const Dev& d, const uint64_t* a, int64_t cnt, int l, uint64_t* acoef, uint64_t* xh) {
    using C = CfgFused<LOGN>;
    launch_cfg<C>(d, "k_relin_intt_d2", k_relin_intt_d2<C>, dim3((unsigned)cnt, l + 1), a, (const uint64_t*)nullptr, l,
                  acoef, *d.mt);
    launch_cfg<C>(d, "k_relin_modup", k_relin_modup<C>, dim3((unsigned)cnt, (l + 1) * (l + 1)), (const uint64_t*)acoef,
                  l, d.L, xh, *d.mt);
}

// ... then per element: key products of the (permuted) raised digits with d = (a0, 0) and
// the mod-down (no rescale), as in launch_relin_n's single-polynomial mode.
template <int LOGN>
void launch_relin_finish_n(const Dev& d, const uint64_t* a, int64_t cnt, int l, const uint64_t* rlk,
                           const uint64_t* rlk_c, uint64_t* xh, uint64_t* acc, uint64_t* r, uint64_t* s, uint64_t* out) {
    using C = CfgFused<LOGN>;
    const uint64_t* b = nullptr;
    launch_relin_mac(d, a, b, cnt, l, xh, rlk, rlk_c, acc);
    launch_cfg<C>(d, "k_relin_moddown_intt", k_relin_moddown_intt<C, false>, dim3((unsigned)cnt, 2), a, b, l,
                  (const uint64_t*)acc, d.L, 0, r, s, *d.mt, d.cc);
    using CE = CfgEpi<LOGN>;
    launch_cfg_x<CE>(d, "k_relin_moddown_ntt", k_relin_moddown_ntt<CE, false>, dim3((unsigned)cnt, 2, l + 1),
                     CE::STAGE_EPI ? CE::M * 8 : 0, a, b, l, (const uint64_t*)acc, (const uint64_t*)r, (const uint64_t*)s,
                     d.L, 0, out, b, b, *d.mt, d.cc);
}

#define EDL_INSTANTIATE_NTT(LOGN)                                                                                   \
    template void launch_ntt_limbs_n<LOGN>(const Dev&, uint64_t*, int64_t, int, const PrimeMap&, bool);            \
    template void launch_rescale_intt_n<LOGN>(const Dev&, const uint64_t*, int64_t, int, const ulonglong2*,         \
                                              uint64_t*, const ulonglong2*, uint64_t*);                             \
    template void launch_rescale_ntt_n<LOGN>(const Dev&, const uint64_t*, int64_t, int, const ulonglong2*,          \
                                             const uint64_t*, const uint64_t*, uint64_t*, int);                     \
    template void launch_relin_n<LOGN>(const Dev&, const uint64_t*, const uint64_t*, int64_t, int, bool,            \
                                       const uint64_t*, const uint64_t*, uint64_t*, uint64_t*, uint64_t*, uint64_t*, \
                                       uint64_t*, uint64_t*, const uint64_t*, const uint64_t*);                \
    template void launch_relin_raise_n<LOGN>(const Dev&, const uint64_t*, int64_t, int, uint64_t*, uint64_t*);     \
    template void launch_relin_finish_n<LOGN>(const Dev&, const uint64_t*, int64_t, int, const uint64_t*,          \
                                              const uint64_t*, uint64_t*, uint64_t*, uint64_t*, uint64_t*, uint64_t*);

}  // namespace edl
