// ntt_kernels.cu -- NTT-based kernels of the hot path (
// K1/K2/K5/K6).  Each CTA transforms whole limbs with ntt_core.cuh and fuses the
// surrounding pointwise work into the transform's prologue/epilogue, so every rescale
// and key-switch touches HBM once per input and once per output limb.
#include "kernels.cuh"
#include "ntt_core.cuh"

namespace edl {

struct PrimeMap {
    int8_t idx[MAXM];
};

// ------------------------------------------------------------------------------------
// K1/K2: plain batched NTT / INTT, in place, data [batch][nl][N], limb j uses pm.idx[j].
template <class C, bool INV>
__global__ void __launch_bounds__(C::T, C::MINB)
k_ntt_limbs(uint64_t* __restrict__ data, int nl, const __grid_constant__ PrimeMap pm, const ModInfo* __restrict__ mods) {
    extern __shared__ uint64_t sm[];
    const int limb = C::bx();
    uint64_t* p = data + (((size_t)blockIdx.y * nl + limb) << C::LOGN);
    const ModInfo m = mods[pm.idx[limb]];
    auto ld = [&](int idx) { return p[idx]; };
    auto st = [&](int idx, uint64_t v) { p[idx] = v; };
    if constexpr (INV) ntt_inv<C>(sm, m, ld, st);
    else ntt_fwd<C>(sm, m, ld, st);
}

// ------------------------------------------------------------------------------------
// K6 rescale, step 1 (O12): r = INTT_{q_l}(c[l] * w_l) for both polys of every ct.  With a
// second constant w2 the same INTT also yields r2 = INTT(c[l] * w2_l) (INTT is linear),
// which the sigma schedule uses for its two scalar products of y (O13 steps 2 and 4).
template <class C>
__global__ void __launch_bounds__(C::T, C::MINB)
k_rescale_intt(const uint64_t* __restrict__ in, int l, const ulonglong2* __restrict__ w,
               uint64_t* __restrict__ r_out, const ulonglong2* __restrict__ w2, uint64_t* __restrict__ r_out2,
               const ModInfo* __restrict__ mods) {
    extern __shared__ uint64_t sm[];
    const int p = C::bx();
    const int64_t c = blockIdx.y;
    const uint64_t* src = in + limb_off(c, p, l, l + 1, C::LOGN);
    uint64_t* dst = r_out + (((size_t)c * 2 + p) << C::LOGN);
    uint64_t* dst2 = r_out2 ? r_out2 + (((size_t)c * 2 + p) << C::LOGN) : nullptr;
    const ModInfo m = mods[l];
    if (w2 == nullptr) {
        const bool has_w = (w != nullptr);
        ulonglong2 wl = has_w ? w[c * (l + 1) + l] : make_ulonglong2(1, 0);
        auto ld = [&](int idx) { return has_w ? shoup_lazy2(src[idx], wl.x, wl.y, m.q) : src[idx]; };
        auto st = [&](int idx, uint64_t v) { dst[idx] = v; };
        ntt_inv<C>(sm, m, ld, st);
    } else {
        const ulonglong2 wa = w[c * (l + 1) + l], wb = w2[c * (l + 1) + l];
        auto ld = [&](int idx) { return src[idx]; };
        auto st = [&](int idx, uint64_t v) {
            dst[idx] = shoup(v, wa.x, wa.y, m.q);
            dst2[idx] = shoup(v, wb.x, wb.y, m.q);
        };
        ntt_inv<C>(sm, m, ld, st);
    }
}

// K6 rescale, step 2: out_i = (c_i w_i - NTT_i([r]_{q_l} mod q_i)) q_l^{-1} (+ bias_i).
template <class C>
__global__ void __launch_bounds__(C::T, C::MINB)
k_rescale_ntt(const uint64_t* __restrict__ in, int l, const ulonglong2* __restrict__ w,
              const uint64_t* __restrict__ r, const uint64_t* __restrict__ bias, uint64_t* __restrict__ out, int nlo,
              const ModInfo* __restrict__ mods, const ChainConsts* __restrict__ cc) {
    extern __shared__ uint64_t sm[];
    const int i = C::bx(), p = blockIdx.y;
    const int64_t c = blockIdx.z;
    const ModInfo m = mods[i];
    const uint64_t ql = mods[l].q;
    const uint64_t ql_mod = cc->qmod[l][i];
    const ulonglong2 qlinv = cc->qinv[l][i];
    const uint64_t* rr = r + (((size_t)c * 2 + p) << C::LOGN);
    const uint64_t* src = in + limb_off(c, p, i, l + 1, C::LOGN);
    uint64_t* dst = out + limb_off(c, p, i, nlo, C::LOGN);
    const bool has_w = (w != nullptr);
    const ulonglong2 wi = has_w ? w[c * (l + 1) + i] : make_ulonglong2(1, 0);
    const uint64_t b = (bias != nullptr && p == 0) ? bias[c * l + i] : 0;
    auto ld = [&](int idx) { return center_mod(rr[idx], ql, ql_mod, m); };
    auto st = [&](int idx, uint64_t x) {
        uint64_t a = src[idx];
        if (has_w) a = shoup(a, wi.x, wi.y, m.q);
        uint64_t v = shoup(submod(a, x, m.q) , qlinv.x, qlinv.y, m.q);
        dst[idx] = addmod(v, b, m.q);
    };
    ntt_fwd<C>(sm, m, ld, st);
}

// ------------------------------------------------------------------------------------
// K5 relinearisation (O11) of the tensor product d = a (x) b at level l, in 4 launches:
//   M1 acoef_j = INTT_{q_j}(a1_j b1_j)                                   [cnt][l+1]
//   M2 acc_{c,t} = sum_j NTT_t(acoef_j mod t) * rlk_j[c][t]  (t = q_0..q_l, P; the
//      t == q_j term reuses d2_j directly)                                [cnt][2][l+2]
//   M3 r_c = INTT_P(acc_{c,P}); if rescaling also
//      s_c = INTT_{q_l}(d_c,l + acc_{c,l} P^-1) - [r_c]_{q_l} P^-1  (= INTT of the
//      relinearised limb l, by linearity)                                 [cnt][2]
//   M4 out_{c,i} = d_c,i + (acc_{c,i} - NTT_i([r_c]_{q_i})) P^-1                 (no rescale)
//      out_{c,i} = (d_c,i + acc_{c,i} P^-1 - NTT_i([r_c]_{q_i} P^-1 + [s_c]_{q_i})) q_l^-1
//      which is bit-identical to mod-down followed by O12 rescale (all steps are exact
//      Z_q-linear maps of the same centered lifts).
__device__ __forceinline__ uint64_t tensor_comp(const uint64_t* a, const uint64_t* b, int64_t c, int cp, int i,
                                                int nl, int logn, int idx, const ModInfo& m) {
    const uint64_t a0 = a[limb_off(c, 0, i, nl, logn) + idx];
    const uint64_t b1 = b[limb_off(c, 1, i, nl, logn) + idx];
    const uint64_t b0 = b[limb_off(c, 0, i, nl, logn) + idx];
    if (cp == 0) return mulmod(a0, b0, m);
    const uint64_t a1 = a[limb_off(c, 1, i, nl, logn) + idx];
    U128 s = mul_wide(a0, b1);
    mac128(s, a1, b0);
    return barrett128(s, m);
}

template <class C>
__global__ void __launch_bounds__(C::T, C::MINB)
k_relin_intt_d2(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b, int l,
                uint64_t* __restrict__ acoef, const ModInfo* __restrict__ mods) {
    extern __shared__ uint64_t sm[];
    const int j = C::bx();
    const int64_t c = blockIdx.y;
    const ModInfo m = mods[j];
    const uint64_t* a1 = a + limb_off(c, 1, j, l + 1, C::LOGN);
    const uint64_t* b1 = b + limb_off(c, 1, j, l + 1, C::LOGN);
    uint64_t* dst = acoef + (((size_t)c * (l + 1) + j) << C::LOGN);
    auto ld = [&](int idx) { return mulmod(a1[idx], b1[idx], m); };
    auto st = [&](int idx, uint64_t v) { dst[idx] = v; };
    ntt_inv<C>(sm, m, ld, st);
}

template <class C>
__global__ void __launch_bounds__(C::T, C::MINB)
k_relin_ks_mac(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b, int l,
               const uint64_t* __restrict__ acoef, const uint64_t* __restrict__ rlk,
               const uint64_t* __restrict__ rlk_s, int L, uint64_t* __restrict__ acc,
               const ModInfo* __restrict__ mods) {
    extern __shared__ uint64_t sm[];
    const int ti = C::bx();                 // 0..l data targets, l+1 = P
    const int64_t c = blockIdx.y;
    const int t = (ti == l + 1) ? (L + 1) : ti;
    const ModInfo m = mods[t];
    uint64_t* acc0 = acc + ((((size_t)c * 2 + 0) * (l + 2) + ti) << C::LOGN);
    uint64_t* acc1 = acc + ((((size_t)c * 2 + 1) * (l + 2) + ti) << C::LOGN);
    for (int j = 0; j <= l; j++) {
        const size_t r0 = (((size_t)j * 2 + 0) * (L + 2) + t) << C::LOGN;
        const size_t r1 = (((size_t)j * 2 + 1) * (L + 2) + t) << C::LOGN;
        auto epi = [&](int idx, uint64_t x) {
            uint64_t p0 = shoup(x, rlk[r0 + idx], rlk_s[r0 + idx], m.q);
            uint64_t p1 = shoup(x, rlk[r1 + idx], rlk_s[r1 + idx], m.q);
            if (j == 0) {
                acc0[idx] = p0;
                acc1[idx] = p1;
            } else {
                acc0[idx] = addmod(acc0[idx], p0, m.q);
                acc1[idx] = addmod(acc1[idx], p1, m.q);
            }
        };
        if (ti == j) {
            const uint64_t* a1 = a + limb_off(c, 1, j, l + 1, C::LOGN);
            const uint64_t* b1 = b + limb_off(c, 1, j, l + 1, C::LOGN);
#pragma unroll 4
            for (int r = 0; r < C::E; r++) {
                const int idx = C::idx(r);
                epi(idx, mulmod(a1[idx], b1[idx], m));
            }
        } else {
            const uint64_t* src = acoef + (((size_t)c * (l + 1) + j) << C::LOGN);
            const bool need_red = mods[j].q > 4 * m.q;   // the forward NTT accepts [0, 4q)
            auto ld = [&](int idx) {
                uint64_t v = src[idx];
                return need_red ? reduce64(v, m) : v;
            };
            ntt_fwd<C>(sm, m, ld, epi);
        }
    }
}

template <class C>
__global__ void __launch_bounds__(C::T, C::MINB)
k_relin_moddown_intt(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b, int l,
                     const uint64_t* __restrict__ acc, int L, int rescale, uint64_t* __restrict__ r_out,
                     uint64_t* __restrict__ s_out, const ModInfo* __restrict__ mods,
                     const ChainConsts* __restrict__ cc) {
    extern __shared__ uint64_t sm[];
    const int cp = C::bx();
    const int64_t c = blockIdx.y;
    const ModInfo mp = mods[L + 1];
    const uint64_t* accP = acc + ((((size_t)c * 2 + cp) * (l + 2) + (l + 1)) << C::LOGN);
    uint64_t* rdst = r_out + (((size_t)c * 2 + cp) << C::LOGN);
    {
        auto ld = [&](int idx) { return accP[idx]; };
        auto st = [&](int idx, uint64_t v) { rdst[idx] = v; };
        ntt_inv<C>(sm, mp, ld, st);
    }
    if (!rescale) return;
    const ModInfo ml = mods[l];
    const ulonglong2 pinv = cc->qinv[L + 1][l];
    const uint64_t pmod = cc->qmod[L + 1][l];
    const uint64_t* accl = acc + ((((size_t)c * 2 + cp) * (l + 2) + l) << C::LOGN);
    uint64_t* sdst = s_out + (((size_t)c * 2 + cp) << C::LOGN);
    auto ld = [&](int idx) {
        uint64_t d = tensor_comp(a, b, c, cp, l, l + 1, C::LOGN, idx, ml);
        return addmod(d, shoup(accl[idx], pinv.x, pinv.y, ml.q), ml.q);
    };
    auto st = [&](int idx, uint64_t y) {
        uint64_t z = shoup(center_mod(rdst[idx], mp.q, pmod, ml), pinv.x, pinv.y, ml.q);
        sdst[idx] = submod(y, z, ml.q);
    };
    ntt_inv<C>(sm, ml, ld, st);
}

template <class C>
__global__ void __launch_bounds__(C::T, C::MINB)
k_relin_moddown_ntt(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b, int l,
                    const uint64_t* __restrict__ acc, const uint64_t* __restrict__ r,
                    const uint64_t* __restrict__ s, int L, int rescale, uint64_t* __restrict__ out,
                    const ModInfo* __restrict__ mods, const ChainConsts* __restrict__ cc) {
    extern __shared__ uint64_t sm[];
    const int i = C::bx(), cp = blockIdx.y;
    const int64_t c = blockIdx.z;
    const ModInfo m = mods[i];
    const uint64_t P = mods[L + 1].q;
    const uint64_t pmod = cc->qmod[L + 1][i];
    const ulonglong2 pinv = cc->qinv[L + 1][i];
    const uint64_t* rr = r + (((size_t)c * 2 + cp) << C::LOGN);
    const uint64_t* ss = s + (((size_t)c * 2 + cp) << C::LOGN);
    const uint64_t* acci = acc + ((((size_t)c * 2 + cp) * (l + 2) + i) << C::LOGN);
    const int nlo = rescale ? l : l + 1;
    uint64_t* dst = out + limb_off(c, cp, i, nlo, C::LOGN);
    if (rescale) {
        const uint64_t ql = mods[l].q;
        const uint64_t qlmod = cc->qmod[l][i];
        const ulonglong2 qlinv = cc->qinv[l][i];
        auto ld = [&](int idx) {
            uint64_t u = shoup(center_mod(rr[idx], P, pmod, m), pinv.x, pinv.y, m.q);
            return addmod(u, center_mod(ss[idx], ql, qlmod, m), m.q);
        };
        auto st = [&](int idx, uint64_t x) {
            uint64_t d = tensor_comp(a, b, c, cp, i, l + 1, C::LOGN, idx, m);
            uint64_t v = addmod(d, shoup(acci[idx], pinv.x, pinv.y, m.q), m.q);
            dst[idx] = shoup(submod(v, x, m.q), qlinv.x, qlinv.y, m.q);
        };
        ntt_fwd<C>(sm, m, ld, st);
    } else {
        auto ld = [&](int idx) { return center_mod(rr[idx], P, pmod, m); };
        auto st = [&](int idx, uint64_t x) {
            uint64_t d = tensor_comp(a, b, c, cp, i, l + 1, C::LOGN, idx, m);
            dst[idx] = addmod(d, shoup(submod(acci[idx], x, m.q), pinv.x, pinv.y, m.q), m.q);
        };
        ntt_fwd<C>(sm, m, ld, st);
    }
}

// ------------------------------------------------------------------------------------
// Host launchers.  Grids are [limb-like x K, ...]: the K CTAs of one limb form a cluster.
bool set_smem_attrs(int /*logn*/) { return true; }   // set lazily by launch_cfg

void launch_ntt_limbs(const Dev& d, uint64_t* data, int64_t batch, int nl, const int* prime_idx_host, bool inverse) {
    PrimeMap pm;
    for (int j = 0; j < nl && j < MAXM; j++) pm.idx[j] = (int8_t)prime_idx_host[j];
    EDL_DISPATCH_LOGN(d.logn, {
        using C = CfgPlain<LOGN>;
        const dim3 grid(nl, (unsigned)batch);
        if (inverse) launch_cfg<C>(d, "k_ntt_limbs", k_ntt_limbs<C, true>, grid, data, nl, pm, d.mods);
        else launch_cfg<C>(d, "k_ntt_limbs", k_ntt_limbs<C, false>, grid, data, nl, pm, d.mods);
    });
}

void launch_rescale_intt(const Dev& d, const uint64_t* in, int64_t cnt, int l, const ulonglong2* w, uint64_t* r_out,
                         const ulonglong2* w2, uint64_t* r_out2) {
    EDL_DISPATCH_LOGN(d.logn, {
        using C = CfgFused<LOGN>;
        launch_cfg<C>(d, "k_rescale_intt", k_rescale_intt<C>, dim3(2, (unsigned)cnt), in, l, w, r_out, w2, r_out2, d.mods);
    });
}

void launch_rescale_ntt(const Dev& d, const uint64_t* in, int64_t cnt, int l, const ulonglong2* w,
                        const uint64_t* r, const uint64_t* bias, uint64_t* out, int lo) {
    const int nlo = (lo < 0 || lo > l - 1) ? l : lo + 1;
    EDL_DISPATCH_LOGN(d.logn, {
        using C = CfgFused<LOGN>;
        launch_cfg<C>(d, "k_rescale_ntt", k_rescale_ntt<C>, dim3(nlo, 2, (unsigned)cnt), in, l, w, r, bias, out, nlo, d.mods,
                      d.cc);
    });
}

size_t relin_scratch_words(int64_t cnt, int l, int logn) {
    return (size_t)cnt * (((size_t)(l + 1) + 2 * (size_t)(l + 2) + 4) << logn);
}

void launch_relin(const Dev& d, const uint64_t* a, const uint64_t* b, int64_t cnt, int l, bool rescale,
                  const uint64_t* rlk, const uint64_t* rlk_s, uint64_t* scratch, uint64_t* out) {
    uint64_t* acoef = scratch;
    uint64_t* acc = acoef + ((size_t)cnt * (l + 1) << d.logn);
    uint64_t* r = acc + ((size_t)cnt * 2 * (l + 2) << d.logn);
    uint64_t* s = r + ((size_t)cnt * 2 << d.logn);
    const int rs = rescale ? 1 : 0;
    EDL_DISPATCH_LOGN(d.logn, {
        using C = CfgFused<LOGN>;
        launch_cfg<C>(d, "k_relin_intt_d2", k_relin_intt_d2<C>, dim3(l + 1, (unsigned)cnt), a, b, l, acoef, d.mods);
        launch_cfg<C>(d, "k_relin_ks_mac", k_relin_ks_mac<C>, dim3(l + 2, (unsigned)cnt), a, b, l, (const uint64_t*)acoef, rlk,
                      rlk_s, d.L, acc, d.mods);
        launch_cfg<C>(d, "k_relin_moddown_intt", k_relin_moddown_intt<C>, dim3(2, (unsigned)cnt), a, b, l,
                      (const uint64_t*)acc, d.L, rs, r, s, d.mods, d.cc);
        launch_cfg<C>(d, "k_relin_moddown_ntt", k_relin_moddown_ntt<C>, dim3(rescale ? l : l + 1, 2, (unsigned)cnt), a, b,
                      l, (const uint64_t*)acc, (const uint64_t*)r, (const uint64_t*)s, d.L, rs, out, d.mods, d.cc);
    });
}

}  // namespace edl
