// rng.cu -- Philox4x32-10 sampling, key generation, public-key encryption and the
// device half of decryption (client-side steps a1/a12).
//
// Counter layout (c0, c1, c2, c3) = (coefficient, object id, limb, domain tag), key =
// (seed lo, seed hi).  Samples are drawn on the fly inside the NTT prologues, so the
// secret/error polynomials never touch HBM in coefficient form.
#pragma once
#include "kernels.cuh"
#include "ntt_core.cuh"

namespace edl {

enum : uint32_t { TAG_S = 1, TAG_PK_A = 2, TAG_PK_E = 3, TAG_RLK_A = 4, TAG_RLK_E = 5, TAG_ENC_V = 6, TAG_ENC_E0 = 7,
                  TAG_ENC_E1 = 8, TAG_GK_A = 9, TAG_GK_E = 10, TAG_SK_A = 11, TAG_SK_E = 12 };

// NTT-domain index of sigma_g: evaluation point psi^{2 brv(k)+1} maps to psi^{(2 brv(k)+1) g}
// (NEXT f1), so sigma_g(a)[k] = a[src_g(k)].
__device__ __forceinline__ int galois_src(int k, uint32_t g, int logn) {
    const uint32_t two_n = 2u << logn;
    const uint32_t bk = __brev((uint32_t)k) >> (32 - logn);
    const uint32_t e = (uint32_t)(((uint64_t)(2 * bk + 1) * g) % two_n);
    return (int)(__brev((e - 1) >> 1) >> (32 - logn));
}

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; r++) {
        if (r > 0) {
            k.x += 0x9E3779B9u;
            k.y += 0xBB67AE85u;
        }
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    }
    return c;
}

__device__ __forceinline__ uint4 draw(uint64_t seed, uint32_t coef, uint32_t obj, uint32_t limb, uint32_t tag) {
    return philox4x32_10(make_uint4(coef, obj, limb, tag), make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
}

__device__ __forceinline__ int ternary_of(uint4 x) { return (int)(x.x % 3u) - 1; }
__device__ __forceinline__ int cbd_of(uint4 x) { return __popc(x.x & 0x1FFFFFu) - __popc(x.y & 0x1FFFFFu); }

__device__ __forceinline__ uint64_t uniform_of(uint4 x, const ModInfo& m) {
    U128 u;
    u.lo = (uint64_t)x.x | ((uint64_t)x.y << 32);
    u.hi = (uint64_t)x.z | ((uint64_t)x.w << 32);
    return barrett128(u, m);
}

__device__ __forceinline__ uint64_t small_mod(int v, uint64_t q) { return v >= 0 ? (uint64_t)v : q - (uint64_t)(-v); }

__device__ __forceinline__ uint64_t signed_mod(int64_t v, const ModInfo& m) {
    if (v >= 0) return reduce64((uint64_t)v, m);
    uint64_t r = reduce64((uint64_t)(-(v + 1)) + 1, m);   // |v| without overflow at INT64_MIN
    return r == 0 ? 0 : m.q - r;
}

// floor(w * 2^64 / q) by restoring division (key generation only).
static __device__ uint64_t shoup_companion(uint64_t w, uint64_t q) {
    uint64_t rem = w, quo = 0;
    for (int b = 0; b < 64; b++) {
        const bool top = (rem >> 63) != 0;
        rem <<= 1;
        quo <<= 1;
        if (top || rem >= q) {
            rem -= q;
            quo |= 1;
        }
    }
    return quo;
}

// companion of a key residue for mulc(): RD(v/q) bits (FP64-quotient limbs) or Shoup
__device__ __forceinline__ uint64_t key_companion(uint64_t v, const ModInfo& m) {
    if (m.fp) return (uint64_t)__double_as_longlong(__ddiv_rd((double)v, (double)m.q));
    return shoup_companion(v, m.q);
}

// ---- keygen: one CTA per modulus (secret), per data limb (pk), per (digit, limb) (rlk)
template <class C>
__global__ void __launch_bounds__(C::T, C::MINB)
k_keygen_s(uint64_t seed, uint64_t* __restrict__ s_hat, const __grid_constant__ ModTable mods) {
    EDL_PDL_ENTRY();
    extern __shared__ uint64_t sm[];
    const int i = C::bx();
    const ModInfo& m = mods[i];
    uint64_t* dst = s_hat + ((size_t)i << C::LOGN);
    auto ld = [&](int idx) { return small_mod(ternary_of(draw(seed, idx, 0, 0, TAG_S)), m.q); };
    auto st = [&](int idx, uint64_t v) { dst[idx] = v; };
    ntt_fwd<C>(sm, m, ld, st);
}

template <class C>
__global__ void __launch_bounds__(C::T, C::MINB)
k_keygen_pk(uint64_t seed, int L, const uint64_t* __restrict__ s_hat, uint64_t* __restrict__ pk,
            const __grid_constant__ ModTable mods) {
    EDL_PDL_ENTRY();
    extern __shared__ uint64_t sm[];
    const int i = C::bx();
    const ModInfo& m = mods[i];
    const uint64_t* s = s_hat + ((size_t)i << C::LOGN);
    uint64_t* b = pk + ((size_t)(0 * (L + 1) + i) << C::LOGN);
    uint64_t* a = pk + ((size_t)(1 * (L + 1) + i) << C::LOGN);
    auto ld = [&](int idx) { return small_mod(cbd_of(draw(seed, idx, 0, 0, TAG_PK_E)), m.q); };
    auto st = [&](int idx, uint64_t e) {
        const uint64_t av = uniform_of(draw(seed, idx, 0, i, TAG_PK_A), m);
        a[idx] = av;
        b[idx] = submod(e, mulmod(av, s[idx], m), m.q);
    };
    ntt_fwd<C>(sm, m, ld, st);
}

template <class C>
__global__ void __launch_bounds__(C::T, C::MINB)
k_keygen_rlk(uint64_t seed, int L, const uint64_t* __restrict__ s_hat, uint64_t* __restrict__ rlk,
             uint64_t* __restrict__ rlk_s, const __grid_constant__ ModTable mods, const ChainConsts* __restrict__ cc) {
    EDL_PDL_ENTRY();
    extern __shared__ uint64_t sm[];
    const int i = C::bx();   // limb 0..L+1 (L+1 = P)
    const int j = blockIdx.y;   // digit 0..L
    const ModInfo& m = mods[i];
    const uint64_t* s = s_hat + ((size_t)i << C::LOGN);
    const size_t ob = ((size_t)(j * 2 + 0) * (L + 2) + i) << C::LOGN;
    const size_t oa = ((size_t)(j * 2 + 1) * (L + 2) + i) << C::LOGN;
    const uint64_t pmod = cc->qmod[L + 1][i];
    auto ld = [&](int idx) { return small_mod(cbd_of(draw(seed, idx, j, 0, TAG_RLK_E)), m.q); };
    auto st = [&](int idx, uint64_t e) {
        const uint64_t av = uniform_of(draw(seed, idx, j, i, TAG_RLK_A), m);
        const uint64_t sv = s[idx];
        uint64_t bv = submod(e, mulmod(av, sv, m), m.q);
        if (i == j) bv = addmod(bv, mulmod(mulmod(sv, sv, m), pmod, m), m.q);
        rlk[ob + idx] = bv;
        rlk[oa + idx] = av;
        rlk_s[ob + idx] = key_companion(bv, m);
        rlk_s[oa + idx] = key_companion(av, m);
    };
    ntt_fwd<C>(sm, m, ld, st);
}

// ---- Galois key for element g (NEXT f1): rlk's digit structure with gadget P sigma_g(s);
// a ~ uniform (tag 9), e ~ CBD (tag 10), object id 64 g + j
template <class C>
__global__ void __launch_bounds__(C::T, C::MINB)
k_keygen_galois(uint64_t seed, int L, uint32_t g, const uint64_t* __restrict__ s_hat, uint64_t* __restrict__ gk,
                uint64_t* __restrict__ gk_c, const __grid_constant__ ModTable mods, const ChainConsts* __restrict__ cc) {
    EDL_PDL_ENTRY();
    extern __shared__ uint64_t sm[];
    const int i = C::bx();      // limb 0..L+1 (L+1 = P)
    const int j = blockIdx.y;   // digit 0..L
    const ModInfo& m = mods[i];
    const uint64_t* s = s_hat + ((size_t)i << C::LOGN);
    const size_t ob = ((size_t)(j * 2 + 0) * (L + 2) + i) << C::LOGN;
    const size_t oa = ((size_t)(j * 2 + 1) * (L + 2) + i) << C::LOGN;
    const uint64_t pmod = cc->qmod[L + 1][i];
    const uint32_t obj = 64u * g + (uint32_t)j;
    auto ld = [&](int idx) { return small_mod(cbd_of(draw(seed, idx, obj, 0, TAG_GK_E)), m.q); };
    auto st = [&](int idx, uint64_t e) {
        const uint64_t av = uniform_of(draw(seed, idx, obj, i, TAG_GK_A), m);
        uint64_t bv = submod(e, mulmod(av, s[idx], m), m.q);
        if (i == j) bv = addmod(bv, mulmod(s[galois_src(idx, g, C::LOGN)], pmod, m), m.q);
        gk[ob + idx] = bv;
        gk[oa + idx] = av;
        gk_c[ob + idx] = key_companion(bv, m);
        gk_c[oa + idx] = key_companion(av, m);
    };
    ntt_fwd<C>(sm, m, ld, st);
}

// ---- plaintext vectors: integer polynomial -> NTT-domain residues, per (vector, limb)
template <class C>
__global__ void __launch_bounds__(C::T, C::MINB)
k_encode_pt(const int64_t* __restrict__ msg, int l, uint64_t* __restrict__ out, const __grid_constant__ ModTable mods) {
    EDL_PDL_ENTRY();
    extern __shared__ uint64_t sm[];
    const int i = blockIdx.y;
    const int64_t c = C::bx();
    const ModInfo& m = mods[i];
    const int64_t* mm = msg + ((size_t)c << C::LOGN);
    uint64_t* dst = out + (((size_t)c * (l + 1) + i) << C::LOGN);
    auto ld = [&](int idx) { return signed_mod(mm[idx], m); };
    auto st = [&](int idx, uint64_t v) { dst[idx] = v; };
    ntt_fwd<C>(sm, m, ld, st);
}

// ---- encrypt (O8): c0 = v*b + NTT(e0 + m), c1 = v*a + NTT(e1), per (ct, limb)
template <class C>
__global__ void __launch_bounds__(C::T, C::MINB)
k_encrypt(const int64_t* __restrict__ msg, int l, int L, uint64_t seed, uint32_t obj0, const uint64_t* __restrict__ pk,
          uint64_t* __restrict__ out, const __grid_constant__ ModTable mods) {
    EDL_PDL_ENTRY();
    extern __shared__ uint64_t sm[];
    const int i = blockIdx.y;
    const int64_t c = C::bx();
    const uint32_t obj = obj0 + (uint32_t)c;
    const ModInfo& m = mods[i];
    const int64_t* mm = msg + ((size_t)c << C::LOGN);
    uint64_t* c0 = out + limb_off(c, 0, i, l + 1, C::LOGN);
    uint64_t* c1 = out + limb_off(c, 1, i, l + 1, C::LOGN);
    const uint64_t* pb = pk + ((size_t)(0 * (L + 1) + i) << C::LOGN);
    const uint64_t* pa = pk + ((size_t)(1 * (L + 1) + i) << C::LOGN);
    {
        auto ld = [&](int idx) { return small_mod(cbd_of(draw(seed, idx, obj, 0, TAG_ENC_E1)), m.q); };
        auto st = [&](int idx, uint64_t v) { c1[idx] = v; };
        ntt_fwd<C>(sm, m, ld, st);
    }
    {
        auto ld = [&](int idx) {
            return addmod(small_mod(cbd_of(draw(seed, idx, obj, 0, TAG_ENC_E0)), m.q), signed_mod(mm[idx], m), m.q);
        };
        auto st = [&](int idx, uint64_t v) { c0[idx] = v; };
        ntt_fwd<C>(sm, m, ld, st);
    }
    {
        auto ld = [&](int idx) { return small_mod(ternary_of(draw(seed, idx, obj, 0, TAG_ENC_V)), m.q); };
        auto st = [&](int idx, uint64_t v) {
            c0[idx] = addmod(c0[idx], mulmod(v, pb[idx], m), m.q);
            c1[idx] = addmod(c1[idx], mulmod(v, pa[idx], m), m.q);
        };
        ntt_fwd<C>(sm, m, ld, st);
    }
}

// ---- secret-key encryption (DESIGN reading Z16): c1_i = a_i = uniform(seed, obj, i, TAG_SK_A)
// drawn directly in the NTT domain, c0_i = NTT_i(m + e) - a_i s_i with e = CBD(eseed, obj,
// TAG_SK_E), where eseed = PRF(secret seed, seed) (host::sk_error_key): only c1 is a public
// function of the wire seed; the error needs the secret key's seed.
template <class C>
__global__ void __launch_bounds__(C::T, C::MINB)
k_encrypt_sk(const int64_t* __restrict__ msg, int l, uint64_t seed, uint64_t eseed, uint32_t obj0,
             const uint64_t* __restrict__ s_hat, uint64_t* __restrict__ out, const __grid_constant__ ModTable mods) {
    EDL_PDL_ENTRY();
    extern __shared__ uint64_t sm[];
    const int i = blockIdx.y;
    const int64_t c = C::bx();
    const uint32_t obj = obj0 + (uint32_t)c;
    const ModInfo& m = mods[i];
    const int64_t* mm = msg + ((size_t)c << C::LOGN);
    uint64_t* c0 = out + limb_off(c, 0, i, l + 1, C::LOGN);
    uint64_t* c1 = out + limb_off(c, 1, i, l + 1, C::LOGN);
    const uint64_t* s = s_hat + ((size_t)i << C::LOGN);
    auto ld = [&](int idx) {
        return addmod(small_mod(cbd_of(draw(eseed, idx, obj, 0, TAG_SK_E)), m.q), signed_mod(mm[idx], m), m.q);
    };
    auto st = [&](int idx, uint64_t v) {
        const uint64_t a = uniform_of(draw(seed, idx, obj, i, TAG_SK_A), m);
        c1[idx] = a;
        c0[idx] = submod(v, mulmod(a, s[idx], m), m.q);
    };
    ntt_fwd<C>(sm, m, ld, st);
}

// ---- decrypt, device half: out[c][i] = INTT(c0 + c1 s)
template <class C>
__global__ void __launch_bounds__(C::T, C::MINB)
k_decrypt(const uint64_t* __restrict__ ct, int l, const uint64_t* __restrict__ s_hat, uint64_t* __restrict__ out,
          const __grid_constant__ ModTable mods) {
    EDL_PDL_ENTRY();
    extern __shared__ uint64_t sm[];
    const int i = blockIdx.y;
    const int64_t c = C::bx();
    const ModInfo& m = mods[i];
    const uint64_t* c0 = ct + limb_off(c, 0, i, l + 1, C::LOGN);
    const uint64_t* c1 = ct + limb_off(c, 1, i, l + 1, C::LOGN);
    const uint64_t* s = s_hat + ((size_t)i << C::LOGN);
    uint64_t* dst = out + (((size_t)c * (l + 1) + i) << C::LOGN);
    auto ld = [&](int idx) { return addmod(c0[idx], mulmod(c1[idx], s[idx], m), m.q); };
    auto st = [&](int idx, uint64_t v) { dst[idx] = v; };
    ntt_inv<C>(sm, m, ld, st);
}

template <int LOGN>
void launch_keygen_n(const Dev& d, uint64_t seed, uint64_t* s_hat, uint64_t* pk, uint64_t* rlk, uint64_t* rlk_s) {
    using C = CfgFused<LOGN>;
    launch_cfg<C>(d, "k_keygen_s", k_keygen_s<C>, dim3(d.L + 2), seed, s_hat, *d.mt);
    launch_cfg<C>(d, "k_keygen_pk", k_keygen_pk<C>, dim3(d.L + 1), seed, d.L, (const uint64_t*)s_hat, pk, *d.mt);
    launch_cfg<C>(d, "k_keygen_rlk", k_keygen_rlk<C>, dim3(d.L + 2, d.L + 1), seed, d.L, (const uint64_t*)s_hat, rlk,
                  rlk_s, *d.mt, d.cc);
}

template <int LOGN>
void launch_encrypt_n(const Dev& d, const int64_t* msg, int64_t cnt, int l, uint64_t seed, uint32_t obj0,
                      const uint64_t* pk, uint64_t* out) {
    using C = CfgFused<LOGN>;
    launch_cfg<C>(d, "k_encrypt", k_encrypt<C>, dim3((unsigned)cnt, l + 1), msg, l, d.L, seed, obj0, pk, out, *d.mt);
}

template <int LOGN>
void launch_encrypt_sk_n(const Dev& d, const int64_t* msg, int64_t cnt, int l, uint64_t seed, uint64_t eseed,
                         uint32_t obj0, const uint64_t* s_hat, uint64_t* out) {
    using C = CfgFused<LOGN>;
    launch_cfg<C>(d, "k_encrypt_sk", k_encrypt_sk<C>, dim3((unsigned)cnt, l + 1), msg, l, seed, eseed, obj0, s_hat, out,
                  *d.mt);
}

template <int LOGN>
void launch_decrypt_n(const Dev& d, const uint64_t* ct, int64_t cnt, int l, const uint64_t* s_hat, uint64_t* out) {
    using C = CfgFused<LOGN>;
    launch_cfg<C>(d, "k_decrypt", k_decrypt<C>, dim3((unsigned)cnt, l + 1), ct, l, s_hat, out, *d.mt);
}

template <int LOGN>
void launch_keygen_galois_n(const Dev& d, uint64_t seed, uint32_t g, const uint64_t* s_hat, uint64_t* gk, uint64_t* gk_c) {
    using C = CfgFused<LOGN>;
    launch_cfg<C>(d, "k_keygen_galois", k_keygen_galois<C>, dim3(d.L + 2, d.L + 1), seed, d.L, g, s_hat, gk, gk_c,
                  *d.mt, d.cc);
}

template <int LOGN>
void launch_encode_pt_n(const Dev& d, const int64_t* msg, int64_t cnt, int l, uint64_t* out) {
    using C = CfgFused<LOGN>;
    launch_cfg<C>(d, "k_encode_pt", k_encode_pt<C>, dim3((unsigned)cnt, l + 1), msg, l, out, *d.mt);
}

#define EDL_INSTANTIATE_RNG(LOGN)                                                                               \
    template void launch_keygen_n<LOGN>(const Dev&, uint64_t, uint64_t*, uint64_t*, uint64_t*, uint64_t*);      \
    template void launch_encrypt_n<LOGN>(const Dev&, const int64_t*, int64_t, int, uint64_t, uint32_t,          \
                                         const uint64_t*, uint64_t*);                                           \
    template void launch_decrypt_n<LOGN>(const Dev&, const uint64_t*, int64_t, int, const uint64_t*, uint64_t*);  \
    template void launch_encrypt_sk_n<LOGN>(const Dev&, const int64_t*, int64_t, int, uint64_t, uint64_t,       \
                                            uint32_t, const uint64_t*, uint64_t*);                              \
    template void launch_keygen_galois_n<LOGN>(const Dev&, uint64_t, uint32_t, const uint64_t*, uint64_t*, uint64_t*); \
    template void launch_encode_pt_n<LOGN>(const Dev&, const int64_t*, int64_t, int, uint64_t*);

}  // namespace edl
