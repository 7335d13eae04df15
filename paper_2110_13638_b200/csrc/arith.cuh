// arith.cuh -- 64-bit modular arithmetic for sm_100a built from 32-bit IMAD.
//
// Residues are uint64 with q < 2^62 (Alg. 8 chains use 40- and 60-bit primes,
// PAPER.md:222-224).  Three multiplication forms are used on the hot path:
//   * Shoup (one operand a precomputed constant w with w' = floor(w 2^64 / q)):
//     result in [0, 2q) -- NTT twiddles, scalar weights, rlk entries.
//   * Barrett on a 128-bit value with ratio floor(2^128 / q): canonical result --
//     variable x variable products and lazily accumulated 128-bit MAC sums.
//   * 128-bit lazy accumulation of full products (MAC layers, key-switch inner product).
#pragma once
#include <cstdint>

// ---- programmatic dependent launch (round 2c) -----------------------------------------
// Every kernel of the library starts with EDL_PDL_ENTRY(): griddepcontrol.wait blocks until
// the preceding kernel of the stream has completed and its memory is visible, so a kernel
// launched with the programmatic-serialization attribute (EDL_PDL, kernels.cuh) may be
// scheduled while its predecessor's last wave still runs without reading or overwriting
// anything early; launched without the attribute both instructions are no-ops.  With
// EDL_PDL_TRIGGER each CTA also signals at entry that the dependent grid may launch (it can
// then become resident as soon as this grid's last CTAs are running).
#ifdef EDL_PDL_TRIGGER
#define EDL_PDL_ENTRY()                                                  \
    do {                                                                 \
        asm volatile("griddepcontrol.wait;" ::: "memory");               \
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); \
    } while (0)
#else
#define EDL_PDL_ENTRY() asm volatile("griddepcontrol.wait;" ::: "memory")
#endif

namespace edl {

struct ModInfo {
    uint64_t q;        // modulus
    uint64_t r_lo;     // floor(2^128 / q), low word
    uint64_t r_hi;     // floor(2^128 / q), high word
    uint64_t two64;    // 2^64 mod q
    uint64_t two64_s;  // Shoup companion of two64
    const ulonglong2* tw_fwd;   // [N] {psi^brv(k), shoup}; fp == 2: [N] binary64 psi^brv(k) (8 bytes each)
    const ulonglong2* tw_inv;   // [N] {psi^-brv(k), shoup}; fp == 2: [N] binary64 (8 bytes each)
    uint64_t ninv, ninv_s;      // N^-1 mod q and Shoup companion
    uint64_t w1ninv, w1ninv_s;  // psi^-brv(1) * N^-1 (last INTT stage), Shoup companion
    uint64_t one_s;             // floor(2^64 / q): Shoup companion of 1 (64-bit reduction)
    uint64_t fp;                // 1: q < 2^46, every constant companion is RD(w/q) as binary64
                                //    (tw_mul_fp / mulc) and variable products use mulmod_fp;
                                // 2: additionally q < 2^44, NTT butterflies on the FP64 pipe
                                //    (twiddle tables hold binary64 {w, RD(w/q)})
    double qinv_d;              // RN(1/q) (mulmod_fp)
    double qinv_rd;             // RD(1/q) (twiddle companions computed on the fly)
};

struct U128 {
    uint64_t lo, hi;
};

__device__ __forceinline__ U128 mul_wide(uint64_t a, uint64_t b) {
    U128 r;
    r.lo = a * b;
    r.hi = __umul64hi(a, b);
    return r;
}

__device__ __forceinline__ void add128(U128& acc, U128 v) {
    asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;"
        : "+l"(acc.lo), "+l"(acc.hi)
        : "l"(v.lo), "l"(v.hi));
}

// acc += a * b (full 128-bit product), mad.lo.cc / madc.hi carry chain.
__device__ __forceinline__ void mac128(U128& acc, uint64_t a, uint64_t b) {
    asm("mad.lo.cc.u64 %0, %2, %3, %0;\n\tmadc.hi.u64 %1, %2, %3, %1;"
        : "+l"(acc.lo), "+l"(acc.hi)
        : "l"(a), "l"(b));
}

// Shoup: w*y mod q in [0, 2q) for any y < 2^64, w < q, ws = floor(w 2^64 / q).
__device__ __forceinline__ uint64_t shoup_lazy(uint64_t y, uint64_t w, uint64_t ws, uint64_t q) {
    uint64_t qt = __umul64hi(y, ws);
    return y * w - qt * q;
}

// Conditional subtraction x >= m ? x - m : x for x, m < 2^63 (every modulus is < 2^61 and
// lazy values stay below 4q): the sign of x - m decides, which lowers to IADD3/IADD3.X/
// ISETP/SEL/SEL on the ALU pipe (the compare-first form adds an IMAD.X on fmaheavy).
__device__ __forceinline__ uint64_t csub(uint64_t x, uint64_t m) {
    const uint64_t d = x - m;
    return ((int64_t)d < 0) ? x : d;
}

// Shoup with an approximate quotient: qt' = y1 s1 + hi(y1 s0) + hi(y0 s1) drops the
// lowest partial product and the carries of the middle ones, so qt - qt' is 0, 1 or 2 and
// the result y w - qt' q lies in [0, 4q).  Costs 3 IMAD.WIDE + 2 IMAD.HI + 4 IMAD on the
// fmaheavy pipe instead of 6 IMAD.WIDE + 4 IMAD (the NTT's binding pipe, round-1 ncu).
__device__ __forceinline__ uint64_t shoup_lazy4(uint64_t y, uint64_t w, uint64_t ws, uint64_t q) {
    const uint32_t y0 = (uint32_t)y, y1 = (uint32_t)(y >> 32);
    const uint32_t s0 = (uint32_t)ws, s1 = (uint32_t)(ws >> 32);
    const uint64_t qt = (uint64_t)y1 * s1 + __umulhi(y1, s0) + __umulhi(y0, s1);
    return y * w - qt * q;
}

// Shoup with a 3-product quotient (round 2): qt' = floor((y1 s1 2^64 + y1 s0 2^32 + y0 s1 2^32)
// / 2^64) computed as hi(y1 s1 + hi(y0 s1) + hi(y1 s0 + lo(y0 s1))) -- three IMAD.WIDE
// instead of __umul64hi's four -- drops y0 s0 / 2^64 < 1 and one fractional carry, so
// qt' is qt or qt - 1 and y w - qt' q lies in [0, 3q) (any y < 2^64).
__device__ __forceinline__ uint64_t shoup_lazy3(uint64_t y, uint64_t w, uint64_t ws, uint64_t q) {
    const uint32_t y0 = (uint32_t)y, y1 = (uint32_t)(y >> 32);
    const uint32_t s0 = (uint32_t)ws, s1 = (uint32_t)(ws >> 32);
    const uint64_t a = (uint64_t)y0 * s1;
    const uint64_t b = (uint64_t)y1 * s0 + (a & 0xFFFFFFFFull);
    const uint64_t qt = (uint64_t)y1 * s1 + (a >> 32) + (b >> 32);
    return y * w - qt * q;
}

// Lazy bound of the Shoup butterflies (ntt_core.cuh): with the 3-product quotient the
// forward keeps values in [0, 8q) and the inverse in [0, 4q) (8q < 2^63 for q < 2^60), the
// same number of conditional subtractions as the exact quotient's [0, 4q) / [0, 2q).
// Measured (C1, B200): the 3-product quotient is slower in the fused kernels (4.54 vs 4.41
// ms per step) although the plain NTT gains 3 %, so it is opt-in (EDL_SHOUP3).
#ifdef EDL_SHOUP3_ON
#define EDL_SHOUP3 1
#endif

// Shoup with the quotient's cross products on the FP64 pipe (round 2c experiment,
// EDL_SHOUP_FQ): with y = yh 2^32 + yl and ws = sh 2^32 + sl,
//   y ws / 2^64 = yh sh + (yh sl + yl sh + yl sl 2^-32) 2^-32,
// yh sh is one exact IMAD.WIDE and the bracket S < 2^65 is summed in binary64 with every
// operation rounded down (s <= S, S - s < 2^13), so E = yh sh + floor(s 2^-32) satisfies
// y ws / 2^64 - 1 - 2^-19 < E <= y ws / 2^64 <= y w / q and, with Shoup's own y / 2^64 < 1/2
// (y < 2^63), y w - E q lies in [0, 1.51 q): the same [0, 2q) contract as shoup_lazy with
// 3 IMAD.WIDE + 4 IMAD on the fmaheavy pipe instead of 6 + 4.  The 32-bit halves become
// binary64 exactly by the 2^52 exponent trick (2^20 exponent: sl 2^-32).
// Measured on B200: register-only butterfly ceiling 774 -> 702 Gbfly/s, C1 3.97 -> 4.45 ms
// (DFMA and IMAD.WIDE do not overlap), so it stays an opt-in switch; bit-exact.
__device__ __forceinline__ uint64_t shoup_lazy_fq(uint64_t y, uint64_t w, uint64_t ws, uint64_t q) {
    const uint32_t yl = (uint32_t)y, yh = (uint32_t)(y >> 32);
    const uint32_t sl = (uint32_t)ws, sh = (uint32_t)(ws >> 32);
    const double m52 = 4503599627370496.0, m20 = 1048576.0;
    const double dyh = __hiloint2double(0x43300000, (int)yh) - m52;
    const double dyl = __hiloint2double(0x43300000, (int)yl) - m52;
    const double dsh = __hiloint2double(0x43300000, (int)sh) - m52;
    const double dsl = __hiloint2double(0x43300000, (int)sl) - m52;
    const double dsl32 = __hiloint2double(0x41300000, (int)sl) - m20;   // sl 2^-32
    double s = __dmul_rd(dyl, dsh);
    s = __fma_rd(dyh, dsl, s);
    s = __fma_rd(dyl, dsl32, s);
    const double t = __fma_rd(s, 2.3283064365386963e-10, m52);   // 2^52 + floor(s 2^-32)
    const uint64_t ti = (uint64_t)__double_as_longlong(t) & 0xFFFFFFFFFFFFFull;
    const uint64_t qt = (uint64_t)yh * sh + ti;
    return y * w - qt * q;
}

// [0, 2q) result for the butterflies.
__device__ __forceinline__ uint64_t shoup_lazy2(uint64_t y, uint64_t w, uint64_t ws, uint64_t q) {
#ifdef EDL_SHOUP_FQ
    return shoup_lazy_fq(y, w, ws, q);
#elif !defined(EDL_APPROX_SHOUP)
    return shoup_lazy(y, w, ws, q);
#else
    return csub(shoup_lazy4(y, w, ws, q), 2 * q);
#endif
}

// Twiddle product in [0, 2q) with the quotient estimated on the otherwise idle FP64 pipe
// (q < 2^50, y < 2^52, wq = RD(w/q) as binary64): y is rebuilt exactly as a double by
// the 2^52 magic-exponent trick, t = fma_rd(y, wq, 2^52) = 2^52 + floor(y wq) with
// floor(y wq) in {qt - 1, qt} for qt = floor(y w / q) (|y (w/q - wq)| < 2^-11), so
// y w - floor(y wq) q lies in [0, 2q); only the two low 64-bit products stay on the
// fmaheavy pipe (the NTT's binding pipe: 22 instead of 36 cycles per warp butterfly).
__device__ __forceinline__ uint64_t tw_mul_fp(uint64_t y, uint64_t w, uint64_t wq_bits, uint64_t q) {
    const double magic = 4503599627370496.0;   // 2^52
    const double yd = __hiloint2double(0x43300000 | (uint32_t)(y >> 32), (uint32_t)y) - magic;
    const double t = __fma_rd(yd, __longlong_as_double((long long)wq_bits), magic);
    const uint64_t qt = (uint64_t)__double_as_longlong(t) & 0xFFFFFFFFFFFFFull;
    return y * w - qt * q;
}


__device__ __forceinline__ uint64_t shoup(uint64_t y, uint64_t w, uint64_t ws, uint64_t q) {
    return csub(shoup_lazy2(y, w, ws, q), q);
}

// Barrett reduction of a 128-bit value x < q * 2^64 ... in practice x < 2^126.
// qest = floor(x * R / 2^128) computed without the lowest partial product; qest is at
// most 2 below floor(x / q), so two conditional subtractions give the canonical value.
__device__ __forceinline__ uint64_t barrett128(U128 x, const ModInfo& m) {
    uint64_t c0 = __umul64hi(x.lo, m.r_lo);
    uint64_t t1lo = x.lo * m.r_hi;
    uint64_t t1hi = __umul64hi(x.lo, m.r_hi);
    uint64_t t2lo = x.hi * m.r_lo;
    uint64_t t2hi = __umul64hi(x.hi, m.r_lo);
    uint64_t s, carry1, carry2;
    // s = c0 + t1lo + t2lo, collecting carries into the quotient word
    asm("add.cc.u64 %0, %3, %4;\n\t"
        "addc.u64 %1, 0, 0;\n\t"
        "add.cc.u64 %0, %0, %5;\n\t"
        "addc.u64 %2, 0, 0;"
        : "=l"(s), "=l"(carry1), "=l"(carry2)
        : "l"(c0), "l"(t1lo), "l"(t2lo));
    (void)s;
    uint64_t qest = x.hi * m.r_hi + t1hi + t2hi + carry1 + carry2;
    uint64_t r = x.lo - qest * m.q;
    r = csub(r, 2 * m.q);
    return csub(r, m.q);
}

__device__ __forceinline__ uint64_t mulmod_barrett(uint64_t a, uint64_t b, const ModInfo& m) {
    return barrett128(mul_wide(a, b), m);
}

__device__ __forceinline__ double u52_to_double(uint64_t a) {   // exact for a < 2^52
    return __hiloint2double(0x43300000 | (uint32_t)(a >> 32), (uint32_t)a) - 4503599627370496.0;
}

// ---- exact binary64 residue arithmetic (ModInfo::fp == 2 moduli, q < 2^44; ntt_core.cuh)
constexpr double F64_RND = 6755399441055744.0;   // 1.5 * 2^52: v + F64_RND - F64_RND = rint(v), |v| < 2^51
constexpr double F64_TWO52 = 4503599627370496.0;

__device__ __forceinline__ double f64_of(uint64_t bits) { return __longlong_as_double((long long)bits); }
__device__ __forceinline__ uint64_t bits_of(double d) { return (uint64_t)__double_as_longlong(d); }

// b w mod q in [-0.625 q, 0.625 q] for |b| < 2^50, w < q, wq = RD(w/q)
__device__ __forceinline__ double f64_mulc(double b, double w, double wq, double q) {
    const double hi = __dmul_rn(b, w);
    const double lo = __fma_rn(b, w, -hi);
    const double qt = __dsub_rn(__fma_rn(b, wq, F64_RND), F64_RND);
    return __dadd_rn(__fma_rn(-qt, q, hi), lo);
}
// Twiddle product without a companion (the NTT butterflies, round 2): b w mod q with the
// quotient taken from the rounded product, qt = rint(RN(b w) RN(1/q)).  For q < 2^44,
// w < q and |b| < 64 q: |RN(b w) - b w| <= 2^-53 |b w| <= 64 q^2 2^-53 and the quotient
// estimate is off from b w / q by at most 64 q 2^-53 + |b w/q| 2^-53 < 0.13, so
// |b w - qt q| <= 0.63 q; hi - qt q is an integer below 2^53 (exact in the FMA) and lo is
// the exact product error.  Same 6 FP64 instructions as f64_mulc, but a twiddle is 8 bytes
// (w only) instead of 16: half the twiddle traffic / shared memory.
__device__ __forceinline__ double f64_mult(double b, double w, double q, double qinv) {
    const double hi = __dmul_rn(b, w);
    const double lo = __fma_rn(b, w, -hi);
    const double qt = __dsub_rn(__fma_rn(hi, qinv, 6755399441055744.0), 6755399441055744.0);
    return __dadd_rn(__fma_rn(-qt, q, hi), lo);
}
// v mod q in [-0.51 q, 0.51 q] for |v| < 2^50 (qinv = RN(1/q))
__device__ __forceinline__ double f64_reduce(double v, double q, double qinv) {
    const double qt = __dsub_rn(__fma_rn(v, qinv, F64_RND), F64_RND);
    return __fma_rn(-qt, q, v);
}
// canonical residue of an exact integer |r| < q, as uint64
__device__ __forceinline__ uint64_t f64_to_canon(double r, double q) {
    const double c = r < 0.0 ? __dadd_rn(q, F64_TWO52) : F64_TWO52;
    return bits_of(__dadd_rn(r, c)) & 0xFFFFFFFFFFFFFull;
}
__device__ __forceinline__ uint64_t f64_from_u(uint64_t v) {   // v < 2^52 -> bits of (double)v
    return bits_of(__hiloint2double(0x43300000 | (uint32_t)(v >> 32), (uint32_t)v) - F64_TWO52);
}

// Variable x variable product for q < 2^50 with the quotient from the FP64 pipe:
// t = fma_rd(fl(a b), RN(1/q), 2^52) gives floor of a b/q within +-1 (relative error
// < 2^-51 of a value < 2^50), so a b - qt q lies in [-q, 2q) and one signed correction
// each way makes it canonical.  16 fmaheavy cycles instead of Barrett's ~60.
__device__ __forceinline__ uint64_t mulmod_fp(uint64_t a, uint64_t b, const ModInfo& m) {
    const double p = u52_to_double(a) * u52_to_double(b);
    const double t = __fma_rd(p, m.qinv_d, 4503599627370496.0);
    const uint64_t qt = (uint64_t)__double_as_longlong(t) & 0xFFFFFFFFFFFFFull;
    int64_t r = (int64_t)(a * b - qt * m.q);
    r = (r < 0) ? r + (int64_t)m.q : r;
    return csub((uint64_t)r, m.q);
}

// Canonical a b mod q (a, b < q): FP64-quotient path for q < 2^50, Barrett otherwise.
// m.fp is uniform across a CTA, so the branch never diverges.
__device__ __forceinline__ uint64_t mulmod(uint64_t a, uint64_t b, const ModInfo& m) {
    return m.fp ? mulmod_fp(a, b, m) : mulmod_barrett(a, b, m);
}

// Constant multiplication y * w with the host-made companion of w for this modulus
// (RD(w/q) bits if m.fp, else the Shoup companion): [0, 2q) (y < 2^52 when m.fp) ...
__device__ __forceinline__ uint64_t mulc_lazy(uint64_t y, ulonglong2 w, const ModInfo& m) {
    return m.fp ? tw_mul_fp(y, w.x, w.y, m.q) : shoup_lazy2(y, w.x, w.y, m.q);
}
// ... and canonical.
__device__ __forceinline__ uint64_t mulc(uint64_t y, ulonglong2 w, const ModInfo& m) {
    return csub(mulc_lazy(y, w, m), m.q);
}

// Canonical reduction of an arbitrary 64-bit value: Shoup multiplication by 1
// (a - floor(a floor(2^64/q) / 2^64) q lies in [0, 2q) for every a < 2^64).
__device__ __forceinline__ uint64_t reduce64(uint64_t a, const ModInfo& m) {
    return csub(a - __umul64hi(a, m.one_s) * m.q, m.q);
}

__device__ __forceinline__ uint64_t addmod(uint64_t a, uint64_t b, uint64_t q) { return csub(a + b, q); }
__device__ __forceinline__ uint64_t submod(uint64_t a, uint64_t b, uint64_t q) { return a >= b ? a - b : a + q - b; }

// Centered lift of r in [0, qf) to (-qf/2, qf/2], reduced into [0, q) where
// qf_mod_q = qf mod q (precomputed).  qf is odd so the half point never occurs.  The
// qf < 2q test is uniform across the CTA (both moduli are per-launch constants), so the
// common case (a 40-bit lift into a 40- or 60-bit limb) costs one conditional subtraction.
__device__ __forceinline__ uint64_t center_mod(uint64_t r, uint64_t qf, uint64_t qf_mod_q, const ModInfo& m) {
    uint64_t rq = (qf < 2 * m.q) ? csub(r, m.q) : reduce64(r, m);
    if (r > (qf >> 1)) rq = submod(rq, qf_mod_q, m.q);
    return rq;
}

}  // namespace edl
