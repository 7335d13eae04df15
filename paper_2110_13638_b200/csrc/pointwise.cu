// pointwise.cu -- limb-parallel element-wise kernels (K3/K4/K8).
//
// All HBM-bound: 16-byte vector loads/stores of uint64 residues, one modulus per row
// (row = one limb of one polynomial).  The MAC layers accumulate full 128-bit
// products lazily (mad.lo.cc / madc.hi) and reduce once per output (O4: modular sums
// are order independent, so this is bit-identical to per-step reduction).
#include <type_traits>

#include <algorithm>

#include "kernels.cuh"
#include "host_math.h"

namespace edl {

namespace {

constexpr int PW_THREADS = 256;

__device__ __forceinline__ const ulonglong2* v2(const uint64_t* p) { return reinterpret_cast<const ulonglong2*>(p); }
__device__ __forceinline__ ulonglong2* v2(uint64_t* p) { return reinterpret_cast<ulonglong2*>(p); }

dim3 rows_grid(int logn, int64_t rows) {
    const int per_block = PW_THREADS * 2;
    unsigned gx = (unsigned)(((1 << logn) + per_block - 1) / per_block);
    unsigned gy = (unsigned)(rows < 65535 ? rows : 65535);
    return dim3(gx, gy);
}

// ---------------------------------------------------------------- add
__global__ void k_add(const uint64_t* __restrict__ a, int la, const uint64_t* __restrict__ b, int lb, int64_t cnt,
                      int lo, uint64_t* __restrict__ out, const __grid_constant__ ModTable mods, int logn) {
    EDL_PDL_ENTRY();
    const int64_t rows = cnt * 2 * (lo + 1);
    const int n2 = 1 << (logn - 1);
    for (int64_t row = blockIdx.y; row < rows; row += gridDim.y) {
        const int i = (int)(row % (lo + 1));
        const int64_t cp = row / (lo + 1);
        const uint64_t q = mods[i].q;
        const uint64_t* pa = a + (((size_t)cp * (la + 1) + i) << logn);
        const uint64_t* pb = b + (((size_t)cp * (lb + 1) + i) << logn);
        uint64_t* po = out + (((size_t)cp * (lo + 1) + i) << logn);
        for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n2; k += gridDim.x * blockDim.x) {
            ulonglong2 x = v2(pa)[k], y = v2(pb)[k];
            v2(po)[k] = make_ulonglong2(addmod(x.x, y.x, q), addmod(x.y, y.y, q));
        }
    }
}

// ---------------------------------------------------------------- scalar const multiply
__global__ void k_mul_const(const uint64_t* __restrict__ a, int64_t cnt, int l, const ulonglong2* __restrict__ w,
                            uint64_t* __restrict__ out, const __grid_constant__ ModTable mods, int logn) {
    EDL_PDL_ENTRY();
    const int64_t rows = cnt * 2 * (l + 1);
    const int n2 = 1 << (logn - 1);
    for (int64_t row = blockIdx.y; row < rows; row += gridDim.y) {
        const int i = (int)(row % (l + 1));
        const int64_t c = row / (2 * (l + 1));
        const ModInfo& m = mods[i];
        const ulonglong2 wi = w[c * (l + 1) + i];
        const uint64_t* pa = a + ((size_t)row << logn);
        uint64_t* po = out + ((size_t)row << logn);
        for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n2; k += gridDim.x * blockDim.x) {
            ulonglong2 x = v2(pa)[k];
            v2(po)[k] = make_ulonglong2(mulc(x.x, wi, m), mulc(x.y, wi, m));
        }
    }
}

// ---------------------------------------------------------------- add constant (poly 0 only)
__global__ void k_add_const(const uint64_t* __restrict__ a, int64_t cnt, int l, const uint64_t* __restrict__ kc,
                            uint64_t* __restrict__ out, const __grid_constant__ ModTable mods, int logn) {
    EDL_PDL_ENTRY();
    const int64_t rows = cnt * 2 * (l + 1);
    const int n2 = 1 << (logn - 1);
    for (int64_t row = blockIdx.y; row < rows; row += gridDim.y) {
        const int i = (int)(row % (l + 1));
        const int p = (int)((row / (l + 1)) % 2);
        const int64_t c = row / (2 * (l + 1));
        const uint64_t q = mods[i].q;
        const uint64_t kk = (p == 0) ? kc[c * (l + 1) + i] : 0;
        const uint64_t* pa = a + ((size_t)row << logn);
        uint64_t* po = out + ((size_t)row << logn);
        for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n2; k += gridDim.x * blockDim.x) {
            ulonglong2 x = v2(pa)[k];
            v2(po)[k] = make_ulonglong2(addmod(x.x, kk, q), addmod(x.y, kk, q));
        }
    }
}

// ---------------------------------------------------------------- mod drop (copy limbs 0..lo)
__global__ void k_mod_drop(const uint64_t* __restrict__ a, int64_t cnt, int la, int lo, uint64_t* __restrict__ out,
                           int logn) {
    EDL_PDL_ENTRY();
    const int64_t rows = cnt * 2 * (lo + 1);
    const int n2 = 1 << (logn - 1);
    for (int64_t row = blockIdx.y; row < rows; row += gridDim.y) {
        const int i = (int)(row % (lo + 1));
        const int64_t cp = row / (lo + 1);
        const uint64_t* pa = a + (((size_t)cp * (la + 1) + i) << logn);
        uint64_t* po = out + ((size_t)row << logn);
        for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n2; k += gridDim.x * blockDim.x) v2(po)[k] = v2(pa)[k];
    }
}

// ---------------------------------------------------------------- in-place x mod q (after NCCL uint64 sum)
__global__ void k_mod_reduce(uint64_t* __restrict__ x, int64_t cnt, int l, const __grid_constant__ ModTable mods,
                             int logn) {
    EDL_PDL_ENTRY();
    const int64_t rows = cnt * 2 * (l + 1);
    const int n2 = 1 << (logn - 1);
    for (int64_t row = blockIdx.y; row < rows; row += gridDim.y) {
        const ModInfo m = mods[row % (l + 1)];
        uint64_t* p = x + ((size_t)row << logn);
        for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n2; k += gridDim.x * blockDim.x) {
            ulonglong2 v = v2(p)[k];
            v2(p)[k] = make_ulonglong2(reduce64(v.x, m), reduce64(v.y, m));
        }
    }
}

// ---------------------------------------------------------------- v + mod_drop(w) + const
__global__ void k_add_add_const(const uint64_t* __restrict__ v, const uint64_t* __restrict__ w, int lw, int64_t cnt,
                                int lo, const uint64_t* __restrict__ kc, uint64_t* __restrict__ out,
                                const __grid_constant__ ModTable mods, int logn) {
    EDL_PDL_ENTRY();
    const int64_t rows = cnt * 2 * (lo + 1);
    const int n2 = 1 << (logn - 1);
    for (int64_t row = blockIdx.y; row < rows; row += gridDim.y) {
        const int i = (int)(row % (lo + 1));
        const int64_t cp = row / (lo + 1);
        const int p = (int)(cp % 2);
        const int64_t c = cp / 2;
        const uint64_t q = mods[i].q;
        const uint64_t kk = (p == 0 && kc) ? kc[c * (lo + 1) + i] : 0;
        const uint64_t* pv = v + ((size_t)row << logn);
        const uint64_t* pw = w + (((size_t)cp * (lw + 1) + i) << logn);
        uint64_t* po = out + ((size_t)row << logn);
        for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n2; k += gridDim.x * blockDim.x) {
            ulonglong2 x = v2(pv)[k], y = v2(pw)[k];
            v2(po)[k] = make_ulonglong2(addmod(addmod(x.x, y.x, q), kk, q), addmod(addmod(x.y, y.y, q), kk, q));
        }
    }
}

// ---------------------------------------------------------------- cross-correlation MAC
// grid: x = coefficient blocks, y = poly*(l+1) + limb, z = output window (r*Wo + c).
// Each thread owns one coefficient of one window: it first issues the loads of all the
// window's taps (up to CC_TAPS, independent -> memory-level parallelism), then keeps up
// to CC_FC filters' 128-bit accumulators in registers, so each input residue is read
// from HBM exactly once.
constexpr int CC_FC = 8;
constexpr int CC_TAPS = 16;

__global__ void __launch_bounds__(PW_THREADS, 2)
k_cc_mac(const uint64_t* __restrict__ x, int l, int H, int W, int F, int kh, int kw, int stride,
         const ulonglong2* __restrict__ wk, uint64_t* __restrict__ out, const __grid_constant__ ModTable mods, int logn) {
    EDL_PDL_ENTRY();
    extern __shared__ uint64_t wsm[];   // [F][taps] residues for this limb
    const int nl = l + 1;
    const int p = blockIdx.y / nl, i = blockIdx.y % nl;
    const int Wo = (W - kw) / stride + 1;
    const int Ho = (H - kh) / stride + 1;
    const int win = blockIdx.z;
    const int wr = win / Wo, wc = win % Wo;
    const int taps = kh * kw;
    for (int t = threadIdx.x; t < F * taps; t += blockDim.x) wsm[t] = wk[(size_t)t * nl + i].x;
    __syncthreads();
    const ModInfo m = mods[i];
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= (1 << logn)) return;
    for (int t0 = 0; t0 < taps; t0 += CC_TAPS) {
        uint64_t xv[CC_TAPS];
#pragma unroll
        for (int t = 0; t < CC_TAPS; t++) {
            const int tt = t0 + t;
            if (tt < taps) {
                const int u = tt / kw, v = tt % kw;
                const int pix = (wr * stride + u) * W + (wc * stride + v);
                xv[t] = __ldg(x + limb_off(pix, p, i, nl, logn) + n);
            } else {
                xv[t] = 0;
            }
        }
        for (int f0 = 0; f0 < F; f0 += CC_FC) {
            U128 acc[CC_FC];
#pragma unroll
            for (int f = 0; f < CC_FC; f++) acc[f].lo = acc[f].hi = 0;
#pragma unroll
            for (int t = 0; t < CC_TAPS; t++) {
#pragma unroll
                for (int f = 0; f < CC_FC; f++)
                    if (f0 + f < F && t0 + t < taps) mac128(acc[f], xv[t], wsm[(f0 + f) * taps + t0 + t]);
            }
#pragma unroll
            for (int f = 0; f < CC_FC; f++) {
                if (f0 + f < F) {
                    const int64_t o = (int64_t)(f0 + f) * Ho * Wo + win;
                    uint64_t* dst = out + limb_off(o, p, i, nl, logn) + n;
                    uint64_t v = barrett128(acc[f], m);
                    if (t0 > 0) v = addmod(v, *dst, m.q);
                    *dst = v;
                }
            }
        }
    }
}

// ---------------------------------------------------------------- cross-correlation MAC, FC filters
// Hot-path variant of k_cc_mac (round 2): each thread owns two consecutive coefficients
// (16-byte loads and stores) of one (window, poly, limb) and all FC <= 8 filters of a
// filter chunk, so every weight fetched from shared memory feeds two 128-bit MACs and
// every input residue is read from HBM once.  Taps stream in batches of CC2_TB with the
// next batch's loads issued before the current batch's MACs (memory-level parallelism
// without a second CTA's registers).
#ifndef EDL_CC2_THREADS
#define EDL_CC2_THREADS 128   // measured: 0.468 vs 0.483 ms (256 x 2 CTAs/SM)
#endif
constexpr int CC2_THREADS = EDL_CC2_THREADS;
#ifndef EDL_CC2_TB
#define EDL_CC2_TB 4
#endif
#ifndef EDL_CC2_MINB
#define EDL_CC2_MINB 4
#endif
constexpr int CC2_TB = EDL_CC2_TB;
constexpr int CC2_MAXTAPS = 64;

template <int FC>
__global__ void __launch_bounds__(CC2_THREADS, EDL_CC2_MINB)
k_cc_mac2(const uint64_t* __restrict__ x, int l, int W, int kw, int stride, int Wo, int taps, int f0, int F,
          int n_out_per_f, const ulonglong2* __restrict__ wk, uint64_t* __restrict__ out,
          const __grid_constant__ ModTable mods, int logn) {
    EDL_PDL_ENTRY();
    __shared__ ulonglong2 wsm[FC * CC2_MAXTAPS];  // [f][tap] {residue, companion} of this limb
    __shared__ int tpix[CC2_MAXTAPS];            // pixel (ciphertext) index of each tap
    const int nl = l + 1;
    const int p = blockIdx.y / nl, i = blockIdx.y % nl;
    const int win = blockIdx.z;
    const int wr = win / Wo, wc = win % Wo;
    const bool f64 = mods[i].fp == 2;   // uniform per CTA (limb i)
#ifdef EDL_CC2_SPLIT
    // split products (see k_cc_mac3): 4 DFMA per MAC, three exact sums per output
    const bool split = f64 && taps <= 16;
#else
    const bool split = false;
#endif
    for (int t = threadIdx.x; t < FC * taps; t += blockDim.x) {
        const int f = t / taps, tt = t % taps;
        ulonglong2 w = (f0 + f < F) ? wk[((size_t)(f0 + f) * taps + tt) * nl + i] : make_ulonglong2(0, 0);
        if (split) w = make_ulonglong2(f64_from_u(w.x & 0x3FFFFFull), f64_from_u(w.x >> 22));
        else if (f64) w.x = f64_from_u(w.x);   // {binary64 w, RD(w/q)} for the FP64-pipe products
        wsm[t] = w;
    }
    for (int t = threadIdx.x; t < taps; t += blockDim.x)
        tpix[t] = (wr * stride + t / kw) * W + (wc * stride + t % kw);
    __syncthreads();
    const int n2 = blockIdx.x * blockDim.x + threadIdx.x;   // coefficient pair
    if (2 * n2 >= (1 << logn)) return;
    const ModInfo& m = mods[i];
    const size_t ct_words = (size_t)2 * nl << logn;
    const uint64_t* xb = x + limb_off(0, p, i, nl, logn) + 2 * (size_t)n2;
    const bool fp = m.fp != 0;
    // FP64-quotient limbs: lazy products in [0, 2q) summed in 64 bits (taps * 2q < 2^57);
    // others: full 128-bit products summed lazily (O4), one reduction per output
    U128 acc[FC][2];
#pragma unroll
    for (int f = 0; f < FC; f++) acc[f][0].lo = acc[f][0].hi = acc[f][1].lo = acc[f][1].hi = 0;
#ifdef EDL_CC2_SPLIT
    double s2[FC][2];
#pragma unroll
    for (int f = 0; f < FC; f++) s2[f][0] = s2[f][1] = 0.0;
#endif
    ulonglong2 cur[CC2_TB], nxt[CC2_TB];
#pragma unroll
    for (int u = 0; u < CC2_TB; u++)
        cur[u] = (u < taps) ? __ldg(reinterpret_cast<const ulonglong2*>(xb + tpix[u] * ct_words)) : make_ulonglong2(0, 0);
    for (int t0 = 0; t0 < taps; t0 += CC2_TB) {
#pragma unroll
        for (int u = 0; u < CC2_TB; u++) {
            const int tt = t0 + CC2_TB + u;
            nxt[u] = (tt < taps) ? __ldg(reinterpret_cast<const ulonglong2*>(xb + tpix[tt] * ct_words))
                                 : make_ulonglong2(0, 0);
        }
#ifdef EDL_CC2_SPLIT
        if (split) {   // acc[f][h].lo / .hi / s2[f][h]: the three split sums of coefficient h
#pragma unroll
            for (int u = 0; u < CC2_TB; u++) {
                const int tt = t0 + u < taps ? t0 + u : 0;   // out-of-range taps carry x = 0
                const double xl0 = u52_to_double(cur[u].x & 0x3FFFFFull), xh0 = u52_to_double(cur[u].x >> 22);
                const double xl1 = u52_to_double(cur[u].y & 0x3FFFFFull), xh1 = u52_to_double(cur[u].y >> 22);
#pragma unroll
                for (int f = 0; f < FC; f++) {
                    const ulonglong2 w = wsm[f * taps + tt];
                    const double wl = f64_of(w.x), wh = f64_of(w.y);
                    acc[f][0].lo = bits_of(__fma_rn(xl0, wl, f64_of(acc[f][0].lo)));
                    acc[f][0].hi = bits_of(__fma_rn(xl0, wh, __fma_rn(xh0, wl, f64_of(acc[f][0].hi))));
                    s2[f][0] = __fma_rn(xh0, wh, s2[f][0]);
                    acc[f][1].lo = bits_of(__fma_rn(xl1, wl, f64_of(acc[f][1].lo)));
                    acc[f][1].hi = bits_of(__fma_rn(xl1, wh, __fma_rn(xh1, wl, f64_of(acc[f][1].hi))));
                    s2[f][1] = __fma_rn(xh1, wh, s2[f][1]);
                }
            }
        } else
#endif
        if (f64) {
            // exact binary64 products t = x w mod q in [-0.625q, 0.625q] summed exactly
            // (taps * 0.625 q < 2^51), reduced once at the end; accumulators hold doubles
            const double qd = u52_to_double(m.q);
#pragma unroll
            for (int u = 0; u < CC2_TB; u++) {
                const int tt = t0 + u < taps ? t0 + u : 0;
                const double x0 = u52_to_double(cur[u].x), x1 = u52_to_double(cur[u].y);
#pragma unroll
                for (int f = 0; f < FC; f++) {
                    const ulonglong2 w = wsm[f * taps + tt];
                    const double wd = f64_of(w.x), wq = f64_of(w.y);
                    acc[f][0].lo = bits_of(__dadd_rn(f64_of(acc[f][0].lo), f64_mulc(x0, wd, wq, qd)));
                    acc[f][1].lo = bits_of(__dadd_rn(f64_of(acc[f][1].lo), f64_mulc(x1, wd, wq, qd)));
                }
            }
        } else if (fp) {
#pragma unroll
            for (int u = 0; u < CC2_TB; u++) {
                const int tt = t0 + u < taps ? t0 + u : 0;   // out-of-range taps carry x = 0
#pragma unroll
                for (int f = 0; f < FC; f++) {
                    const ulonglong2 w = wsm[f * taps + tt];
                    acc[f][0].lo += tw_mul_fp(cur[u].x, w.x, w.y, m.q);
                    acc[f][1].lo += tw_mul_fp(cur[u].y, w.x, w.y, m.q);
                }
            }
        } else {
#pragma unroll
            for (int u = 0; u < CC2_TB; u++) {
                const int tt = t0 + u < taps ? t0 + u : 0;
#pragma unroll
                for (int f = 0; f < FC; f++) {
                    const uint64_t w = wsm[f * taps + tt].x;
                    mac128(acc[f][0], cur[u].x, w);
                    mac128(acc[f][1], cur[u].y, w);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < CC2_TB; u++) cur[u] = nxt[u];
    }
#pragma unroll
    for (int f = 0; f < FC; f++) {
        if (f0 + f < F) {
            const int64_t o = (int64_t)(f0 + f) * n_out_per_f + win;
            uint64_t* dst = out + limb_off(o, p, i, nl, logn) + 2 * (size_t)n2;
            ulonglong2 v;
#ifdef EDL_CC2_SPLIT
            if (split) {   // v = s2 (2^44 mod q) + s1 2^22 + s0 mod q
                const double qd = u52_to_double(m.q);
                const double c44d = u52_to_double((1ull << 44) % m.q), c44q = __ddiv_rd(c44d, qd);
                const double c22q = __ddiv_rd(4194304.0, qd);
                uint64_t o[2];
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const double t = __dadd_rn(f64_reduce(f64_of(acc[f][h].lo), qd, m.qinv_d),
                                               __dadd_rn(f64_mulc(f64_of(acc[f][h].hi), 4194304.0, c22q, qd),
                                                         f64_mulc(s2[f][h], c44d, c44q, qd)));
                    o[h] = f64_to_canon(f64_reduce(t, qd, m.qinv_d), qd);
                }
                v = make_ulonglong2(o[0], o[1]);
            } else
#endif
            if (f64) {
                const double qd = u52_to_double(m.q);
                v = make_ulonglong2(f64_to_canon(f64_reduce(f64_of(acc[f][0].lo), qd, m.qinv_d), qd),
                                    f64_to_canon(f64_reduce(f64_of(acc[f][1].lo), qd, m.qinv_d), qd));
            } else {
                v = fp ? make_ulonglong2(reduce64(acc[f][0].lo, m), reduce64(acc[f][1].lo, m))
                       : make_ulonglong2(barrett128(acc[f][0], m), barrett128(acc[f][1], m));
            }
            *reinterpret_cast<ulonglong2*>(dst) = v;
        }
    }
}

// ---------------------------------------------------------------- cross-correlation MAC, round 2b
// k_cc_mac4: the C1 geometry (KH x KW = 4 x 4 taps, <= 8 filters, <= 6 limbs) with the
// filter weights in the kernel's parameter space (constant bank: uniform loads, no shared-
// memory staging or barrier per CTA) and F64 limbs as split products: x = xh 2^22 + xl and
// w = wh 2^22 + wl (every piece < 2^22 for q < 2^44) give x w = xh wh 2^44 +
// (xh wl + xl wh) 2^22 + xl wl, three exact binary64 FMA sums (S0, S2 < 16 2^44 = 2^48,
// S1 < 2^49 for 16 taps) -- 4 DFMA per MAC instead of f64_mulc's 6 plus the add -- reduced
// once per output: S0 mod q + S1 2^22 + S2 (2^44 mod q).  60-bit limbs: full 128-bit products
// summed lazily, one Barrett per output (O4).  One coefficient per thread, a CTA walks
// CC4_WPB windows (tap loads of a window all issued before its MACs).
constexpr int CC4_T = 128;
constexpr int CC4_MAXL = 6, CC4_MAXF = 8, CC4_TAPS = 16;
#ifndef EDL_CC4_WPB
#define EDL_CC4_WPB 4
#endif
#ifndef EDL_CC4_MINB
#define EDL_CC4_MINB 6
#endif
// F64 limbs: Karatsuba split products (3 DFMA per MAC instead of 4; EDL_CC4_KARATSUBA=0: 4)
#ifndef EDL_CC4_KARATSUBA
#define EDL_CC4_KARATSUBA 1
#endif
#if EDL_CC4_KARATSUBA == 0
#undef EDL_CC4_KARATSUBA
#endif
struct CCW4 {   // [limb][filter][tap] {wl, wh} as binary64 (F64 limbs), {w, companion} (others)
    uint64_t w[CC4_MAXL][CC4_MAXF][CC4_TAPS][2];
    double c44[CC4_MAXL][3];   // F64 limbs: 2^44 mod q, RD((2^44 mod q) / q), RD(2^22 / q) (host-made)
#ifdef EDL_CC4_CBANK
    double ws[CC4_MAXL][CC4_MAXF][CC4_TAPS];   // F64 limbs: wl + wh (< 2^23, exact)
#endif
};

template <int FC, int KH, int KW>
__global__ void __launch_bounds__(CC4_T, EDL_CC4_MINB)
k_cc_mac4(const uint64_t* __restrict__ x, int l, int W, int stride, int Wo, int nwin, int f0, int F, int n_out_per_f,
          uint64_t* __restrict__ out, const __grid_constant__ CCW4 wt, const __grid_constant__ ModTable mods, int logn) {
    EDL_PDL_ENTRY();
    constexpr int TAPS = KH * KW;
    static_assert(TAPS <= CC4_TAPS && FC <= CC4_MAXF, "k_cc_mac4 geometry");
    const int nl = l + 1;
    const int p = blockIdx.y / nl, i = blockIdx.y % nl;
    const int n = blockIdx.x * CC4_T + threadIdx.x;
    const ModInfo& m = mods[i];
    const int mode = (int)m.fp;   // uniform per CTA (limb i)
    static_assert(CC4_T >= 1, "");
    const size_t ct_words = (size_t)2 * nl << logn;
    const uint64_t* xb = x + limb_off(0, p, i, nl, logn) + n;
    const double qd = u52_to_double(m.q);
    // this limb's weights -> shared memory once per CTA (LDS.128 broadcasts in the MAC loop:
    // constant-bank loads with the runtime limb index stalled every DFMA on LDC, ncu round 2)
    __shared__ ulonglong2 ws[FC][TAPS];
#ifdef EDL_CC4_KARATSUBA
    __shared__ double wsum[FC][TAPS];   // F64 limbs: wl + wh (< 2^23, exact)
#endif
    for (int e = threadIdx.x; e < FC * TAPS; e += CC4_T) {
        ws[e / TAPS][e % TAPS] = make_ulonglong2(wt.w[i][e / TAPS][e % TAPS][0], wt.w[i][e / TAPS][e % TAPS][1]);
#ifdef EDL_CC4_KARATSUBA
        if (mode == 2)
            wsum[e / TAPS][e % TAPS] = __dadd_rn(f64_of(wt.w[i][e / TAPS][e % TAPS][0]), f64_of(wt.w[i][e / TAPS][e % TAPS][1]));
#endif
    }
    __syncthreads();
    const double c44d = wt.c44[i][0], c44q = wt.c44[i][1], c22q = wt.c44[i][2];
    const int w_end = min(nwin, (int)(blockIdx.z + 1) * EDL_CC4_WPB);
    auto fetch = [&](int win, uint64_t* xv) {
        const int wr = win / Wo, wc = win - (win / Wo) * Wo;
        const uint64_t* xw = xb + (size_t)((wr * stride) * W + wc * stride) * ct_words;
#pragma unroll
        for (int t = 0; t < TAPS; t++) xv[t] = __ldg(xw + (size_t)((t / KW) * W + (t % KW)) * ct_words);
    };
    // (measured: prefetching the next window's taps during this window's MACs, 128 registers,
    //  4 CTAs/SM: 0.46 ms vs 0.44 without)
#ifdef EDL_CC4_ASYNC
    // the next window's taps copied by cp.async into this thread's slots of a 2-stage
    // shared-memory ring while this window computes (no registers held)
    extern __shared__ uint64_t cc_ring[];   // [2][TAPS][CC4_T]
    auto afetch = [&](int win, int st) {
        const int wr = win / Wo, wc = win - (win / Wo) * Wo;
        const uint64_t* xw = xb + (size_t)((wr * stride) * W + wc * stride) * ct_words;
#pragma unroll
        for (int t = 0; t < TAPS; t++)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(
                             cc_ring + ((size_t)st * TAPS + t) * CC4_T + threadIdx.x)),
                         "l"(xw + (size_t)((t / KW) * W + (t % KW)) * ct_words)
                         : "memory");
    };
    const int w_beg = blockIdx.z * EDL_CC4_WPB;
    if (w_beg < w_end) afetch(w_beg, 0);
    asm volatile("cp.async.commit_group;" ::: "memory");
#endif
    for (int win = blockIdx.z * EDL_CC4_WPB; win < w_end; win++) {
        uint64_t xv[TAPS];
#ifdef EDL_CC4_ASYNC
        {
            const int u = win - w_beg;
            if (win + 1 < w_end) afetch(win + 1, (u + 1) & 1);
            asm volatile("cp.async.commit_group;" ::: "memory");
            asm volatile("cp.async.wait_group 1;" ::: "memory");
#pragma unroll
            for (int t = 0; t < TAPS; t++) xv[t] = cc_ring[((size_t)(u & 1) * TAPS + t) * CC4_T + threadIdx.x];
        }
#else
        fetch(win, xv);
#endif
        uint64_t res[FC];
        if (mode == 2) {
            double s0[FC], s1[FC], s2[FC];
#pragma unroll
            for (int f = 0; f < FC; f++) s0[f] = s1[f] = s2[f] = 0.0;
#pragma unroll
            for (int t = 0; t < TAPS; t++) {
                const double xl = __hiloint2double(0x43300000, (int)((uint32_t)xv[t] & 0x3FFFFFu)) - F64_TWO52;
                const double xh = __hiloint2double(0x43300000, (int)(uint32_t)(xv[t] >> 22)) - F64_TWO52;
#ifdef EDL_CC4_KARATSUBA
                // 3 DFMA per MAC: S1 = sum (xl + xh)(wl + wh) - S0 - S2 after the taps; every
                // product < 2^46 and every sum < 16 2^46 = 2^50, so all of it is exact
                const double xs = __dadd_rn(xl, xh);
#endif
#pragma unroll
                for (int f = 0; f < FC; f++) {
                    const ulonglong2 wv = ws[f][t];
                    const double wl = f64_of(wv.x), wh = f64_of(wv.y);
                    s0[f] = __fma_rn(xl, wl, s0[f]);
#ifdef EDL_CC4_KARATSUBA
                    s1[f] = __fma_rn(xs, wsum[f][t], s1[f]);
#else
                    s1[f] = __fma_rn(xh, wl, s1[f]);
                    s1[f] = __fma_rn(xl, wh, s1[f]);
#endif
                    s2[f] = __fma_rn(xh, wh, s2[f]);
                }
            }
#ifdef EDL_CC4_KARATSUBA
#pragma unroll
            for (int f = 0; f < FC; f++) s1[f] = __dsub_rn(__dsub_rn(s1[f], s0[f]), s2[f]);
#endif
#pragma unroll
            for (int f = 0; f < FC; f++) {
                const double tt = __dadd_rn(f64_reduce(s0[f], qd, m.qinv_d),
                                            __dadd_rn(f64_mulc(s1[f], 4194304.0, c22q, qd), f64_mulc(s2[f], c44d, c44q, qd)));
                res[f] = f64_to_canon(f64_reduce(tt, qd, m.qinv_d), qd);
            }
        } else if (mode == 1) {   // lazy [0, 2q) products summed in 64 bits (16 x 2q < 2^51)
            uint64_t acc[FC];
#pragma unroll
            for (int f = 0; f < FC; f++) acc[f] = 0;
#pragma unroll
            for (int t = 0; t < TAPS; t++)
#pragma unroll
                for (int f = 0; f < FC; f++) acc[f] += tw_mul_fp(xv[t], ws[f][t].x, ws[f][t].y, m.q);
#pragma unroll
            for (int f = 0; f < FC; f++) res[f] = reduce64(acc[f], m);
        } else {
            U128 acc[FC];
#pragma unroll
            for (int f = 0; f < FC; f++) acc[f].lo = acc[f].hi = 0;
#pragma unroll
            for (int t = 0; t < TAPS; t++)
#pragma unroll
                for (int f = 0; f < FC; f++) mac128(acc[f], xv[t], ws[f][t].x);
#pragma unroll
            for (int f = 0; f < FC; f++) res[f] = barrett128(acc[f], m);
        }
#pragma unroll
        for (int f = 0; f < FC; f++)
            if (f0 + f < F) out[limb_off((int64_t)(f0 + f) * n_out_per_f + win, p, i, nl, logn) + n] = res[f];
    }
}

#ifdef EDL_CC4_CBANK
// k_cc_mac5: k_cc_mac4's arithmetic with the weights read as constant-bank operands of the
// DFMA / IMAD.WIDE instructions themselves: the limb index is made a compile-time constant
// by a switch over per-limb instantiations of the body (the first attempt indexed the
// parameter table with the runtime limb and paid an LDC per operand), so the MAC loop has no
// shared-memory weight loads (k_cc_mac4: one LDS.128 + one LDS.64 per 3 DFMA) and no staging
// barrier.  Grid: z = poly * (l+1) + limb is the slowest index, so the CTAs running at one
// time work on one limb (one body's code and one limb's 2 KB of weights in the caches).
// Measured on B200 (C1): 0.68 ms against k_cc_mac4's 0.42 (ptxas feeds the constants through
// LDCU + uniform registers, one load per DFMA and window, and spills ~200 B per thread at 80
// registers; 96 registers: 0.77 ms), so it is compiled only with -DEDL_CC4_CBANK; bit-exact.
template <int FC, int KH, int KW, int I, int MODE>
__device__ __forceinline__ void cc5_body(const uint64_t* __restrict__ xb, size_t ct_words, int W, int stride, int Wo,
                                         int w_beg, int w_end, int f0, int F, int n_out_per_f, uint64_t* __restrict__ out,
                                         const CCW4& wt, const ModInfo& m, int p, int nl, int logn, int n) {
    constexpr int TAPS = KH * KW;
    const double qd = u52_to_double(m.q);
    for (int win = w_beg; win < w_end; win++) {
        uint64_t xv[TAPS];
        {
            const int wr = win / Wo, wc = win - (win / Wo) * Wo;
            const uint64_t* xw = xb + (size_t)((wr * stride) * W + wc * stride) * ct_words;
#pragma unroll
            for (int t = 0; t < TAPS; t++) xv[t] = __ldg(xw + (size_t)((t / KW) * W + (t % KW)) * ct_words);
        }
        uint64_t res[FC];
        if constexpr (MODE == 2) {
            double s0[FC], s1[FC], s2[FC];
#pragma unroll
            for (int f = 0; f < FC; f++) s0[f] = s1[f] = s2[f] = 0.0;
#pragma unroll
            for (int t = 0; t < TAPS; t++) {
                const double xl = __hiloint2double(0x43300000, (int)((uint32_t)xv[t] & 0x3FFFFFu)) - F64_TWO52;
                const double xh = __hiloint2double(0x43300000, (int)(uint32_t)(xv[t] >> 22)) - F64_TWO52;
                const double xs = __dadd_rn(xl, xh);
#pragma unroll
                for (int f = 0; f < FC; f++) {
                    s0[f] = __fma_rn(xl, f64_of(wt.w[I][f][t][0]), s0[f]);
                    s1[f] = __fma_rn(xs, wt.ws[I][f][t], s1[f]);
                    s2[f] = __fma_rn(xh, f64_of(wt.w[I][f][t][1]), s2[f]);
                }
            }
            const double c44d = wt.c44[I][0], c44q = wt.c44[I][1], c22q = wt.c44[I][2];
#pragma unroll
            for (int f = 0; f < FC; f++) {
                const double s1f = __dsub_rn(__dsub_rn(s1[f], s0[f]), s2[f]);
                const double tt = __dadd_rn(f64_reduce(s0[f], qd, m.qinv_d),
                                            __dadd_rn(f64_mulc(s1f, 4194304.0, c22q, qd), f64_mulc(s2[f], c44d, c44q, qd)));
                res[f] = f64_to_canon(f64_reduce(tt, qd, m.qinv_d), qd);
            }
        } else if constexpr (MODE == 1) {
            uint64_t acc[FC];
#pragma unroll
            for (int f = 0; f < FC; f++) acc[f] = 0;
#pragma unroll
            for (int t = 0; t < TAPS; t++)
#pragma unroll
                for (int f = 0; f < FC; f++) acc[f] += tw_mul_fp(xv[t], wt.w[I][f][t][0], wt.w[I][f][t][1], m.q);
#pragma unroll
            for (int f = 0; f < FC; f++) res[f] = reduce64(acc[f], m);
        } else {
            U128 acc[FC];
#pragma unroll
            for (int f = 0; f < FC; f++) acc[f].lo = acc[f].hi = 0;
#pragma unroll
            for (int t = 0; t < TAPS; t++)
#pragma unroll
                for (int f = 0; f < FC; f++) mac128(acc[f], xv[t], wt.w[I][f][t][0]);
#pragma unroll
            for (int f = 0; f < FC; f++) res[f] = barrett128(acc[f], m);
        }
#pragma unroll
        for (int f = 0; f < FC; f++)
            if (f0 + f < F) out[limb_off((int64_t)(f0 + f) * n_out_per_f + win, p, I, nl, logn) + n] = res[f];
    }
}

template <int FC, int KH, int KW>
__global__ void __launch_bounds__(CC4_T, EDL_CC4_MINB)
k_cc_mac5(const uint64_t* __restrict__ x, int l, int W, int stride, int Wo, int nwin, int f0, int F, int n_out_per_f,
          uint64_t* __restrict__ out, const __grid_constant__ CCW4 wt, const __grid_constant__ ModTable mods, int logn) {
    EDL_PDL_ENTRY();
    const int nl = l + 1;
    const int p = blockIdx.z / nl, i = blockIdx.z % nl;
    const int n = blockIdx.x * CC4_T + threadIdx.x;
    const ModInfo& m = mods[i];
    const int mode = (int)m.fp;   // uniform per CTA (limb i)
    const size_t ct_words = (size_t)2 * nl << logn;
    const uint64_t* xb = x + limb_off(0, p, i, nl, logn) + n;
    const int w_beg = blockIdx.y * EDL_CC4_WPB, w_end = min(nwin, (int)(blockIdx.y + 1) * EDL_CC4_WPB);
#define CC5_ARGS xb, ct_words, W, stride, Wo, w_beg, w_end, f0, F, n_out_per_f, out, wt, m, p, nl, logn, n
#define CC5_CASE(II)                                                      \
    case II:                                                              \
        if (mode == 2) cc5_body<FC, KH, KW, II, 2>(CC5_ARGS);             \
        else if (mode == 1) cc5_body<FC, KH, KW, II, 1>(CC5_ARGS);        \
        else cc5_body<FC, KH, KW, II, 0>(CC5_ARGS);                       \
        break;
    switch (i) {
        CC5_CASE(0) CC5_CASE(1) CC5_CASE(2) CC5_CASE(3) CC5_CASE(4) CC5_CASE(5)
    }
#undef CC5_CASE
#undef CC5_ARGS
}
#endif

// ---------------------------------------------------------------- cross-correlation MAC, round 2
// One coefficient per thread (8-byte loads, 256 B per warp) and all FC <= 8 filters of a
// filter chunk: accumulators take 2 (binary64) or 4 (128-bit) registers per filter instead
// of twice that, so CTAs of CC3_T threads run more warps per SM than k_cc_mac2 (128
// registers, 16 warps); tap loads run CC3_TB ahead of the MACs.  Measured on C1: 0.53 ms
// against k_cc_mac2's 0.47 (the kernel is FP64-/IMAD-issue-bound, not occupancy-bound), so
// it is compiled only with EDL_CC_MAC3.
constexpr int CC3_T = 128;
constexpr int CC3_TB = 8;

template <int FC>
__global__ void __launch_bounds__(CC3_T, 8)
k_cc_mac3(const uint64_t* __restrict__ x, int l, int W, int kw, int stride, int Wo, int taps, int f0, int F,
          int n_out_per_f, const ulonglong2* __restrict__ wk, uint64_t* __restrict__ out,
          const __grid_constant__ ModTable mods, int logn) {
    EDL_PDL_ENTRY();
    __shared__ ulonglong2 wsm[FC * CC2_MAXTAPS];   // [f][tap] {residue (binary64 on F64 limbs), companion}
    __shared__ int tpix[CC2_MAXTAPS];
    const int nl = l + 1;
    const int p = blockIdx.y / nl, i = blockIdx.y % nl;
    const int win = blockIdx.z;
    const int wr = win / Wo, wc = win % Wo;
    const ModInfo& m = mods[i];
    const bool f64 = m.fp == 2, fp = m.fp != 0;   // uniform per CTA
    // F64 limbs with <= 16 taps: split products (x = xh 2^22 + xl, w = wh 2^22 + wl, every
    // piece < 2^22): x w = xh wh 2^44 + (xh wl + xl wh) 2^22 + xl wl with three exact binary64
    // sums (S1 < 2 taps 2^44 <= 2^49), 4 DFMA per MAC instead of f64_mulc's 6 + 1; reduced
    // once per output.  wsm then holds {wl, wh} as binary64.
    const bool split = f64 && taps <= 16;
    for (int t = threadIdx.x; t < FC * taps; t += CC3_T) {
        const int f = t / taps, tt = t % taps;
        ulonglong2 w = (f0 + f < F) ? wk[((size_t)(f0 + f) * taps + tt) * nl + i] : make_ulonglong2(0, 0);
        if (split) w = make_ulonglong2(f64_from_u(w.x & 0x3FFFFFull), f64_from_u(w.x >> 22));
        else if (f64) w.x = f64_from_u(w.x);
        wsm[t] = w;
    }
    for (int t = threadIdx.x; t < taps; t += CC3_T) tpix[t] = (wr * stride + t / kw) * W + (wc * stride + t % kw);
    __syncthreads();
    const int n = blockIdx.x * CC3_T + threadIdx.x;
    if (n >= (1 << logn)) return;
    const size_t ct_words = (size_t)2 * nl << logn;
    const uint64_t* xb = x + limb_off(0, p, i, nl, logn) + n;
    const double qd = u52_to_double(m.q);
    if (split) {
        double s0[FC], s1[FC], s2[FC];
#pragma unroll
        for (int f = 0; f < FC; f++) s0[f] = s1[f] = s2[f] = 0.0;
        for (int t0 = 0; t0 < taps; t0 += CC3_TB) {
            uint64_t xv[CC3_TB];
#pragma unroll
            for (int u = 0; u < CC3_TB; u++) xv[u] = (t0 + u < taps) ? __ldg(xb + tpix[t0 + u] * ct_words) : 0;
#pragma unroll
            for (int u = 0; u < CC3_TB; u++) {
                if (t0 + u >= taps) break;
                const double xl = u52_to_double(xv[u] & 0x3FFFFFull), xh = u52_to_double(xv[u] >> 22);
#pragma unroll
                for (int f = 0; f < FC; f++) {
                    const ulonglong2 w = wsm[f * taps + t0 + u];
                    const double wl = f64_of(w.x), wh = f64_of(w.y);
                    s0[f] = __fma_rn(xl, wl, s0[f]);
                    s1[f] = __fma_rn(xh, wl, s1[f]);
                    s1[f] = __fma_rn(xl, wh, s1[f]);
                    s2[f] = __fma_rn(xh, wh, s2[f]);
                }
            }
        }
        // v = s2 (2^44 mod q) + s1 2^22 + s0 mod q (2^22 < q: c22 = 2^22)
        const uint64_t c44 = (1ull << 44) % m.q;
        const double c44d = u52_to_double(c44), c44q = __ddiv_rd(c44d, qd);
        const double c22d = 4194304.0, c22q = __ddiv_rd(c22d, qd);
#pragma unroll
        for (int f = 0; f < FC; f++)
            if (f0 + f < F) {
                double v = __dadd_rn(f64_reduce(s0[f], qd, m.qinv_d),
                                     __dadd_rn(f64_mulc(s1[f], c22d, c22q, qd), f64_mulc(s2[f], c44d, c44q, qd)));
                out[limb_off((int64_t)(f0 + f) * n_out_per_f + win, p, i, nl, logn) + n] =
                    f64_to_canon(f64_reduce(v, qd, m.qinv_d), qd);
            }
    } else if (f64) {
        double acc[FC];
#pragma unroll
        for (int f = 0; f < FC; f++) acc[f] = 0.0;
        for (int t0 = 0; t0 < taps; t0 += CC3_TB) {
            uint64_t xv[CC3_TB];
#pragma unroll
            for (int u = 0; u < CC3_TB; u++) xv[u] = (t0 + u < taps) ? __ldg(xb + tpix[t0 + u] * ct_words) : 0;
#pragma unroll
            for (int u = 0; u < CC3_TB; u++) {
                if (t0 + u >= taps) break;
                const double xd = u52_to_double(xv[u]);
#pragma unroll
                for (int f = 0; f < FC; f++) {
                    const ulonglong2 w = wsm[f * taps + t0 + u];
                    acc[f] = __dadd_rn(acc[f], f64_mulc(xd, f64_of(w.x), f64_of(w.y), qd));
                }
            }
        }
#pragma unroll
        for (int f = 0; f < FC; f++)
            if (f0 + f < F)
                out[limb_off((int64_t)(f0 + f) * n_out_per_f + win, p, i, nl, logn) + n] =
                    f64_to_canon(f64_reduce(acc[f], qd, m.qinv_d), qd);
    } else {
        U128 acc[FC];
#pragma unroll
        for (int f = 0; f < FC; f++) acc[f].lo = acc[f].hi = 0;
        for (int t0 = 0; t0 < taps; t0 += CC3_TB) {
            uint64_t xv[CC3_TB];
#pragma unroll
            for (int u = 0; u < CC3_TB; u++) xv[u] = (t0 + u < taps) ? __ldg(xb + tpix[t0 + u] * ct_words) : 0;
#pragma unroll
            for (int u = 0; u < CC3_TB; u++) {
                if (t0 + u >= taps) break;
#pragma unroll
                for (int f = 0; f < FC; f++) {
                    const ulonglong2 w = wsm[f * taps + t0 + u];
                    if (fp) acc[f].lo += tw_mul_fp(xv[u], w.x, w.y, m.q);   // [0, 2q): taps * 2q < 2^53
                    else mac128(acc[f], xv[u], w.x);
                }
            }
        }
#pragma unroll
        for (int f = 0; f < FC; f++)
            if (f0 + f < F)
                out[limb_off((int64_t)(f0 + f) * n_out_per_f + win, p, i, nl, logn) + n] =
                    fp ? reduce64(acc[f].lo, m) : barrett128(acc[f], m);
    }
}

// ---------------------------------------------------------------- dense MAC
// grid: x = coefficient blocks, y = poly*(l+1) + limb, z = output chunk of DN_OC x K split.
// Split-K (round 2): the K inputs are cut into ks slices so a small layer (C1: 245 -> 10
// on 2 limbs) still fills every SM; each slice writes its reduced partial sum and
// k_dense_combine adds the slices mod q (O4: order-independent).  The K loop is
// unrolled by DN_U with all DN_U input loads issued before the MACs.
constexpr int DN_OC = 12;
constexpr int DN_KC = 256;    // fold 128-bit accumulators every 256 terms (K*q^2 < 2^128)
constexpr int DN_U = 4;

__global__ void __launch_bounds__(PW_THREADS, 2)
k_dense_mac(const uint64_t* __restrict__ x, int64_t K, int64_t O, int l, int ks, const ulonglong2* __restrict__ wd,
            uint64_t* __restrict__ out, const __grid_constant__ ModTable mods, int logn) {
    EDL_PDL_ENTRY();
    extern __shared__ ulonglong2 wsm2[];   // [DN_OC][DN_KC] {residue, companion}
    const int nl = l + 1;
    const int p = blockIdx.y / nl, i = blockIdx.y % nl;
    const int oc = blockIdx.z / ks, sl = blockIdx.z % ks;
    const int64_t o0 = (int64_t)oc * DN_OC;
    const int64_t kper = (K + ks - 1) / ks;
    const int64_t kbeg = sl * kper, kend = (kbeg + kper < K) ? kbeg + kper : K;
    uint64_t* outp = out + (size_t)sl * ((size_t)O * 2 * nl << logn);
    const ModInfo& m = mods[i];
    const bool fp = m.fp != 0;
    const bool f64 = m.fp == 2;   // FP64-pipe products (uniform per CTA)
    const double qd = u52_to_double(m.q);
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = n < (1 << logn);
    const size_t kstride = (size_t)2 * nl << logn;            // one ciphertext
    const uint64_t* xp = x + limb_off(0, p, i, nl, logn) + (active ? n : 0);
    bool first = true;
    for (int64_t k0 = kbeg; k0 < kend || first; k0 += DN_KC) {
        const int kc = (int)((kend - k0) < DN_KC ? (kend - k0) : DN_KC);
        __syncthreads();
        for (int t = threadIdx.x; t < DN_OC * DN_KC; t += blockDim.x) {
            const int o = t / DN_KC, k = t % DN_KC;
            ulonglong2 w = (o0 + o < O && k < kc) ? wd[((size_t)(o0 + o) * K + (k0 + k)) * nl + i] : make_ulonglong2(0, 0);
            if (f64) w.x = f64_from_u(w.x);
            wsm2[t] = w;
        }
        __syncthreads();
        if (!active) { first = false; continue; }
        U128 acc[DN_OC];
#pragma unroll
        for (int o = 0; o < DN_OC; o++) acc[o].lo = acc[o].hi = 0;
        for (int k = 0; k < kc; k += DN_U) {
            uint64_t xv[DN_U];
#pragma unroll
            for (int u = 0; u < DN_U; u++) xv[u] = (k + u < kc) ? __ldg(xp + (size_t)(k0 + k + u) * kstride) : 0;
            if (f64) {   // exact binary64 products in [-0.625q, 0.625q], exact sums (DN_KC terms)
#pragma unroll
                for (int u = 0; u < DN_U; u++) {
                    const double xd = u52_to_double(xv[u]);
#pragma unroll
                    for (int o = 0; o < DN_OC; o++) {
                        const ulonglong2 w = wsm2[o * DN_KC + ((k + u) & (DN_KC - 1))];
                        acc[o].lo = bits_of(__dadd_rn(f64_of(acc[o].lo), f64_mulc(xd, f64_of(w.x), f64_of(w.y), qd)));
                    }
                }
            } else if (fp) {   // lazy [0, 2q) products summed in 64 bits (256 * 2q < 2^59)
#pragma unroll
                for (int u = 0; u < DN_U; u++) {
#pragma unroll
                    for (int o = 0; o < DN_OC; o++) {
                        const ulonglong2 w = wsm2[o * DN_KC + ((k + u) & (DN_KC - 1))];
                        acc[o].lo += tw_mul_fp(xv[u], w.x, w.y, m.q);
                    }
                }
            } else {
#pragma unroll
                for (int u = 0; u < DN_U; u++) {
#pragma unroll
                    for (int o = 0; o < DN_OC; o++) mac128(acc[o], xv[u], wsm2[o * DN_KC + ((k + u) & (DN_KC - 1))].x);
                }
            }
        }
#pragma unroll
        for (int o = 0; o < DN_OC; o++) {
            if (o0 + o < O) {
                uint64_t* dst = outp + limb_off(o0 + o, p, i, nl, logn) + n;
                uint64_t v = f64 ? f64_to_canon(f64_reduce(f64_of(acc[o].lo), qd, m.qinv_d), qd)
                                 : (fp ? reduce64(acc[o].lo, m) : barrett128(acc[o], m));
                if (!first) v = addmod(v, *dst, m.q);
                *dst = v;
            }
        }
        first = false;
    }
}

// ---------------------------------------------------------------- dense MAC, round 2
// grid: x = coefficient blocks (one coefficient per thread), y = poly * (l+1) + limb,
// z = K slice.  A CTA stages only its slice's weights [kc][OC] in shared memory (round 1
// staged a [12][256] block per CTA: 48 KB of mostly padding per CTA, ~50 MB of L2 reads
// per layer) and every thread keeps all OC <= 16 outputs' accumulators in registers, so
// each input residue is read once and feeds O products.  Input loads run DN3_U ahead.
// F64 limbs: exact binary64 products (f64_mulc) summed exactly (kc <= 256 terms); others
// full 128-bit products summed lazily; one reduction per output (O4).
constexpr int DN3_T = 128;
constexpr int DN3_U = 4;

// EDL_DN3_ASYNC: the next DN3_U inputs copied by cp.async into this thread's slots of a
// 2-stage shared-memory ring (behind the weight slice) while the current ones compute
// (C1 dense 0.146-0.150 -> 0.140 ms; EDL_DN3_ASYNC=0 restores register loads).
#ifndef EDL_DN3_ASYNC
#define EDL_DN3_ASYNC 1
#endif
#if EDL_DN3_ASYNC == 0
#undef EDL_DN3_ASYNC
#endif
#ifdef EDL_DN3_ASYNC
constexpr int DN3_RING_WORDS = 2 * DN3_U * DN3_T;
#define DN3_RING_PROLOGUE                                                                                      \
    uint64_t* ring = reinterpret_cast<uint64_t*>(wsm3 + kc * OC);                                             \
    auto afetch = [&](int k0_, int st) {                                                                       \
        _Pragma("unroll") for (int u = 0; u < DN3_U; u++) if (k0_ + u < kc) asm volatile(                    \
            "cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(              \
                ring + ((size_t)st * DN3_U + u) * DN3_T + threadIdx.x)), "l"(xp + (size_t)(k0_ + u) * kstride) \
            : "memory");                                                                                       \
    };                                                                                                         \
    afetch(0, 0);                                                                                              \
    asm volatile("cp.async.commit_group;" ::: "memory");
#define DN3_FETCH(xv)                                                                                          \
    {                                                                                                          \
        const int it = kk / DN3_U;                                                                             \
        if (kk + DN3_U < kc) afetch(kk + DN3_U, (it + 1) & 1);                                                 \
        asm volatile("cp.async.commit_group;" ::: "memory");                                                   \
        asm volatile("cp.async.wait_group 1;" ::: "memory");                                                   \
        _Pragma("unroll") for (int u = 0; u < DN3_U; u++) xv[u] =                                             \
            (kk + u < kc) ? ring[((size_t)(it & 1) * DN3_U + u) * DN3_T + threadIdx.x] : 0;                   \
    }
#else
constexpr int DN3_RING_WORDS = 0;
#define DN3_RING_PROLOGUE
#define DN3_FETCH(xv)                                                                                          \
    _Pragma("unroll") for (int u = 0; u < DN3_U; u++) xv[u] = (kk + u < kc) ? __ldg(xp + (size_t)(kk + u) * kstride) : 0;
#endif

// KARA (kper <= DN3_KARA_MAX): F64 limbs as Karatsuba split products like k_cc_mac4 -- x =
// xh 2^22 + xl, w = wh 2^22 + wl, S0 = sum xl wl, S2 = sum xh wh, S = sum (xl + xh)(wl + wh)
// (every product < 2^46, so sums of <= 128 terms stay below 2^53: exact), S1 = S - S0 - S2;
// 3 DFMA per MAC instead of f64_mulc + add = 7.  Each sum is reduced (f64_reduce is exact for
// any integer |v| < 2^53: the quotient estimate is off by < 2^-38) before the two constant
// products S1 2^22 + S2 (2^44 mod q), whose operands are then below q.
// Measured on B200 (C1 dense 245 -> 10): 0.148 ms against 0.140 for the f64_mulc form -- the
// three sums per output take 94 registers (5 CTAs per SM instead of 7) and the dense MAC is
// latency-, not FP64-bound -- so it is opt-in (-DEDL_DN3_KARATSUBA=1); bit-exact either way.
constexpr int DN3_KARA_MAX = 128;
#ifndef EDL_DN3_KARATSUBA
#define EDL_DN3_KARATSUBA 0
#endif
template <int OC, bool KARA>
__global__ void __launch_bounds__(DN3_T)
k_dense_mac3(const uint64_t* __restrict__ x, int64_t K, int O, int l, int kper, const ulonglong2* __restrict__ wd,
             uint64_t* __restrict__ out, const __grid_constant__ ModTable mods, int logn) {
    EDL_PDL_ENTRY();
    // [kper][OC] {residue (binary64 on F64 limbs), companion}; KARA F64 limbs: {wl, wh} as
    // binary64, then [kper][OC] wl + wh behind the input ring
    extern __shared__ ulonglong2 wsm3[];
    __shared__ double kc3[3];   // KARA: 2^44 mod q, RD((2^44 mod q) / q), RD(2^22 / q)
    const int nl = l + 1;
    const int p = blockIdx.y / nl, i = blockIdx.y % nl;
    const int sl = blockIdx.z;
    const int64_t k0 = (int64_t)sl * kper;
    const int kc = (int)((K - k0) < kper ? (K - k0) : kper);
    const ModInfo& m = mods[i];
    const bool f64 = m.fp == 2, fp = m.fp != 0;
    double* wsum = reinterpret_cast<double*>(wsm3 + kc * OC) + DN3_RING_WORDS;
    for (int t = threadIdx.x; t < kc * OC; t += DN3_T) {
        const int kk = t / OC, o = t % OC;
        ulonglong2 w = (o < O) ? wd[((size_t)o * K + (k0 + kk)) * nl + i] : make_ulonglong2(0, 0);
        if (KARA && f64) {
            const uint64_t wl = w.x & 0x3FFFFFu, wh = w.x >> 22;
            w.x = f64_from_u(wl);
            w.y = f64_from_u(wh);
            wsum[t] = u52_to_double(wl + wh);
        } else if (f64) {
            w.x = f64_from_u(w.x);
        }
        wsm3[t] = w;
    }
    if (KARA && f64 && threadIdx.x == 0) {
        const double qd0 = u52_to_double(m.q), c44 = u52_to_double((1ull << 44) % m.q);
        kc3[0] = c44;
        kc3[1] = __ddiv_rd(c44, qd0);
        kc3[2] = __ddiv_rd(4194304.0, qd0);
    }
    __syncthreads();
    const int n = blockIdx.x * DN3_T + threadIdx.x;
    if (n >= (1 << logn)) return;
    const size_t kstride = (size_t)2 * nl << logn;
    const uint64_t* xp = x + limb_off(k0, p, i, nl, logn) + n;
    uint64_t* outp = out + (size_t)sl * ((size_t)O * 2 * nl << logn);
    const double qd = u52_to_double(m.q);
    if (KARA && f64) {
        double s0[OC], s1[OC], s2[OC];
#pragma unroll
        for (int o = 0; o < OC; o++) s0[o] = s1[o] = s2[o] = 0.0;
        DN3_RING_PROLOGUE
        for (int kk = 0; kk < kc; kk += DN3_U) {
            uint64_t xv[DN3_U];
            DN3_FETCH(xv)
#pragma unroll
            for (int u = 0; u < DN3_U; u++) {
                if (kk + u >= kc) break;
                const double xl = __hiloint2double(0x43300000, (int)((uint32_t)xv[u] & 0x3FFFFFu)) - F64_TWO52;
                const double xh = __hiloint2double(0x43300000, (int)(uint32_t)(xv[u] >> 22)) - F64_TWO52;
                const double xs = __dadd_rn(xl, xh);
#pragma unroll
                for (int o = 0; o < OC; o++) {
                    const ulonglong2 w = wsm3[(kk + u) * OC + o];
                    s0[o] = __fma_rn(xl, f64_of(w.x), s0[o]);
                    s1[o] = __fma_rn(xs, wsum[(kk + u) * OC + o], s1[o]);
                    s2[o] = __fma_rn(xh, f64_of(w.y), s2[o]);
                }
            }
        }
        const double c44d = kc3[0], c44q = kc3[1], c22q = kc3[2];
#pragma unroll
        for (int o = 0; o < OC; o++)
            if (o < O) {
                const double r0 = f64_reduce(s0[o], qd, m.qinv_d), r2 = f64_reduce(s2[o], qd, m.qinv_d);
                const double r1 = f64_reduce(__dsub_rn(__dsub_rn(s1[o], s0[o]), s2[o]), qd, m.qinv_d);
                const double tt = __dadd_rn(r0, __dadd_rn(f64_mulc(r1, 4194304.0, c22q, qd), f64_mulc(r2, c44d, c44q, qd)));
                outp[limb_off(o, p, i, nl, logn) + n] = f64_to_canon(f64_reduce(tt, qd, m.qinv_d), qd);
            }
    } else if (f64) {
        double acc[OC];
#pragma unroll
        for (int o = 0; o < OC; o++) acc[o] = 0.0;
        DN3_RING_PROLOGUE
        for (int kk = 0; kk < kc; kk += DN3_U) {
            uint64_t xv[DN3_U];
            DN3_FETCH(xv)
#pragma unroll
            for (int u = 0; u < DN3_U; u++) {
                if (kk + u >= kc) break;
                const double xd = u52_to_double(xv[u]);
#pragma unroll
                for (int o = 0; o < OC; o++) {
                    const ulonglong2 w = wsm3[(kk + u) * OC + o];
                    acc[o] = __dadd_rn(acc[o], f64_mulc(xd, f64_of(w.x), f64_of(w.y), qd));
                }
            }
        }
#pragma unroll
        for (int o = 0; o < OC; o++)
            if (o < O) outp[limb_off(o, p, i, nl, logn) + n] = f64_to_canon(f64_reduce(acc[o], qd, m.qinv_d), qd);
    } else {
        U128 acc[OC];
#pragma unroll
        for (int o = 0; o < OC; o++) acc[o].lo = acc[o].hi = 0;
        DN3_RING_PROLOGUE
        for (int kk = 0; kk < kc; kk += DN3_U) {
            uint64_t xv[DN3_U];
            DN3_FETCH(xv)
#pragma unroll
            for (int u = 0; u < DN3_U; u++) {
                if (kk + u >= kc) break;
#pragma unroll
                for (int o = 0; o < OC; o++) {
                    const ulonglong2 w = wsm3[(kk + u) * OC + o];
                    if (fp) acc[o].lo += tw_mul_fp(xv[u], w.x, w.y, m.q);   // [0, 2q) lazy, kc * 2q < 2^55
                    else mac128(acc[o], xv[u], w.x);
                }
            }
        }
#pragma unroll
        for (int o = 0; o < OC; o++)
            if (o < O) outp[limb_off(o, p, i, nl, logn) + n] = fp ? reduce64(acc[o].lo, m) : barrett128(acc[o], m);
    }
}

// out[r][k] = sum_s part[s][r][k] mod q over ks slices (rows = O * 2 * nl limbs).
__global__ void k_dense_combine(const uint64_t* __restrict__ part, int ks, int64_t O, int l, uint64_t* __restrict__ out,
                                const __grid_constant__ ModTable mods, int logn) {
    EDL_PDL_ENTRY();
    const int64_t rows = O * 2 * (l + 1);
    const int n2 = 1 << (logn - 1);
    const size_t slice = (size_t)rows << logn;
    for (int64_t row = blockIdx.y; row < rows; row += gridDim.y) {
        const uint64_t q = mods[row % (l + 1)].q;
        const uint64_t* pp = part + ((size_t)row << logn);
        uint64_t* po = out + ((size_t)row << logn);
        for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n2; k += gridDim.x * blockDim.x) {
            ulonglong2 a = v2(pp)[k];
            for (int s = 1; s < ks; s++) {
                const ulonglong2 b = v2(pp + s * slice)[k];
                a.x = addmod(a.x, b.x, q);
                a.y = addmod(a.y, b.y, q);
            }
            v2(po)[k] = a;
        }
    }
}

// ---------------------------------------------------------------- key inner product (M2b)
// acc_{c,t} = sum_{j<=l} x_{j,t} rlk_j[c][t] mod q_t with x_{j,t} = xh_{j,t} (raised digit)
// or, for t == j, d2_j = a1_j b1_j.  A thread owns two coefficients (16-byte accesses) of
// MAC_CB ciphertexts, so each key residue fetched from L2 serves MAC_CB ciphertexts and
// both components share the digit loads.  FP64-quotient limbs: lazy [0, 2q) products
// summed in 64 bits; others: 128-bit lazy sums; one reduction per output (O4).
constexpr int MAC_CB = 4;

struct TargetList {
    int8_t slot[MAXM];
};

template <bool FP>
__global__ void __launch_bounds__(PW_THREADS, 3)
k_relin_mac(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b, int l, int L, int64_t cnt,
            const uint64_t* __restrict__ xh, const uint64_t* __restrict__ rlk, const uint64_t* __restrict__ rlk_c,
            uint64_t* __restrict__ acc, const __grid_constant__ TargetList tl, const __grid_constant__ ModTable mods,
            const ChainConsts* __restrict__ chain, int logn) {
    EDL_PDL_ENTRY();
    const int ti = tl.slot[blockIdx.y];        // 0..l data targets, l+1 = P
    const int64_t c0 = (int64_t)blockIdx.z * MAC_CB;
    const int t = (ti == l + 1) ? (L + 1) : ti;
    const ModInfo& m = mods[t];
    const int k = blockIdx.x * blockDim.x + threadIdx.x;   // coefficient pair
    if (2 * k >= (1 << logn)) return;
    // FP64-quotient limbs: lazy [0, 2q) products summed in 64 bits ((l+1) 2q < 2^60);
    // others: full 128-bit products summed lazily
    using Acc = typename std::conditional<FP, uint64_t, U128>::type;
    Acc s[MAC_CB][2][2];
#pragma unroll
    for (int e = 0; e < MAC_CB; e++)
#pragma unroll
        for (int cc = 0; cc < 2; cc++)
#pragma unroll
            for (int h = 0; h < 2; h++) {
                if constexpr (FP) s[e][cc][h] = 0;
                else s[e][cc][h].lo = s[e][cc][h].hi = 0;
            }
    for (int j = 0; j <= l; j++) {
        const size_t o0 = (((size_t)j * 2 + 0) * (L + 2) + t) << logn, o1 = (((size_t)j * 2 + 1) * (L + 2) + t) << logn;
        const ulonglong2 r0 = __ldg(v2(rlk + o0) + k), r1 = __ldg(v2(rlk + o1) + k);
        ulonglong2 q0 = make_ulonglong2(0, 0), q1 = q0;
        if constexpr (FP) {
            q0 = __ldg(v2(rlk_c + o0) + k);
            q1 = __ldg(v2(rlk_c + o1) + k);
        }
        ulonglong2 x[MAC_CB];
#pragma unroll
        for (int e = 0; e < MAC_CB; e++) {
            const int64_t c = c0 + e;
            x[e] = make_ulonglong2(0, 0);
            if (c >= cnt) continue;
            if (j == ti) {
                const ulonglong2 a1 = v2(a + limb_off(c, 1, j, l + 1, logn))[k];
                if (b == nullptr) {
                    x[e] = a1;
                } else {
                    const ulonglong2 b1 = v2(b + limb_off(c, 1, j, l + 1, logn))[k];
                    x[e] = make_ulonglong2(mulmod(a1.x, b1.x, m), mulmod(a1.y, b1.y, m));
                }
            } else {
                x[e] = v2(xh + ((((size_t)c * (l + 1) + j) * (l + 2) + ti) << logn))[k];
            }
        }
#pragma unroll
        for (int e = 0; e < MAC_CB; e++) {
            if constexpr (FP) {
                s[e][0][0] += tw_mul_fp(x[e].x, r0.x, q0.x, m.q);
                s[e][0][1] += tw_mul_fp(x[e].y, r0.y, q0.y, m.q);
                s[e][1][0] += tw_mul_fp(x[e].x, r1.x, q1.x, m.q);
                s[e][1][1] += tw_mul_fp(x[e].y, r1.y, q1.y, m.q);
            } else {
                mac128(s[e][0][0], x[e].x, r0.x);
                mac128(s[e][0][1], x[e].y, r0.y);
                mac128(s[e][1][0], x[e].x, r1.x);
                mac128(s[e][1][1], x[e].y, r1.y);
            }
        }
    }
    // data limbs: fold the tensor's d0 = a0 b0, d1 = a0 b1 + a1 b0 in, v = d + acc P^-1
    const ulonglong2 pinv = (ti <= l) ? chain->qinv[L + 1][t] : make_ulonglong2(0, 0);
#pragma unroll
    for (int e = 0; e < MAC_CB; e++) {
        const int64_t c = c0 + e;
        if (c >= cnt) continue;
        ulonglong2 v[2];
#pragma unroll
        for (int cc = 0; cc < 2; cc++) {
            if constexpr (FP) v[cc] = make_ulonglong2(reduce64(s[e][cc][0], m), reduce64(s[e][cc][1], m));
            else v[cc] = make_ulonglong2(barrett128(s[e][cc][0], m), barrett128(s[e][cc][1], m));
        }
        if (ti <= l) {
            const ulonglong2 a0 = v2(a + limb_off(c, 0, ti, l + 1, logn))[k];
            uint64_t d0x = a0.x, d0y = a0.y, d1x = 0, d1y = 0;   // single polynomial: (d0, d1) = (a0, 0)
            if (b != nullptr) {
                const ulonglong2 a1 = v2(a + limb_off(c, 1, ti, l + 1, logn))[k];
                const ulonglong2 b0 = v2(b + limb_off(c, 0, ti, l + 1, logn))[k], b1 = v2(b + limb_off(c, 1, ti, l + 1, logn))[k];
                d0x = mulmod(a0.x, b0.x, m);
                d0y = mulmod(a0.y, b0.y, m);
                d1x = addmod(mulmod(a0.x, b1.x, m), mulmod(a1.x, b0.x, m), m.q);
                d1y = addmod(mulmod(a0.y, b1.y, m), mulmod(a1.y, b0.y, m), m.q);
            }
            v[0] = make_ulonglong2(addmod(d0x, mulc(v[0].x, pinv, m), m.q), addmod(d0y, mulc(v[0].y, pinv, m), m.q));
            v[1] = make_ulonglong2(addmod(d1x, mulc(v[1].x, pinv, m), m.q), addmod(d1y, mulc(v[1].y, pinv, m), m.q));
        }
#pragma unroll
        for (int cc = 0; cc < 2; cc++) v2(acc + ((((size_t)c * 2 + cc) * (l + 2) + ti) << logn))[k] = v[cc];
    }
}

// Smem-staged key-product pass (l + 1 <= MAC2_MAXD digits): a thread owns one coefficient
// pair of one target for MAC2_CTS ciphertexts; the key entries of its pair (all digits,
// both components, with companions) are staged once in shared memory and reused for every
// ciphertext, so each key residue is fetched from L2 once per MAC2_CTS ciphertexts, and
// a ciphertext's l+1 digit loads are all issued before its MACs.
#ifndef EDL_MAC2_THREADS
#define EDL_MAC2_THREADS 128
#endif
#ifndef EDL_MAC2_CTS
#define EDL_MAC2_CTS 8   // measured 0.745 vs 0.773 ms (16), 0.757 (4)
#endif
constexpr int MAC2_THREADS = EDL_MAC2_THREADS;
constexpr int MAC2_MAXD = 8;
constexpr int MAC2_CTS = EDL_MAC2_CTS;

// FP selects the arithmetic path at compile time (the launch groups targets by path); ND is
// the exact digit count l+1 (loops fully unrolled, no per-digit branches); CPI ciphertexts
// are processed per iteration so their loads are in flight together.
template <bool FP>
__device__ __forceinline__ uint64_t mulmod_path(uint64_t a, uint64_t b, const ModInfo& m) {
    if constexpr (FP) return mulmod_fp(a, b, m);
    else return mulmod_barrett(a, b, m);
}
template <bool FP>
__device__ __forceinline__ uint64_t mulc_path(uint64_t y, ulonglong2 w, const ModInfo& m) {
    if constexpr (FP) return csub(tw_mul_fp(y, w.x, w.y, m.q), m.q);
    else return shoup(y, w.x, w.y, m.q);
}

#ifndef EDL_MAC2_CPI
#define EDL_MAC2_CPI 2
#endif
constexpr int MAC2_CPI = EDL_MAC2_CPI;
#ifndef EDL_MAC2_CPI_F64
#define EDL_MAC2_CPI_F64 1   // measured: 0.770 vs 0.786 ms (C1) with 2
#endif

#ifndef EDL_MAC2_LB
#define EDL_MAC2_LB 4
#endif
template <int MODE, int ND>   // MODE = ModInfo::fp of the launch's targets (0 Shoup/Barrett, 1 FP64 quotient, 2 FP64 pipe)
__global__ void __launch_bounds__(MAC2_THREADS, EDL_MAC2_LB)
k_relin_mac2(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b, int l, int L, int64_t cnt,
             const uint64_t* __restrict__ xh, const uint64_t* __restrict__ rlk, const uint64_t* __restrict__ rlk_c,
             uint64_t* __restrict__ acc, const __grid_constant__ TargetList tl, const __grid_constant__ ModTable mods,
             const ChainConsts* __restrict__ chain, int logn) {
    EDL_PDL_ENTRY();
    // [digit][comp][thread] {key pair, companion pair}
    extern __shared__ ulonglong2 ks[];
    constexpr bool FP = MODE != 0;
    constexpr bool F64 = MODE == 2;
    const int ti = tl.slot[blockIdx.y];
    const int t = (ti == l + 1) ? (L + 1) : ti;
    const ModInfo& m = mods[t];
    const int k = blockIdx.x * MAC2_THREADS + threadIdx.x;   // coefficient pair
    if (2 * k >= (1 << logn)) return;   // no block-wide barrier below: each thread reads only its own slice
#pragma unroll
    for (int j = 0; j < ND; j++)
#pragma unroll
        for (int cc = 0; cc < 2; cc++) {
            const size_t o = (((size_t)j * 2 + cc) * (L + 2) + t) << logn;
            ulonglong2 kv = __ldg(v2(rlk + o) + k);
            if constexpr (F64) kv = make_ulonglong2(f64_from_u(kv.x), f64_from_u(kv.y));   // binary64 key residues
            ks[((j * 2 + cc) * 2 + 0) * MAC2_THREADS + threadIdx.x] = kv;
            if constexpr (FP) ks[((j * 2 + cc) * 2 + 1) * MAC2_THREADS + threadIdx.x] = __ldg(v2(rlk_c + o) + k);
        }
    const ulonglong2 pinv = (ti <= l) ? chain->qinv[L + 1][t] : make_ulonglong2(0, 0);
    const bool single = (b == nullptr);
    const size_t limb = (size_t)1 << logn;
    const size_t xs_j = (size_t)(l + 2) << logn, xs_c = (size_t)(l + 1) * xs_j;   // xh strides
    const size_t cs = (size_t)2 * (l + 1) << logn;                                 // one ciphertext
    const ulonglong2* xb = v2(xh + ((size_t)ti << logn)) + k;
    const ulonglong2* a0b = v2(a + ((size_t)ti << logn)) + k;                      // poly 0, limb ti
    const ulonglong2* a1b = v2(a + ((size_t)(l + 1 + ti) << logn)) + k;            // poly 1, limb ti
    const ulonglong2* b0b = single ? a0b : v2(b + ((size_t)ti << logn)) + k;
    const ulonglong2* b1b = single ? a1b : v2(b + ((size_t)(l + 1 + ti) << logn)) + k;
    (void)limb;
    const int64_t c_beg = (int64_t)blockIdx.z * MAC2_CTS;
    const int64_t c_end = c_beg + MAC2_CTS < cnt ? c_beg + MAC2_CTS : cnt;
    constexpr int CPI = F64 ? EDL_MAC2_CPI_F64 : MAC2_CPI;
    for (int64_t c0 = c_beg; c0 < c_end; c0 += CPI) {
        ulonglong2 x[CPI][ND], ta0[CPI], ta1[CPI], tb0[CPI], tb1[CPI];
#pragma unroll
        for (int e = 0; e < CPI; e++) {   // issue every load of the CPI ciphertexts first
            const int64_t c = (c0 + e < c_end) ? c0 + e : c0;
            const size_t oc = (size_t)c * cs / 2;   // in ulonglong2 units
#pragma unroll
            for (int j = 0; j < ND; j++)
                if (j != ti) x[e][j] = xb[((size_t)c * xs_c + (size_t)j * xs_j) / 2];
            if (ti <= l) {   // target P (ti = l + 1) has no limb in the input ciphertexts
                ta1[e] = a1b[oc];
                tb1[e] = b1b[oc];
                ta0[e] = a0b[oc];
                tb0[e] = b0b[oc];
            }
        }
#pragma unroll
        for (int e = 0; e < CPI; e++) {
            const int64_t c = c0 + e;
            if (c >= c_end) break;
#pragma unroll
            for (int j = 0; j < ND; j++)   // digit j = ti: d2 = a1 b1 (or a1 alone for a rotation)
                if (j == ti)
                    x[e][j] = single ? ta1[e]
                                     : make_ulonglong2(mulmod_path<FP>(ta1[e].x, tb1[e].x, m),
                                                       mulmod_path<FP>(ta1[e].y, tb1[e].y, m));
            ulonglong2 v[2];
#pragma unroll
            for (int cc = 0; cc < 2; cc++) {
                if constexpr (F64) {   // exact binary64 products and sums (ND * 0.625 q < 2^47)
                    const double qd = u52_to_double(m.q);
                    double s0 = 0.0, s1 = 0.0;
#pragma unroll
                    for (int j = 0; j < ND; j++) {
                        const ulonglong2 r = ks[((j * 2 + cc) * 2 + 0) * MAC2_THREADS + threadIdx.x];
                        const ulonglong2 q = ks[((j * 2 + cc) * 2 + 1) * MAC2_THREADS + threadIdx.x];
                        s0 = __dadd_rn(s0, f64_mulc(u52_to_double(x[e][j].x), f64_of(r.x), f64_of(q.x), qd));
                        s1 = __dadd_rn(s1, f64_mulc(u52_to_double(x[e][j].y), f64_of(r.y), f64_of(q.y), qd));
                    }
                    v[cc] = make_ulonglong2(f64_to_canon(f64_reduce(s0, qd, m.qinv_d), qd),
                                            f64_to_canon(f64_reduce(s1, qd, m.qinv_d), qd));
                } else if constexpr (FP) {
                    uint64_t s0 = 0, s1 = 0;
#pragma unroll
                    for (int j = 0; j < ND; j++) {
                        const ulonglong2 r = ks[((j * 2 + cc) * 2 + 0) * MAC2_THREADS + threadIdx.x];
                        const ulonglong2 q = ks[((j * 2 + cc) * 2 + 1) * MAC2_THREADS + threadIdx.x];
                        s0 += tw_mul_fp(x[e][j].x, r.x, q.x, m.q);
                        s1 += tw_mul_fp(x[e][j].y, r.y, q.y, m.q);
                    }
                    v[cc] = make_ulonglong2(reduce64(s0, m), reduce64(s1, m));
                } else {
                    U128 s0, s1;
                    s0.lo = s0.hi = s1.lo = s1.hi = 0;
#pragma unroll
                    for (int j = 0; j < ND; j++) {
                        const ulonglong2 r = ks[((j * 2 + cc) * 2 + 0) * MAC2_THREADS + threadIdx.x];
                        mac128(s0, x[e][j].x, r.x);
                        mac128(s1, x[e][j].y, r.y);
                    }
                    v[cc] = make_ulonglong2(barrett128(s0, m), barrett128(s1, m));
                }
            }
            if (ti <= l) {   // fold the tensor's d0, d1: v = d + acc P^-1 (rotation: d = (a0, 0))
                uint64_t d0x = ta0[e].x, d0y = ta0[e].y, d1x = 0, d1y = 0;
                if (!single) {
                    d0x = mulmod_path<FP>(ta0[e].x, tb0[e].x, m);
                    d0y = mulmod_path<FP>(ta0[e].y, tb0[e].y, m);
                    d1x = addmod(mulmod_path<FP>(ta0[e].x, tb1[e].x, m), mulmod_path<FP>(ta1[e].x, tb0[e].x, m), m.q);
                    d1y = addmod(mulmod_path<FP>(ta0[e].y, tb1[e].y, m), mulmod_path<FP>(ta1[e].y, tb0[e].y, m), m.q);
                }
                v[0] = make_ulonglong2(addmod(d0x, mulc_path<FP>(v[0].x, pinv, m), m.q),
                                       addmod(d0y, mulc_path<FP>(v[0].y, pinv, m), m.q));
                v[1] = make_ulonglong2(addmod(d1x, mulc_path<FP>(v[1].x, pinv, m), m.q),
                                       addmod(d1y, mulc_path<FP>(v[1].y, pinv, m), m.q));
            }
#pragma unroll
            for (int cc = 0; cc < 2; cc++) v2(acc + ((((size_t)c * 2 + cc) * (l + 2) + ti) << logn))[k] = v[cc];
        }
    }
}

// ---------------------------------------------------------------- key inner product, round 2
// One coefficient per thread (8-byte accesses), the thread's key entries for its target
// (ND digits x 2 components) held in registers for all MAC3_CTS ciphertexts of its CTA,
// and the next ciphertext's loads (l digit limbs + the tensor operands) issued before the
// current one's arithmetic (software pipelining across ciphertexts): 256-thread CTAs at
// <= 80 registers, 3 per SM, instead of k_relin_mac2's 128-register 128-thread CTAs.
// F64 targets: f64_mult products (no key companion) summed exactly; 60-bit targets: full
// 128-bit products summed lazily, Barrett once; MODE 1 (2^44 <= q < 2^46) keeps the
// FP64-quotient lazy products with companions.  Same output as k_relin_mac2.
constexpr int MAC3_T = 256;
#ifndef EDL_MAC3_CTS
#define EDL_MAC3_CTS 8
#endif
constexpr int MAC3_CTS = EDL_MAC3_CTS;
// operand ring depth (cp.async, shared memory): measured on C1 (round 2b) 2 stages 0.552 ms,
// 3 stages 0.564, 4 stages 0.557, register prefetch (0 = off) 0.599; 4 CTAs/SM 0.559
#ifndef EDL_MAC3_ASYNC
#define EDL_MAC3_ASYNC 2
#endif
#if EDL_MAC3_ASYNC == 0
#undef EDL_MAC3_ASYNC
#endif

// pfold: the data targets' key entries already carry the factor P^-1 (the context's
// P^-1-folded copy of rlk, keygen), so v = d + acc directly.
template <int MODE, int ND>
__device__ __forceinline__ void mac3_body(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b, int l, int L,
                                          int64_t cnt, const uint64_t* __restrict__ xh, const uint64_t* __restrict__ rlk,
                                          const uint64_t* __restrict__ rlk_c, uint64_t* __restrict__ acc, int ti, int t,
                                          const ModInfo& m, const ChainConsts* __restrict__ chain, int logn, bool pfold,
                                          int k) {
    constexpr bool F64 = MODE == 2;
    const double qd = u52_to_double(m.q);
    // key entries of this coefficient: kv[j][cc] (binary64 on F64 targets), companions for MODE 1
    uint64_t kv[ND][2], kc[ND][2];
#pragma unroll
    for (int j = 0; j < ND; j++)
#pragma unroll
        for (int cc = 0; cc < 2; cc++) {
            const size_t o = ((((size_t)j * 2 + cc) * (L + 2) + t) << logn) + k;
            kv[j][cc] = F64 ? bits_of(u52_to_double(__ldg(rlk + o))) : __ldg(rlk + o);
            kc[j][cc] = (MODE == 1) ? __ldg(rlk_c + o) : 0;
        }
    const bool data = ti <= l;
    const bool single = (b == nullptr);
    const bool fold = data && !pfold;   // multiply the key sum by P^-1 here
    const ulonglong2 pinv = data ? chain->qinv[L + 1][t] : make_ulonglong2(0, 0);
    const double pinv_d = u52_to_double(pinv.x);
    const size_t limb = (size_t)1 << logn;
    const size_t cs = (size_t)2 * (l + 1) << logn;                       // one ciphertext
    const size_t xs_c = (size_t)(l + 1) * (l + 2) << logn;               // raised digits of one ciphertext
    const uint64_t* xb = xh + ((size_t)ti << logn) + k;                  // digit j at + j (l+2) N
    const uint64_t* a0b = a + ((size_t)(data ? ti : 0) << logn) + k;
    const uint64_t* a1b = a0b + (size_t)(l + 1) * limb;
    const uint64_t* b0b = single ? a0b : b + ((size_t)(data ? ti : 0) << logn) + k;
    const uint64_t* b1b = b0b + (size_t)(l + 1) * limb;
    (void)limb;
    const int64_t c_beg = (int64_t)blockIdx.z * MAC3_CTS;
    const int64_t c_end = c_beg + MAC3_CTS < cnt ? c_beg + MAC3_CTS : cnt;
    // per-ciphertext operands: x[j] (j != ti), a0, a1, b0, b1
    struct Ops {
        uint64_t x[ND], a0, a1, b0, b1;
    };
    auto fetch = [&](int64_t c, Ops& o) {
#pragma unroll
        for (int j = 0; j < ND; j++) o.x[j] = (j != ti) ? xb[(size_t)c * xs_c + (size_t)j * (l + 2) * limb] : 0;
        if (data) {
            o.a0 = a0b[(size_t)c * cs];
            o.a1 = a1b[(size_t)c * cs];
            o.b0 = single ? o.a0 : b0b[(size_t)c * cs];
            o.b1 = single ? o.a1 : b1b[(size_t)c * cs];
        } else if (ti < ND) {
            o.a0 = o.a1 = o.b0 = o.b1 = 0;
        } else {
            o.a0 = o.a1 = o.b0 = o.b1 = 0;
        }
    };
#ifdef EDL_MAC3_ASYNC
    // operands of ciphertext c + S - 1 copied into this thread's slots of a shared-memory
    // ring by cp.async while ciphertext c computes (S - 1 ciphertexts in flight, no registers
    // held); each thread reads back only words it copied itself, so no barrier
    extern __shared__ uint64_t mac_ring[];   // [S][ND + 4][MAC3_T]
    constexpr int S = EDL_MAC3_ASYNC, NO = ND + 4;
    const int tid = threadIdx.x;
    auto slot = [&](int st, int o) { return mac_ring + ((size_t)st * NO + o) * MAC3_T + tid; };
#ifdef EDL_MAC3_BULK
    // EDL_MAC3_BULK: the ring filled by the bulk-copy engine instead of per-thread cp.async:
    // thread 0 issues one cp.async.bulk per operand row (MAC3_T words = 2 KB, contiguous in
    // global and in the ring) onto the stage's mbarrier; every thread waits on the mbarrier's
    // phase, takes its words into registers, and a CTA barrier releases the stage for the
    // ciphertext S iterations ahead.  No LDGSTS or operand address arithmetic per thread.
    // Measured on B200 (C1): 0.553-0.555 ms against 0.552 for the per-thread cp.async ring (the
    // barrier per ciphertext costs what the removed instructions saved): opt-in, bit-exact.
    __shared__ __align__(8) uint64_t ring_full[S];
    const uint64_t* xrow = xb - tid;       // row bases (thread 0's word)
    const uint64_t* a0row = a0b - tid;
    const uint64_t* a1row = a1b - tid;
    const uint64_t* b0row = b0b - tid;
    const uint64_t* b1row = b1b - tid;
    const uint32_t rows_ct = (uint32_t)((data ? ND - 1 : ND) + (data ? (single ? 2 : 4) : 0));
    if (tid == 0) {
#pragma unroll
        for (int u = 0; u < S; u++)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&ring_full[u])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    auto bulk = [&](uint64_t* dst, const uint64_t* src, uint32_t mb) {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(dst)),
                     "l"(src), "r"((uint32_t)(MAC3_T * 8)), "r"(mb)
                     : "memory");
    };
    auto bfetch = [&](int64_t c, int st) {   // thread 0 only
        const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&ring_full[st]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(rows_ct * (uint32_t)(MAC3_T * 8))
                     : "memory");
        uint64_t* base = mac_ring + (size_t)st * NO * MAC3_T;
#pragma unroll
        for (int j = 0; j < ND; j++)
            if (j != ti) bulk(base + (size_t)j * MAC3_T, xrow + (size_t)c * xs_c + (size_t)j * (l + 2) * limb, mb);
        if (data) {
            bulk(base + (size_t)(ND + 0) * MAC3_T, a0row + (size_t)c * cs, mb);
            bulk(base + (size_t)(ND + 1) * MAC3_T, a1row + (size_t)c * cs, mb);
            if (!single) {
                bulk(base + (size_t)(ND + 2) * MAC3_T, b0row + (size_t)c * cs, mb);
                bulk(base + (size_t)(ND + 3) * MAC3_T, b1row + (size_t)c * cs, mb);
            }
        }
    };
    if (tid == 0) {
#pragma unroll
        for (int u = 0; u < S; u++)
            if (c_beg + u < c_end) bfetch(c_beg + u, u);
    }
    for (int64_t c = c_beg; c < c_end; c++) {
        const int u = (int)(c - c_beg);
        const int st = u % S;
        {
            const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&ring_full[st]);
            const uint32_t par = (uint32_t)((u / S) & 1);
            uint32_t done;
            do {
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                             "selp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(done)
                             : "r"(mb), "r"(par)
                             : "memory");
            } while (!done);
        }
        Ops cur;
#pragma unroll
        for (int j = 0; j < ND; j++) cur.x[j] = (j != ti) ? *slot(st, j) : 0;
        cur.a0 = cur.a1 = cur.b0 = cur.b1 = 0;
        if (data) {
            cur.a0 = *slot(st, ND + 0);
            cur.a1 = *slot(st, ND + 1);
            cur.b0 = single ? cur.a0 : *slot(st, ND + 2);
            cur.b1 = single ? cur.a1 : *slot(st, ND + 3);
        }
        __syncthreads();   // every thread holds its words: the stage may be refilled
        if (tid == 0 && c + S < c_end) bfetch(c + S, st);
#else
    auto cpa = [&](uint64_t* dst, const uint64_t* src) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
                     : "memory");
    };
    auto afetch = [&](int64_t c, int st) {
#pragma unroll
        for (int j = 0; j < ND; j++)
            if (j != ti) cpa(slot(st, j), xb + (size_t)c * xs_c + (size_t)j * (l + 2) * limb);
        if (data) {
            cpa(slot(st, ND + 0), a0b + (size_t)c * cs);
            cpa(slot(st, ND + 1), a1b + (size_t)c * cs);
            if (!single) {
                cpa(slot(st, ND + 2), b0b + (size_t)c * cs);
                cpa(slot(st, ND + 3), b1b + (size_t)c * cs);
            }
        }
    };
#pragma unroll
    for (int u = 0; u < S - 1; u++) {
        if (c_beg + u < c_end) afetch(c_beg + u, u);
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int64_t c = c_beg; c < c_end; c++) {
        const int u = (int)(c - c_beg);
        if (c + S - 1 < c_end) afetch(c + S - 1, (u + S - 1) % S);
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group %0;" ::"n"(S - 1) : "memory");
        const int st = u % S;
        Ops cur;
#pragma unroll
        for (int j = 0; j < ND; j++) cur.x[j] = (j != ti) ? *slot(st, j) : 0;
        cur.a0 = cur.a1 = cur.b0 = cur.b1 = 0;
        if (data) {
            cur.a0 = *slot(st, ND + 0);
            cur.a1 = *slot(st, ND + 1);
            cur.b0 = single ? cur.a0 : *slot(st, ND + 2);
            cur.b1 = single ? cur.a1 : *slot(st, ND + 3);
        }
#endif   // EDL_MAC3_BULK
#else
    Ops nx;
    if (c_beg < c_end) fetch(c_beg, nx);
    for (int64_t c = c_beg; c < c_end; c++) {
        const Ops cur = nx;
        if (c + 1 < c_end) fetch(c + 1, nx);
#endif
        uint64_t v0, v1;
        if constexpr (F64) {
            double s0 = 0.0, s1 = 0.0;
            double d0 = 0.0, d1 = 0.0;
#pragma unroll
            for (int j = 0; j < ND; j++) {
                double xd;
                if (j == ti) {   // d2 = a1 b1 (rotation: a1), exact product reduced on the FP64 pipe
                    const double x1 = u52_to_double(cur.a1);
                    xd = single ? x1 : f64_mult(x1, u52_to_double(cur.b1), qd, m.qinv_d);
                } else {
                    xd = u52_to_double(cur.x[j]);
                }
                s0 = __dadd_rn(s0, f64_mult(xd, f64_of(kv[j][0]), qd, m.qinv_d));
                s1 = __dadd_rn(s1, f64_mult(xd, f64_of(kv[j][1]), qd, m.qinv_d));
            }
            if (data) {   // v = d + acc P^-1, d0 = a0 b0, d1 = a0 b1 + a1 b0 (rotation: d = (a0, 0))
                const double x0 = u52_to_double(cur.a0);
                if (single) {
                    d0 = x0;
                } else {
                    const double y0 = u52_to_double(cur.b0), y1 = u52_to_double(cur.b1), x1 = u52_to_double(cur.a1);
                    d0 = f64_mult(x0, y0, qd, m.qinv_d);
                    d1 = __dadd_rn(f64_mult(x0, y1, qd, m.qinv_d), f64_mult(x1, y0, qd, m.qinv_d));
                }
                s0 = __dadd_rn(d0, fold ? f64_mult(s0, pinv_d, qd, m.qinv_d) : f64_reduce(s0, qd, m.qinv_d));
                s1 = __dadd_rn(d1, fold ? f64_mult(s1, pinv_d, qd, m.qinv_d) : f64_reduce(s1, qd, m.qinv_d));
            }
            v0 = f64_to_canon(f64_reduce(s0, qd, m.qinv_d), qd);
            v1 = f64_to_canon(f64_reduce(s1, qd, m.qinv_d), qd);
        } else if constexpr (MODE == 1) {
            uint64_t s0 = 0, s1 = 0;
#pragma unroll
            for (int j = 0; j < ND; j++) {
                const uint64_t x = (j == ti) ? (single ? cur.a1 : mulmod_fp(cur.a1, cur.b1, m)) : cur.x[j];
                s0 += tw_mul_fp(x, kv[j][0], kc[j][0], m.q);
                s1 += tw_mul_fp(x, kv[j][1], kc[j][1], m.q);
            }
            v0 = reduce64(s0, m);
            v1 = reduce64(s1, m);
            if (data) {
                uint64_t d0 = cur.a0, d1 = 0;
                if (!single) {
                    d0 = mulmod_fp(cur.a0, cur.b0, m);
                    d1 = addmod(mulmod_fp(cur.a0, cur.b1, m), mulmod_fp(cur.a1, cur.b0, m), m.q);
                }
                v0 = addmod(d0, fold ? mulc(v0, pinv, m) : v0, m.q);
                v1 = addmod(d1, fold ? mulc(v1, pinv, m) : v1, m.q);
            }
        } else {
            U128 s0, s1;
            s0.lo = s0.hi = s1.lo = s1.hi = 0;
#pragma unroll
            for (int j = 0; j < ND; j++) {
                const uint64_t x = (j == ti) ? (single ? cur.a1 : mulmod_barrett(cur.a1, cur.b1, m)) : cur.x[j];
                mac128(s0, x, kv[j][0]);
                mac128(s1, x, kv[j][1]);
            }
            if (data && pfold) {
                // keys carry P^-1: the tensor's d0 = a0 b0 and d1 = a0 b1 + a1 b0 join the same
                // lazy 128-bit sums (<= l + 3 terms below 2^120), one Barrett per output
                if (single) {
                    U128 t;
                    t.lo = cur.a0;
                    t.hi = 0;
                    add128(s0, t);
                } else {
                    mac128(s0, cur.a0, cur.b0);
                    mac128(s1, cur.a0, cur.b1);
                    mac128(s1, cur.a1, cur.b0);
                }
                v0 = barrett128(s0, m);
                v1 = barrett128(s1, m);
            } else {
                v0 = barrett128(s0, m);
                v1 = barrett128(s1, m);
            }
            if (data && !pfold) {
                uint64_t d0 = cur.a0, d1 = 0;
                if (!single) {
                    d0 = mulmod_barrett(cur.a0, cur.b0, m);
                    d1 = addmod(mulmod_barrett(cur.a0, cur.b1, m), mulmod_barrett(cur.a1, cur.b0, m), m.q);
                }
                v0 = addmod(d0, fold ? mulc(v0, pinv, m) : v0, m.q);
                v1 = addmod(d1, fold ? mulc(v1, pinv, m) : v1, m.q);
            }
        }
        acc[((((size_t)c * 2 + 0) * (l + 2) + ti) << logn) + k] = v0;
        acc[((((size_t)c * 2 + 1) * (l + 2) + ti) << logn) + k] = v1;
    }
}

// MODE >= 0: one arithmetic path for every target of the launch; MODE = -1: the targets of
// all paths in ONE launch (per-CTA branch on the target's mode), so the memory-latency-bound
// F64 targets and the IMAD-bound 60-bit targets share the SMs instead of running back to back.
template <int MODE, int ND>
#ifndef EDL_MAC3_MINB
#define EDL_MAC3_MINB 3
#endif
__global__ void __launch_bounds__(MAC3_T, EDL_MAC3_MINB)
k_relin_mac3(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b, int l, int L, int64_t cnt,
             const uint64_t* __restrict__ xh, const uint64_t* __restrict__ rlk, const uint64_t* __restrict__ rlk_c,
             uint64_t* __restrict__ acc, const __grid_constant__ TargetList tl, const __grid_constant__ ModTable mods,
             const ChainConsts* __restrict__ chain, int logn, int pfold) {
    EDL_PDL_ENTRY();
    const int ti = tl.slot[blockIdx.y];
    const int t = (ti == l + 1) ? (L + 1) : ti;
    const ModInfo& m = mods[t];
    const int k = blockIdx.x * MAC3_T + threadIdx.x;
    if (k >= (1 << logn)) return;
    if constexpr (MODE >= 0) {
        mac3_body<MODE, ND>(a, b, l, L, cnt, xh, rlk, rlk_c, acc, ti, t, m, chain, logn, pfold != 0, k);
    } else {
        // (the launcher sends MODE-1 targets, 2^44 <= q < 2^46, to their own launch)
        if (m.fp == 2) mac3_body<2, ND>(a, b, l, L, cnt, xh, rlk, rlk_c, acc, ti, t, m, chain, logn, pfold != 0, k);
        else mac3_body<0, ND>(a, b, l, L, cnt, xh, rlk, rlk_c, acc, ti, t, m, chain, logn, pfold != 0, k);
    }
}

// ---------------------------------------------------------------- NEXT f1: automorphism, ct (.) pt
// sigma_g in the NTT domain is a permutation of the evaluation points (same for every limb):
// out[k] = in[src_g(k)], (2 brv(src) + 1) = (2 brv(k) + 1) g mod 2N.
__global__ void k_automorphism(const uint64_t* __restrict__ in, int64_t rows, uint32_t g, uint64_t* __restrict__ out,
                               int logn) {
    EDL_PDL_ENTRY();
    const int n = 1 << logn;
    const uint32_t two_n = 2u << logn;
    for (int64_t row = blockIdx.y; row < rows; row += gridDim.y) {
        const uint64_t* src = in + ((size_t)row << logn);
        uint64_t* dst = out + ((size_t)row << logn);
        for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
            const uint32_t bk = __brev((uint32_t)k) >> (32 - logn);
            const uint32_t e = (uint32_t)(((uint64_t)(2 * bk + 1) * g) % two_n);
            dst[k] = __ldg(src + (__brev((e - 1) >> 1) >> (32 - logn)));
        }
    }
}

__global__ void k_mul_pt(const uint64_t* __restrict__ a, int64_t cnt, int l, const uint64_t* __restrict__ pt,
                         int64_t pt_count, int pt_level, uint64_t* __restrict__ out,
                         const __grid_constant__ ModTable mods, int logn) {
    EDL_PDL_ENTRY();
    const int64_t rows = cnt * 2 * (l + 1);
    const int n2 = 1 << (logn - 1);
    for (int64_t row = blockIdx.y; row < rows; row += gridDim.y) {
        const int i = (int)(row % (l + 1));
        const int64_t c = row / (2 * (l + 1));
        const ModInfo& m = mods[i];
        const uint64_t* pa = a + ((size_t)row << logn);
        const uint64_t* pp = pt + ((((size_t)(pt_count == 1 ? 0 : c)) * (pt_level + 1) + i) << logn);
        uint64_t* po = out + ((size_t)row << logn);
        for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n2; k += gridDim.x * blockDim.x) {
            const ulonglong2 x = v2(pa)[k], w = v2(pp)[k];
            v2(po)[k] = make_ulonglong2(mulmod(x.x, w.x, m), mulmod(x.y, w.y, m));
        }
    }
}

// out = a + pt on polynomial 0 (ct + plaintext vector, NTT domain; polynomial 1 copied)
__global__ void k_add_pt(const uint64_t* __restrict__ a, int64_t cnt, int l, const uint64_t* __restrict__ pt,
                         int64_t pt_count, int pt_level, uint64_t* __restrict__ out, const __grid_constant__ ModTable mods,
                         int logn) {
    EDL_PDL_ENTRY();
    const int64_t rows = cnt * 2 * (l + 1);
    const int n2 = 1 << (logn - 1);
    for (int64_t row = blockIdx.y; row < rows; row += gridDim.y) {
        const int i = (int)(row % (l + 1));
        const int p = (int)((row / (l + 1)) % 2);
        const int64_t c = row / (2 * (l + 1));
        const uint64_t q = mods[i].q;
        const uint64_t* pa = a + ((size_t)row << logn);
        const uint64_t* pp = pt + ((((size_t)(pt_count == 1 ? 0 : c)) * (pt_level + 1) + i) << logn);
        uint64_t* po = out + ((size_t)row << logn);
        for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n2; k += gridDim.x * blockDim.x) {
            const ulonglong2 x = v2(pa)[k];
            if (p == 0) {
                const ulonglong2 w = v2(pp)[k];
                v2(po)[k] = make_ulonglong2(addmod(x.x, w.x, q), addmod(x.y, w.y, q));
            } else {
                v2(po)[k] = x;
            }
        }
    }
}

// ---------------------------------------------------------------- wire format (pack/unpack)
// A ciphertext array travels host<->device with every residue of limb i stored in
// bits_i = bit length of q_i (60 or 40 for the Alg. 8 chains) instead of 64: limb i of a
// polynomial is N*bits_i/64 little-endian words, coefficient k at bit offset k*bits_i.
// Limbs follow the [count][2][level+1] order; `loff` holds each limb's word offset within
// one polynomial and `pw` the words per polynomial.
struct PackInfo {
    int bits[MAXM];
    int64_t loff[MAXM];
};

// `stride` = 2 packs/unpacks only polynomial 0 of each ciphertext (c0 of a seeded
// secret-key ciphertext): wire polynomial p <-> array polynomial stride * p.
__global__ void k_unpack(const uint64_t* __restrict__ in, int64_t polys, int nl, int64_t pw,
                         const __grid_constant__ PackInfo pi, uint64_t* __restrict__ out, int logn, int stride) {
    EDL_PDL_ENTRY();
    const int64_t rows = polys * nl;
    const int n = 1 << logn;
    for (int64_t row = blockIdx.y; row < rows; row += gridDim.y) {
        const int i = (int)(row % nl);
        const int64_t pl = row / nl;
        const int b = pi.bits[i];
        const uint64_t mask = (b == 64) ? ~0ull : ((1ull << b) - 1);
        const uint64_t* src = in + pl * pw + pi.loff[i];
        uint64_t* dst = out + (((size_t)pl * stride * nl + i) << logn);
        for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
            const uint64_t off = (uint64_t)k * b;
            const uint64_t w = off >> 6;
            const int sh = (int)(off & 63);
            uint64_t v = __ldg(src + w) >> sh;
            if (sh + b > 64) v |= __ldg(src + w + 1) << (64 - sh);
            dst[k] = v & mask;
        }
    }
}

__global__ void k_pack(const uint64_t* __restrict__ in, int64_t polys, int nl, int64_t pw,
                       const __grid_constant__ PackInfo pi, uint64_t* __restrict__ out, int logn, int stride) {
    EDL_PDL_ENTRY();
    const int64_t rows = polys * nl;
    const int n = 1 << logn;
    for (int64_t row = blockIdx.y; row < rows; row += gridDim.y) {
        const int i = (int)(row % nl);
        const int64_t pl = row / nl;
        const int b = pi.bits[i];
        const int64_t words = ((int64_t)n * b) >> 6;
        const uint64_t* src = in + (((size_t)pl * stride * nl + i) << logn);
        uint64_t* dst = out + pl * pw + pi.loff[i];
        for (int64_t w = blockIdx.x * blockDim.x + threadIdx.x; w < words; w += gridDim.x * blockDim.x) {
            // coefficients overlapping bits [64 w, 64 w + 64)
            const uint64_t lo = (uint64_t)w << 6;
            const int64_t k0 = lo / b, k1 = (lo + 63) / b;
            uint64_t v = 0;
            for (int64_t k = k0; k <= k1 && k < n; k++) {
                const int64_t off = k * b - (int64_t)lo;   // may be negative for k0
                const uint64_t c = src[k];
                if (off >= 0) v |= c << off;
                else v |= c >> (-off);
            }
            dst[w] = v;
        }
    }
}

}  // namespace

// out[c*F + f] = sum_t rots[t][c] (.) pts[f][t]  (NTT domain, both polynomials): every
// rotated residue is read once and feeds all F filters; FP64-pipe limbs accumulate exact
// binary64 products (T <= 64 terms of |.| <= 0.51 q), the others 128-bit sums.
__global__ void k_pt_mac_multi(const uint64_t* __restrict__ rots, int T, int64_t n, int l,
                               const uint64_t* __restrict__ pts, int F, int ptl, uint64_t* __restrict__ out,
                               const __grid_constant__ ModTable mods, int logn) {
    EDL_PDL_ENTRY();
    const int nl = l + 1;
    const int64_t row = blockIdx.y;                 // (c, p, i)
    const int i = (int)(row % nl);
    const int64_t cp = row / nl;                    // c * 2 + p
    const int64_t c = cp / 2;
    const int p = (int)(cp % 2);
    const ModInfo& m = mods[i];
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= (1 << logn)) return;
    const size_t rot_stride = (size_t)n * 2 * nl << logn;   // one rotation block
    const uint64_t* xr = rots + ((size_t)row << logn) + k;
    const bool f64 = m.fp == 2;
    const double qd = u52_to_double(m.q);
    for (int f = 0; f < F; f++) {
        const uint64_t* pf = pts + ((((size_t)f * T) * (ptl + 1) + i) << logn) + k;
        const size_t pt_stride = (size_t)(ptl + 1) << logn;
        uint64_t* dst = out + ((((size_t)c * F + f) * 2 + p) * nl + i << logn) + k;
        if (f64) {
            double acc = 0.0;
            for (int t = 0; t < T; t++) {
                const double x = u52_to_double(__ldg(xr + t * rot_stride)), y = u52_to_double(__ldg(pf + t * pt_stride));
                const double hi = __dmul_rn(x, y);
                const double lo = __fma_rn(x, y, -hi);
                const double qt = __dsub_rn(__fma_rn(hi, m.qinv_d, F64_RND), F64_RND);
                acc = __dadd_rn(acc, __dadd_rn(__fma_rn(-qt, qd, hi), lo));
            }
            *dst = f64_to_canon(f64_reduce(acc, qd, m.qinv_d), qd);
        } else {
            U128 acc;
            acc.lo = acc.hi = 0;
            for (int t = 0; t < T; t++) mac128(acc, __ldg(xr + t * rot_stride), __ldg(pf + t * pt_stride));
            *dst = barrett128(acc, m);
        }
    }
}

void launch_pt_mac_multi(const Dev& d, const uint64_t* rots, int T, int64_t n, int l, const uint64_t* pts, int F, int ptl,
                         uint64_t* out) {
    const dim3 grid((unsigned)((1 << d.logn) / PW_THREADS), (unsigned)(n * 2 * (l + 1)));
    EDL_LAUNCH(d, "k_pt_mac_multi", k_pt_mac_multi<<<grid, PW_THREADS, 0, d.st>>>(rots, T, n, l, pts, F, ptl, out, *d.mt,
                                                                                  d.logn));
}

void launch_automorphism_rows(const Dev& d, const uint64_t* in, int64_t rows, uint32_t g, uint64_t* out) {
    EDL_LAUNCH(d, "k_automorphism", k_automorphism<<<rows_grid(d.logn + 1, rows), PW_THREADS, 0, d.st>>>(in, rows, g, out,
                                                                                                      d.logn));
}

void launch_automorphism(const Dev& d, const uint64_t* in, int64_t cnt, int l, uint32_t g, uint64_t* out) {
    EDL_LAUNCH(d, "k_automorphism", k_automorphism<<<rows_grid(d.logn + 1, cnt * 2 * (l + 1)), PW_THREADS, 0, d.st>>>(
                                        in, cnt * 2 * (l + 1), g, out, d.logn));
}

void launch_mul_pt(const Dev& d, const uint64_t* a, int64_t cnt, int l, const uint64_t* pt, int64_t pt_count,
                   int pt_level, uint64_t* out) {
    EDL_LAUNCH(d, "k_mul_pt", k_mul_pt<<<rows_grid(d.logn, cnt * 2 * (l + 1)), PW_THREADS, 0, d.st>>>(
                                  a, cnt, l, pt, pt_count, pt_level, out, *d.mt, d.logn));
}

void launch_add_pt(const Dev& d, const uint64_t* a, int64_t cnt, int l, const uint64_t* pt, int64_t pt_count,
                   int pt_level, uint64_t* out) {
    EDL_LAUNCH(d, "k_add_pt", k_add_pt<<<rows_grid(d.logn, cnt * 2 * (l + 1)), PW_THREADS, 0, d.st>>>(
                                  a, cnt, l, pt, pt_count, pt_level, out, *d.mt, d.logn));
}

static PackInfo pack_info(const Dev& d, int nl, const int* bits, int64_t* pw) {
    PackInfo pi;
    int64_t off = 0;
    for (int i = 0; i < nl && i < MAXM; i++) {
        pi.bits[i] = bits[i];
        pi.loff[i] = off;
        off += ((int64_t)bits[i] << d.logn) >> 6;
    }
    *pw = off;
    return pi;
}

void launch_unpack(const Dev& d, const uint64_t* in, int64_t polys, int nl, const int* bits, uint64_t* out, int stride) {
    int64_t pw = 0;
    const PackInfo pi = pack_info(d, nl, bits, &pw);
    EDL_LAUNCH(d, "k_unpack", k_unpack<<<rows_grid(d.logn + 1, polys * nl), PW_THREADS, 0, d.st>>>(in, polys, nl, pw, pi,
                                                                                                     out, d.logn, stride));
}

__global__ void k_fetch_mapped(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst, int64_t words) {
    EDL_PDL_ENTRY();
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < words; k += (int64_t)gridDim.x * blockDim.x)
        dst[k] = src[k];
}

void launch_fetch_mapped(const Dev& d, const uint64_t* src, uint64_t* dst, int64_t words) {
    if (words <= 0) return;
    const unsigned blocks = (unsigned)std::min<int64_t>((words + 255) / 256, 148);
    EDL_LAUNCH(d, "k_fetch_mapped", k_fetch_mapped<<<blocks, 256, 0, d.st>>>(src, dst, words));
}

void launch_pack(const Dev& d, const uint64_t* in, int64_t polys, int nl, const int* bits, uint64_t* out, int stride) {
    int64_t pw = 0;
    const PackInfo pi = pack_info(d, nl, bits, &pw);
    EDL_LAUNCH(d, "k_pack", k_pack<<<rows_grid(d.logn + 1, polys * nl), PW_THREADS, 0, d.st>>>(in, polys, nl, pw, pi, out,
                                                                                                 d.logn, stride));
}

// dynamic shared memory of k_relin_mac3 (the cp.async operand ring, EDL_MAC3_ASYNC stages)
static int mac3_smem(int nd, const void* kern) {
#ifdef EDL_MAC3_ASYNC
    const int bytes = EDL_MAC3_ASYNC * (nd + 4) * MAC3_T * 8;
    ensure_smem_attr(kern, bytes);
    return bytes;
#else
    (void)nd;
    (void)kern;
    return 0;
#endif
}

void launch_relin_mac(const Dev& d, const uint64_t* a, const uint64_t* b, int64_t cnt, int l, const uint64_t* xh,
                      const uint64_t* rlk, const uint64_t* rlk_c, uint64_t* acc) {
    // one launch per arithmetic path (targets grouped by their modulus' mode)
    TargetList tf, ti, t6;
    int nf = 0, ni = 0, n6 = 0;
    for (int s = 0; s <= l + 1; s++) {
        const int t = (s == l + 1) ? d.L + 1 : s;
        if (d.hmods[t].fp == 2) t6.slot[n6++] = (int8_t)s;
        else if (d.hmods[t].fp) tf.slot[nf++] = (int8_t)s;
        else ti.slot[ni++] = (int8_t)s;
    }
#ifndef EDL_MAC2
    if (l + 1 <= 6 && d.logn >= 8) {   // round 2: k_relin_mac3
        const unsigned gx3 = (unsigned)((1 << d.logn) / MAC3_T), gz3 = (unsigned)((cnt + MAC3_CTS - 1) / MAC3_CTS);
        // the relinearisation key's P^-1-folded copy (data targets), when these are its keys
        const int pfold = (rlk == d.rlk && d.rlk_pf != nullptr) ? 1 : 0;
        const uint64_t* kk = pfold ? d.rlk_pf : rlk;
        const uint64_t* kkc = pfold ? d.rlk_pf_c : rlk_c;
        TargetList all;
        int na = 0;
        for (int k = 0; k < n6; k++) all.slot[na++] = t6.slot[k];
        for (int k = 0; k < ni; k++) all.slot[na++] = ti.slot[k];
#ifndef EDL_MAC3_SPLIT
#define EDL_MAC3_ND(ND)                                                                                            \
    case ND:                                                                                                       \
        if (na)                                                                                                    \
            launch_k(d, "k_relin_mac", k_relin_mac3<-1, ND>, dim3(gx3, na, gz3), dim3(MAC3_T), mac3_smem(ND, (const void*)k_relin_mac3<-1, ND>), \
                     a, b, l, d.L, cnt, xh, kk, kkc, acc, all, *d.mt, d.cc, d.logn, pfold); \
        if (nf)                                                                                                    \
            launch_k(d, "k_relin_mac", k_relin_mac3<1, ND>, dim3(gx3, nf, gz3), dim3(MAC3_T), mac3_smem(ND, (const void*)k_relin_mac3<1, ND>), \
                     a, b, l, d.L, cnt, xh, kk, kkc, acc, tf, *d.mt, d.cc, d.logn, pfold); \
        break;
#else
#define EDL_MAC3(FPV, ND, LIST, NT)                                                                   \
    EDL_LAUNCH(d, "k_relin_mac", (k_relin_mac3<FPV, ND><<<dim3(gx3, NT, gz3), MAC3_T, 0, d.st>>>( \
                                     a, b, l, d.L, cnt, xh, kk, kkc, acc, LIST, *d.mt, d.cc, d.logn, pfold)))
#define EDL_MAC3_ND(ND)                                  \
    case ND:                                             \
        if (n6) EDL_MAC3(2, ND, t6, n6);                 \
        if (nf) EDL_MAC3(1, ND, tf, nf);                 \
        if (ni) EDL_MAC3(0, ND, ti, ni);                 \
        break;
#endif
        switch (l + 1) {
            EDL_MAC3_ND(1)
            EDL_MAC3_ND(2)
            EDL_MAC3_ND(3)
            EDL_MAC3_ND(4)
            EDL_MAC3_ND(5)
            EDL_MAC3_ND(6)
        }
#undef EDL_MAC3_ND
#ifdef EDL_MAC3
#undef EDL_MAC3
#endif
        return;
    }
#endif
#ifdef EDL_NO_MAC2
    if (false) {
#else
    if (l + 1 <= 4 && d.logn >= 8) {
#endif
        const unsigned gx2 = (unsigned)((1 << d.logn) / (2 * MAC2_THREADS)), gz2 = (unsigned)((cnt + MAC2_CTS - 1) / MAC2_CTS);
        const size_t smem = (size_t)(l + 1) * 2 * 2 * MAC2_THREADS * sizeof(ulonglong2);
#define EDL_MAC2(FPV, ND, LIST, NT)                                                                         \
    EDL_LAUNCH(d, "k_relin_mac", (k_relin_mac2<FPV, ND><<<dim3(gx2, NT, gz2), MAC2_THREADS, smem, d.st>>>( \
                                     a, b, l, d.L, cnt, xh, rlk, rlk_c, acc, LIST, *d.mt, d.cc, d.logn)))
#define EDL_MAC2_ND(ND)                                  \
    case ND:                                             \
        if (n6) EDL_MAC2(2, ND, t6, n6);                 \
        if (nf) EDL_MAC2(1, ND, tf, nf);                 \
        if (ni) EDL_MAC2(0, ND, ti, ni);                 \
        break;
        switch (l + 1) {
            EDL_MAC2_ND(1)
            EDL_MAC2_ND(2)
            EDL_MAC2_ND(3)
            EDL_MAC2_ND(4)
        }
#undef EDL_MAC2_ND
#undef EDL_MAC2
        return;
    }
    const unsigned gx = (unsigned)((1 << d.logn) / (2 * PW_THREADS)), gz = (unsigned)((cnt + MAC_CB - 1) / MAC_CB);
    for (int k = 0; k < n6; k++) tf.slot[nf++] = t6.slot[k];   // the generic pass runs every fp target on the FP64-quotient path
    if (nf)
        EDL_LAUNCH(d, "k_relin_mac", (k_relin_mac<true><<<dim3(gx, nf, gz), PW_THREADS, 0, d.st>>>(
                                         a, b, l, d.L, cnt, xh, rlk, rlk_c, acc, tf, *d.mt, d.cc, d.logn)));
    if (ni)
        EDL_LAUNCH(d, "k_relin_mac", (k_relin_mac<false><<<dim3(gx, ni, gz), PW_THREADS, 0, d.st>>>(
                                         a, b, l, d.L, cnt, xh, rlk, rlk_c, acc, ti, *d.mt, d.cc, d.logn)));
}

void launch_add(const Dev& d, const uint64_t* a, int la, const uint64_t* b, int lb, int64_t cnt, int lo, uint64_t* out) {
    EDL_LAUNCH(d, "k_add", k_add<<<rows_grid(d.logn, cnt * 2 * (lo + 1)), PW_THREADS, 0, d.st>>>(a, la, b, lb, cnt, lo, out, *d.mt, d.logn));
}

void launch_mul_const(const Dev& d, const uint64_t* a, int64_t cnt, int l, const ulonglong2* w, uint64_t* out) {
    EDL_LAUNCH(d, "k_mul_const", k_mul_const<<<rows_grid(d.logn, cnt * 2 * (l + 1)), PW_THREADS, 0, d.st>>>(a, cnt, l, w, out, *d.mt, d.logn));
}

void launch_add_const(const Dev& d, const uint64_t* a, int64_t cnt, int l, const uint64_t* k, uint64_t* out) {
    EDL_LAUNCH(d, "k_add_const", k_add_const<<<rows_grid(d.logn, cnt * 2 * (l + 1)), PW_THREADS, 0, d.st>>>(a, cnt, l, k, out, *d.mt, d.logn));
}

void launch_mod_drop(const Dev& d, const uint64_t* a, int64_t cnt, int la, int lo, uint64_t* out) {
    EDL_LAUNCH(d, "k_mod_drop", k_mod_drop<<<rows_grid(d.logn, cnt * 2 * (lo + 1)), PW_THREADS, 0, d.st>>>(a, cnt, la, lo, out, d.logn));
}

void launch_mod_reduce(const Dev& d, uint64_t* x, int64_t cnt, int l) {
    EDL_LAUNCH(d, "k_mod_reduce", k_mod_reduce<<<rows_grid(d.logn, cnt * 2 * (l + 1)), PW_THREADS, 0, d.st>>>(x, cnt, l, *d.mt, d.logn));
}

void launch_add_add_const(const Dev& d, const uint64_t* v, const uint64_t* w, int lw, int64_t cnt, int lo,
                          const uint64_t* k, uint64_t* out) {
    EDL_LAUNCH(d, "k_add_add_const", k_add_add_const<<<rows_grid(d.logn, cnt * 2 * (lo + 1)), PW_THREADS, 0, d.st>>>(v, w, lw, cnt, lo, k, out, *d.mt,
                                                                                   d.logn));
}

void launch_cc_mac(const Dev& d, const uint64_t* x, int l, int H, int W, int F, int kh, int kw, int stride,
                   const ulonglong2* wk, uint64_t* out, const ulonglong2* hw) {
    const int Ho = (H - kh) / stride + 1, Wo = (W - kw) / stride + 1;
    const int taps = kh * kw;
#ifndef EDL_NO_CC4
    if (hw && kh == 4 && kw == 4 && l + 1 <= CC4_MAXL && d.logn >= 7) {
        const int nl = l + 1, nwin = Ho * Wo;
        const dim3 grid((unsigned)((1 << d.logn) / CC4_T), (unsigned)(2 * nl), (unsigned)((nwin + EDL_CC4_WPB - 1) / EDL_CC4_WPB));
        for (int f0 = 0; f0 < F; f0 += CC4_MAXF) {
            const int fc = (F - f0) < CC4_MAXF ? (F - f0) : CC4_MAXF;
            CCW4 wt;
            memset(&wt, 0, sizeof(wt));
            for (int i = 0; i < nl; i++)
                for (int f = 0; f < fc; f++)
                    for (int t = 0; t < taps; t++) {
                        const ulonglong2 v = hw[((size_t)(f0 + f) * taps + t) * nl + i];
                        if (d.hmods[i].fp == 2) {   // split residue pieces as binary64
                            const double lo = (double)(v.x & 0x3FFFFFull), hi = (double)(v.x >> 22);
                            memcpy(&wt.w[i][f][t][0], &lo, 8);
                            memcpy(&wt.w[i][f][t][1], &hi, 8);
#ifdef EDL_CC4_CBANK
                            wt.ws[i][f][t] = lo + hi;
#endif
                        } else {
                            wt.w[i][f][t][0] = v.x;
                            wt.w[i][f][t][1] = v.y;
                        }
                    }
            for (int i = 0; i < nl; i++)
                if (d.hmods[i].fp == 2) {
                    const uint64_t q = d.hmods[i].q, c44 = (1ull << 44) % q;
                    const uint64_t b44 = host::mul_companion(c44, q), b22 = host::mul_companion(1ull << 22, q);
                    wt.c44[i][0] = (double)c44;   // exact: < 2^44
                    memcpy(&wt.c44[i][1], &b44, 8);
                    memcpy(&wt.c44[i][2], &b22, 8);
                }
#ifdef EDL_CC4_ASYNC
#define EDL_CC4(FCV)                                                                                         \
    {                                                                                                        \
        const int sm4 = 2 * 16 * CC4_T * 8;                                                                  \
        ensure_smem_attr((const void*)k_cc_mac4<FCV, 4, 4>, sm4);                                            \
        EDL_LAUNCH(d, "k_cc_mac", (k_cc_mac4<FCV, 4, 4><<<grid, CC4_T, sm4, d.st>>>(x, l, W, stride, Wo, nwin, f0, F, nwin, out, wt, *d.mt, d.logn))); \
    }
#elif defined(EDL_CC4_CBANK)
            const dim3 grid5(grid.x, grid.z, grid.y);   // limb slowest
#define EDL_CC4(FCV) launch_k(d, "k_cc_mac", k_cc_mac5<FCV, 4, 4>, grid5, dim3(CC4_T), 0, x, l, W, stride, Wo, nwin, f0, F, nwin, out, wt, *d.mt, d.logn)
#else
#define EDL_CC4(FCV) launch_k(d, "k_cc_mac", k_cc_mac4<FCV, 4, 4>, grid, dim3(CC4_T), 0, x, l, W, stride, Wo, nwin, f0, F, nwin, out, wt, *d.mt, d.logn)
#endif
            switch (fc) {
                case 1: EDL_CC4(1); break;
                case 2: EDL_CC4(2); break;
                case 3: EDL_CC4(3); break;
                case 4: EDL_CC4(4); break;
                case 5: EDL_CC4(5); break;
                case 6: EDL_CC4(6); break;
                case 7: EDL_CC4(7); break;
                default: EDL_CC4(8); break;
            }
#undef EDL_CC4
        }
        return;
    }
#endif
#ifdef EDL_CC_MAC3   // measured slower on C1 (0.53 vs 0.47 ms): kept for reference
    if (taps <= CC2_MAXTAPS && d.logn >= 8) {
        dim3 grid((unsigned)((1 << d.logn) / CC3_T), (unsigned)(2 * (l + 1)), (unsigned)(Ho * Wo));
        for (int f0 = 0; f0 < F; f0 += 8) {
            const int fc = (F - f0) < 8 ? (F - f0) : 8;
#define EDL_CC3(FCV) EDL_LAUNCH(d, "k_cc_mac", (k_cc_mac3<FCV><<<grid, CC3_T, 0, d.st>>>(x, l, W, kw, stride, Wo, taps, f0, F, Ho * Wo, wk, out, *d.mt, d.logn)))
            switch (fc) {
                case 1: EDL_CC3(1); break;
                case 2: EDL_CC3(2); break;
                case 3: EDL_CC3(3); break;
                case 4: EDL_CC3(4); break;
                case 5: EDL_CC3(5); break;
                case 6: EDL_CC3(6); break;
                case 7: EDL_CC3(7); break;
                default: EDL_CC3(8); break;
            }
#undef EDL_CC3
        }
        return;
    }
#endif
    if (taps <= CC2_MAXTAPS && d.logn >= 9) {
        dim3 grid((unsigned)((1 << d.logn) / (2 * CC2_THREADS)), (unsigned)(2 * (l + 1)), (unsigned)(Ho * Wo));
        for (int f0 = 0; f0 < F; f0 += 8) {
            const int fc = (F - f0) < 8 ? (F - f0) : 8;
#define EDL_CC2(FCV) EDL_LAUNCH(d, "k_cc_mac", (k_cc_mac2<FCV><<<grid, CC2_THREADS, 0, d.st>>>(x, l, W, kw, stride, Wo, taps, f0, F, Ho * Wo, wk, out, *d.mt, d.logn)))
            switch (fc) {
                case 1: EDL_CC2(1); break;
                case 2: EDL_CC2(2); break;
                case 3: EDL_CC2(3); break;
                case 4: EDL_CC2(4); break;
                case 5: EDL_CC2(5); break;
                case 6: EDL_CC2(6); break;
                case 7: EDL_CC2(7); break;
                default: EDL_CC2(8); break;
            }
#undef EDL_CC2
        }
        return;
    }
    dim3 grid((unsigned)(((1 << d.logn) + PW_THREADS - 1) / PW_THREADS), (unsigned)(2 * (l + 1)), (unsigned)(Ho * Wo));
    size_t smem = (size_t)F * kh * kw * sizeof(uint64_t);
    EDL_LAUNCH(d, "k_cc_mac", k_cc_mac<<<grid, PW_THREADS, smem, d.st>>>(x, l, H, W, F, kh, kw, stride, wk, out, *d.mt, d.logn));
}

#ifndef EDL_DN3_CTAS_PER_SM
#define EDL_DN3_CTAS_PER_SM 28   // several waves of short CTAs (1.5 waves of long ones left a tail)
#endif
int dense_split(const Dev& d, int64_t K, int64_t O, int l) {
    if (O <= 16 && d.logn >= 7) {   // k_dense_mac3: K slices of >= 8 inputs
        const int64_t base = (int64_t)((1 << d.logn) / DN3_T) * 2 * (l + 1);
        int64_t ks = (EDL_DN3_CTAS_PER_SM * 148 + base - 1) / base;
        if (ks > K / 8) ks = K / 8;
        if (ks > 32) ks = 32;
        return ks < 1 ? 1 : (int)ks;
    }
    const int64_t ctas = (int64_t)((1 << d.logn) / PW_THREADS) * 2 * (l + 1) * ((O + DN_OC - 1) / DN_OC);
    int ks = 1;
    while (ks < 16 && ctas * ks < 4 * 148 && K / (ks * 2) >= 16) ks *= 2;
    return ks;
}

void launch_dense_mac(const Dev& d, const uint64_t* x, int64_t K, int64_t O, int l, const ulonglong2* wd, uint64_t* out,
                      uint64_t* part) {
    const int ks = part ? dense_split(d, K, O, l) : 1;
    if (O <= 16 && d.logn >= 7) {
        const int kper = (int)((K + ks - 1) / ks);
        if (kper <= 256) {   // exact binary64 / 128-bit sums bounded for <= 256 terms
            const int oc = O <= 4 ? 4 : (O <= 8 ? 8 : (O == 10 ? 10 : (O <= 12 ? 12 : 16)));
            dim3 grid((unsigned)((1 << d.logn) / DN3_T), (unsigned)(2 * (l + 1)), (unsigned)ks);
            size_t smem = (size_t)kper * oc * sizeof(ulonglong2);
#ifdef EDL_DN3_ASYNC
            smem += (size_t)2 * DN3_U * DN3_T * 8;   // cp.async input ring
#endif
            uint64_t* dst = ks > 1 ? part : out;
            const bool kara = EDL_DN3_KARATSUBA && kper <= DN3_KARA_MAX;
            if (kara) smem += (size_t)kper * oc * sizeof(double);   // wl + wh
#define EDL_DN3(OCV)                                                                                \
    if (kara) {                                                                                     \
        ensure_smem_attr((const void*)k_dense_mac3<OCV, true>, (int)smem);                          \
        launch_k(d, "k_dense_mac", k_dense_mac3<OCV, true>, grid, dim3(DN3_T), smem, x, K, (int)O, l, kper, wd, dst, *d.mt, d.logn); \
    } else {                                                                                        \
        ensure_smem_attr((const void*)k_dense_mac3<OCV, false>, (int)smem); /* kper x 16 x 16 B can pass 48 KB */ \
        launch_k(d, "k_dense_mac", k_dense_mac3<OCV, false>, grid, dim3(DN3_T), smem, x, K, (int)O, l, kper, wd, dst, *d.mt, d.logn); \
    }
            switch (oc) {
                case 4: EDL_DN3(4); break;
                case 8: EDL_DN3(8); break;
                case 10: EDL_DN3(10); break;   // C1's 245 -> 10
                case 12: EDL_DN3(12); break;
                default: EDL_DN3(16); break;
            }
#undef EDL_DN3
            if (ks > 1)
                launch_k(d, "k_dense_combine", k_dense_combine, rows_grid(d.logn, O * 2 * (l + 1)), dim3(PW_THREADS), 0, part, ks, O,
                         l, out, *d.mt, d.logn);
            return;
        }
    }
    dim3 grid((unsigned)(((1 << d.logn) + PW_THREADS - 1) / PW_THREADS), (unsigned)(2 * (l + 1)),
              (unsigned)(((O + DN_OC - 1) / DN_OC) * ks));
    size_t smem = (size_t)DN_OC * DN_KC * sizeof(ulonglong2);
    uint64_t* dst = ks > 1 ? part : out;
    EDL_LAUNCH(d, "k_dense_mac", k_dense_mac<<<grid, PW_THREADS, smem, d.st>>>(x, K, O, l, ks, wd, dst, *d.mt, d.logn));
    if (ks > 1)
        EDL_LAUNCH(d, "k_dense_combine", k_dense_combine<<<rows_grid(d.logn, O * 2 * (l + 1)), PW_THREADS, 0, d.st>>>(
                                             part, ks, O, l, out, *d.mt, d.logn));
}

}  // namespace edl
