// host_math.cpp -- see host_math.h.  Compiled with -ffp-contract=off so double
// arithmetic (encode, scale bookkeeping) rounds exactly as written.
#include "host_math.h"

#include <cfenv>
#include <cstring>

#include <cmath>
#include <set>

namespace edl {
namespace host {

uint64_t mulmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a * b) % q); }

uint64_t powmod(uint64_t a, uint64_t e, uint64_t q) {
    uint64_t r = 1 % q;
    a %= q;
    while (e) {
        if (e & 1) r = mulmod(r, a, q);
        a = mulmod(a, a, q);
        e >>= 1;
    }
    return r;
}

uint64_t invmod(uint64_t a, uint64_t q) { return powmod(a, q - 2, q); }

bool is_prime(uint64_t n) {
    if (n < 2) return false;
    static const uint64_t bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    for (uint64_t p : bases) {
        if (n % p == 0) return n == p;
    }
    uint64_t d = n - 1;
    int s = 0;
    while ((d & 1) == 0) {
        d >>= 1;
        s++;
    }
    for (uint64_t a : bases) {
        uint64_t x = powmod(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (int r = 1; r < s; r++) {
            x = mulmod(x, x, n);
            if (x == n - 1) {
                comp = false;
                break;
            }
        }
        if (comp) return false;
    }
    return true;
}

uint64_t shoup_companion(uint64_t w, uint64_t q) { return (uint64_t)(((u128)w << 64) / q); }

bool select_primes(const int* bits, int n_bits, int logn, uint64_t* out) {
    std::set<uint64_t> used;
    const uint64_t two_n = 2ull << logn;
    for (int k = 0; k < n_bits; k++) {
        const int b = bits[k];
        if (b < 2 || b > 60) return false;   // q < 2^60: MAC folds of 256 full products stay below 2^128
        const uint64_t top = (b == 64) ? ~0ull : ((1ull << b) - 1);
        uint64_t cand = top / two_n * two_n + 1;
        while (true) {
            if (cand < two_n) return false;
            if (cand <= top && !used.count(cand) && is_prime(cand)) break;
            cand -= two_n;
        }
        used.insert(cand);
        out[k] = cand;
    }
    return true;
}

// Philox4x32-10 (Salmon et al. 2011), host copy of the device generator (rng_kernels.cuh).
void philox4x32_10(const uint32_t ctr[4], uint64_t key, uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
    for (int r = 0; r < 10; r++) {
        if (r > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0, n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        c0 = n0;
        c1 = (uint32_t)p1;
        c2 = n2;
        c3 = (uint32_t)p0;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
}

uint64_t sk_error_key(uint64_t sk_seed, uint64_t enc_seed) {
    const uint32_t ctr[4] = {(uint32_t)enc_seed, (uint32_t)(enc_seed >> 32), 0u, 13u};
    uint32_t w[4];
    philox4x32_10(ctr, sk_seed, w);
    return (uint64_t)w[0] | ((uint64_t)w[1] << 32);
}

// SHA-256 (FIPS 180-4) of a short message, for key identifiers.
static void sha256(const uint8_t* msg, size_t len, uint8_t out[32]) {
    static const uint32_t K[64] = {
        0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5, 0xd807aa98,
        0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174, 0xe49b69c1, 0xefbe4786,
        0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da, 0x983e5152, 0xa831c66d, 0xb00327c8,
        0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967, 0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13,
        0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85, 0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819,
        0xd6990624, 0xf40e3585, 0x106aa070, 0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a,
        0x5b9cca4f, 0x682e6ff3, 0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7,
        0xc67178f2};
    uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a, 0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    std::vector<uint8_t> m(msg, msg + len);
    m.push_back(0x80);
    while (m.size() % 64 != 56) m.push_back(0);
    const uint64_t bits = (uint64_t)len * 8;
    for (int k = 7; k >= 0; k--) m.push_back((uint8_t)(bits >> (8 * k)));
    auto rotr = [](uint32_t x, int n) { return (x >> n) | (x << (32 - n)); };
    for (size_t blk = 0; blk < m.size(); blk += 64) {
        uint32_t w[64];
        for (int t = 0; t < 16; t++)
            w[t] = ((uint32_t)m[blk + 4 * t] << 24) | ((uint32_t)m[blk + 4 * t + 1] << 16) |
                   ((uint32_t)m[blk + 4 * t + 2] << 8) | m[blk + 4 * t + 3];
        for (int t = 16; t < 64; t++) {
            const uint32_t s0 = rotr(w[t - 15], 7) ^ rotr(w[t - 15], 18) ^ (w[t - 15] >> 3);
            const uint32_t s1 = rotr(w[t - 2], 17) ^ rotr(w[t - 2], 19) ^ (w[t - 2] >> 10);
            w[t] = w[t - 16] + s0 + w[t - 7] + s1;
        }
        uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
        for (int t = 0; t < 64; t++) {
            const uint32_t t1 = hh + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) + K[t] + w[t];
            const uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
            hh = g;
            g = f;
            f = e;
            e = d + t1;
            d = c;
            c = b;
            b = a;
            a = t1 + t2;
        }
        h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
    }
    for (int k = 0; k < 8; k++)
        for (int j = 0; j < 4; j++) out[4 * k + j] = (uint8_t)(h[k] >> (24 - 8 * j));
}

uint64_t key_identifier(uint64_t seed) {
    uint8_t msg[16] = {'e', 'd', 'l', '-', 'k', 'e', 'y', '\0'};
    for (int k = 0; k < 8; k++) msg[8 + k] = (uint8_t)(seed >> (8 * k));
    uint8_t d[32];
    sha256(msg, sizeof(msg), d);
    uint64_t id = 0;
    for (int k = 0; k < 8; k++) id |= (uint64_t)d[k] << (8 * k);
    return id ? id : 1;
}

uint64_t minimal_psi(uint64_t q, int logn) {
    const uint64_t n = 1ull << logn, two_n = 2 * n;
    uint64_t y = 0;
    for (uint64_t x = 2;; x++) {
        y = powmod(x, (q - 1) / two_n, q);
        if (powmod(y, n, q) == q - 1) break;
    }
    uint64_t best = q, yt = y;
    const uint64_t y2 = mulmod(y, y, q);
    for (uint64_t t = 0; t < n; t++) {
        if (yt < best) best = yt;
        yt = mulmod(yt, y2, q);
    }
    return best;
}

void parameterise(int c, int s, double p, std::vector<int>& bits, int& logn) {
    bits.assign(c + 2, s);                       // m = [s for i in range(c+2)]
    bits[0] = (int)(bits[0] * p);                // m[0] = int(m[0]*p)
    bits[c + 1] = (int)(bits[c + 1] * p);        // m[-1] = int(m[-1]*p)
    long b = 27, sum = 0;
    for (int v : bits) sum += v;
    while (b < sum) b *= 2;                      // while b < sum(m): b *= 2
    const long n = (long)(1024.0 * ((double)b / 27.0));   // int(1024 * (b/27))
    logn = 0;
    while ((1L << logn) < n) logn++;
}

static uint32_t bitrev(uint32_t x, int bits) {
    uint32_t r = 0;
    for (int i = 0; i < bits; i++) {
        r = (r << 1) | (x & 1);
        x >>= 1;
    }
    return r;
}

// floor-ish w/q as a binary64 rounded toward -infinity (w, q < 2^53 are exact doubles and
// IEEE division is correctly rounded in the current mode).
static uint64_t quotient_rd_bits(uint64_t w, uint64_t q) {
    const int old = std::fegetround();
    std::fesetround(FE_DOWNWARD);
    volatile double a = (double)w, b = (double)q;
    volatile double r = a / b;
    std::fesetround(old);
    uint64_t bits;
    double rr = r;
    std::memcpy(&bits, &rr, 8);
    return bits;
}

// q < 2^46: the FP64-quotient products need inputs below 2^52, and the forward NTT lets
// its values grow by 2q per stage without reduction (at most (4 + 2*16) q < 2^52 for
// N <= 2^16).
bool fp_quotient_prime(uint64_t q) { return q < (1ull << 46); }

// q < 2^44: NTT butterflies on the FP64 pipe keep every intermediate below 2^50
// (ntt_core.cuh F64 path bounds: forward < 15 q, inverse < 64 q).
bool f64_ntt_prime(uint64_t q) {
#ifdef EDL_NO_F64
    (void)q;
    return false;
#else
    return q < (1ull << 44);
#endif
}

uint64_t mul_companion(uint64_t w, uint64_t q) { return fp_quotient_prime(q) ? quotient_rd_bits(w, q) : shoup_companion(w, q); }

void twiddle_table(uint64_t q, uint64_t psi, int logn, bool inverse, std::vector<uint64_t>& out2) {
    const uint64_t n = 1ull << logn;
    const uint64_t base = inverse ? invmod(psi, q) : psi;
    const bool f64 = f64_ntt_prime(q);
    out2.assign(2 * n, 0);
    uint64_t p = 1;
    for (uint64_t k = 0; k < n; k++) {
        const uint32_t r = bitrev((uint32_t)k, logn);
        if (f64) {
            const double pd = (double)p;   // exact: p < 2^44
            std::memcpy(&out2[2 * r], &pd, 8);
        } else {
            out2[2 * r] = p;
        }
        out2[2 * r + 1] = f64 ? quotient_rd_bits(p, q) : shoup_companion(p, q);
        p = mulmod(p, base, q);
    }
}

// ---- canonical embedding (O5) with an in-house radix-2 complex FFT ----
typedef std::complex<double> cd;

static void fft(std::vector<cd>& a, int logn, int sign) {
    const size_t n = a.size();
    for (size_t i = 0; i < n; i++) {
        const size_t j = bitrev((uint32_t)i, logn);
        if (i < j) std::swap(a[i], a[j]);
    }
    for (size_t len = 2; len <= n; len <<= 1) {
        const size_t half = len / 2;
        const size_t step = n / len;
        for (size_t i = 0; i < n; i += len) {
            for (size_t k = 0; k < half; k++) {
                // twiddle exp(sign * 2 pi i * k*step / n), evaluated directly (no recurrence)
                const double ang = sign * 2.0 * M_PI * (double)(k * step) / (double)n;
                const cd w(std::cos(ang), std::sin(ang));
                const cd u = a[i + k];
                const cd v = a[i + k + half] * w;
                a[i + k] = u + v;
                a[i + k + half] = u - v;
            }
        }
    }
}

void encode(const double* z, int64_t n_slots, int logn, double scale, int64_t* m_out) {
    const int64_t n = 1LL << logn;
    const uint64_t two_n = 2ull * n;
    std::vector<cd> v(n, cd(0, 0));
    uint64_t e = 1;
    for (int64_t j = 0; j < n / 2; j++) {
        const double zj = j < n_slots ? z[j] : 0.0;
        v[(e - 1) / 2] = cd(zj, 0.0);
        v[(two_n - e - 1) / 2] = cd(zj, -0.0);
        e = e * 5 % two_n;
    }
    fft(v, logn, -1);   // w_k = sum_t v_t exp(-2 pi i t k / N)
    for (int64_t k = 0; k < n; k++) {
        const cd wk = v[k] / (double)n;
        const double ang = -M_PI * (double)k / (double)n;
        const double u = wk.real() * std::cos(ang) - wk.imag() * std::sin(ang);
        m_out[k] = (int64_t)std::nearbyint(scale * u);
    }
}

void decode(const int64_t* m, int logn, double scale, int64_t n_out, double* z_out) {
    const int64_t n = 1LL << logn;
    const uint64_t two_n = 2ull * n;
    std::vector<cd> v(n);
    for (int64_t k = 0; k < n; k++) {
        const double ang = M_PI * (double)k / (double)n;
        v[k] = cd((double)m[k] * std::cos(ang), (double)m[k] * std::sin(ang));
    }
    fft(v, logn, +1);   // v_t = sum_k (m_k zeta^k) exp(+2 pi i t k / N)
    uint64_t e = 1;
    for (int64_t j = 0; j < n_out; j++) {
        z_out[j] = v[(e - 1) / 2].real() / scale;
        e = e * 5 % two_n;
    }
}

void crt_lift(const uint64_t* r, int nl, const uint64_t* q, int logn, int64_t* out) {
    const int64_t n = 1LL << logn;
    if (nl == 1) {
        for (int64_t k = 0; k < n; k++) {
            const uint64_t v = r[k];
            out[k] = v > q[0] / 2 ? (int64_t)v - (int64_t)q[0] : (int64_t)v;
        }
        return;
    }
    // m = sum_i y_i Qhat_i - round(sum_i y_i / q_i) Q, evaluated mod 2^64
    std::vector<uint64_t> qhat_inv(nl), qhat_mod64(nl);
    uint64_t Q_mod64 = 1;
    for (int i = 0; i < nl; i++) Q_mod64 *= q[i];
    for (int i = 0; i < nl; i++) {
        uint64_t inv = 1, m64 = 1;
        for (int j = 0; j < nl; j++) {
            if (j == i) continue;
            inv = mulmod(inv, q[j] % q[i], q[i]);
            m64 *= q[j];
        }
        qhat_inv[i] = invmod(inv, q[i]);
        qhat_mod64[i] = m64;
    }
    for (int64_t k = 0; k < n; k++) {
        uint64_t acc = 0;
        double frac = 0.0;
        for (int i = 0; i < nl; i++) {
            const uint64_t y = mulmod(r[(size_t)i * n + k], qhat_inv[i], q[i]);
            acc += y * qhat_mod64[i];
            frac += (double)y / (double)q[i];
        }
        const uint64_t v = (uint64_t)(int64_t)std::nearbyint(frac);
        out[k] = (int64_t)(acc - v * Q_mod64);
    }
}

}  // namespace host
}  // namespace edl
