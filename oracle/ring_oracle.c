/*
 * oracle/ring_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU reference for the integer ring arithmetic
 * underneath the RNS-CKKS hot path of arXiv 2110.13638 (EDLaaS).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load this library.  It shares no code, header, table or constant generator with
 * the CUDA path under paper_2110_13638_b200/.
 *
 * The paper runs CKKS through MS-SEAL on CPUs ("all operations are
 * conducted on CPUs", §Methodology) and prints no ring arithmetic; every routine
 * here is textbook RNS-CKKS background (PAPER.md:459/463 cite CKKS), with each free
 * choice fixed by SURVEY.md §8(c) (O3, O4, O6) and listed in DESIGN.md.
 *
 * Every modular product is (unsigned __int128)a*b % q: no Shoup, no Barrett, no
 * lazy ranges.  Every residue in and out is canonical in [0, q).
 */
#include <stdint.h>
#include <stddef.h>

typedef unsigned __int128 u128;
typedef __int128 i128;

/* (a*b) mod q, the plain definition.  O4. */
uint64_t orc_mulmod(uint64_t a, uint64_t b, uint64_t q) {
#if defined(__x86_64__)
    /* Same value as (u128)a*b % q: the 128-by-64 hardware divide.  Callers pass
       canonical a, b < q, so the
       high word is < q and divq cannot overflow). */
    uint64_t hi, lo, quo, rem;
    __asm__("mulq %3" : "=a"(lo), "=d"(hi) : "a"(a), "r"(b));
    __asm__("divq %4" : "=a"(quo), "=d"(rem) : "a"(lo), "d"(hi), "r"(q));
    (void)quo;
    return rem;
#else
    return (uint64_t)(((u128)a * (u128)b) % (u128)q);
#endif
}

/* a, b canonical in [0, q), q < 2^62: one conditional correction suffices. */
static uint64_t addmod(uint64_t a, uint64_t b, uint64_t q) {
    uint64_t s = a + b;
    return s >= q ? s - q : s;
}

static uint64_t submod(uint64_t a, uint64_t b, uint64_t q) {
    return a >= b ? a - b : a + q - b;
}

uint64_t orc_powmod(uint64_t a, uint64_t e, uint64_t q) {
    uint64_t r = 1 % q;
    a %= q;
    while (e) {
        if (e & 1) r = orc_mulmod(r, a, q);
        a = orc_mulmod(a, a, q);
        e >>= 1;
    }
    return r;
}

/* Inverse by Fermat (q prime). */
uint64_t orc_invmod(uint64_t a, uint64_t q) { return orc_powmod(a, q - 2, q); }

static uint32_t bitrev(uint32_t x, int bits) {
    uint32_t r = 0;
    for (int i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

static int ilog2(int64_t n) { int l = 0; while ((1LL << l) < n) l++; return l; }

/*
 * O3: forward negacyclic NTT, in place, natural order in, bit-reversed order out:
 *   A[k] = sum_j a_j * psi^{(2*brv(k)+1)*j}  mod q.
 * Textbook iterative Cooley-Tukey decimation in time with stage twiddle psi^{brv(m+i)}.
 * The twiddle table is rebuilt on every call (this is the oracle; it is not tuned).
 * `rows` limbs of length n are transformed, row r with modulus q[r] and root psi[r].
 */
void orc_ntt_fwd(uint64_t* a, int64_t rows, int64_t n, const uint64_t* q, const uint64_t* psi,
                 uint64_t* scratch /* n words */) {
    int logn = ilog2(n);
    for (int64_t r = 0; r < rows; r++) {
        uint64_t qq = q[r];
        uint64_t* x = a + r * n;
        /* scratch[k] = psi^{brv(k)} */
        uint64_t p = 1;
        for (int64_t k = 0; k < n; k++) { scratch[bitrev((uint32_t)k, logn)] = p; p = orc_mulmod(p, psi[r], qq); }
        int64_t t = n;
        for (int64_t m = 1; m < n; m <<= 1) {
            t >>= 1;
            for (int64_t i = 0; i < m; i++) {
                int64_t j1 = 2 * i * t;
                uint64_t S = scratch[m + i];
                for (int64_t j = j1; j < j1 + t; j++) {
                    uint64_t U = x[j];
                    uint64_t V = orc_mulmod(x[j + t], S, qq);
                    x[j] = addmod(U, V, qq);
                    x[j + t] = submod(U, V, qq);
                }
            }
        }
    }
}

/*
 * O3: inverse of orc_ntt_fwd: textbook Gentleman-Sande decimation in frequency with
 * stage twiddle psi^{-brv(h+i)}, bit-reversed in, natural out, then times n^{-1}.
 */
void orc_ntt_inv(uint64_t* a, int64_t rows, int64_t n, const uint64_t* q, const uint64_t* psi,
                 uint64_t* scratch) {
    int logn = ilog2(n);
    for (int64_t r = 0; r < rows; r++) {
        uint64_t qq = q[r];
        uint64_t* x = a + r * n;
        uint64_t psi_inv = orc_invmod(psi[r], qq);
        uint64_t p = 1;
        for (int64_t k = 0; k < n; k++) { scratch[bitrev((uint32_t)k, logn)] = p; p = orc_mulmod(p, psi_inv, qq); }
        int64_t t = 1;
        for (int64_t m = n; m > 1; m >>= 1) {
            int64_t h = m >> 1;
            int64_t j1 = 0;
            for (int64_t i = 0; i < h; i++) {
                uint64_t S = scratch[h + i];
                for (int64_t j = j1; j < j1 + t; j++) {
                    uint64_t U = x[j];
                    uint64_t V = x[j + t];
                    x[j] = addmod(U, V, qq);
                    x[j + t] = orc_mulmod(submod(U, V, qq), S, qq);
                }
                j1 += 2 * t;
            }
            t <<= 1;
        }
        uint64_t ninv = orc_invmod((uint64_t)(n % qq), qq);
        for (int64_t j = 0; j < n; j++) x[j] = orc_mulmod(x[j], ninv, qq);
    }
}

/* ---- element-wise modular arithmetic on one limb (O4, O10, O11) ---- */
void orc_vec_mul(uint64_t* out, const uint64_t* a, const uint64_t* b, int64_t n, uint64_t q) {
    for (int64_t i = 0; i < n; i++) out[i] = orc_mulmod(a[i], b[i], q);
}
void orc_vec_mul_scalar(uint64_t* out, const uint64_t* a, uint64_t s, int64_t n, uint64_t q) {
    for (int64_t i = 0; i < n; i++) out[i] = orc_mulmod(a[i], s, q);
}
void orc_vec_add(uint64_t* out, const uint64_t* a, const uint64_t* b, int64_t n, uint64_t q) {
    for (int64_t i = 0; i < n; i++) out[i] = addmod(a[i], b[i], q);
}
void orc_vec_sub(uint64_t* out, const uint64_t* a, const uint64_t* b, int64_t n, uint64_t q) {
    for (int64_t i = 0; i < n; i++) out[i] = submod(a[i], b[i], q);
}
void orc_vec_add_scalar(uint64_t* out, const uint64_t* a, uint64_t s, int64_t n, uint64_t q) {
    for (int64_t i = 0; i < n; i++) out[i] = addmod(a[i], s, q);
}
/* out[i] = a[i] mod q for arbitrary 64-bit a (plain unsigned reduction, O11 step 2). */
void orc_vec_mod(uint64_t* out, const uint64_t* a, int64_t n, uint64_t q) {
    for (int64_t i = 0; i < n; i++) out[i] = a[i] % q;
}
/* out[i] = signed(a[i]) mod q, a holds int64 values (error / message polys). */
void orc_vec_from_signed(uint64_t* out, const int64_t* a, int64_t n, uint64_t q) {
    for (int64_t i = 0; i < n; i++) {
        i128 v = (i128)a[i] % (i128)q;
        if (v < 0) v += q;
        out[i] = (uint64_t)v;
    }
}
/*
 * O11 step 4 / O12: centered lift of r in [0, q_from) to (-q_from/2, q_from/2], then
 * reduce into [0, q_to).  q_from is odd, so the half point is never hit.
 */
void orc_vec_center_mod(uint64_t* out, const uint64_t* r, int64_t n, uint64_t q_from, uint64_t q_to) {
    for (int64_t i = 0; i < n; i++) {
        i128 v = (i128)r[i];
        if (r[i] > (q_from - 1) / 2) v -= (i128)q_from;
        v %= (i128)q_to;
        if (v < 0) v += q_to;
        out[i] = (uint64_t)v;
    }
}

/* ---- O6: Philox4x32-10 (Salmon et al., SC'11), counter-based ---- */
static void philox_round(uint32_t c[4], const uint32_t k[2]) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k[0];
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c[3] ^ k[1];
    uint32_t n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
}

void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    uint32_t k[2] = {key[0], key[1]};
    for (int r = 0; r < 10; r++) {
        if (r > 0) { k[0] += 0x9E3779B9u; k[1] += 0xBB67AE85u; }
        philox_round(c, k);
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

static void philox_at(uint64_t seed, uint32_t coef, uint32_t obj, uint32_t limb, uint32_t tag, uint32_t x[4]) {
    uint32_t ctr[4] = {coef, obj, limb, tag};
    uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    orc_philox4x32_10(ctr, key, x);
}

/* O6 uniform sampler: u = x0 + 2^32 x1 + 2^64 x2 + 2^96 x3, then u mod q. */
void orc_sample_uniform(uint64_t* out, int64_t n, uint64_t seed, uint32_t obj, uint32_t limb,
                        uint32_t tag, uint64_t q) {
    for (int64_t k = 0; k < n; k++) {
        uint32_t x[4];
        philox_at(seed, (uint32_t)k, obj, limb, tag, x);
        u128 u = (u128)x[0] | ((u128)x[1] << 32) | ((u128)x[2] << 64) | ((u128)x[3] << 96);
        out[k] = (uint64_t)(u % (u128)q);
    }
}

/* O6 ternary sampler: (x0 mod 3) - 1, limb field 0. */
void orc_sample_ternary(int64_t* out, int64_t n, uint64_t seed, uint32_t obj, uint32_t tag) {
    for (int64_t k = 0; k < n; k++) {
        uint32_t x[4];
        philox_at(seed, (uint32_t)k, obj, 0, tag, x);
        out[k] = (int64_t)(x[0] % 3u) - 1;
    }
}

static int popcount32(uint32_t v) { int c = 0; while (v) { c += (int)(v & 1u); v >>= 1; } return c; }

/* O6 error sampler, centered binomial eta=21: popcount(x0 & 0x1FFFFF) - popcount(x1 & 0x1FFFFF). */
void orc_sample_cbd(int64_t* out, int64_t n, uint64_t seed, uint32_t obj, uint32_t tag) {
    for (int64_t k = 0; k < n; k++) {
        uint32_t x[4];
        philox_at(seed, (uint32_t)k, obj, 0, tag, x);
        out[k] = (int64_t)popcount32(x[0] & 0x1FFFFFu) - (int64_t)popcount32(x[1] & 0x1FFFFFu);
    }
}
