// host_math.h -- host-side number theory and the CKKS canonical-embedding transform.
// Independent of oracle/ (which is test infrastructure); pinned against it by tests.
#pragma once
#include <complex>
#include <cstdint>
#include <vector>

namespace edl {
namespace host {

typedef unsigned __int128 u128;

uint64_t mulmod(uint64_t a, uint64_t b, uint64_t q);
uint64_t powmod(uint64_t a, uint64_t e, uint64_t q);
uint64_t invmod(uint64_t a, uint64_t q);
bool is_prime(uint64_t n);
uint64_t shoup_companion(uint64_t w, uint64_t q);
// O2: largest unused primes p < 2^b, p = 1 mod 2N, in chain order
bool select_primes(const int* bits, int n_bits, int logn, uint64_t* out);
// Philox4x32-10 (the device generator's host copy): counter ctr[4], key (lo, hi) of `key`
void philox4x32_10(const uint32_t ctr[4], uint64_t key, uint32_t out[4]);
// Philox key of the secret-key encryption error: PRF(secret seed, enc_seed) =
// words 0,1 of Philox_{sk_seed}(enc_seed lo, enc_seed hi, 0, 13).  The error thus depends
// on key material the wire never carries (c1 is the only function of enc_seed alone).
uint64_t sk_error_key(uint64_t sk_seed, uint64_t enc_seed);
// Public key identifier: first 8 bytes (little-endian) of SHA-256("edl-key\0" || seed le64),
// a one-way function of the key seed (never the seed itself); never 0.
uint64_t key_identifier(uint64_t seed);
// O3: minimal primitive 2N-th root of unity mod q
uint64_t minimal_psi(uint64_t q, int logn);
// Alg. 8: returns chain bits (c+2 entries) and log2 N
void parameterise(int c, int s, double p, std::vector<int>& bits, int& logn);

// psi^{brv(k)} (or psi^{-brv(k)}) table, interleaved {w, w'}: [N] pairs
// {psi^(+-brv(k)), floor(w 2^64/q)} (Shoup butterflies), or for f64_ntt_prime(q) the
// binary64 bits of {w, RD(w/q)} used by the FP64-pipe butterflies (ntt_core.cuh).
void twiddle_table(uint64_t q, uint64_t psi, int logn, bool inverse, std::vector<uint64_t>& out2);
bool fp_quotient_prime(uint64_t q);
bool f64_ntt_prime(uint64_t q);
// companion of a constant w for the device's mulc(): RD(w/q) bits or floor(w 2^64/q)
uint64_t mul_companion(uint64_t w, uint64_t q);

// O5 encode: slots z[n_slots] -> m[N] = rint(scale * u_k)
void encode(const double* z, int64_t n_slots, int logn, double scale, int64_t* m_out);
// O5 decode: coefficients m[N] (int64) -> slots z[n_out]
void decode(const int64_t* m, int logn, double scale, int64_t n_out, double* z_out);
// centered CRT lift of residues r[nl][N] (coefficient domain) into int64 (|m| < 2^62)
void crt_lift(const uint64_t* r, int nl, const uint64_t* q, int logn, int64_t* out);

}  // namespace host
}  // namespace edl
