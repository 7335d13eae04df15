/*
 * edl.h -- C-ABI of the B200-native hot path of arXiv 2110.13638 (EDLaaS: "Fully
 * Homomorphic Encryption Over Neural Network Graphs").
 *
 * What crosses this boundary: homomorphic forward inference of the
 * paper's node-centric network over RNS-CKKS ciphertexts -- cross-correlation and
 * dense layers as ciphertext x plaintext multiply-accumulate, the
 * polynomial sigmoid as ciphertext x ciphertext multiply with relinearisation
 * and rescale between levels -- plus the
 * client-side keygen / encode / encrypt / decrypt the paper delegates to MS-SEAL
 * (PAPER.md:85).  Every step runs in the library's sm_100a kernels; there is no CPU
 * fallback.
 *
 * Conventions:
 *  - A ciphertext array (edl_cts) is `count` ciphertexts at one level `level`, stored
 *    contiguously in DEVICE memory as uint64 [count][2][level+1][N], NTT domain (the
 *    bit-reversed evaluation order of SURVEY O3), every residue canonical in [0, q_i).
 *    The caller (e.g. torch) allocates it: edl_cts_bytes(count, level, log_n) bytes.
 *  - `scale` is the CKKS scale (double), `key_id` identifies the secret key.
 *  - The library owns keys, twiddle tables and scratch inside edl_ctx.
 *  - All device work is enqueued on the context's stream (edl_ctx_create / set_stream)
 *    and is asynchronous, except calls that take or return HOST buffers (edl_encode,
 *    edl_encrypt, edl_decrypt*, edl_keygen), which synchronise the stream.
 *  - Errors are synchronous status codes from argument validation (below); CUDA
 *    launch/runtime errors surface as EDL_ERR_CUDA at the next call that checks.
 *    edl_last_error() returns a message for the last failure on that context.
 *  - `out` buffers must not alias inputs unless the function says so.
 */
#ifndef EDL_H
#define EDL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t edl_status;

enum {
    EDL_OK = 0,
    EDL_ERR_ARG = -1,         /* bad argument / unsupported configuration            */
    EDL_ERR_LEVEL = -2,       /* LevelExhausted: no prime left to rescale by */
    EDL_ERR_SCALE = -3,       /* operand scales differ by more than 2^-30 relative    */
    EDL_ERR_KEY = -4,         /* KeyMismatch: operands under different keys */
    EDL_ERR_SHAPE = -5,       /* ShapeMismatch: counts / layer shapes disagree         */
    EDL_ERR_CAPACITY = -6,    /* more values than N/2 slots              */
    EDL_ERR_CUDA = -7,        /* CUDA runtime error                                    */
    EDL_ERR_NOKEY = -8        /* operation needs keys: call edl_keygen first           */
};

#define EDL_MAX_PRIMES 32

/* CKKS parameter set.  bits[] is the full coefficient-modulus chain of Alg. 8
 * INCLUDING the special prime as its last entry (reading R1);
 * q[0..n_data-1] are the data primes, p_special the key-switching prime (rule O2:
 * largest unused prime below 2^bits with p = 1 mod 2N), psi[k] the minimal
 * primitive 2N-th root of unity mod q[k] (psi[n_data] is P's). */
typedef struct {
    int32_t log_n;
    int32_t n_data;               /* number of data primes = L+1 */
    int32_t n_bits;               /* entries in bits[] = n_data + 1 */
    int32_t scale_bits;
    int32_t bits[EDL_MAX_PRIMES + 1];
    uint64_t q[EDL_MAX_PRIMES];
    uint64_t p_special;
    uint64_t psi[EDL_MAX_PRIMES + 1];
} edl_params;

typedef struct edl_ctx edl_ctx;

typedef struct {
    uint64_t* data;      /* device pointer, [count][2][level+1][N] uint64 */
    int64_t count;
    int32_t level;
    int32_t reserved;
    double scale;
    uint64_t key_id;
} edl_cts;

/* Alg. 8 "parameterise(c, s, p)" followed by prime rule O2 and root
 * rule O3.  depth = c >= 0, scale_bits = s (default 40), special_mult = p (default 1.5).
 * Errors: EDL_ERR_ARG if depth < 0 or the chain exceeds EDL_MAX_PRIMES. */
edl_status edl_params_from_depth(int32_t depth, int32_t scale_bits, double special_mult, edl_params* out);

/* Explicit chain (microbench C2): bits[0..n_bits-1], last entry = special prime. */
edl_status edl_params_from_bits(int32_t log_n, const int32_t* bits, int32_t n_bits, int32_t scale_bits,
                                edl_params* out);

/* Bytes of a ciphertext array: 2 * (level+1) * 2^log_n * 8 * count. */
size_t edl_cts_bytes(int64_t count, int32_t level, int32_t log_n);

/* Environment switches read at context creation (diagnostics; results never change):
 * EDL_NVTX=1 wraps every layer-level call in an NVTX range named after the call; EDL_PDL=0
 * turns programmatic dependent launch off; EDL_KS_SPLIT=0 keeps key switches on one stream;
 * EDL_KS_FUSED=1 / EDL_RAISE_FUSED=1 / EDL_KS_CHUNK=<n> select measured-and-rejected key-switch
 * variants. */
/* Create a context on CUDA `device`, enqueueing on `cuda_stream` (a cudaStream_t; NULL =
 * legacy default stream).  Uploads twiddle tables.  log_n must be in [10, 16] (N > 2^13
 * runs one limb per thread-block cluster) and compiled into the build (EDL_LOGNS_MASK);
 * every modulus must be below 2^60 (the MAC kernels fold up to 256 full 128-bit products
 * before reducing).  EDL_ERR_ARG otherwise. */
edl_status edl_ctx_create(const edl_params* params, int32_t device, void* cuda_stream, edl_ctx** out);
void edl_ctx_destroy(edl_ctx* ctx);
edl_status edl_ctx_set_stream(edl_ctx* ctx, void* cuda_stream);
const char* edl_last_error(const edl_ctx* ctx);
/* Number of kernels the library launched on this context since creation. */
int64_t edl_launch_count(const edl_ctx* ctx);
/* Per-launch CUDA-event timing on the context stream (enable != 0), resetting records. */
edl_status edl_profile(edl_ctx* ctx, int32_t enable);
/* Aggregate recorded launches by kernel name: writes up to max_entries rows of total
 * milliseconds (ms) and launch counts (counts); names are '\n'-separated into `names`.
 * Synchronises the stream.  Returns the number of rows (>= 0) or an error status. */
int32_t edl_profile_read(edl_ctx* ctx, char* names, size_t names_len, double* ms, int64_t* counts,
                         int32_t max_entries);

/* O7 key generation from Philox4x32-10(seed): secret s (ternary), public key over
 * q_0..q_L, relinearisation key over q_0..q_L, P.  The seed is secret key material: the
 * context keeps it on the host (secret-key encryption's error PRF) and never exposes it.
 * key_id := the first 8 bytes of SHA-256("edl-key\0" || seed) (edl_key_id), a one-way
 * function of the seed, equal on every rank that generated the same key.  Galois keys of
 * a previous key are freed.  Synchronises. */
edl_status edl_keygen(edl_ctx* ctx, uint64_t seed);
/* The current key's identifier (0 before edl_keygen). */
uint64_t edl_key_id(const edl_ctx* ctx);

/* O5 encode on the host: slots [n_vec][n_slots] doubles -> int64 coefficient polys
 * poly_out [n_vec][N] (host), m_k = rint(scale * u_k).  EDL_ERR_CAPACITY if
 * n_slots > N/2.  Unused slots are zero. */
edl_status edl_encode(edl_ctx* ctx, const double* slots, int64_t n_vec, int64_t n_slots, double scale,
                      int64_t* poly_out);

/* O8 public-key encryption of integer polys (DEVICE pointer int64 [n_vec][N]) at
 * `level` with scale `scale`; ciphertext c uses Philox object id obj0 + c.  out->data
 * must hold edl_cts_bytes(n_vec, level); out's metadata is filled in.  enc_seed is the
 * encryptor's secret randomness (v, e0, e1 are functions of (enc_seed, object id)): a pair
 * (enc_seed, object id) must never be used twice under one key, or the two ciphertexts
 * differ by exactly (m - m', 0). */
edl_status edl_encrypt_poly(edl_ctx* ctx, const int64_t* poly_dev, int64_t n_vec, int32_t level, double scale,
                            uint64_t enc_seed, uint32_t obj0, edl_cts* out);

/* Secret-key encryption (DESIGN reading Z16; the client owns s in EDLaaS, PAPER.md:258-260,
 * 314-316): for ciphertext c (Philox object id obj0 + c) and limb i,
 *   c1_i = uniform(enc_seed, obj0 + c, limb i, tag 11)      (drawn in the NTT domain),
 *   c0_i = NTT_i(m + e) - c1_i s_i,   e = CBD(k_e, obj0 + c, tag 12),
 *   k_e = words 0,1 of Philox_{key seed}(enc_seed lo, enc_seed hi, 0, 13)  (a PRF keyed by
 *         the secret key's seed, so the error is NOT a function of the public enc_seed),
 * so c0 + c1 s = m + e exactly and only c1 is a public function of (enc_seed, obj0 + c):
 * such ciphertexts can cross PCIe as c0 plus the seed (edl_cts_pack_c0 /
 * edl_cts_unpack_seeded).  (enc_seed, object id) must never repeat under one key.
 * Arguments, layout and errors as edl_encrypt_poly.  Asynchronous. */
edl_status edl_encrypt_poly_sk(edl_ctx* ctx, const int64_t* poly_dev, int64_t n_vec, int32_t level, double scale,
                               uint64_t enc_seed, uint32_t obj0, edl_cts* out);

/* Host convenience: encode (host) + copy + encrypt at the top level L, scale 2^scale_bits. */
edl_status edl_encrypt(edl_ctx* ctx, const double* slots, int64_t n_vec, int64_t n_slots, uint64_t enc_seed,
                       uint32_t obj0, edl_cts* out);

/* Decrypt + centered CRT lift: poly_out [count][N] int64 (host).  Valid while the
 * decrypted coefficients satisfy |m| < 2^62.  Synchronises. */
edl_status edl_decrypt_poly(edl_ctx* ctx, const edl_cts* in, int64_t* poly_out);
/* Decrypt + decode: slots_out [count][n_slots] doubles (host).  Synchronises. */
edl_status edl_decrypt(edl_ctx* ctx, const edl_cts* in, double* slots_out, int64_t n_slots);

/* ---- ciphertext arithmetic (meta-object rules) ---- */
/* out = a + b; the higher-level operand is mod-dropped to the lower level first.
 * Scales must agree within 2^-30 relative; out takes a's scale. */
edl_status edl_ct_add(edl_ctx* ctx, const edl_cts* a, const edl_cts* b, edl_cts* out);
/* out_c = a_c * rint(w[c] * pt_scale) (w: host doubles [count]); no rescale; scale *= pt_scale. */
edl_status edl_ct_pt_mul(edl_ctx* ctx, const edl_cts* a, const double* w, double pt_scale, edl_cts* out);
/* out_c = a_c + rint(c[c] * a.scale) on the constant coefficient (host doubles [count]). */
edl_status edl_ct_pt_add(edl_ctx* ctx, const edl_cts* a, const double* c, edl_cts* out);
/* Tensor + relinearisation (key-switch with the special prime, O11); never rescales. */
edl_status edl_ct_ct_mul_relin(edl_ctx* ctx, const edl_cts* a, const edl_cts* b, edl_cts* out);
/* Divide by the last prime with rounding (O12).  EDL_ERR_LEVEL at level 0. */
edl_status edl_rescale(edl_ctx* ctx, const edl_cts* in, edl_cts* out);
/* Keep limbs 0..level (scale unchanged).  out may alias in only if level == in->level. */
edl_status edl_mod_drop(edl_ctx* ctx, const edl_cts* in, int32_t level, edl_cts* out);

/* ---- layer nodes (O13) ---- */
/* Biased cross-correlation (Eq. cnn) in the batch-in-slots layout:
 * x = H*W ciphertexts (pixel-major), k = host doubles [F][kh][kw], bias [F] (or NULL).
 * out = F*Ho*Wo ciphertexts ([f][r][c] order) at level x.level-1:
 * Rescale(sum_taps x * const(k, q_l)) + const(b). */
edl_status edl_cross_correlate(edl_ctx* ctx, const edl_cts* x, int32_t H, int32_t W, const double* k, int32_t F,
                               int32_t kh, int32_t kw, int32_t stride, const double* bias, edl_cts* out);
/* Polynomial activation: coeffs c_0..c_degree.  Schedules:
 *   degree 3 with c_2 = 0: sigma_a = 0.5 + 0.197x - 0.004x^3, 2 levels;
 *   degree 2 (0, 0, 1): x^2 (C0), 1 level;
 *   degree 2 general: c0 + c1 x + c2 x^2, e.g. ReLU_a = 4/(3 pi q) x^2 + x/2 + q/(3 pi)
 *     (PAPER.md:416), 2 levels: Rescale(Rescale(Relin(x x)) * c2) + drop(Rescale(x * c1)) + c0;
 *   degree 1: c0 + c1 x, e.g. the linear sigmoid 0.5 + 0.197x, 1 level.
 * Output level: x.level - levels; EDL_ERR_LEVEL if x.level is too low; others EDL_ERR_ARG. */
edl_status edl_poly_activation(edl_ctx* ctx, const edl_cts* x, const double* coeffs, int32_t degree, edl_cts* out);
/* Dense: out_o = Rescale(sum_k x_k * const(Wt[o][k], q_l)) + const(b_o).
 * Wt host doubles [O][K] (K = x->count), b [O] or NULL.  defer_rescale != 0 returns the
 * un-rescaled accumulators (level x.level, for the C4 NCCL combine), ignoring b. */
edl_status edl_dense(edl_ctx* ctx, const edl_cts* x, const double* Wt, const double* b, int32_t O,
                     int32_t defer_rescale, edl_cts* out);
/* Finish a deferred dense after the rank partials were summed as uint64 (north_star's
 * NCCL uint64 allreduce): in place x mod q_i (O15). */
edl_status edl_mod_reduce(edl_ctx* ctx, edl_cts* inout);
/* Rescale + bias of combined dense accumulators (b host doubles [count] or NULL). */
edl_status edl_dense_finish(edl_ctx* ctx, const edl_cts* acc, const double* b, edl_cts* out);

/* ---- microbench / test entry points ---- */
/* In-place forward (inverse != 0: inverse) NTT of n_polys * (level+1) limbs laid out
 * [n_polys][level+1][N] (device); limb j uses q_j (j == n_data means P). */
edl_status edl_ntt(edl_ctx* ctx, uint64_t* limbs, int64_t n_polys, int32_t level, int32_t inverse);
/* Key switch with the relinearisation key (C2 microbench; O11 on its own):
 * for every ciphertext (d0, d2) of `d` (level l, NTT domain) -- d2 a polynomial under s^2 --
 * out = (d0 + ks_0, ks_1) with (ks_0, ks_1) = ModDown(sum_j NTT_t([INTT_{q_j} d2_j] mod t)
 * rlk_j), the same pipeline as edl_ct_ct_mul_relin without the tensor product, so
 * decrypt(out) = d0 + d2 s^2 (+ key-switch noise).  out: caller-allocated (count, level),
 * must not alias d; scale and key_id copied from d.  Errors: EDL_ERR_NOKEY, EDL_ERR_ARG.
 * Asynchronous. */
edl_status edl_keyswitch_bench(edl_ctx* ctx, const edl_cts* d, edl_cts* out);
/* Raw Philox4x32-10 words for host counters ctr[n][4] with key (seed lo, seed hi). */
edl_status edl_philox(edl_ctx* ctx, uint64_t seed, const uint32_t* ctr_host, int64_t n, uint32_t* out_host);
/* ---- NEXT f1: the paper's one-image-per-ciphertext layout (kernel masquerading,
 * PAPER.md:279-292): Galois rotations and plaintext vectors ----
 * Rotation by r slots (left; negative r: right) = the automorphism sigma_g, g = 5^r mod 2N
 * (a permutation of NTT-domain residues), then the key switch of sigma_g(c1) back to s
 * with a Galois key that has the relinearisation key's digit structure and gadget term
 * P sigma_g(s) (Philox tags 9/10, object 64 g + digit).  Bit-exact with oracle/galois.py.
 * edl_galois_keygen: keys for each rotation in steps[0..n) (after edl_keygen; the keys live
 *   in the context, ~2 x (L+1)(L+2) 2 N x 8 bytes each).  EDL_ERR_NOKEY without a secret key.
 * edl_rotate: out = in rotated by `steps` slots, same level and scale.  EDL_ERR_NOKEY if no
 *   Galois key for that rotation; out must not alias in.
 * edl_encode_pt: host slots [n_vec][n_slots] -> device NTT-domain plaintexts
 *   pt_out [n_vec][level+1][N] at `scale` (O5 encode, then NTT per limb).  Synchronises.
 * edl_encode_pt_poly: device integer polynomials [n_vec][N] -> pt_out (the bit-exact entry
 *   point, like edl_encrypt_poly: host encoders differ by +-1 in rounding, reading Z1).
 * edl_ct_pt_vec_mul: out = a (.) pt (both polys, NTT domain), scale a.scale * pt_scale, no
 *   rescale; pt_count = 1 (broadcast) or a.count, pt_level >= a.level (else EDL_ERR_LEVEL).
 * edl_export_galois_key: copy the key of rotation `steps` to host ([L+1][2][L+2][N]). */
edl_status edl_galois_keygen(edl_ctx* ctx, uint64_t seed, const int32_t* steps, int32_t n_steps);
edl_status edl_rotate(edl_ctx* ctx, const edl_cts* in, int32_t steps, edl_cts* out);
/* Hoisted rotations (background; oracle/galois.py rotate_hoisted): the digits of c1 are
 * raised to the key-switch basis ONCE (d2 INTT + modulus raise) and every rotation
 * steps[k] applies sigma_g to the raised digits and to c0, then runs the key products and
 * the mod-down: the n_steps outputs cost one raise plus n_steps (permute + MAC + mod-down)
 * instead of n_steps full key switches.  Results decrypt to the rotated slots and differ
 * from edl_rotate's in the key-switch noise only (the lift of sigma_g-negated digit
 * coefficients).  outs[k]: caller-allocated, edl_cts_bytes(count, level) each, must not
 * alias `in`.  Errors: EDL_ERR_NOKEY (a missing Galois key), EDL_ERR_ARG.  Asynchronous. */
edl_status edl_rotate_hoisted(edl_ctx* ctx, const edl_cts* in, const int32_t* steps, int32_t n_steps, edl_cts* outs);
edl_status edl_encode_pt(edl_ctx* ctx, const double* slots, int64_t n_vec, int64_t n_slots, double scale, int32_t level,
                         uint64_t* pt_out);
edl_status edl_encode_pt_poly(edl_ctx* ctx, const int64_t* poly, int64_t n_vec, int32_t level, uint64_t* pt_out);
edl_status edl_ct_pt_vec_mul(edl_ctx* ctx, const edl_cts* a, const uint64_t* pt, int64_t pt_count, int32_t pt_level,
                             double pt_scale, edl_cts* out);
/* ct + plaintext vector (NEXT f1, the packed dense's per-block bias):
 * out_c = (a_c0 + pt_c, a_c1) in the NTT domain; pt [pt_count][pt_level+1][N] device
 * residues from edl_encode_pt(_poly) encoded at a's scale (the caller's choice: the
 * scale is not checked), pt_count = 1 (broadcast) or a.count, pt_level >= a.level.
 * out: caller-allocated (a's count and level), may alias a; scale = a.scale.
 * Errors: EDL_ERR_SHAPE (pt_count), EDL_ERR_LEVEL (pt_level < a.level), EDL_ERR_ARG.
 * Asynchronous. */
edl_status edl_ct_pt_vec_add(edl_ctx* ctx, const edl_cts* a, const uint64_t* pt, int64_t pt_count, int32_t pt_level,
                             edl_cts* out);
/* Multi-plaintext MAC (NEXT f1, the tap-by-tap masked CC over hoisted rotations):
 * rots holds T blocks of n ciphertexts ([T][n][2][level+1][N], count = T n); pts holds
 * F x T NTT-domain plaintexts ([F][T][pt_level+1][N]); out[c F + f] = sum_t rots[t][c] (.)
 * pts[f][t] for both polynomials, scale rots.scale * pt_scale, no rescale (out: n F
 * ciphertexts at rots' level, caller-allocated).  Errors: EDL_ERR_SHAPE (count not a
 * multiple of T), EDL_ERR_LEVEL, EDL_ERR_ARG (T > 64 or null buffers).  Asynchronous. */
edl_status edl_ct_pt_mac_multi(edl_ctx* ctx, const edl_cts* rots, int32_t T, const uint64_t* pts, int32_t F,
                               int32_t pt_level, double pt_scale, edl_cts* out);
edl_status edl_export_galois_key(edl_ctx* ctx, int32_t steps, uint64_t* host_out, size_t words);

/* ---- NEXT f3: client encode / decode on the device (O5 canonical embedding) ----
 * edl_encode_device: device slots [n_vec][n_slots] (float64) -> device integer polynomials
 *   [n_vec][N], m_k = rint(scale u_k) with u the inverse canonical embedding (slot j <->
 *   zeta^{5^j}); a four-step fp64 DFT of length N.  Same +-1 contract with the oracle as
 *   edl_encode (reading Z1).  Feed the result to edl_encrypt_poly.  Asynchronous.
 * edl_decrypt_device: in (count ciphertexts) -> device slots [count][n_slots] (float64):
 *   m = c0 + c1 s, INTT, exact mod-2^64 CRT lift to signed integers (valid while |m| < 2^63,
 *   i.e. for every in-range CKKS message), forward embedding, / scale.  Asynchronous.
 * Errors: EDL_ERR_CAPACITY if n_slots > N/2; EDL_ERR_NOKEY without a secret key. */
edl_status edl_encode_device(edl_ctx* ctx, const double* slots, int64_t n_vec, int64_t n_slots, double scale,
                             int64_t* poly_out);
edl_status edl_decrypt_device(edl_ctx* ctx, const edl_cts* in, double* slots_out, int64_t n_slots);

/* ---- wire format (client <-> server transfer of ciphertext arrays) ----
 * Every residue of limb i is stored in bits_i = bit length of q_i bits (60 or 40 for the
 * Alg. 8 chains) instead of 64: per polynomial, limb i occupies
 * N*bits_i/64 little-endian 64-bit words and coefficient k sits at bit offset k*bits_i;
 * polynomials follow the [count][2] order of edl_cts, limbs 0..level inside each.  For C1
 * (60 + 4 x 40 bits) this is 27.5 instead of 40 bytes per coefficient pair-limb-set:
 * 0.69x the PCIe bytes of the 64-bit layout.
 * edl_cts_packed_bytes: size of `count` ciphertexts at `level` (0 on bad arguments).
 * edl_cts_pack: device array `in` -> device buffer `packed` (caller-allocated, that size).
 * edl_cts_unpack: device buffer `packed` -> device array `out` (caller-allocated,
 *   edl_cts_bytes), setting out's count/level/scale/key_id.  Residues must be canonical
 *   (< q_i), which every library output is.  Asynchronous on the context's stream.
 * Errors: EDL_ERR_ARG on null buffers or a level outside 0..L. */
size_t edl_cts_packed_bytes(const edl_ctx* ctx, int64_t count, int32_t level);
edl_status edl_cts_pack(edl_ctx* ctx, const edl_cts* in, void* packed);
edl_status edl_cts_unpack(edl_ctx* ctx, const void* packed, int64_t count, int32_t level, double scale,
                          uint64_t key_id, edl_cts* out);

/* Seeded wire format for secret-key ciphertexts: only c0 travels, in the packed layout
 * above (half of edl_cts_packed_bytes); the receiver regenerates c1 from the seed.
 * edl_cts_seeded_bytes: size of `count` ciphertexts at `level` (0 on bad arguments).
 * edl_cts_pack_c0: device array `in` -> device buffer (caller-allocated, that size): the
 *   c0 polynomials of every ciphertext (c1 is not read).
 * edl_cts_unpack_seeded: device buffer -> device array `out` (edl_cts_bytes): c0 unpacked,
 *   c1_i[k] = uniform(enc_seed, obj0 + c, limb i, tag 11) regenerated on the device (the
 *   arguments the ciphertexts were encrypted with by edl_encrypt_poly_sk).  Sets out's
 *   metadata.  Asynchronous.  Errors: EDL_ERR_ARG on null buffers or a bad level. */
size_t edl_cts_seeded_bytes(const edl_ctx* ctx, int64_t count, int32_t level);
edl_status edl_cts_pack_c0(edl_ctx* ctx, const edl_cts* in, void* packed);
edl_status edl_cts_unpack_seeded(edl_ctx* ctx, const void* packed, int64_t count, int32_t level, double scale,
                                 uint64_t key_id, uint64_t enc_seed, uint32_t obj0, edl_cts* out);

/* Host wire path (the EDLaaS server's receive / reply side, PAPER.md:85 client-server split;
 * DESIGN.md §7b): ciphertexts arrive in HOST memory in a wire format and results return to
 * HOST memory; the context owns two device staging slots and a copy stream, so the transfer
 * of batch k+1 overlaps the compute of batch k.
 * edl_wire_upload: enqueue the copy of `bytes` (a multiple of 8) of host memory `host`
 *   (pinned memory for an asynchronous copy; it must stay valid until the slot's unpack has
 *   run) into staging slot `slot` (0 or 1) on the copy stream, after the last unpack that
 *   read the slot; returns at once.  The slot's device buffer is (re)allocated when `bytes`
 *   exceeds its capacity (this synchronises).
 * edl_cts_unpack_host / edl_cts_unpack_seeded_host: edl_cts_unpack / edl_cts_unpack_seeded
 *   reading staging slot `slot`: the context's stream waits for the slot's copy, unpacks into
 *   the device array `out`, and frees the slot for the next upload.  Asynchronous.
 * edl_cts_download: enqueue the device -> host copy of a ciphertext array (64-bit layout,
 *   edl_cts_bytes) into `host_out` on the context's stream; the bytes are valid after
 *   edl_ctx_sync.
 * Errors: EDL_ERR_ARG on a bad slot, null buffers, a size that is not a multiple of 8, or a
 *   slot holding fewer bytes than the array needs; EDL_ERR_CUDA when the copy cannot be queued. */
edl_status edl_wire_upload(edl_ctx* ctx, int32_t slot, const void* host, size_t bytes);
edl_status edl_cts_unpack_host(edl_ctx* ctx, int32_t slot, int64_t count, int32_t level, double scale, uint64_t key_id,
                               edl_cts* out);
edl_status edl_cts_unpack_seeded_host(edl_ctx* ctx, int32_t slot, int64_t count, int32_t level, double scale,
                                      uint64_t key_id, uint64_t enc_seed, uint32_t obj0, edl_cts* out);
edl_status edl_cts_download(edl_ctx* ctx, const edl_cts* x, void* host_out);
/* Block the calling host thread until everything queued on the context's streams (compute,
 * side and copy stream) has completed; reports a pending CUDA error as EDL_ERR_CUDA. */
edl_status edl_ctx_sync(edl_ctx* ctx);

/* Integer-pipe ceiling: lazy Shoup 64-bit modular multiplications per second measured
 * by a register-only kernel on all SMs (the "alu" roofline peak). */
edl_status edl_modmul_peak(edl_ctx* ctx, int32_t iters, double* modmul_per_s);

/* Butterfly ceiling of the NTT's arithmetic for modulus `prime_index` (0..L data primes,
 * L+1 = P): a register-only kernel of independent Harvey Cooley-Tukey butterflies
 * on every SM, through the same twiddle-product path the NTT kernels
 * take for that modulus (FP64 quotient if q < 2^50, Shoup otherwise).  Writes butterflies
 * per second to *bfly_per_s.  Synchronises.  EDL_ERR_ARG on a bad index or iters <= 0. */
edl_status edl_bfly_peak(edl_ctx* ctx, int32_t prime_index, int32_t iters, double* bfly_per_s);
/* Raw pipe probes anchoring the butterfly and MAC ceilings: lane-operations per second of
 * register-only chains of DFMA (which = 0, the FP64 pipe), 32x32->64 IMAD.WIDE.U32
 * (which = 1, the integer multiply the Shoup butterflies are built from), the F64 modular
 * MAC acc += x w mod q (which = 2, the MAC layers' 40-bit path) or the 128-bit lazy MAC
 * acc += x w (which = 3, their 60-bit path), on every SM (8 CTAs of 256 threads per SM,
 * 8 independent chains per thread).  EDL_ERR_ARG for another `which`.  Synchronises. */
edl_status edl_pipe_peak(edl_ctx* ctx, int32_t which, int32_t iters, double* ops_per_s);
/* Copy the secret key s_hat [L+2][N], public key [2][L+1][N] or rlk [L+1][2][L+2][N]
 * to host (which: 0, 1, 2).  For parity tests. */
edl_status edl_export_key(edl_ctx* ctx, int32_t which, uint64_t* host_out, size_t words);

#ifdef __cplusplus
}
#endif
#endif /* EDL_H */
