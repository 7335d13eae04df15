// kernels.cuh -- launch interface between the C-ABI host code (api.cu) and the
// sm_100a kernels.  Ciphertext arrays are uint64 [count][2][level+1][N] (NTT domain,
// canonical residues), SURVEY §8(a) layout.
#pragma once
#include <cstdlib>
#include <cuda_runtime.h>
#include <cstdint>
#include <vector>
#include "arith.cuh"

namespace edl {

constexpr int MAXM = 34;   // max moduli (data primes + P)

// Per-chain constants used by rescale / mod-down epilogues.
struct ChainConsts {
    int L;                           // highest data level; P is modulus index L+1
    uint64_t qmod[MAXM][MAXM];       // qmod[a][b] = q_a mod q_b
    ulonglong2 qinv[MAXM][MAXM];     // qinv[a][b] = q_a^{-1} mod q_b (a != b) with Shoup
};

__host__ __device__ inline size_t limb_off(int64_t ct, int poly, int limb, int nl, int logn) {
    return ((((size_t)ct * 2 + poly) * (size_t)nl) + (size_t)limb) << logn;
}

// Launch accounting + optional per-launch CUDA-event timing (edl_profile).
struct Prof {
    struct Rec {
        const char* name;
        cudaEvent_t a, b;
    };
    bool on = false;
    bool sync_check = std::getenv("EDL_DEBUG_SYNC") != nullptr;   // debug: synchronise + check after every launch
    const char* last = nullptr;
    int64_t launches = 0;
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    cudaEvent_t ev();
    void begin(const char* name, cudaStream_t st);
    void end(cudaStream_t st);
    void reset();
    ~Prof();
};

// All moduli of a context as one kernel parameter (constant bank: uniform loads, no
// vector registers held for the per-limb constants).
struct ModTable {
    ModInfo m[MAXM];
    __host__ __device__ const ModInfo& operator[](int i) const { return m[i]; }
};

struct Dev {
    const ModInfo* mods;        // [L+2] (device)
    const ModTable* mt;         // host copy passed by value to every kernel
    const ModInfo* hmods;       // [L+2] (host copy: launch-time decisions such as the arithmetic path)
    const ChainConsts* cc;
    int logn;
    int L;
    cudaStream_t st;
    Prof* prof;
    bool ks_fused = false;      // key switch: fused modulus raise + key products (k_relin_ks, N = 2^14)
    bool raise_fused = false;   // key switch: fused d2 INTT + modulus raise (k_relin_raise, N = 2^14)
    // relinearisation key and its copy with P^-1 folded into the data limbs (keygen):
    // the key-product pass uses the copy when it is handed `rlk`
    const uint64_t* rlk = nullptr;
    const uint64_t* rlk_pf = nullptr;
    const uint64_t* rlk_pf_c = nullptr;
};

// Supported ring degrees: 2^10 .. 2^16 (N > 2^13 runs one limb per thread-block cluster).
// EDL_LOGNS_MASK (bit k = 2^k supported) trims development builds; default: all.
#ifndef EDL_LOGNS_MASK
#define EDL_LOGNS_MASK 0x1FC00
#endif
#define EDL_LOGN_CASE(K, ...) \
    case K: { constexpr int LOGN = K; if constexpr (((EDL_LOGNS_MASK) >> K) & 1) { __VA_ARGS__; } } break;
#define EDL_DISPATCH_LOGN(logn, ...)        \
    switch (logn) {                          \
        EDL_LOGN_CASE(10, __VA_ARGS__)       \
        EDL_LOGN_CASE(11, __VA_ARGS__)       \
        EDL_LOGN_CASE(12, __VA_ARGS__)       \
        EDL_LOGN_CASE(13, __VA_ARGS__)       \
        EDL_LOGN_CASE(14, __VA_ARGS__)       \
        EDL_LOGN_CASE(15, __VA_ARGS__)       \
        EDL_LOGN_CASE(16, __VA_ARGS__)       \
        default: break;                      \
    }

void ensure_smem_attr(const void* kern, int bytes);

// Programmatic dependent launch (arith.cuh EDL_PDL_ENTRY; on unless EDL_PDL=0 in the
// environment, read once): the launch may overlap the tail of the stream's previous kernel.
// Off while per-launch profiling brackets every launch with events (they serialise anyway).
// Measured (C1, B200, round 2c): 4.024 -> 4.002 ms per step; with an early trigger
// (griddepcontrol.launch_dependents at CTA entry, EDL_PDL_TRIGGER) 4.03: the waiting
// dependent CTAs take SM slots the other stream's kernels would use.
bool pdl_enabled();
inline int pdl_attr(const Dev& d, cudaLaunchAttribute* at) {
    if (!pdl_enabled() || d.prof->on) return 0;
    at->id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at->val.programmaticStreamSerializationAllowed = 1;
    return 1;
}
// A plain (non-cluster) launch with the PDL attribute: the <<<>>> form of the hot kernels.
template <typename... KArgs, typename... Args>
void launch_k(const Dev& d, const char* name, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = d.st;
    cudaLaunchAttribute at[1];
    cfg.numAttrs = pdl_attr(d, at);
    cfg.attrs = at;
    d.prof->begin(name, d.st);
    cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
    d.prof->end(d.st);
}

// Launch an NTT-family kernel with config C: grid.x is multiplied by the cluster size
// C::K (consecutive blocks form one limb's cluster), block = C::T threads, dynamic shared
// memory C::SMEM_BYTES.
template <class C, typename... KArgs, typename... Args>
void launch_cfg_x(const Dev& d, const char* name, void (*kern)(KArgs...), dim3 grid, int extra_smem, Args... args) {
    const int smem = C::SMEM_BYTES + extra_smem;
    ensure_smem_attr((const void*)kern, smem);
    grid.x *= C::K;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(C::T, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = d.st;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (C::K > 1) {
        at[na].id = cudaLaunchAttributeClusterDimension;
        at[na].val.clusterDim.x = C::K;
        at[na].val.clusterDim.y = 1;
        at[na].val.clusterDim.z = 1;
        na++;
    }
    na += pdl_attr(d, at + na);
    cfg.attrs = at;
    cfg.numAttrs = na;
    d.prof->begin(name, d.st);
    cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
    d.prof->end(d.st);
}
template <class C, typename... KArgs, typename... Args>
void launch_cfg(const Dev& d, const char* name, void (*kern)(KArgs...), dim3 grid, Args... args) {
    launch_cfg_x<C>(d, name, kern, grid, 0, args...);
}

// Persistent cluster launch: as many clusters of C::K CTAs as can be co-resident (at most
// one per work item), block = C::T threads, dynamic shared memory = the transform buffer
// plus the rank's twiddle table (C::M entries of 16 bytes).
template <class C, typename... KArgs, typename... Args>
void launch_persist(const Dev& d, const char* name, void (*kern)(KArgs...), int64_t items, Args... args) {
    const int smem = C::SMEM_BYTES + C::M * 16;
    ensure_smem_attr((const void*)kern, smem);
    static thread_local std::vector<std::pair<const void*, int>> occ;
    int ncl = 0;
    for (auto& e : occ)
        if (e.first == (const void*)kern) ncl = e.second;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(C::T, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = d.st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C::K;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (ncl == 0) {
        cfg.gridDim = dim3(C::K * 1024, 1, 1);
        if (cudaOccupancyMaxActiveClusters(&ncl, (void*)kern, &cfg) != cudaSuccess || ncl < 1) ncl = 1;
        occ.emplace_back((const void*)kern, ncl);
    }
    const int64_t g = items < ncl ? items : ncl;
    if (g <= 0) return;
    cfg.gridDim = dim3((unsigned)(g * C::K), 1, 1);
    d.prof->begin(name, d.st);
    cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
    d.prof->end(d.st);
}

#define EDL_LAUNCH(d, name, ...)                         \
    do {                                                  \
        (d).prof->begin(name, (d).st);                    \
        __VA_ARGS__;                                      \
        (d).prof->end((d).st);                            \
    } while (0)

// ---- per-degree launchers (defined in ntt_kernels.cuh / rng_kernels.cuh, instantiated in
// ntt_inst_<logN>.cu) ----
struct PrimeMap {
    int8_t idx[MAXM];
};
template <int LOGN>
void launch_ntt_limbs_n(const Dev& d, uint64_t* data, int64_t batch, int nl, const PrimeMap& pm, bool inverse);
template <int LOGN>
void launch_rescale_intt_n(const Dev& d, const uint64_t* in, int64_t cnt, int l, const ulonglong2* w, uint64_t* r_out,
                           const ulonglong2* w2, uint64_t* r_out2);
template <int LOGN>
void launch_rescale_ntt_n(const Dev& d, const uint64_t* in, int64_t cnt, int l, const ulonglong2* w, const uint64_t* r,
                          const uint64_t* bias, uint64_t* out, int nlo);
template <int LOGN>
void launch_relin_n(const Dev& d, const uint64_t* a, const uint64_t* b, int64_t cnt, int l, bool rescale,
                    const uint64_t* rlk, const uint64_t* rlk_c, uint64_t* acoef, uint64_t* xh, uint64_t* acc, uint64_t* r,
                    uint64_t* s, uint64_t* out, const uint64_t* add_w, const uint64_t* add_k);
// key inner product of the relinearisation (pointwise.cu): acc [cnt][2][l+2][N] from the
// raised digits xh [cnt][l+1][l+2][N], the tensor's d2 (a1 b1) and rlk [L+1][2][L+2][N]
void launch_relin_mac(const Dev& d, const uint64_t* a, const uint64_t* b, int64_t cnt, int l, const uint64_t* xh,
                      const uint64_t* rlk, const uint64_t* rlk_c, uint64_t* acc);
template <int LOGN>
void launch_keygen_n(const Dev& d, uint64_t seed, uint64_t* s_hat, uint64_t* pk, uint64_t* rlk, uint64_t* rlk_s);
template <int LOGN>
void launch_encrypt_n(const Dev& d, const int64_t* msg, int64_t cnt, int l, uint64_t seed, uint32_t obj0,
                      const uint64_t* pk, uint64_t* out);
template <int LOGN>
void launch_encrypt_sk_n(const Dev& d, const int64_t* msg, int64_t cnt, int l, uint64_t seed, uint64_t eseed,
                         uint32_t obj0, const uint64_t* s_hat, uint64_t* out);
template <int LOGN>
void launch_keygen_galois_n(const Dev& d, uint64_t seed, uint32_t g, const uint64_t* s_hat, uint64_t* gk, uint64_t* gk_c);
template <int LOGN>
void launch_encode_pt_n(const Dev& d, const int64_t* msg, int64_t cnt, int l, uint64_t* out);
template <int LOGN>
void launch_decrypt_n(const Dev& d, const uint64_t* ct, int64_t cnt, int l, const uint64_t* s_hat, uint64_t* out);

// ---- NTT family (ntt_kernels.cu) ----
void launch_ntt_limbs(const Dev& d, uint64_t* data, int64_t batch, int nl, const int* prime_idx_host, bool inverse);
// rescale: r_out [cnt][2][N] <- INTT_{q_l}(in[.][.][l] * w_l) ; w may be null
void launch_rescale_intt(const Dev& d, const uint64_t* in, int64_t cnt, int l, const ulonglong2* w, uint64_t* r_out,
                         const ulonglong2* w2 = nullptr, uint64_t* r_out2 = nullptr);
// out [cnt][2][lo+1][N] <- (in_i * w_i - NTT_i([r]_{q_l} mod q_i)) * q_l^{-1} (+ bias_i on poly 0),
// i <= lo; lo = -1 means the full rescaled level l-1 (a smaller lo fuses a mod-drop)
void launch_rescale_ntt(const Dev& d, const uint64_t* in, int64_t cnt, int l, const ulonglong2* w,
                        const uint64_t* r, const uint64_t* bias, uint64_t* out, int lo = -1);
// relinearisation of the tensor a (x) b at level l (+ optional rescale by q_l)
// add_w / add_k (rescale only, optional): out += add_w (a ciphertext array at the output
// level) + add_k[c][i] on polynomial 0, fused into the last kernel's epilogue
void launch_relin(const Dev& d, const uint64_t* a, const uint64_t* b, int64_t cnt, int l, bool rescale,
                  const uint64_t* rlk, const uint64_t* rlk_s, uint64_t* scratch, uint64_t* out,
                  const uint64_t* add_w = nullptr, const uint64_t* add_k = nullptr);
size_t relin_scratch_words(int64_t cnt, int l, int logn);
template <int LOGN>
void launch_relin_raise_n(const Dev& d, const uint64_t* a, int64_t cnt, int l, uint64_t* acoef, uint64_t* xh);
template <int LOGN>
void launch_relin_finish_n(const Dev& d, const uint64_t* a, int64_t cnt, int l, const uint64_t* rlk,
                           const uint64_t* rlk_c, uint64_t* xh, uint64_t* acc, uint64_t* r, uint64_t* s, uint64_t* out);
// hoisted rotations on the relin scratch layout: raise c1 of `a` once, finish per element
// (the raised digits at the scratch's xh slot, already permuted by the caller)
void launch_relin_raise(const Dev& d, const uint64_t* a, int64_t cnt, int l, uint64_t* scratch);
void launch_relin_finish(const Dev& d, const uint64_t* a, int64_t cnt, int l, const uint64_t* rlk, const uint64_t* rlk_s,
                         uint64_t* scratch, uint64_t* out);
// pointer to the raised digits [cnt][l+1][l+2][N] inside a relin scratch block
uint64_t* relin_scratch_xh(uint64_t* scratch, int64_t cnt, int l, int logn);
// out [n*F] = sum_t rots[t] (.) pts[f][t]; rots [T][n][2][l+1][N], pts [F][T][ptl+1][N]
void launch_pt_mac_multi(const Dev& d, const uint64_t* rots, int T, int64_t n, int l, const uint64_t* pts, int F, int ptl,
                         uint64_t* out);
// sigma_g on `rows` NTT-domain rows of N residues
void launch_automorphism_rows(const Dev& d, const uint64_t* in, int64_t rows, uint32_t g, uint64_t* out);

// ---- pointwise family (pointwise.cu) ----
// out [cnt][2][lo+1] = a (level la) + b (level lb), lo <= min(la, lb)
void launch_add(const Dev& d, const uint64_t* a, int la, const uint64_t* b, int lb, int64_t cnt, int lo, uint64_t* out);
// out = a * w[c][i] (Shoup consts [cnt][l+1])
void launch_mul_const(const Dev& d, const uint64_t* a, int64_t cnt, int l, const ulonglong2* w, uint64_t* out);
// out = a + k[c][i] on poly 0 (consts [cnt][l+1]); out may alias a
void launch_add_const(const Dev& d, const uint64_t* a, int64_t cnt, int l, const uint64_t* k, uint64_t* out);
// out (level lo) = limbs 0..lo of a (level la)
void launch_mod_drop(const Dev& d, const uint64_t* a, int64_t cnt, int la, int lo, uint64_t* out);
// in place: x mod q_i
void launch_mod_reduce(const Dev& d, uint64_t* x, int64_t cnt, int l);
// v (level lo) + w (level lw >= lo) + k[c][i] on poly 0 -> out (level lo)
void launch_add_add_const(const Dev& d, const uint64_t* v, const uint64_t* w, int lw, int64_t cnt, int lo,
                          const uint64_t* k, uint64_t* out);
// cross-correlation MAC: out[f*Ho*Wo + r*Wo + c] = sum_{u,v} x[(r*st+u)*W + c*st+v] * wk[f][u*kw+v][i]
void launch_cc_mac(const Dev& d, const uint64_t* x, int l, int H, int W, int F, int kh, int kw, int stride,
                   const ulonglong2* wk /*[F][kh*kw][l+1] {residue, companion}*/, uint64_t* out,
                   const ulonglong2* hw = nullptr /*host copy of wk: 4x4 taps go to k_cc_mac4*/);
// dense MAC: out[o] = sum_k x[k] * wd[o][k][i]  (x: K cts, out: O cts, level l)
// part: scratch for split-K partial sums (dense_split(...) * O * 2 * (l+1) * N words) or null
void launch_dense_mac(const Dev& d, const uint64_t* x, int64_t K, int64_t O, int l, const ulonglong2* wd, uint64_t* out,
                      uint64_t* part = nullptr);
int dense_split(const Dev& d, int64_t K, int64_t O, int l);

// NEXT f1: Galois key [L+1][2][L+2][N] (+ companions) for element g; NTT-domain plaintexts
// [cnt][l+1][N] from integer polynomials; sigma_g of ct arrays; ct (.) plaintext vectors
void launch_keygen_galois(const Dev& d, uint64_t seed, uint32_t g, const uint64_t* s_hat, uint64_t* gk, uint64_t* gk_c);
void launch_encode_pt(const Dev& d, const int64_t* msg, int64_t cnt, int l, uint64_t* out);
void launch_automorphism(const Dev& d, const uint64_t* in, int64_t cnt, int l, uint32_t g, uint64_t* out);
// out = a (.) pt ; pt [pt_count][pt_level+1][N], pt_count = 1 (broadcast) or cnt, pt_level >= l
void launch_mul_pt(const Dev& d, const uint64_t* a, int64_t cnt, int l, const uint64_t* pt, int64_t pt_count,
                   int pt_level, uint64_t* out);

// out = a + pt on polynomial 0 (pt as in launch_mul_pt)
void launch_add_pt(const Dev& d, const uint64_t* a, int64_t cnt, int l, const uint64_t* pt, int64_t pt_count,
                   int pt_level, uint64_t* out);

// NEXT f3 (fft.cu): device canonical embedding; scratch fft_scratch_bytes(n_vec, logn)
size_t fft_scratch_bytes(int64_t n_vec, int logn);
void launch_encode_slots(const Dev& d, const double* z, int64_t n_vec, int64_t n_slots, double scale, int64_t* m,
                         void* scratch);
void launch_decode_slots(const Dev& d, const uint64_t* r, int64_t n_vec, int nl, const uint64_t* q,
                         const uint64_t* qhat_inv, const uint64_t* qhat64, uint64_t Q64, int64_t n_slots, double scale,
                         double* z, void* scratch);

// wire format: residues of limb i in bits[i] bits (pointwise.cu); polys = count * 2
void launch_unpack(const Dev& d, const uint64_t* in, int64_t polys, int nl, const int* bits, uint64_t* out,
                   int stride = 1);
void launch_pack(const Dev& d, const uint64_t* in, int64_t polys, int nl, const int* bits, uint64_t* out,
                 int stride = 1);
// dst[0..words) = src (mapped pinned host memory read by the SMs: no DMA engine)
void launch_fetch_mapped(const Dev& d, const uint64_t* src, uint64_t* dst, int64_t words);

// ---- randomness / keys / encryption (rng.cu) ----
void launch_keygen(const Dev& d, uint64_t seed, uint64_t* s_hat /*[L+2][N]*/, uint64_t* pk /*[2][L+1][N]*/,
                   uint64_t* rlk /*[L+1][2][L+2][N]*/, uint64_t* rlk_s, uint64_t* scratch);
// rlk_pf[j][c][t] = rlk[j][c][t] P^-1 mod q_t for data limbs t <= L (rlk for t = P), with
// mulc() companions (the key-product pass's P^-1 fold moved into the key)
void launch_fold_pinv(const Dev& d, const uint64_t* rlk, uint64_t* rlk_pf, uint64_t* rlk_pf_c);
void launch_encrypt(const Dev& d, const int64_t* msg /*[cnt][N]*/, int64_t cnt, int l, uint64_t seed, uint32_t obj0,
                    const uint64_t* pk, uint64_t* out);
// secret-key encryption (reading Z16) and the server-side regeneration of its seeded c1
void launch_encrypt_sk(const Dev& d, const int64_t* msg, int64_t cnt, int l, uint64_t seed, uint64_t eseed,
                       uint32_t obj0, const uint64_t* s_hat, uint64_t* out);
void launch_expand_sk_a(const Dev& d, uint64_t* ct, int64_t cnt, int l, uint64_t seed, uint32_t obj0);
// m_hat = c0 + c1 s, INTT -> coefficient residues [cnt][l+1][N]
void launch_decrypt(const Dev& d, const uint64_t* ct, int64_t cnt, int l, const uint64_t* s_hat, uint64_t* out);
void launch_philox_words(const Dev& d, uint64_t seed, const uint32_t* ctr /*[n][4]*/, int64_t n, uint32_t* out);

void launch_bfly_peak(const Dev& d, uint64_t q, bool fp, const ulonglong2* tw, int iters, int blocks, uint64_t* sink);
void launch_modmul_peak(const Dev& d, uint64_t q, uint64_t w, uint64_t ws, int iters, int blocks, uint64_t* sink);
// which = 0: DFMA chains, 1: IMAD.WIDE.U32 chains (8 per thread, 256 threads per CTA)
void launch_pipe_probe(const Dev& d, int which, int iters, int blocks, uint64_t* sink);

bool set_smem_attrs(int logn);

}  // namespace edl
