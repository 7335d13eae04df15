// rng.cu -- host dispatch of key generation, encryption and decryption (rng_kernels.cuh,
// instantiated per ring degree in ntt_inst_<logN>.cu) and the raw Philox word kernel.
#include "rng_kernels.cuh"

namespace edl {

__global__ void k_philox_words(uint64_t seed, const uint32_t* __restrict__ ctr, int64_t n, uint32_t* __restrict__ out) {
    EDL_PDL_ENTRY();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    uint4 r = draw(seed, ctr[4 * t], ctr[4 * t + 1], ctr[4 * t + 2], ctr[4 * t + 3]);
    out[4 * t] = r.x;
    out[4 * t + 1] = r.y;
    out[4 * t + 2] = r.z;
    out[4 * t + 3] = r.w;
}

void launch_keygen(const Dev& d, uint64_t seed, uint64_t* s_hat, uint64_t* pk, uint64_t* rlk, uint64_t* rlk_s,
                   uint64_t* /*scratch*/) {
    EDL_DISPATCH_LOGN(d.logn, launch_keygen_n<LOGN>(d, seed, s_hat, pk, rlk, rlk_s));
}

void launch_encrypt(const Dev& d, const int64_t* msg, int64_t cnt, int l, uint64_t seed, uint32_t obj0,
                    const uint64_t* pk, uint64_t* out) {
    EDL_DISPATCH_LOGN(d.logn, launch_encrypt_n<LOGN>(d, msg, cnt, l, seed, obj0, pk, out));
}

void launch_encrypt_sk(const Dev& d, const int64_t* msg, int64_t cnt, int l, uint64_t seed, uint64_t eseed,
                       uint32_t obj0, const uint64_t* s_hat, uint64_t* out) {
    EDL_DISPATCH_LOGN(d.logn, launch_encrypt_sk_n<LOGN>(d, msg, cnt, l, seed, eseed, obj0, s_hat, out));
}

// Seeded public component of secret-key ciphertexts: c1[c][i][k] = uniform(seed, k, obj0 + c, i, TAG_SK_A).
__global__ void k_expand_sk_a(uint64_t* __restrict__ ct, int64_t cnt, int l, uint64_t seed, uint32_t obj0,
                              const __grid_constant__ ModTable mods, int logn) {
    EDL_PDL_ENTRY();
    const int64_t rows = cnt * (l + 1);
    const int n = 1 << logn;
    for (int64_t row = blockIdx.y; row < rows; row += gridDim.y) {
        const int i = (int)(row % (l + 1));
        const int64_t c = row / (l + 1);
        const ModInfo& m = mods[i];
        uint64_t* c1 = ct + limb_off(c, 1, i, l + 1, logn);
        for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
            c1[k] = uniform_of(draw(seed, (uint32_t)k, obj0 + (uint32_t)c, (uint32_t)i, TAG_SK_A), m);
    }
}

void launch_expand_sk_a(const Dev& d, uint64_t* ct, int64_t cnt, int l, uint64_t seed, uint32_t obj0) {
    const int64_t rows = cnt * (l + 1);
    const dim3 grid((unsigned)((1 << d.logn) / 256), (unsigned)(rows < 65535 ? rows : 65535));
    EDL_LAUNCH(d, "k_expand_sk_a", k_expand_sk_a<<<grid, 256, 0, d.st>>>(ct, cnt, l, seed, obj0, *d.mt, d.logn));
}

__global__ void k_fold_pinv(const uint64_t* __restrict__ rlk, uint64_t* __restrict__ pf, uint64_t* __restrict__ pfc,
                            int L, const __grid_constant__ ModTable mods, const ChainConsts* __restrict__ cc, int logn) {
    EDL_PDL_ENTRY();
    const int64_t rows = (int64_t)(L + 1) * 2 * (L + 2);
    const int n = 1 << logn;
    for (int64_t row = blockIdx.y; row < rows; row += gridDim.y) {
        const int t = (int)(row % (L + 2));
        const ModInfo& m = mods[t];
        const ulonglong2 pinv = (t <= L) ? cc->qinv[L + 1][t] : make_ulonglong2(1, 0);
        const uint64_t* src = rlk + ((size_t)row << logn);
        for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
            const uint64_t v = (t <= L) ? mulc(src[k], pinv, m) : src[k];
            pf[((size_t)row << logn) + k] = v;
            pfc[((size_t)row << logn) + k] = key_companion(v, m);
        }
    }
}

void launch_fold_pinv(const Dev& d, const uint64_t* rlk, uint64_t* rlk_pf, uint64_t* rlk_pf_c) {
    const int64_t rows = (int64_t)(d.L + 1) * 2 * (d.L + 2);
    const dim3 grid((unsigned)((1 << d.logn) / 256), (unsigned)(rows < 65535 ? rows : 65535));
    EDL_LAUNCH(d, "k_fold_pinv", k_fold_pinv<<<grid, 256, 0, d.st>>>(rlk, rlk_pf, rlk_pf_c, d.L, *d.mt, d.cc, d.logn));
}

void launch_keygen_galois(const Dev& d, uint64_t seed, uint32_t g, const uint64_t* s_hat, uint64_t* gk, uint64_t* gk_c) {
    EDL_DISPATCH_LOGN(d.logn, launch_keygen_galois_n<LOGN>(d, seed, g, s_hat, gk, gk_c));
}

void launch_encode_pt(const Dev& d, const int64_t* msg, int64_t cnt, int l, uint64_t* out) {
    EDL_DISPATCH_LOGN(d.logn, launch_encode_pt_n<LOGN>(d, msg, cnt, l, out));
}

void launch_decrypt(const Dev& d, const uint64_t* ct, int64_t cnt, int l, const uint64_t* s_hat, uint64_t* out) {
    EDL_DISPATCH_LOGN(d.logn, launch_decrypt_n<LOGN>(d, ct, cnt, l, s_hat, out));
}

void launch_philox_words(const Dev& d, uint64_t seed, const uint32_t* ctr, int64_t n, uint32_t* out) {
    const int th = 256;
    EDL_LAUNCH(d, "k_philox_words", k_philox_words<<<(unsigned)((n + th - 1) / th), th, 0, d.st>>>(seed, ctr, n, out));
}

}  // namespace edl
