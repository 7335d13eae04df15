// rng.cu -- host dispatch of key generation, encryption and decryption (rng_kernels.cuh,
// instantiated per ring degree in ntt_inst_<logN>.cu) and the raw Philox word kernel.
#include "rng_kernels.cuh"

namespace edl {

__global__ void k_philox_words(uint64_t seed, const uint32_t* __restrict__ ctr, int64_t n, uint32_t* __restrict__ out) {
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
