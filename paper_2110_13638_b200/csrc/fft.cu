// fft.cu -- client-side CKKS canonical embedding on the GPU (O5).
//
//   encode: v_{(e_j-1)/2} = v_{N-1-(e_j-1)/2} = z_j (e_j = 5^j mod 2N), w = DFT_N(v),
//           u_k = Re(w_k exp(-i pi k / N)) / N,  m_k = rint(Delta u_k)   (round half even)
//   decode: v_t = sum_k m_k exp(i pi k / N) exp(2 pi i t k / N),  z_j = Re(v_{(e_j-1)/2}) / Delta
//
// The length-N complex DFT (N up to 2^16 doubles: more than one CTA's shared memory)
// runs as a four-step transform N = 128 x (N/128): 128-point DFTs down the columns, the
// exp(+-2 pi i k1 c / N) twist, then (N/128)-point DFTs along the rows, each a radix-2
// FFT on a shared-memory copy of its column/row with a sincospi root table (fp64).  The encoder's +-1 contract with the oracle (reading Z1) is checked in the
// GPU tests.  Decrypted coefficients are lifted from residues to signed 64-bit integers
// with the same exact-mod-2^64 CRT as the host path.
#include "kernels.cuh"

namespace edl {

namespace {

constexpr int FFT_N1 = 128;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// 5^j mod 2N by square-and-multiply
__device__ __forceinline__ uint32_t pow5(uint32_t j, uint32_t two_n) {
    uint64_t r = 1, b = 5;
    while (j) {
        if (j & 1) r = r * b % two_n;
        b = b * b % two_n;
        j >>= 1;
    }
    return (uint32_t)r;
}

__global__ void k_encode_prep(const double* __restrict__ z, int64_t n_vec, int64_t n_slots, int logn,
                              double2* __restrict__ v) {
    EDL_PDL_ENTRY();
    const int64_t n = 1LL << logn;
    const int64_t b = blockIdx.y;
    double2* vb = v + b * n;
    for (int64_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n / 2; j += gridDim.x * blockDim.x) {
        const double zj = j < n_slots ? z[b * n_slots + j] : 0.0;
        const uint32_t e = pow5((uint32_t)j, (uint32_t)(2 * n));
        const int64_t t = (e - 1) / 2;
        vb[t] = make_double2(zj, 0.0);
        vb[n - 1 - t] = make_double2(zj, 0.0);
    }
}

// In-place radix-2 DFT of length L = 2^logL held in shared memory, X[k] = sum_r x[r] w^{rk},
// w = exp(sign 2 pi i / L): bit-reversal permutation, then logL Cooley-Tukey stages with the
// roots root[k] = w^k (k < L/2) from a shared table.  All threads of the block take part.
__device__ void fft_smem(double2* a, const double2* root, int L, int logL) {
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
        const int j = (int)(__brev((uint32_t)i) >> (32 - logL));
        if (i < j) {
            const double2 t = a[i];
            a[i] = a[j];
            a[j] = t;
        }
    }
    __syncthreads();
    for (int s = 0; s < logL; s++) {
        const int half = 1 << s;
        for (int t = threadIdx.x; t < L / 2; t += blockDim.x) {
            const int k = t & (half - 1);
            const int i0 = ((t >> s) << (s + 1)) + k;
            const double2 w = root[k << (logL - 1 - s)];
            const double2 u = a[i0], v = cmul(a[i0 + half], w);
            a[i0] = make_double2(u.x + v.x, u.y + v.y);
            a[i0 + half] = make_double2(u.x - v.x, u.y - v.y);
        }
        __syncthreads();
    }
}

// stage 1: for vector b, column c < n2: X1[k1][c] = twist^(k1 c) sum_r x[r n2 + c] w128^(r k1)
__global__ void __launch_bounds__(FFT_N1) k_fft_cols(const double2* __restrict__ in, double2* __restrict__ out, int logn,
                                                     int sign) {
    EDL_PDL_ENTRY();
    __shared__ double2 col[FFT_N1];
    __shared__ double2 root[FFT_N1 / 2];
    const int64_t n = 1LL << logn;
    const int n2 = (int)(n / FFT_N1);
    const int c = blockIdx.x;
    const int64_t b = blockIdx.y;
    const int k1 = threadIdx.x;
    col[k1] = in[b * n + (int64_t)k1 * n2 + c];
    double s, co;
    if (k1 < FFT_N1 / 2) {
        sincospi(2.0 * (double)k1 / FFT_N1, &s, &co);
        root[k1] = make_double2(co, sign * s);
    }
    __syncthreads();
    fft_smem(col, root, FFT_N1, 7);
    sincospi(2.0 * (double)(((int64_t)k1 * c) % n) / (double)n, &s, &co);
    out[b * n + (int64_t)k1 * n2 + c] = cmul(col[k1], make_double2(co, sign * s));
}

// stage 2: for vector b, row k1: X[k1 + 128 k2] = sum_c X1[k1][c] w_{n2}^(c k2)
__global__ void k_fft_rows(const double2* __restrict__ in, double2* __restrict__ out, int logn, int sign) {
    EDL_PDL_ENTRY();
    extern __shared__ double2 sh[];   // row [n2] then roots [n2 / 2]
    const int64_t n = 1LL << logn;
    const int n2 = (int)(n / FFT_N1);
    const int log2n2 = logn - 7;
    double2* row = sh;
    double2* root = sh + n2;
    const int k1 = blockIdx.x;
    const int64_t b = blockIdx.y;
    for (int c = threadIdx.x; c < n2; c += blockDim.x) {
        row[c] = in[b * n + (int64_t)k1 * n2 + c];
        if (c < n2 / 2) {
            double s, co;
            sincospi(2.0 * (double)c / (double)n2, &s, &co);
            root[c] = make_double2(co, sign * s);
        }
    }
    __syncthreads();
    fft_smem(row, root, n2, log2n2);
    for (int k2 = threadIdx.x; k2 < n2; k2 += blockDim.x) out[b * n + k1 + (int64_t)FFT_N1 * k2] = row[k2];
}

__global__ void k_encode_finish(const double2* __restrict__ w, int64_t n_vec, int logn, double scale,
                                int64_t* __restrict__ m) {
    EDL_PDL_ENTRY();
    const int64_t n = 1LL << logn;
    const int64_t b = blockIdx.y;
    for (int64_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        double s, co;
        sincospi(-(double)k / (double)n, &s, &co);
        const double2 x = w[b * n + k];
        const double u = (x.x * co - x.y * s) / (double)n;
        m[b * n + k] = __double2ll_rn(scale * u);
    }
}

// decode: residues [n_vec][nl][N] (coefficient domain) -> centered int64 -> twisted complex
__global__ void k_decode_prep(const uint64_t* __restrict__ r, int64_t n_vec, int nl, const uint64_t* __restrict__ q,
                              const uint64_t* __restrict__ qhat_inv, const uint64_t* __restrict__ qhat64,
                              uint64_t Q64, int logn, double2* __restrict__ v) {
    EDL_PDL_ENTRY();
    const int64_t n = 1LL << logn;
    const int64_t b = blockIdx.y;
    for (int64_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        int64_t mk;
        if (nl == 1) {
            const uint64_t x = r[b * n + k];
            mk = x > q[0] / 2 ? (int64_t)x - (int64_t)q[0] : (int64_t)x;
        } else {
            // m = sum_i y_i Qhat_i - round(sum_i y_i / q_i) Q  (mod 2^64, exact for |m| < 2^63)
            uint64_t acc = 0;
            double frac = 0.0;
            for (int i = 0; i < nl; i++) {
                const uint64_t x = r[(b * nl + i) * n + k];
                const uint64_t y = (uint64_t)(((unsigned __int128)x * qhat_inv[i]) % q[i]);
                acc += y * qhat64[i];
                frac += (double)y / (double)q[i];
            }
            acc -= (uint64_t)llrint(frac) * Q64;
            mk = (int64_t)acc;
        }
        double s, co;
        sincospi((double)k / (double)n, &s, &co);
        v[b * n + k] = make_double2((double)mk * co, (double)mk * s);
    }
}

__global__ void k_decode_finish(const double2* __restrict__ v, int64_t n_vec, int64_t n_slots, int logn, double scale,
                                double* __restrict__ z) {
    EDL_PDL_ENTRY();
    const int64_t n = 1LL << logn;
    const int64_t b = blockIdx.y;
    for (int64_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n_slots; j += gridDim.x * blockDim.x) {
        const uint32_t e = pow5((uint32_t)j, (uint32_t)(2 * n));
        z[b * n_slots + j] = v[b * n + (e - 1) / 2].x / scale;
    }
}

void launch_dft(const Dev& d, double2* buf, double2* tmp, int64_t n_vec, int sign) {
    const int64_t n = 1LL << d.logn;
    const int n2 = (int)(n / FFT_N1);
    EDL_LAUNCH(d, "k_fft_cols", k_fft_cols<<<dim3(n2, (unsigned)n_vec), FFT_N1, 0, d.st>>>(buf, tmp, d.logn, sign));
    EDL_LAUNCH(d, "k_fft_rows", k_fft_rows<<<dim3(FFT_N1, (unsigned)n_vec), 128, (n2 + n2 / 2) * sizeof(double2), d.st>>>(
                                    tmp, buf, d.logn, sign));
}

}  // namespace

size_t fft_scratch_bytes(int64_t n_vec, int logn) { return (size_t)2 * n_vec * ((size_t)16 << logn); }

void launch_encode_slots(const Dev& d, const double* z, int64_t n_vec, int64_t n_slots, double scale, int64_t* m,
                         void* scratch) {
    const int64_t n = 1LL << d.logn;
    double2* v = reinterpret_cast<double2*>(scratch);
    double2* tmp = v + n_vec * n;
    const dim3 g((unsigned)((n / 2 + 255) / 256), (unsigned)n_vec);
    EDL_LAUNCH(d, "k_encode_prep", k_encode_prep<<<g, 256, 0, d.st>>>(z, n_vec, n_slots, d.logn, v));
    launch_dft(d, v, tmp, n_vec, -1);
    EDL_LAUNCH(d, "k_encode_finish", k_encode_finish<<<dim3((unsigned)((n + 255) / 256), (unsigned)n_vec), 256, 0, d.st>>>(
                                         v, n_vec, d.logn, scale, m));
}

void launch_decode_slots(const Dev& d, const uint64_t* r, int64_t n_vec, int nl, const uint64_t* q,
                         const uint64_t* qhat_inv, const uint64_t* qhat64, uint64_t Q64, int64_t n_slots, double scale,
                         double* z, void* scratch) {
    const int64_t n = 1LL << d.logn;
    double2* v = reinterpret_cast<double2*>(scratch);
    double2* tmp = v + n_vec * n;
    EDL_LAUNCH(d, "k_decode_prep", k_decode_prep<<<dim3((unsigned)((n + 255) / 256), (unsigned)n_vec), 256, 0, d.st>>>(
                                       r, n_vec, nl, q, qhat_inv, qhat64, Q64, d.logn, v));
    launch_dft(d, v, tmp, n_vec, +1);
    EDL_LAUNCH(d, "k_decode_finish",
               k_decode_finish<<<dim3((unsigned)((n_slots + 255) / 256 + 1), (unsigned)n_vec), 256, 0, d.st>>>(
                   v, n_vec, n_slots, d.logn, scale, z));
}

}  // namespace edl
