// ntt_kernels.cu -- host dispatch of the NTT-family kernels (ntt_kernels.cuh) over the
// supported ring degrees; the per-degree launchers are instantiated in ntt_inst_<logN>.cu.
#include "kernels.cuh"

namespace edl {

bool set_smem_attrs(int /*logn*/) { return true; }   // set lazily by launch_cfg

void launch_ntt_limbs(const Dev& d, uint64_t* data, int64_t batch, int nl, const int* prime_idx_host, bool inverse) {
    PrimeMap pm;
    for (int j = 0; j < nl && j < MAXM; j++) pm.idx[j] = (int8_t)prime_idx_host[j];
    EDL_DISPATCH_LOGN(d.logn, launch_ntt_limbs_n<LOGN>(d, data, batch, nl, pm, inverse));
}

void launch_rescale_intt(const Dev& d, const uint64_t* in, int64_t cnt, int l, const ulonglong2* w, uint64_t* r_out,
                         const ulonglong2* w2, uint64_t* r_out2) {
    EDL_DISPATCH_LOGN(d.logn, launch_rescale_intt_n<LOGN>(d, in, cnt, l, w, r_out, w2, r_out2));
}

void launch_rescale_ntt(const Dev& d, const uint64_t* in, int64_t cnt, int l, const ulonglong2* w,
                        const uint64_t* r, const uint64_t* bias, uint64_t* out, int lo) {
    const int nlo = (lo < 0 || lo > l - 1) ? l : lo + 1;
    EDL_DISPATCH_LOGN(d.logn, launch_rescale_ntt_n<LOGN>(d, in, cnt, l, w, r, bias, out, nlo));
}

size_t relin_scratch_words(int64_t cnt, int l, int logn) {
    return (size_t)cnt * (((size_t)(l + 1) + (size_t)(l + 1) * (l + 2) + 2 * (size_t)(l + 2) + 4) << logn);
}

void launch_relin(const Dev& d, const uint64_t* a, const uint64_t* b, int64_t cnt, int l, bool rescale,
                  const uint64_t* rlk, const uint64_t* rlk_s, uint64_t* scratch, uint64_t* out, const uint64_t* add_w,
                  const uint64_t* add_k) {
    uint64_t* acoef = scratch;
    uint64_t* xh = acoef + ((size_t)cnt * (l + 1) << d.logn);
    uint64_t* acc = xh + ((size_t)cnt * (l + 1) * (l + 2) << d.logn);
    uint64_t* r = acc + ((size_t)cnt * 2 * (l + 2) << d.logn);
    uint64_t* s = r + ((size_t)cnt * 2 << d.logn);
    EDL_DISPATCH_LOGN(d.logn, launch_relin_n<LOGN>(d, a, b, cnt, l, rescale, rlk, rlk_s, acoef, xh, acc, r, s, out, add_w, add_k));
}

uint64_t* relin_scratch_xh(uint64_t* scratch, int64_t cnt, int l, int logn) {
    return scratch + ((size_t)cnt * (l + 1) << logn);
}

void launch_relin_raise(const Dev& d, const uint64_t* a, int64_t cnt, int l, uint64_t* scratch) {
    uint64_t* acoef = scratch;
    uint64_t* xh = relin_scratch_xh(scratch, cnt, l, d.logn);
    EDL_DISPATCH_LOGN(d.logn, launch_relin_raise_n<LOGN>(d, a, cnt, l, acoef, xh));
}

void launch_relin_finish(const Dev& d, const uint64_t* a, int64_t cnt, int l, const uint64_t* rlk, const uint64_t* rlk_s,
                         uint64_t* scratch, uint64_t* out) {
    uint64_t* xh = relin_scratch_xh(scratch, cnt, l, d.logn);
    uint64_t* acc = xh + ((size_t)cnt * (l + 1) * (l + 2) << d.logn);
    uint64_t* r = acc + ((size_t)cnt * 2 * (l + 2) << d.logn);
    uint64_t* s = r + ((size_t)cnt * 2 << d.logn);
    EDL_DISPATCH_LOGN(d.logn, launch_relin_finish_n<LOGN>(d, a, cnt, l, rlk, rlk_s, xh, acc, r, s, out));
}

}  // namespace edl
