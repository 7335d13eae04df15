// api.cu -- the C-ABI (include/edl.h): argument validation, CKKS level/scale
// bookkeeping (meta-object rules), layer schedules and kernel
// orchestration on the context's stream.  No arithmetic on ciphertexts happens here:
// every residue is produced by the sm_100a kernels in *.cu.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>   // header-only; ranges are emitted only with EDL_NVTX=1

#include <cfenv>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <unordered_map>
#include <string>
#include <vector>

#include "../../include/edl.h"
#include "host_math.h"
#include "kernels.cuh"

using namespace edl;

struct edl_ctx {
    edl_params prm;
    int logn = 0;
    int64_t N = 0;
    int L = 0;              // top data level
    int device = 0;
    cudaStream_t st = nullptr;
    cudaStream_t st2 = nullptr;              // side stream for independent branches of a schedule
    cudaEvent_t fork = nullptr, join = nullptr;
    // host wire path (edl_wire_upload / edl_cts_unpack*_host): two device staging buffers
    // filled on the context's own copy stream
    cudaStream_t cst = nullptr;
    void* wire[2] = {nullptr, nullptr};
    size_t wire_cap[2] = {0, 0};
    size_t wire_len[2] = {0, 0};
    cudaEvent_t wire_copied[2] = {nullptr, nullptr}, wire_used[2] = {nullptr, nullptr};
    bool wire_busy[2] = {false, false};   // an unpack has been queued on the slot since its last upload
    std::vector<ModInfo> h_mods;
    ModInfo* d_mods = nullptr;
    ModTable h_mt;
    ChainConsts* h_cc = nullptr;
    ChainConsts* d_cc = nullptr;
    uint64_t* d_tw = nullptr;
    uint64_t* d_s = nullptr;
    uint64_t* d_pk = nullptr;
    uint64_t* d_rlk = nullptr;
    uint64_t* d_rlk_s = nullptr;
    uint64_t* d_rlk_pf = nullptr;     // rlk with P^-1 folded into the data limbs (+ companions)
    uint64_t* d_rlk_pf_c = nullptr;
    std::map<uint32_t, std::pair<uint64_t*, uint64_t*>> gkeys;   // Galois element -> (key, companions)
    bool has_key = false;
    uint64_t key_id = 0;       // host::key_identifier(seed): public, one-way in the seed
    uint64_t sk_seed = 0;      // secret: the key seed (secret-key encryption's error PRF)
    uint64_t* d_scratch = nullptr;
    size_t scratch_words = 0;
    uint8_t* h_pin = nullptr;       // mapped pinned staging ring (host view)
    uint8_t* h_pin_dev = nullptr;   // ... and its device view
    uint8_t* d_const = nullptr;     // device cache of constant tables (bump-allocated)
    size_t const_cap = 0, const_off = 0;     // staging ring
    size_t cache_cap = 0, cache_off = 0;     // device cache
    struct CacheEnt {
        size_t off;
        std::vector<uint8_t> bytes;
    };
    std::unordered_multimap<uint64_t, CacheEnt> cache;   // content hash -> device copy
    std::string err;
    mutable Prof prof;
    // Key-switch variant (N = 2^14): the fused target-major kernel k_relin_ks (modulus raise
    // and key products in one pass, accumulators in shared memory) or the two-kernel
    // k_relin_modup + k_relin_mac (default: measured faster on B200).
    // EDL_KS_FUSED=1 in the environment at context creation selects the fused kernel.
    bool ks_fused = false;
    // Key switches of many ciphertexts in chunks of ks_chunk (EDL_KS_CHUNK, 0 = two halves)
    // alternating over the two streams, so each chunk's raised digits stay in L2.
    int64_t ks_chunk = 0;
    // d2 INTT + modulus raise in one kernel (EDL_RAISE_FUSED=1, N = 2^14)
    bool raise_fused = false;
    // EDL_NVTX=1: an NVTX range around every layer-level C-ABI call (ncu --nvtx filters, timelines)
    bool nvtx = false;
    // EDL_KS_SPLIT=0: key switches as one launch sequence on the main stream instead of two
    // halves on the two streams (experiments with several contexts in flight)
    bool ks_split = true;

    Dev dev() const {
        Dev d;
        d.mods = d_mods;
        d.mt = &h_mt;
        d.hmods = h_mods.data();
        d.cc = d_cc;
        d.logn = logn;
        d.L = L;
        d.st = st;
        d.prof = &prof;
        d.ks_fused = ks_fused;
        d.raise_fused = raise_fused;
        d.rlk = d_rlk;
        d.rlk_pf = ks_fused ? nullptr : d_rlk_pf;   // the fused kernel applies P^-1 itself
        d.rlk_pf_c = d_rlk_pf_c;
        return d;
    }
    uint64_t modulus(int idx) const { return idx <= L ? prm.q[idx] : prm.p_special; }
};

namespace edl {
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("EDL_PDL");   // default on; EDL_PDL=0 turns it off
        return e == nullptr || e[0] != '0';
    }();
    return on;
}
void ensure_smem_attr(const void* kern, int bytes) {   // raise (never lower) a kernel's dynamic smem limit
    static std::vector<std::pair<const void*, int>> done;
    for (auto& e : done)
        if (e.first == kern) {
            if (bytes > e.second) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
                e.second = bytes;
            }
            return;
        }
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    done.emplace_back(kern, bytes);
}

cudaEvent_t Prof::ev() {
    if (used == pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        pool.push_back(e);
    }
    return pool[used++];
}
void Prof::begin(const char* name, cudaStream_t st) {
    launches++;
    last = name;
    if (!on) return;
    Rec r;
    r.name = name;
    r.a = ev();
    r.b = ev();
    cudaEventRecord(r.a, st);
    recs.push_back(r);
}
void Prof::end(cudaStream_t st) {
    if (sync_check) {
        const cudaError_t e = cudaStreamSynchronize(st);
        const cudaError_t l = cudaGetLastError();
        if (e != cudaSuccess || l != cudaSuccess)
            std::fprintf(stderr, "edl: kernel %s failed: %s\n", last ? last : "?",
                         cudaGetErrorString(e != cudaSuccess ? e : l));
    }
    if (!on || recs.empty()) return;
    cudaEventRecord(recs.back().b, st);
}
void Prof::reset() {
    recs.clear();
    used = 0;
}
Prof::~Prof() {
    for (auto e : pool) cudaEventDestroy(e);
}
}  // namespace edl

namespace {

edl_status fail(edl_ctx* c, edl_status code, const char* msg) {
    if (c) c->err = msg;
    return code;
}

edl_status cuda_check(edl_ctx* c, const char* where) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        if (c) c->err = std::string(where) + ": " + cudaGetErrorString(e);
        return EDL_ERR_CUDA;
    }
    return EDL_OK;
}

// Grow-only scratch; growing synchronises the stream so in-flight kernels finish first.
uint64_t* scratch(edl_ctx* c, size_t words) {
    if (words > c->scratch_words) {
        cudaStreamSynchronize(c->st);
        if (c->d_scratch) cudaFree(c->d_scratch);
        size_t w = words + words / 4;
        if (cudaMalloc(&c->d_scratch, w * 8) != cudaSuccess) {
            c->d_scratch = nullptr;
            c->scratch_words = 0;
            return nullptr;
        }
        c->scratch_words = w;
    }
    return c->d_scratch;
}

// Small constant tables (encoded weights): staged through a mapped pinned ring and pulled
// into the device ring by a copy kernel on the stream (zero-copy PCIe reads by the SMs),
// not by the DMA engine: a large host->device transfer the caller overlaps with compute
// (the next batch's ciphertexts) would otherwise hold the constants -- and the whole
// stream behind them -- in the engine's queue.  Wrapping synchronises the stream, so a
// slot is never overwritten while an earlier copy or kernel may still read it.
// Tables are cached on the device by content (a served model's encoded weights repeat
// every batch): a hit costs a host hash + compare and no transfer at all.  A full cache
// is dropped after synchronising the stream (queued kernels may still read it).
template <class T>
const T* upload(edl_ctx* c, const std::vector<T>& v) {
    static_assert(sizeof(T) % 8 == 0, "constant tables are 64-bit words");
    const size_t raw = v.size() * sizeof(T);
    const size_t bytes = (raw + 255) & ~size_t(255);
    if (bytes > c->const_cap || bytes > c->cache_cap) return nullptr;
    const uint8_t* src = reinterpret_cast<const uint8_t*>(v.data());
    uint64_t h = 1469598103934665603ull ^ raw;
    for (size_t k = 0; k < raw / 8; k++) {
        uint64_t w;
        std::memcpy(&w, src + 8 * k, 8);
        h = (h ^ w) * 1099511628211ull;
        h ^= h >> 29;
    }
    auto range = c->cache.equal_range(h);
    for (auto it = range.first; it != range.second; ++it)
        if (it->second.bytes.size() == raw && std::memcmp(it->second.bytes.data(), src, raw) == 0)
            return reinterpret_cast<const T*>(c->d_const + it->second.off);
    if (c->cache_off + bytes > c->cache_cap) {
        cudaStreamSynchronize(c->st);
        c->cache.clear();
        c->cache_off = 0;
    }
    if (c->const_off + bytes > c->const_cap) {
        cudaStreamSynchronize(c->st);
        c->const_off = 0;
    }
    std::memcpy(c->h_pin + c->const_off, src, raw);
    uint8_t* d = c->d_const + c->cache_off;
    launch_fetch_mapped(c->dev(), reinterpret_cast<const uint64_t*>(c->h_pin_dev + c->const_off),
                        reinterpret_cast<uint64_t*>(d), (int64_t)(raw / 8));
    c->const_off += bytes;
    c->cache.emplace(h, edl_ctx::CacheEnt{c->cache_off, std::vector<uint8_t>(src, src + raw)});
    c->cache_off += bytes;
    return reinterpret_cast<const T*>(d);
}

// Key switch of a ciphertext batch split in two halves on the context's two streams: the
// five-kernel pipeline of one half (ALU-bound transforms) overlaps the other's memory-bound
// key-product pass and both halves' wave tails.  The halves use disjoint slices of every
// per-ciphertext array (inputs, scratch, output), so they are independent; the main stream
// joins the side stream before returning.  Profiling keeps one stream.
void relin_split(edl_ctx* c, const Dev& d, const uint64_t* a, const uint64_t* b, int64_t cnt, int l, bool rescale,
                 const uint64_t* rlk, const uint64_t* rlk_s, uint64_t* scr, uint64_t* out,
                 const uint64_t* add_w = nullptr, const uint64_t* add_k = nullptr) {
    const int64_t c0 = cnt / 2;
    if (c->prof.on || c0 < 8 || !c->ks_split) {
        launch_relin(d, a, b, cnt, l, rescale, rlk, rlk_s, scr, out, add_w, add_k);
        return;
    }
    const int nlo = rescale ? l : l + 1;
    const size_t in_w = (size_t)2 * (l + 1) << c->logn, out_w = (size_t)2 * (rescale ? l : l + 1) << c->logn;
    Dev d2 = d;
    d2.st = c->st2;
    if (c->ks_chunk > 0 && cnt > 2 * c->ks_chunk) {
        // L2-sized chunks alternating over the two streams: a chunk's raised digits
        // (chunk x (l+1)(l+2) limbs) stay in L2 between the modulus raise and the key products
        const int64_t ch = c->ks_chunk;
        cudaEventRecord(c->fork, c->st);
        cudaStreamWaitEvent(c->st2, c->fork, 0);
        const size_t sw = relin_scratch_words(ch, l, c->logn);
        int k = 0;
        for (int64_t s0 = 0; s0 < cnt; s0 += ch, k++) {
            const int64_t n = (cnt - s0) < ch ? (cnt - s0) : ch;
            const Dev& dd = (k & 1) ? d2 : d;
            launch_relin(dd, a + s0 * in_w, b ? b + s0 * in_w : nullptr, n, l, rescale, rlk, rlk_s, scr + (k & 1) * sw,
                         out + s0 * out_w, add_w ? add_w + s0 * out_w : nullptr, add_k ? add_k + s0 * nlo : nullptr);
        }
        cudaEventRecord(c->join, c->st2);
        cudaStreamWaitEvent(c->st, c->join, 0);
        return;
    }
    // (measured: starting the second half only after the first half's d2 INTT, to pair
    // transforms with the key-product pass, is slower than the halves side by side)
    cudaEventRecord(c->fork, c->st);
    cudaStreamWaitEvent(c->st2, c->fork, 0);
    launch_relin(d, a, b, c0, l, rescale, rlk, rlk_s, scr, out, add_w, add_k);
    launch_relin(d2, a + c0 * in_w, b ? b + c0 * in_w : nullptr, cnt - c0, l, rescale, rlk, rlk_s,
                 scr + relin_scratch_words(c0, l, c->logn), out + c0 * out_w, add_w ? add_w + c0 * out_w : nullptr,
                 add_k ? add_k + c0 * nlo : nullptr);
    cudaEventRecord(c->join, c->st2);
    cudaStreamWaitEvent(c->st, c->join, 0);
}

// NVTX range over one C-ABI call (host side: the kernels it launches fall inside it on a timeline
// and under `ncu --nvtx --nvtx-include <name>/`); a no-op unless the context was created with
// EDL_NVTX=1.
struct NvtxRange {
    bool on;
    NvtxRange(const edl_ctx* c, const char* name) : on(c && c->nvtx) {
        if (on) nvtxRangePushA(name);
    }
    ~NvtxRange() {
        if (on) nvtxRangePop();
    }
};

bool scales_match(double a, double b) { return std::fabs(a - b) <= std::ldexp(1.0, -30) * std::fmax(a, b); }

// O10: a constant encodes to rint(value * scale) (one IEEE multiply, round-half-even).
int64_t const_int(double value, double scale) { return (int64_t)std::nearbyint(value * scale); }

uint64_t signed_mod(int64_t v, uint64_t q) {
    __int128 r = (__int128)v % (__int128)q;
    if (r < 0) r += q;
    return (uint64_t)r;
}

size_t ct_words(const edl_ctx* c, int64_t cnt, int l) { return (size_t)cnt * 2 * (l + 1) * (size_t)c->N; }

edl_status check_ct(edl_ctx* c, const edl_cts* a) {
    if (!a || (!a->data && a->count > 0)) return fail(c, EDL_ERR_ARG, "null ciphertext array");
    if (a->count < 0) return fail(c, EDL_ERR_ARG, "negative count");
    if (a->level < 0 || a->level > c->L) return fail(c, EDL_ERR_ARG, "level out of range");
    if (c->has_key && a->key_id != c->key_id) return fail(c, EDL_ERR_KEY, "KeyMismatch: ciphertext key differs");
    return EDL_OK;
}

void set_meta(edl_cts* out, int64_t count, int level, double scale, uint64_t key) {
    out->count = count;
    out->level = level;
    out->scale = scale;
    out->key_id = key;
}

// Scalar constants (per ciphertext) -> Shoup pairs [cnt][l+1]
std::vector<ulonglong2> shoup_consts(const edl_ctx* c, const std::vector<int64_t>& ints, int l) {
    std::vector<ulonglong2> w(ints.size() * (l + 1));
    for (size_t k = 0; k < ints.size(); k++)
        for (int i = 0; i <= l; i++) {
            const uint64_t q = c->prm.q[i];
            const uint64_t r = signed_mod(ints[k], q);
            w[k * (l + 1) + i] = make_ulonglong2(r, host::mul_companion(r, q));
        }
    return w;
}

// Constants with their mulc() companions -> [count][nl] {residue, companion}
std::vector<ulonglong2> residue_pairs(const edl_ctx* c, const std::vector<int64_t>& ints, int nl) {
    std::vector<ulonglong2> r(ints.size() * nl);
    for (size_t k = 0; k < ints.size(); k++)
        for (int i = 0; i < nl; i++) {
            const uint64_t v = signed_mod(ints[k], c->prm.q[i]);
            r[k * nl + i] = make_ulonglong2(v, host::mul_companion(v, c->prm.q[i]));
        }
    return r;
}

std::vector<uint64_t> residues(const edl_ctx* c, const std::vector<int64_t>& ints, int nl) {
    std::vector<uint64_t> r(ints.size() * nl);
    for (size_t k = 0; k < ints.size(); k++)
        for (int i = 0; i < nl; i++) r[k * nl + i] = signed_mod(ints[k], c->prm.q[i]);
    return r;
}

}  // namespace

extern "C" {

edl_status edl_params_from_bits(int32_t log_n, const int32_t* bits, int32_t n_bits, int32_t scale_bits,
                                edl_params* out) {
    if (!out || !bits || n_bits < 2 || n_bits > EDL_MAX_PRIMES + 1 || log_n < 1 || log_n > 17) return EDL_ERR_ARG;
    std::memset(out, 0, sizeof(*out));
    out->log_n = log_n;
    out->n_bits = n_bits;
    out->n_data = n_bits - 1;
    out->scale_bits = scale_bits;
    std::vector<int> b(bits, bits + n_bits);
    std::vector<uint64_t> primes(n_bits);
    if (!host::select_primes(b.data(), n_bits, log_n, primes.data())) return EDL_ERR_ARG;
    for (int k = 0; k < n_bits; k++) out->bits[k] = bits[k];
    for (int k = 0; k < n_bits - 1; k++) out->q[k] = primes[k];
    out->p_special = primes[n_bits - 1];
    for (int k = 0; k < n_bits; k++) out->psi[k] = host::minimal_psi(primes[k], log_n);
    return EDL_OK;
}

edl_status edl_params_from_depth(int32_t depth, int32_t scale_bits, double special_mult, edl_params* out) {
    if (depth < 0 || depth + 2 > EDL_MAX_PRIMES + 1 || !out) return EDL_ERR_ARG;
    std::vector<int> bits;
    int logn = 0;
    host::parameterise(depth, scale_bits, special_mult, bits, logn);
    return edl_params_from_bits(logn, bits.data(), (int32_t)bits.size(), scale_bits, out);
}

size_t edl_cts_bytes(int64_t count, int32_t level, int32_t log_n) {
    return (size_t)count * 2 * (size_t)(level + 1) * ((size_t)1 << log_n) * 8;
}

edl_status edl_ctx_create(const edl_params* p, int32_t device, void* stream, edl_ctx** out) {
    if (!p || !out) return EDL_ERR_ARG;
    *out = nullptr;
    if (p->log_n < 10 || p->log_n > 16 || p->n_data < 1 || p->n_data > EDL_MAX_PRIMES) return EDL_ERR_ARG;
    if (!(((EDL_LOGNS_MASK) >> p->log_n) & 1)) return EDL_ERR_ARG;   // ring degree not compiled into this build
    // every modulus < 2^60: the MAC kernels fold up to 256 full 128-bit products (256 q^2 < 2^128)
    for (int k = 0; k < p->n_data; k++)
        if (p->q[k] >= (1ull << 60)) return EDL_ERR_ARG;
    if (p->p_special >= (1ull << 60)) return EDL_ERR_ARG;
    if (cudaSetDevice(device) != cudaSuccess) return EDL_ERR_CUDA;
    edl_ctx* c = new edl_ctx();
    c->prm = *p;
    c->logn = p->log_n;
    c->N = 1LL << p->log_n;
    c->L = p->n_data - 1;
    c->device = device;
    c->st = (cudaStream_t)stream;
    {
        const char* e = std::getenv("EDL_KS_FUSED");
        c->ks_fused = e && e[0] == '1';
        const char* rf = std::getenv("EDL_RAISE_FUSED");
        c->raise_fused = rf && rf[0] == '1';
        const char* k = std::getenv("EDL_KS_CHUNK");
        c->ks_chunk = k ? std::atoll(k) : 0;
        const char* nv = std::getenv("EDL_NVTX");
        c->nvtx = nv && nv[0] == '1';
        const char* sp = std::getenv("EDL_KS_SPLIT");
        c->ks_split = !(sp && sp[0] == '0');
    }
    const int nm = c->L + 2;
    // twiddle tables: per modulus [fwd N][inv N] of {w, w'}
    const size_t tw_words = (size_t)nm * 4 * c->N;
    if (cudaMalloc(&c->d_tw, tw_words * 8) != cudaSuccess) {
        delete c;
        return EDL_ERR_CUDA;
    }
    c->h_mods.resize(nm);
    std::vector<uint64_t> tf, ti;
    for (int k = 0; k < nm; k++) {
        const uint64_t q = c->modulus(k);
        const uint64_t psi = p->psi[k];
        host::twiddle_table(q, psi, c->logn, false, tf);
        host::twiddle_table(q, psi, c->logn, true, ti);
        uint64_t* dfwd = c->d_tw + (size_t)k * 4 * c->N;
        uint64_t* dinv = dfwd + 2 * c->N;
        if (host::f64_ntt_prime(q)) {   // FP64-pipe butterflies: compact [N] binary64 w (f64_mult, no companion)
            std::vector<uint64_t> cf(c->N), ci(c->N);
            for (int64_t j = 0; j < c->N; j++) {
                cf[j] = tf[2 * j];
                ci[j] = ti[2 * j];
            }
            cudaMemcpy(dfwd, cf.data(), cf.size() * 8, cudaMemcpyHostToDevice);
            cudaMemcpy(dinv, ci.data(), ci.size() * 8, cudaMemcpyHostToDevice);
        } else {
            cudaMemcpy(dfwd, tf.data(), tf.size() * 8, cudaMemcpyHostToDevice);
            cudaMemcpy(dinv, ti.data(), ti.size() * 8, cudaMemcpyHostToDevice);
        }
        ModInfo m;
        std::memset(&m, 0, sizeof(m));
        m.q = q;
        const host::u128 ratio = (~(host::u128)0) / q;   // floor((2^128-1)/q) = floor(2^128/q), q odd
        m.r_lo = (uint64_t)ratio;
        m.r_hi = (uint64_t)(ratio >> 64);
        m.two64 = (uint64_t)((((host::u128)1) << 64) % q);
        m.two64_s = host::shoup_companion(m.two64, q);
        m.one_s = host::shoup_companion(1, q);   // floor(2^64 / q)
        m.fp = host::fp_quotient_prime(q) ? (host::f64_ntt_prime(q) ? 2 : 1) : 0;
        m.tw_fwd = reinterpret_cast<const ulonglong2*>(dfwd);
        m.tw_inv = reinterpret_cast<const ulonglong2*>(dinv);
        m.ninv = host::invmod((uint64_t)c->N % q, q);
        m.ninv_s = host::mul_companion(m.ninv, q);
        uint64_t w1 = ti[2 * 1];   // psi^-brv(1): table word (binary64 bits on the F64 path)
        if (m.fp == 2) {
            double wd;
            std::memcpy(&wd, &w1, 8);
            w1 = (uint64_t)wd;
        }
        m.w1ninv = host::mulmod(w1, m.ninv, q);
        m.w1ninv_s = host::mul_companion(m.w1ninv, q);
        m.qinv_d = 1.0 / (double)q;
        {
            const int old = std::fegetround();
            std::fesetround(FE_DOWNWARD);
            volatile double one = 1.0, qd = (double)q;
            volatile double r = one / qd;
            std::fesetround(old);
            m.qinv_rd = r;
        }
        c->h_mods[k] = m;
    }
    c->h_cc = new ChainConsts();
    std::memset(c->h_cc, 0, sizeof(ChainConsts));
    c->h_cc->L = c->L;
    for (int a = 0; a < nm; a++)
        for (int b = 0; b < nm; b++) {
            const uint64_t qa = c->modulus(a), qb = c->modulus(b);
            c->h_cc->qmod[a][b] = qa % qb;
            if (a != b) {
                const uint64_t inv = host::invmod(qa % qb, qb);
                c->h_cc->qinv[a][b] = make_ulonglong2(inv, host::mul_companion(inv, qb));
            }
        }
    cudaMalloc(&c->d_mods, nm * sizeof(ModInfo));
    cudaMemcpy(c->d_mods, c->h_mods.data(), nm * sizeof(ModInfo), cudaMemcpyHostToDevice);
    std::memset(&c->h_mt, 0, sizeof(c->h_mt));
    for (int k = 0; k < nm && k < MAXM; k++) c->h_mt.m[k] = c->h_mods[k];
    cudaMalloc(&c->d_cc, sizeof(ChainConsts));
    cudaMemcpy(c->d_cc, c->h_cc, sizeof(ChainConsts), cudaMemcpyHostToDevice);
    c->const_cap = 16u << 20;
    c->cache_cap = 64u << 20;
    if (cudaHostAlloc(&c->h_pin, c->const_cap, cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->h_pin_dev), c->h_pin, 0) != cudaSuccess) {
        edl_ctx_destroy(c);
        return EDL_ERR_CUDA;
    }
    cudaMalloc(&c->d_const, c->cache_cap);
    if (cudaStreamCreateWithFlags(&c->st2, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming) != cudaSuccess) {
        edl_ctx_destroy(c);
        return EDL_ERR_CUDA;
    }
    if (!set_smem_attrs(c->logn)) {
        edl_ctx_destroy(c);
        return EDL_ERR_CUDA;
    }
    if (cuda_check(c, "ctx_create") != EDL_OK) {
        edl_ctx_destroy(c);
        return EDL_ERR_CUDA;
    }
    *out = c;
    return EDL_OK;
}

void edl_ctx_destroy(edl_ctx* c) {
    if (!c) return;
    cudaStreamSynchronize(c->st);
    cudaFree(c->d_tw);
    cudaFree(c->d_mods);
    cudaFree(c->d_cc);
    cudaFree(c->d_s);
    cudaFree(c->d_pk);
    cudaFree(c->d_rlk);
    cudaFree(c->d_rlk_s);
    cudaFree(c->d_rlk_pf);
    cudaFree(c->d_rlk_pf_c);
    for (auto& kv : c->gkeys) {
        cudaFree(kv.second.first);
        cudaFree(kv.second.second);
    }
    cudaFree(c->d_scratch);
    cudaFree(c->d_const);
    for (int k = 0; k < 2; k++) {
        cudaFree(c->wire[k]);
        if (c->wire_copied[k]) cudaEventDestroy(c->wire_copied[k]);
        if (c->wire_used[k]) cudaEventDestroy(c->wire_used[k]);
    }
    if (c->cst) cudaStreamDestroy(c->cst);
    if (c->st2) cudaStreamDestroy(c->st2);
    if (c->fork) cudaEventDestroy(c->fork);
    if (c->join) cudaEventDestroy(c->join);
    if (c->h_pin) cudaFreeHost(c->h_pin);
    delete c->h_cc;
    delete c;
}

edl_status edl_ctx_set_stream(edl_ctx* c, void* stream) {
    if (!c) return EDL_ERR_ARG;
    cudaStreamSynchronize(c->st);
    c->st = (cudaStream_t)stream;
    return EDL_OK;
}

const char* edl_last_error(const edl_ctx* c) { return c ? c->err.c_str() : "null context"; }
int64_t edl_launch_count(const edl_ctx* c) { return c ? c->prof.launches : 0; }
uint64_t edl_key_id(const edl_ctx* c) { return (c && c->has_key) ? c->key_id : 0; }

edl_status edl_profile(edl_ctx* c, int32_t enable) {
    if (!c) return EDL_ERR_ARG;
    cudaStreamSynchronize(c->st);
    c->prof.reset();
    c->prof.on = enable != 0;
    return EDL_OK;
}

int32_t edl_profile_read(edl_ctx* c, char* names, size_t names_len, double* ms, int64_t* counts, int32_t max_entries) {
    if (!c) return EDL_ERR_ARG;
    if (cudaStreamSynchronize(c->st) != cudaSuccess) return cuda_check(c, "profile_read");
    std::vector<std::string> keys;
    std::vector<double> tot;
    std::vector<int64_t> cnt;
    for (auto& r : c->prof.recs) {
        float t = 0.f;
        cudaEventElapsedTime(&t, r.a, r.b);
        size_t k = 0;
        while (k < keys.size() && keys[k] != r.name) k++;
        if (k == keys.size()) {
            keys.push_back(r.name);
            tot.push_back(0.0);
            cnt.push_back(0);
        }
        tot[k] += t;
        cnt[k] += 1;
    }
    std::string joined;
    int32_t n = 0;
    for (size_t k = 0; k < keys.size() && n < max_entries; k++, n++) {
        if (ms) ms[n] = tot[k];
        if (counts) counts[n] = cnt[k];
        joined += keys[k];
        joined += "\n";
    }
    if (names && names_len) {
        std::strncpy(names, joined.c_str(), names_len - 1);
        names[names_len - 1] = 0;
    }
    return n;
}

edl_status edl_keygen(edl_ctx* c, uint64_t seed) {
    if (!c) return EDL_ERR_ARG;
    const int nm = c->L + 2;
    const size_t N = c->N;
    if (!c->d_s) {
        if (cudaMalloc(&c->d_s, nm * N * 8) != cudaSuccess ||
            cudaMalloc(&c->d_pk, 2 * (size_t)(c->L + 1) * N * 8) != cudaSuccess ||
            cudaMalloc(&c->d_rlk, (size_t)(c->L + 1) * 2 * nm * N * 8) != cudaSuccess ||
            cudaMalloc(&c->d_rlk_s, (size_t)(c->L + 1) * 2 * nm * N * 8) != cudaSuccess ||
            cudaMalloc(&c->d_rlk_pf, (size_t)(c->L + 1) * 2 * nm * N * 8) != cudaSuccess ||
            cudaMalloc(&c->d_rlk_pf_c, (size_t)(c->L + 1) * 2 * nm * N * 8) != cudaSuccess)
            return fail(c, EDL_ERR_CUDA, "keygen: out of device memory");
    }
    // Galois keys belong to the previous secret: drop them (edl_galois_keygen regenerates)
    cudaStreamSynchronize(c->st);
    for (auto& kv : c->gkeys) {
        cudaFree(kv.second.first);
        cudaFree(kv.second.second);
    }
    c->gkeys.clear();
    launch_keygen(c->dev(), seed, c->d_s, c->d_pk, c->d_rlk, c->d_rlk_s, nullptr);
    launch_fold_pinv(c->dev(), c->d_rlk, c->d_rlk_pf, c->d_rlk_pf_c);
    if (cudaStreamSynchronize(c->st) != cudaSuccess) return cuda_check(c, "keygen");
    c->has_key = true;
    c->key_id = host::key_identifier(seed);
    c->sk_seed = seed;
    return cuda_check(c, "keygen");
}

edl_status edl_encode(edl_ctx* c, const double* slots, int64_t n_vec, int64_t n_slots, double scale,
                      int64_t* poly_out) {
    if (!c || (!slots && n_vec > 0) || (!poly_out && n_vec > 0) || n_vec < 0 || n_slots < 0)
        return fail(c, EDL_ERR_ARG, "encode: bad arguments");
    if (n_slots > c->N / 2) return fail(c, EDL_ERR_CAPACITY, "CapacityError: n_slots > N/2");
    for (int64_t v = 0; v < n_vec; v++) host::encode(slots + v * n_slots, n_slots, c->logn, scale, poly_out + v * c->N);
    return EDL_OK;
}

edl_status edl_encrypt_poly(edl_ctx* c, const int64_t* poly, int64_t n_vec, int32_t level, double scale,
                            uint64_t enc_seed, uint32_t obj0, edl_cts* out) {
    NvtxRange nvtx_(c, "edl_encrypt_poly");
    if (!c || !out || (!poly && n_vec > 0) || n_vec < 0) return fail(c, EDL_ERR_ARG, "encrypt: bad arguments");
    if (!c->has_key) return fail(c, EDL_ERR_NOKEY, "encrypt: no key");
    if (level < 0 || level > c->L) return fail(c, EDL_ERR_LEVEL, "encrypt: level out of range");
    if (!out->data && n_vec > 0) return fail(c, EDL_ERR_ARG, "encrypt: null output");
    if (n_vec > 0) {
        launch_encrypt(c->dev(), poly, n_vec, level, enc_seed, obj0, c->d_pk, out->data);
    }
    set_meta(out, n_vec, level, scale, c->key_id);
    return cuda_check(c, "encrypt");
}

edl_status edl_encrypt_poly_sk(edl_ctx* c, const int64_t* poly, int64_t n_vec, int32_t level, double scale,
                               uint64_t enc_seed, uint32_t obj0, edl_cts* out) {
    NvtxRange nvtx_(c, "edl_encrypt_poly_sk");
    if (!c || !out || (!poly && n_vec > 0) || n_vec < 0) return fail(c, EDL_ERR_ARG, "encrypt_sk: bad arguments");
    if (!c->has_key) return fail(c, EDL_ERR_NOKEY, "encrypt_sk: no key");
    if (level < 0 || level > c->L) return fail(c, EDL_ERR_LEVEL, "encrypt_sk: level out of range");
    if (!out->data && n_vec > 0) return fail(c, EDL_ERR_ARG, "encrypt_sk: null output");
    if (n_vec > 0)
        launch_encrypt_sk(c->dev(), poly, n_vec, level, enc_seed, host::sk_error_key(c->sk_seed, enc_seed), obj0, c->d_s,
                          out->data);
    set_meta(out, n_vec, level, scale, c->key_id);
    return cuda_check(c, "encrypt_sk");
}

edl_status edl_encrypt(edl_ctx* c, const double* slots, int64_t n_vec, int64_t n_slots, uint64_t enc_seed,
                       uint32_t obj0, edl_cts* out) {
    if (!c) return EDL_ERR_ARG;
    const double scale = std::ldexp(1.0, c->prm.scale_bits);
    std::vector<int64_t> polys((size_t)n_vec * c->N);
    edl_status s = edl_encode(c, slots, n_vec, n_slots, scale, polys.data());
    if (s != EDL_OK) return s;
    int64_t* d = reinterpret_cast<int64_t*>(scratch(c, polys.size()));
    if (!d && n_vec > 0) return fail(c, EDL_ERR_CUDA, "encrypt: scratch");
    cudaMemcpyAsync(d, polys.data(), polys.size() * 8, cudaMemcpyHostToDevice, c->st);
    s = edl_encrypt_poly(c, d, n_vec, c->L, scale, enc_seed, obj0, out);
    cudaStreamSynchronize(c->st);
    return s;
}

edl_status edl_decrypt_poly(edl_ctx* c, const edl_cts* in, int64_t* poly_out) {
    if (!c || !poly_out) return EDL_ERR_ARG;
    if (!c->has_key) return fail(c, EDL_ERR_NOKEY, "decrypt: no key");
    edl_status s = check_ct(c, in);
    if (s != EDL_OK) return s;
    const int l = in->level;
    const size_t words = (size_t)in->count * (l + 1) * c->N;
    uint64_t* d = scratch(c, words);
    if (!d && words) return fail(c, EDL_ERR_CUDA, "decrypt: scratch");
    std::vector<uint64_t> h(words);
    if (in->count > 0) {
        launch_decrypt(c->dev(), in->data, in->count, l, c->d_s, d);
        cudaMemcpyAsync(h.data(), d, words * 8, cudaMemcpyDeviceToHost, c->st);
    }
    if (cudaStreamSynchronize(c->st) != cudaSuccess) return cuda_check(c, "decrypt");
    for (int64_t k = 0; k < in->count; k++)
        host::crt_lift(h.data() + (size_t)k * (l + 1) * c->N, l + 1, c->prm.q, c->logn, poly_out + k * c->N);
    return cuda_check(c, "decrypt");
}

edl_status edl_decrypt(edl_ctx* c, const edl_cts* in, double* slots_out, int64_t n_slots) {
    if (!c || !in || !slots_out) return EDL_ERR_ARG;
    if (n_slots > c->N / 2) return fail(c, EDL_ERR_CAPACITY, "CapacityError: n_slots > N/2");
    std::vector<int64_t> polys((size_t)in->count * c->N);
    edl_status s = edl_decrypt_poly(c, in, polys.data());
    if (s != EDL_OK) return s;
    for (int64_t k = 0; k < in->count; k++)
        host::decode(polys.data() + k * c->N, c->logn, in->scale, n_slots, slots_out + k * n_slots);
    return EDL_OK;
}

// ---- NEXT f3: client encode / decrypt+decode on the device ----
edl_status edl_encode_device(edl_ctx* c, const double* slots, int64_t n_vec, int64_t n_slots, double scale,
                             int64_t* poly_out) {
    if (!c || n_vec < 0 || n_slots < 0 || (n_vec > 0 && (!slots || !poly_out)))
        return fail(c, EDL_ERR_ARG, "encode_device: bad arguments");
    if (n_slots > c->N / 2) return fail(c, EDL_ERR_CAPACITY, "CapacityError: n_slots > N/2");
    if (c->logn < 8) return fail(c, EDL_ERR_ARG, "encode_device: N >= 256 required");
    if (n_vec == 0) return EDL_OK;
    void* tmp = scratch(c, fft_scratch_bytes(n_vec, c->logn) / 8);
    if (!tmp) return fail(c, EDL_ERR_CUDA, "encode_device: scratch");
    launch_encode_slots(c->dev(), slots, n_vec, n_slots, scale, poly_out, tmp);
    return cuda_check(c, "encode_device");
}

edl_status edl_decrypt_device(edl_ctx* c, const edl_cts* in, double* slots_out, int64_t n_slots) {
    if (!c || !in || (in->count > 0 && !slots_out)) return EDL_ERR_ARG;
    if (!c->has_key) return fail(c, EDL_ERR_NOKEY, "decrypt: no key");
    edl_status s = check_ct(c, in);
    if (s != EDL_OK) return s;
    if (n_slots > c->N / 2) return fail(c, EDL_ERR_CAPACITY, "CapacityError: n_slots > N/2");
    if (c->logn < 8) return fail(c, EDL_ERR_ARG, "decrypt_device: N >= 256 required");
    if (in->count == 0) return EDL_OK;
    const int l = in->level, nl = l + 1;
    // exact-mod-2^64 CRT constants (as host::crt_lift)
    std::vector<uint64_t> tab(3 * nl);
    uint64_t Q64 = 1;
    for (int i = 0; i < nl; i++) Q64 *= c->prm.q[i];
    for (int i = 0; i < nl; i++) {
        uint64_t inv = 1, m64 = 1;
        for (int j = 0; j < nl; j++) {
            if (j == i) continue;
            inv = host::mulmod(inv, c->prm.q[j] % c->prm.q[i], c->prm.q[i]);
            m64 *= c->prm.q[j];
        }
        tab[i] = c->prm.q[i];
        tab[nl + i] = host::invmod(inv, c->prm.q[i]);
        tab[2 * nl + i] = m64;
    }
    const uint64_t* dtab = upload(c, tab);
    if (!dtab) return fail(c, EDL_ERR_CAPACITY, "CapacityError: constant table exceeds the staging ring");
    const size_t words = (size_t)in->count * nl * c->N;
    uint64_t* res = scratch(c, words + fft_scratch_bytes(in->count, c->logn) / 8);
    if (!res) return fail(c, EDL_ERR_CUDA, "decrypt_device: scratch");
    Dev d = c->dev();
    launch_decrypt(d, in->data, in->count, l, c->d_s, res);
    launch_decode_slots(d, res, in->count, nl, dtab, dtab + nl, dtab + 2 * nl, Q64, n_slots, in->scale, slots_out,
                        res + words);
    return cuda_check(c, "decrypt_device");
}

edl_status edl_ct_add(edl_ctx* c, const edl_cts* a, const edl_cts* b, edl_cts* out) {
    if (!c || !out) return EDL_ERR_ARG;
    edl_status s;
    if ((s = check_ct(c, a)) != EDL_OK || (s = check_ct(c, b)) != EDL_OK) return s;
    if (a->key_id != b->key_id) return fail(c, EDL_ERR_KEY, "KeyMismatch");
    if (a->count != b->count) return fail(c, EDL_ERR_SHAPE, "ShapeMismatch: counts differ");
    if (!scales_match(a->scale, b->scale)) return fail(c, EDL_ERR_SCALE, "scale mismatch on add");
    const int lo = a->level < b->level ? a->level : b->level;
    if (a->count > 0) {
        launch_add(c->dev(), a->data, a->level, b->data, b->level, a->count, lo, out->data);
    }
    set_meta(out, a->count, lo, a->scale, a->key_id);
    return cuda_check(c, "ct_add");
}

edl_status edl_ct_pt_mul(edl_ctx* c, const edl_cts* a, const double* w, double pt_scale, edl_cts* out) {
    if (!c || !out || (!w && a && a->count > 0)) return EDL_ERR_ARG;
    edl_status s = check_ct(c, a);
    if (s != EDL_OK) return s;
    std::vector<int64_t> ints(a->count);
    for (int64_t k = 0; k < a->count; k++) ints[k] = const_int(w[k], pt_scale);
    if (a->count > 0) {
        const ulonglong2* dw = upload(c, shoup_consts(c, ints, a->level));
        if (!dw) return fail(c, EDL_ERR_CAPACITY, "CapacityError: constant table exceeds the staging ring");
        launch_mul_const(c->dev(), a->data, a->count, a->level, dw, out->data);
    }
    set_meta(out, a->count, a->level, a->scale * pt_scale, a->key_id);
    return cuda_check(c, "ct_pt_mul");
}

edl_status edl_ct_pt_add(edl_ctx* c, const edl_cts* a, const double* cst, edl_cts* out) {
    if (!c || !out || (!cst && a && a->count > 0)) return EDL_ERR_ARG;
    edl_status s = check_ct(c, a);
    if (s != EDL_OK) return s;
    std::vector<int64_t> ints(a->count);
    for (int64_t k = 0; k < a->count; k++) ints[k] = const_int(cst[k], a->scale);
    if (a->count > 0) {
        const uint64_t* dk = upload(c, residues(c, ints, a->level + 1));
        if (!dk) return fail(c, EDL_ERR_CAPACITY, "CapacityError: constant table exceeds the staging ring");
        launch_add_const(c->dev(), a->data, a->count, a->level, dk, out->data);
    }
    set_meta(out, a->count, a->level, a->scale, a->key_id);
    return cuda_check(c, "ct_pt_add");
}

edl_status edl_mod_drop(edl_ctx* c, const edl_cts* in, int32_t level, edl_cts* out) {
    if (!c || !out) return EDL_ERR_ARG;
    edl_status s = check_ct(c, in);
    if (s != EDL_OK) return s;
    if (level < 0 || level > in->level) return fail(c, EDL_ERR_LEVEL, "mod_drop: cannot raise the level");
    if (!(out->data == in->data && level == in->level) && in->count > 0) {
        if (out->data == in->data) return fail(c, EDL_ERR_ARG, "mod_drop: out aliases in");
        launch_mod_drop(c->dev(), in->data, in->count, in->level, level, out->data);
    }
    set_meta(out, in->count, level, in->scale, in->key_id);
    return cuda_check(c, "mod_drop");
}

edl_status edl_rescale(edl_ctx* c, const edl_cts* in, edl_cts* out) {
    NvtxRange nvtx_(c, "edl_rescale");
    if (!c || !out) return EDL_ERR_ARG;
    edl_status s = check_ct(c, in);
    if (s != EDL_OK) return s;
    const int l = in->level;
    if (l < 1) return fail(c, EDL_ERR_LEVEL, "LevelExhausted: rescale at level 0");
    if (in->count > 0 && out->data == in->data) return fail(c, EDL_ERR_ARG, "rescale: out aliases in");
    if (in->count > 0) {
        uint64_t* r = scratch(c, (size_t)in->count * 2 * c->N);
        if (!r) return fail(c, EDL_ERR_CUDA, "rescale: scratch");
        launch_rescale_intt(c->dev(), in->data, in->count, l, nullptr, r);
        launch_rescale_ntt(c->dev(), in->data, in->count, l, nullptr, r, nullptr, out->data);
    }
    set_meta(out, in->count, l - 1, in->scale / (double)c->prm.q[l], in->key_id);
    return cuda_check(c, "rescale");
}

edl_status edl_ct_ct_mul_relin(edl_ctx* c, const edl_cts* a, const edl_cts* b, edl_cts* out) {
    NvtxRange nvtx_(c, "edl_ct_ct_mul_relin");
    if (!c || !out) return EDL_ERR_ARG;
    if (!c->has_key) return fail(c, EDL_ERR_NOKEY, "mul_relin: no relinearisation key");
    edl_status s;
    if ((s = check_ct(c, a)) != EDL_OK || (s = check_ct(c, b)) != EDL_OK) return s;
    if (a->key_id != b->key_id) return fail(c, EDL_ERR_KEY, "KeyMismatch");
    if (a->count != b->count) return fail(c, EDL_ERR_SHAPE, "ShapeMismatch: counts differ");
    if (a->count > 0 && (out->data == a->data || out->data == b->data))
        return fail(c, EDL_ERR_ARG, "mul_relin: out aliases input");
    const int l = a->level < b->level ? a->level : b->level;
    const int64_t cnt = a->count;
    if (cnt > 0) {
        const size_t drop_a = a->level > l ? ct_words(c, cnt, l) : 0;
        const size_t drop_b = b->level > l ? ct_words(c, cnt, l) : 0;
        uint64_t* base = scratch(c, relin_scratch_words(cnt, l, c->logn) + drop_a + drop_b);
        if (!base) return fail(c, EDL_ERR_CUDA, "mul_relin: scratch");
        const uint64_t* pa = a->data;
        const uint64_t* pb = b->data;
        uint64_t* extra = base + relin_scratch_words(cnt, l, c->logn);
        if (drop_a) {
            launch_mod_drop(c->dev(), a->data, cnt, a->level, l, extra);
            pa = extra;
            extra += drop_a;
        }
        if (drop_b) {
            launch_mod_drop(c->dev(), b->data, cnt, b->level, l, extra);
            pb = extra;
        }
        relin_split(c, c->dev(), pa, pb, cnt, l, false, c->d_rlk, c->d_rlk_s, base, out->data);
    }
    set_meta(out, cnt, l, a->scale * b->scale, a->key_id);
    return cuda_check(c, "mul_relin");
}

edl_status edl_cross_correlate(edl_ctx* c, const edl_cts* x, int32_t H, int32_t W, const double* k, int32_t F,
                               int32_t kh, int32_t kw, int32_t stride, const double* bias, edl_cts* out) {
    NvtxRange nvtx_(c, "edl_cross_correlate");
    if (!c || !out || !k) return EDL_ERR_ARG;
    edl_status s = check_ct(c, x);
    if (s != EDL_OK) return s;
    if (H <= 0 || W <= 0 || F <= 0 || kh <= 0 || kw <= 0 || stride <= 0 || kh > H || kw > W)
        return fail(c, EDL_ERR_SHAPE, "cross_correlate: bad geometry");
    if (x->count != (int64_t)H * W) return fail(c, EDL_ERR_SHAPE, "cross_correlate: x must hold H*W ciphertexts");
    const int l = x->level;
    if (l < 1) return fail(c, EDL_ERR_LEVEL, "LevelExhausted");
    const int Ho = (H - kh) / stride + 1, Wo = (W - kw) / stride + 1;
    const int64_t cnt = (int64_t)F * Ho * Wo;
    const int taps = kh * kw;
    const double pt_scale = (double)c->prm.q[l];
    std::vector<int64_t> wi((size_t)F * taps);
    for (int f = 0; f < F; f++)
        for (int t = 0; t < taps; t++) wi[(size_t)f * taps + t] = const_int(k[(size_t)f * taps + t], pt_scale);
    const double s_after = (x->scale * pt_scale) / (double)c->prm.q[l];
    uint64_t* acc = scratch(c, ct_words(c, cnt, l) + (size_t)cnt * 2 * c->N);
    if (!acc) return fail(c, EDL_ERR_CUDA, "cross_correlate: scratch");
    uint64_t* r = acc + ct_words(c, cnt, l);
    const std::vector<ulonglong2> hw = residue_pairs(c, wi, l + 1);
    const ulonglong2* dw = upload(c, hw);
    if (!dw) return fail(c, EDL_ERR_CAPACITY, "CapacityError: constant table exceeds the staging ring");
    const uint64_t* db = nullptr;
    if (bias) {
        std::vector<int64_t> bi(cnt);
        for (int64_t o = 0; o < cnt; o++) bi[o] = const_int(bias[o / (Ho * Wo)], s_after);
        db = upload(c, residues(c, bi, l));
        if (!db) return fail(c, EDL_ERR_CAPACITY, "CapacityError: constant table exceeds the staging ring");
    }
    Dev d = c->dev();
    launch_cc_mac(d, x->data, l, H, W, F, kh, kw, stride, dw, acc, hw.data());
    launch_rescale_intt(d, acc, cnt, l, nullptr, r);
    launch_rescale_ntt(d, acc, cnt, l, nullptr, r, db, out->data);
    set_meta(out, cnt, l - 1, s_after, x->key_id);
    return cuda_check(c, "cross_correlate");
}

edl_status edl_dense(edl_ctx* c, const edl_cts* x, const double* Wt, const double* b, int32_t O,
                     int32_t defer_rescale, edl_cts* out) {
    NvtxRange nvtx_(c, "edl_dense");
    if (!c || !out || !Wt || O <= 0) return EDL_ERR_ARG;
    edl_status s = check_ct(c, x);
    if (s != EDL_OK) return s;
    const int l = x->level;
    const int64_t K = x->count;
    if (K <= 0) return fail(c, EDL_ERR_SHAPE, "dense: no inputs");
    if (!defer_rescale && l < 1) return fail(c, EDL_ERR_LEVEL, "LevelExhausted");
    if (l < 0) return fail(c, EDL_ERR_LEVEL, "dense: bad level");
    const double pt_scale = (double)c->prm.q[l];
    std::vector<int64_t> wi((size_t)O * K);
    for (size_t t = 0; t < wi.size(); t++) wi[t] = const_int(Wt[t], pt_scale);
    const ulonglong2* dw = upload(c, residue_pairs(c, wi, l + 1));
    if (!dw) return fail(c, EDL_ERR_CAPACITY, "CapacityError: dense weight table exceeds the staging ring");
    Dev d = c->dev();
    const size_t part_words = (size_t)dense_split(d, K, O, l) * ct_words(c, O, l);
    if (defer_rescale) {
        uint64_t* part = scratch(c, part_words);
        if (!part) return fail(c, EDL_ERR_CUDA, "dense: scratch");
        launch_dense_mac(d, x->data, K, O, l, dw, out->data, part);
        set_meta(out, O, l, x->scale * pt_scale, x->key_id);
        return cuda_check(c, "dense");
    }
    const double s_after = (x->scale * pt_scale) / (double)c->prm.q[l];
    uint64_t* acc = scratch(c, ct_words(c, O, l) + (size_t)O * 2 * c->N + part_words);
    if (!acc) return fail(c, EDL_ERR_CUDA, "dense: scratch");
    uint64_t* r = acc + ct_words(c, O, l);
    uint64_t* part = r + (size_t)O * 2 * c->N;
    const uint64_t* db = nullptr;
    if (b) {
        std::vector<int64_t> bi(O);
        for (int o = 0; o < O; o++) bi[o] = const_int(b[o], s_after);
        db = upload(c, residues(c, bi, l));
        if (!db) return fail(c, EDL_ERR_CAPACITY, "CapacityError: constant table exceeds the staging ring");
    }
    launch_dense_mac(d, x->data, K, O, l, dw, acc, part);
    launch_rescale_intt(d, acc, O, l, nullptr, r);
    launch_rescale_ntt(d, acc, O, l, nullptr, r, db, out->data);
    set_meta(out, O, l - 1, s_after, x->key_id);
    return cuda_check(c, "dense");
}

static void limb_bits(const edl_ctx* c, int nl, int* bits) {
    for (int i = 0; i < nl; i++) {
        const uint64_t q = c->prm.q[i];
        int b = 0;
        while (b < 64 && (q >> b) != 0) b++;
        bits[i] = b;
    }
}

size_t edl_cts_packed_bytes(const edl_ctx* c, int64_t count, int32_t level) {
    if (!c || count < 0 || level < 0 || level > c->L) return 0;
    int bits[MAXM];
    limb_bits(c, level + 1, bits);
    size_t words = 0;
    for (int i = 0; i <= level; i++) words += ((size_t)bits[i] << c->logn) >> 6;
    return (size_t)count * 2 * words * 8;
}

edl_status edl_cts_pack(edl_ctx* c, const edl_cts* in, void* packed) {
    if (!c) return EDL_ERR_ARG;
    edl_status s = check_ct(c, in);
    if (s != EDL_OK) return s;
    if (in->count > 0 && !packed) return fail(c, EDL_ERR_ARG, "cts_pack: null output");
    if (in->count > 0) {
        int bits[MAXM];
        limb_bits(c, in->level + 1, bits);
        launch_pack(c->dev(), in->data, in->count * 2, in->level + 1, bits, reinterpret_cast<uint64_t*>(packed));
    }
    return cuda_check(c, "cts_pack");
}

edl_status edl_cts_unpack(edl_ctx* c, const void* packed, int64_t count, int32_t level, double scale, uint64_t key_id,
                          edl_cts* out) {
    NvtxRange nvtx_(c, "edl_cts_unpack");
    if (!c || !out || count < 0) return EDL_ERR_ARG;
    if (level < 0 || level > c->L) return fail(c, EDL_ERR_ARG, "cts_unpack: level out of range");
    if (count > 0 && (!packed || !out->data)) return fail(c, EDL_ERR_ARG, "cts_unpack: null buffer");
    if (count > 0) {
        int bits[MAXM];
        limb_bits(c, level + 1, bits);
        launch_unpack(c->dev(), reinterpret_cast<const uint64_t*>(packed), count * 2, level + 1, bits, out->data);
    }
    set_meta(out, count, level, scale, key_id);
    return cuda_check(c, "cts_unpack");
}

size_t edl_cts_seeded_bytes(const edl_ctx* c, int64_t count, int32_t level) {
    return edl_cts_packed_bytes(c, count, level) / 2;
}

edl_status edl_cts_pack_c0(edl_ctx* c, const edl_cts* in, void* packed) {
    if (!c) return EDL_ERR_ARG;
    edl_status s = check_ct(c, in);
    if (s != EDL_OK) return s;
    if (in->count > 0 && !packed) return fail(c, EDL_ERR_ARG, "cts_pack_c0: null output");
    if (in->count > 0) {
        int bits[MAXM];
        limb_bits(c, in->level + 1, bits);
        launch_pack(c->dev(), in->data, in->count, in->level + 1, bits, reinterpret_cast<uint64_t*>(packed), 2);
    }
    return cuda_check(c, "cts_pack_c0");
}

edl_status edl_cts_unpack_seeded(edl_ctx* c, const void* packed, int64_t count, int32_t level, double scale,
                                 uint64_t key_id, uint64_t enc_seed, uint32_t obj0, edl_cts* out) {
    NvtxRange nvtx_(c, "edl_cts_unpack_seeded");
    if (!c || !out || count < 0) return EDL_ERR_ARG;
    if (level < 0 || level > c->L) return fail(c, EDL_ERR_ARG, "cts_unpack_seeded: level out of range");
    if (count > 0 && (!packed || !out->data)) return fail(c, EDL_ERR_ARG, "cts_unpack_seeded: null buffer");
    if (count > 0) {
        int bits[MAXM];
        limb_bits(c, level + 1, bits);
        launch_unpack(c->dev(), reinterpret_cast<const uint64_t*>(packed), count, level + 1, bits, out->data, 2);
        launch_expand_sk_a(c->dev(), out->data, count, level, enc_seed, obj0);
    }
    set_meta(out, count, level, scale, key_id);
    return cuda_check(c, "cts_unpack_seeded");
}

// ---- host wire path: ciphertexts arrive in host memory, results return to host memory ----
edl_status edl_wire_upload(edl_ctx* c, int32_t slot, const void* host, size_t bytes) {
    if (!c || slot < 0 || slot > 1) return EDL_ERR_ARG;
    if (bytes > 0 && !host) return fail(c, EDL_ERR_ARG, "wire_upload: null host buffer");
    if (bytes % 8) return fail(c, EDL_ERR_ARG, "wire_upload: size must be a multiple of 8 bytes");
    cudaSetDevice(c->device);
    if (!c->cst && cudaStreamCreateWithFlags(&c->cst, cudaStreamNonBlocking) != cudaSuccess)
        return fail(c, EDL_ERR_CUDA, "wire_upload: copy stream");
    if (!c->wire_copied[slot]) {
        if (cudaEventCreateWithFlags(&c->wire_copied[slot], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->wire_used[slot], cudaEventDisableTiming) != cudaSuccess)
            return fail(c, EDL_ERR_CUDA, "wire_upload: events");
    }
    if (bytes > c->wire_cap[slot]) {   // first use (or a larger batch): the old buffer may still be read
        cudaStreamSynchronize(c->st);
        cudaStreamSynchronize(c->cst);
        cudaFree(c->wire[slot]);
        c->wire[slot] = nullptr;
        c->wire_cap[slot] = 0;
        if (cudaMalloc(&c->wire[slot], bytes) != cudaSuccess) return fail(c, EDL_ERR_CUDA, "wire_upload: device staging buffer");
        c->wire_cap[slot] = bytes;
        c->wire_busy[slot] = false;
    }
    if (c->wire_busy[slot]) cudaStreamWaitEvent(c->cst, c->wire_used[slot], 0);   // the last unpack of this slot
    if (bytes > 0 && cudaMemcpyAsync(c->wire[slot], host, bytes, cudaMemcpyHostToDevice, c->cst) != cudaSuccess)
        return fail(c, EDL_ERR_CUDA, "wire_upload: cudaMemcpyAsync");
    cudaEventRecord(c->wire_copied[slot], c->cst);
    c->wire_len[slot] = bytes;
    c->wire_busy[slot] = false;
    return EDL_OK;
}

static edl_status wire_ready(edl_ctx* c, int32_t slot, size_t need, const char* what) {
    if (slot < 0 || slot > 1) return EDL_ERR_ARG;
    if (!c->wire_copied[slot] || c->wire_len[slot] < need) return fail(c, EDL_ERR_ARG, what);
    cudaStreamWaitEvent(c->st, c->wire_copied[slot], 0);
    return EDL_OK;
}
static void wire_release(edl_ctx* c, int32_t slot) {
    cudaEventRecord(c->wire_used[slot], c->st);
    c->wire_busy[slot] = true;
}

edl_status edl_cts_unpack_host(edl_ctx* c, int32_t slot, int64_t count, int32_t level, double scale, uint64_t key_id,
                               edl_cts* out) {
    if (!c || !out || count < 0) return EDL_ERR_ARG;
    if (level < 0 || level > c->L) return fail(c, EDL_ERR_ARG, "cts_unpack_host: level out of range");
    edl_status s = wire_ready(c, slot, edl_cts_packed_bytes(c, count, level), "cts_unpack_host: slot holds fewer bytes than the array");
    if (s != EDL_OK) return s;
    s = edl_cts_unpack(c, c->wire[slot], count, level, scale, key_id, out);
    wire_release(c, slot);
    return s;
}

edl_status edl_cts_unpack_seeded_host(edl_ctx* c, int32_t slot, int64_t count, int32_t level, double scale,
                                      uint64_t key_id, uint64_t enc_seed, uint32_t obj0, edl_cts* out) {
    if (!c || !out || count < 0) return EDL_ERR_ARG;
    if (level < 0 || level > c->L) return fail(c, EDL_ERR_ARG, "cts_unpack_seeded_host: level out of range");
    edl_status s = wire_ready(c, slot, edl_cts_seeded_bytes(c, count, level),
                              "cts_unpack_seeded_host: slot holds fewer bytes than the array");
    if (s != EDL_OK) return s;
    s = edl_cts_unpack_seeded(c, c->wire[slot], count, level, scale, key_id, enc_seed, obj0, out);
    wire_release(c, slot);
    return s;
}

edl_status edl_cts_download(edl_ctx* c, const edl_cts* x, void* host_out) {
    if (!c) return EDL_ERR_ARG;
    edl_status s = check_ct(c, x);
    if (s != EDL_OK) return s;
    if (x->count > 0 && !host_out) return fail(c, EDL_ERR_ARG, "cts_download: null host buffer");
    if (x->count > 0 && cudaMemcpyAsync(host_out, x->data, edl_cts_bytes(x->count, x->level, c->logn), cudaMemcpyDeviceToHost,
                                        c->st) != cudaSuccess)
        return fail(c, EDL_ERR_CUDA, "cts_download: cudaMemcpyAsync");
    return EDL_OK;
}

edl_status edl_ctx_sync(edl_ctx* c) {
    if (!c) return EDL_ERR_ARG;
    cudaSetDevice(c->device);
    cudaError_t e = cudaStreamSynchronize(c->st);
    if (e == cudaSuccess && c->st2) e = cudaStreamSynchronize(c->st2);
    if (e == cudaSuccess && c->cst) e = cudaStreamSynchronize(c->cst);
    if (e != cudaSuccess) return fail(c, EDL_ERR_CUDA, cudaGetErrorString(e));
    return cuda_check(c, "ctx_sync");
}

// ---- NEXT f1: Galois rotations and plaintext vectors ----
static uint32_t galois_elt(const edl_ctx* c, int32_t steps) {
    const int64_t half = c->N / 2, two_n = 2 * c->N;
    int64_t r = ((int64_t)steps % half + half) % half;
    uint64_t g = 1, b = 5;
    while (r) {
        if (r & 1) g = (g * b) % (uint64_t)two_n;
        b = (b * b) % (uint64_t)two_n;
        r >>= 1;
    }
    return (uint32_t)g;
}

edl_status edl_galois_keygen(edl_ctx* c, uint64_t seed, const int32_t* steps, int32_t n_steps) {
    if (!c || (n_steps > 0 && !steps) || n_steps < 0) return EDL_ERR_ARG;
    if (!c->has_key) return fail(c, EDL_ERR_NOKEY, "galois_keygen: no secret key");
    const size_t words = (size_t)(c->L + 1) * 2 * (c->L + 2) * c->N;
    for (int32_t k = 0; k < n_steps; k++) {
        const uint32_t g = galois_elt(c, steps[k]);
        if (g == 1 || c->gkeys.count(g)) continue;
        uint64_t *gk = nullptr, *gc = nullptr;
        if (cudaMalloc(&gk, words * 8) != cudaSuccess || cudaMalloc(&gc, words * 8) != cudaSuccess) {
            cudaFree(gk);
            return fail(c, EDL_ERR_CUDA, "galois_keygen: out of memory");
        }
        launch_keygen_galois(c->dev(), seed, g, c->d_s, gk, gc);
        c->gkeys[g] = std::make_pair(gk, gc);
    }
    cudaStreamSynchronize(c->st);
    return cuda_check(c, "galois_keygen");
}

edl_status edl_rotate(edl_ctx* c, const edl_cts* in, int32_t steps, edl_cts* out) {
    NvtxRange nvtx_(c, "edl_rotate");
    if (!c || !out) return EDL_ERR_ARG;
    edl_status s = check_ct(c, in);
    if (s != EDL_OK) return s;
    if (in->count > 0 && out->data == in->data) return fail(c, EDL_ERR_ARG, "rotate: out aliases in");
    const int l = in->level;
    const int64_t cnt = in->count;
    const uint32_t g = galois_elt(c, steps);
    if (cnt > 0) {
        if (g == 1) {
            cudaMemcpyAsync(out->data, in->data, ct_words(c, cnt, l) * 8, cudaMemcpyDeviceToDevice, c->st);
        } else {
            auto it = c->gkeys.find(g);
            if (it == c->gkeys.end()) return fail(c, EDL_ERR_NOKEY, "rotate: no Galois key for this rotation");
            uint64_t* tmp = scratch(c, ct_words(c, cnt, l) + relin_scratch_words(cnt, l, c->logn));
            if (!tmp) return fail(c, EDL_ERR_CUDA, "rotate: scratch");
            Dev d = c->dev();
            launch_automorphism(d, in->data, cnt, l, g, tmp);
            launch_relin(d, tmp, nullptr, cnt, l, false, it->second.first, it->second.second, tmp + ct_words(c, cnt, l),
                         out->data);
        }
    }
    set_meta(out, cnt, l, in->scale, in->key_id);
    return cuda_check(c, "rotate");
}

edl_status edl_rotate_hoisted(edl_ctx* c, const edl_cts* in, const int32_t* steps, int32_t n_steps, edl_cts* outs) {
    NvtxRange nvtx_(c, "edl_rotate_hoisted");
    if (!c || n_steps < 0 || (n_steps > 0 && (!steps || !outs))) return EDL_ERR_ARG;
    edl_status s = check_ct(c, in);
    if (s != EDL_OK) return s;
    const int l = in->level;
    const int64_t cnt = in->count;
    for (int k = 0; k < n_steps; k++) {
        if (cnt > 0 && (!outs[k].data || outs[k].data == in->data))
            return fail(c, EDL_ERR_ARG, "rotate_hoisted: null output or output aliases input");
        const uint32_t g = galois_elt(c, steps[k]);
        if (g != 1 && c->gkeys.find(g) == c->gkeys.end())
            return fail(c, EDL_ERR_NOKEY, "rotate_hoisted: no Galois key for a rotation");
    }
    if (cnt > 0 && n_steps > 0) {
        const size_t ctw = ct_words(c, cnt, l), rs = relin_scratch_words(cnt, l, c->logn);
        const size_t xw = (size_t)cnt * (l + 1) * (l + 2) << c->logn;
        uint64_t* base = scratch(c, ctw + rs + xw);
        if (!base) return fail(c, EDL_ERR_CUDA, "rotate_hoisted: scratch");
        uint64_t* ctg = base;
        uint64_t* scr = base + ctw;
        uint64_t* xh_base = scr + rs;
        uint64_t* xh = relin_scratch_xh(scr, cnt, l, c->logn);
        Dev d = c->dev();
        launch_relin_raise(d, in->data, cnt, l, scr);   // c1's digits raised once
        cudaMemcpyAsync(xh_base, xh, xw * 8, cudaMemcpyDeviceToDevice, c->st);
        for (int k = 0; k < n_steps; k++) {
            const uint32_t g = galois_elt(c, steps[k]);
            if (g == 1) {
                cudaMemcpyAsync(outs[k].data, in->data, ctw * 8, cudaMemcpyDeviceToDevice, c->st);
                continue;
            }
            const auto& key = c->gkeys.find(g)->second;
            launch_automorphism_rows(d, xh_base, (int64_t)cnt * (l + 1) * (l + 2), g, xh);   // sigma_g(raised digits)
            launch_automorphism(d, in->data, cnt, l, g, ctg);                                // sigma_g(c0, c1)
            launch_relin_finish(d, ctg, cnt, l, key.first, key.second, scr, outs[k].data);
        }
    }
    for (int k = 0; k < n_steps; k++) set_meta(&outs[k], cnt, l, in->scale, in->key_id);
    return cuda_check(c, "rotate_hoisted");
}

edl_status edl_encode_pt(edl_ctx* c, const double* slots, int64_t n_vec, int64_t n_slots, double scale, int32_t level,
                         uint64_t* pt_out) {
    if (!c || n_vec < 0 || (n_vec > 0 && (!slots || !pt_out))) return fail(c, EDL_ERR_ARG, "encode_pt: bad arguments");
    if (level < 0 || level > c->L) return fail(c, EDL_ERR_LEVEL, "encode_pt: level out of range");
    if (n_vec == 0) return EDL_OK;
    std::vector<int64_t> polys((size_t)n_vec * c->N);
    edl_status s = edl_encode(c, slots, n_vec, n_slots, scale, polys.data());
    if (s != EDL_OK) return s;
    int64_t* dp = reinterpret_cast<int64_t*>(scratch(c, polys.size()));
    if (!dp) return fail(c, EDL_ERR_CUDA, "encode_pt: scratch");
    cudaMemcpyAsync(dp, polys.data(), polys.size() * 8, cudaMemcpyHostToDevice, c->st);
    launch_encode_pt(c->dev(), dp, n_vec, level, pt_out);
    cudaStreamSynchronize(c->st);
    return cuda_check(c, "encode_pt");
}

edl_status edl_encode_pt_poly(edl_ctx* c, const int64_t* poly, int64_t n_vec, int32_t level, uint64_t* pt_out) {
    if (!c || n_vec < 0 || (n_vec > 0 && (!poly || !pt_out))) return fail(c, EDL_ERR_ARG, "encode_pt_poly: bad arguments");
    if (level < 0 || level > c->L) return fail(c, EDL_ERR_LEVEL, "encode_pt_poly: level out of range");
    if (n_vec > 0) launch_encode_pt(c->dev(), poly, n_vec, level, pt_out);
    return cuda_check(c, "encode_pt_poly");
}

edl_status edl_ct_pt_vec_mul(edl_ctx* c, const edl_cts* a, const uint64_t* pt, int64_t pt_count, int32_t pt_level,
                             double pt_scale, edl_cts* out) {
    if (!c || !out) return EDL_ERR_ARG;
    edl_status s = check_ct(c, a);
    if (s != EDL_OK) return s;
    if (a->count > 0 && !pt) return fail(c, EDL_ERR_ARG, "ct_pt_vec_mul: null plaintext");
    if (pt_count != 1 && pt_count != a->count) return fail(c, EDL_ERR_SHAPE, "ct_pt_vec_mul: plaintext count");
    if (pt_level < a->level) return fail(c, EDL_ERR_LEVEL, "ct_pt_vec_mul: plaintext level below ciphertext level");
    if (a->count > 0) launch_mul_pt(c->dev(), a->data, a->count, a->level, pt, pt_count, pt_level, out->data);
    set_meta(out, a->count, a->level, a->scale * pt_scale, a->key_id);
    return cuda_check(c, "ct_pt_vec_mul");
}

edl_status edl_keyswitch_bench(edl_ctx* c, const edl_cts* d, edl_cts* out) {
    if (!c || !out) return EDL_ERR_ARG;
    if (!c->has_key) return fail(c, EDL_ERR_NOKEY, "keyswitch: no relinearisation key");
    edl_status s = check_ct(c, d);
    if (s != EDL_OK) return s;
    if (d->count > 0 && (!out->data || out->data == d->data)) return fail(c, EDL_ERR_ARG, "keyswitch: bad output");
    const int l = d->level;
    if (d->count > 0) {
        uint64_t* base = scratch(c, relin_scratch_words(d->count, l, c->logn));
        if (!base) return fail(c, EDL_ERR_CUDA, "keyswitch: scratch");
        relin_split(c, c->dev(), d->data, nullptr, d->count, l, false, c->d_rlk, c->d_rlk_s, base, out->data);
    }
    set_meta(out, d->count, l, d->scale, d->key_id);
    return cuda_check(c, "keyswitch");
}

edl_status edl_ct_pt_vec_add(edl_ctx* c, const edl_cts* a, const uint64_t* pt, int64_t pt_count, int32_t pt_level,
                             edl_cts* out) {
    if (!c || !out) return EDL_ERR_ARG;
    edl_status s = check_ct(c, a);
    if (s != EDL_OK) return s;
    if (a->count > 0 && (!pt || !out->data)) return fail(c, EDL_ERR_ARG, "ct_pt_vec_add: null buffer");
    if (pt_count != 1 && pt_count != a->count) return fail(c, EDL_ERR_SHAPE, "ct_pt_vec_add: plaintext count");
    if (pt_level < a->level) return fail(c, EDL_ERR_LEVEL, "ct_pt_vec_add: plaintext level below ciphertext level");
    if (a->count > 0) launch_add_pt(c->dev(), a->data, a->count, a->level, pt, pt_count, pt_level, out->data);
    set_meta(out, a->count, a->level, a->scale, a->key_id);
    return cuda_check(c, "ct_pt_vec_add");
}

edl_status edl_ct_pt_mac_multi(edl_ctx* c, const edl_cts* rots, int32_t T, const uint64_t* pts, int32_t F,
                               int32_t pt_level, double pt_scale, edl_cts* out) {
    if (!c || !out || T < 1 || F < 1 || T > 64) return EDL_ERR_ARG;
    edl_status s = check_ct(c, rots);
    if (s != EDL_OK) return s;
    if (rots->count % T) return fail(c, EDL_ERR_SHAPE, "ct_pt_mac_multi: count not a multiple of T");
    if (pt_level < rots->level) return fail(c, EDL_ERR_LEVEL, "ct_pt_mac_multi: plaintext level below ciphertext level");
    const int64_t n = rots->count / T;
    if (n > 0 && (!pts || !out->data)) return fail(c, EDL_ERR_ARG, "ct_pt_mac_multi: null buffer");
    if (n > 0) launch_pt_mac_multi(c->dev(), rots->data, T, n, rots->level, pts, F, pt_level, out->data);
    set_meta(out, n * F, rots->level, rots->scale * pt_scale, rots->key_id);
    return cuda_check(c, "ct_pt_mac_multi");
}

edl_status edl_mod_reduce(edl_ctx* c, edl_cts* x) {
    if (!c) return EDL_ERR_ARG;
    edl_status s = check_ct(c, x);
    if (s != EDL_OK) return s;
    if (x->count > 0) {
        launch_mod_reduce(c->dev(), x->data, x->count, x->level);
    }
    return cuda_check(c, "mod_reduce");
}

edl_status edl_dense_finish(edl_ctx* c, const edl_cts* acc, const double* b, edl_cts* out) {
    NvtxRange nvtx_(c, "edl_dense_finish");
    if (!c || !out) return EDL_ERR_ARG;
    edl_status s = check_ct(c, acc);
    if (s != EDL_OK) return s;
    const int l = acc->level;
    if (l < 1) return fail(c, EDL_ERR_LEVEL, "LevelExhausted");
    const int64_t O = acc->count;
    const double s_after = acc->scale / (double)c->prm.q[l];
    uint64_t* r = scratch(c, (size_t)O * 2 * c->N);
    if (!r) return fail(c, EDL_ERR_CUDA, "dense_finish: scratch");
    const uint64_t* db = nullptr;
    if (b) {
        std::vector<int64_t> bi(O);
        for (int64_t o = 0; o < O; o++) bi[o] = const_int(b[o], s_after);
        db = upload(c, residues(c, bi, l));
        if (!db) return fail(c, EDL_ERR_CAPACITY, "CapacityError: constant table exceeds the staging ring");
    }
    Dev d = c->dev();
    launch_rescale_intt(d, acc->data, O, l, nullptr, r);
    launch_rescale_ntt(d, acc->data, O, l, nullptr, r, db, out->data);
    set_meta(out, O, l - 1, s_after, acc->key_id);
    return cuda_check(c, "dense_finish");
}

edl_status edl_poly_activation(edl_ctx* c, const edl_cts* x, const double* coeffs, int32_t degree, edl_cts* out) {
    NvtxRange nvtx_(c, "edl_poly_activation");
    if (!c || !out || !coeffs) return EDL_ERR_ARG;
    if (!c->has_key) return fail(c, EDL_ERR_NOKEY, "poly_activation: no relinearisation key");
    edl_status s = check_ct(c, x);
    if (s != EDL_OK) return s;
    if (x->count > 0 && out->data == x->data) return fail(c, EDL_ERR_ARG, "poly_activation: out aliases x");
    const int l = x->level;
    const int64_t cnt = x->count;
    Dev d = c->dev();
    if (degree == 2 && coeffs[0] == 0.0 && coeffs[1] == 0.0 && coeffs[2] == 1.0) {
        if (l < 1) return fail(c, EDL_ERR_LEVEL, "LevelExhausted");
        if (cnt > 0) {
            uint64_t* base = scratch(c, relin_scratch_words(cnt, l, c->logn));
            if (!base) return fail(c, EDL_ERR_CUDA, "poly_activation: scratch");
            relin_split(c, d, x->data, x->data, cnt, l, true, c->d_rlk, c->d_rlk_s, base, out->data);
        }
        set_meta(out, cnt, l - 1, (x->scale * x->scale) / (double)c->prm.q[l], x->key_id);
        return cuda_check(c, "poly_activation");
    }
    if (degree == 1) {   // c0 + c1 y: Rescale(y x c1@q_l) + c0 (PAPER.md:292 linear sigmoid)
        if (l < 1) return fail(c, EDL_ERR_LEVEL, "LevelExhausted");
        const double ql = (double)c->prm.q[l];
        const double Su = (x->scale * ql) / ql;
        if (cnt > 0) {
            uint64_t* r = scratch(c, (size_t)cnt * 2 * c->N);
            if (!r) return fail(c, EDL_ERR_CUDA, "poly_activation: scratch");
            std::vector<int64_t> i1(cnt, const_int(coeffs[1], ql)), i0(cnt, const_int(coeffs[0], Su));
            const ulonglong2* w1 = upload(c, shoup_consts(c, i1, l));
            if (!w1) return fail(c, EDL_ERR_CAPACITY, "CapacityError: constant table exceeds the staging ring");
            const uint64_t* k0 = upload(c, residues(c, i0, l));
            if (!k0) return fail(c, EDL_ERR_CAPACITY, "CapacityError: constant table exceeds the staging ring");
            launch_rescale_intt(d, x->data, cnt, l, w1, r);
            launch_rescale_ntt(d, x->data, cnt, l, w1, r, k0, out->data);
        }
        set_meta(out, cnt, l - 1, Su, x->key_id);
        return cuda_check(c, "poly_activation");
    }
    if (degree == 2) {   // c0 + c1 y + c2 y^2 on 2 levels (PAPER.md:416 ReLU_a), oracle order
        if (l < 2) return fail(c, EDL_ERR_LEVEL, "LevelExhausted");
        const double c0 = coeffs[0], c1 = coeffs[1], c2 = coeffs[2];
        const double ql = (double)c->prm.q[l], qlm1 = (double)c->prm.q[l - 1];
        const double Sy = x->scale;
        const double S2 = (Sy * Sy) / ql;                    // y2 = Rescale(Relin(y*y))
        const double Sa = (S2 * qlm1) / qlm1;                // a = Rescale(y2 * c2@q_{l-1})
        const double p1 = (S2 * ql) / Sy;                    // b = drop(Rescale(y * c1@p1))
        const double Sb = (Sy * p1) / ql;
        if (!scales_match(Sa, Sb)) return fail(c, EDL_ERR_SCALE, "poly_activation: scale drift");
        if (cnt > 0) {
            const size_t wl = ct_words(c, cnt, l - 1), wd = ct_words(c, cnt, l - 2);
            const size_t rs = relin_scratch_words(cnt, l, c->logn);
            uint64_t* base = scratch(c, wl + 2 * wd + 2 * (size_t)cnt * 2 * c->N + rs);
            if (!base) return fail(c, EDL_ERR_CUDA, "poly_activation: scratch");
            uint64_t* y2 = base;
            uint64_t* av = y2 + wl;
            uint64_t* bv = av + wd;
            uint64_t* r = bv + wd;
            uint64_t* r2 = r + (size_t)cnt * 2 * c->N;
            uint64_t* rsc = r2 + (size_t)cnt * 2 * c->N;
            std::vector<int64_t> i2(cnt, const_int(c2, qlm1)), i1(cnt, const_int(c1, p1)), i0(cnt, const_int(c0, Sa));
            const ulonglong2* w2 = upload(c, shoup_consts(c, i2, l - 1));
            if (!w2) return fail(c, EDL_ERR_CAPACITY, "CapacityError: constant table exceeds the staging ring");
            const ulonglong2* w1 = upload(c, shoup_consts(c, i1, l));
            if (!w1) return fail(c, EDL_ERR_CAPACITY, "CapacityError: constant table exceeds the staging ring");
            const uint64_t* k0 = upload(c, residues(c, i0, l - 1));   // output level l-2: l-1 limbs
            if (!k0) return fail(c, EDL_ERR_CAPACITY, "CapacityError: constant table exceeds the staging ring");
            relin_split(c, d, x->data, x->data, cnt, l, true, c->d_rlk, c->d_rlk_s, rsc, y2);
            launch_rescale_intt(d, y2, cnt, l - 1, w2, r);
            launch_rescale_ntt(d, y2, cnt, l - 1, w2, r, nullptr, av);
            launch_rescale_intt(d, x->data, cnt, l, w1, r2);
            launch_rescale_ntt(d, x->data, cnt, l, w1, r2, nullptr, bv, l - 2);
            launch_add_add_const(d, av, bv, l - 2, cnt, l - 2, k0, out->data);
        }
        set_meta(out, cnt, l - 2, Sa, x->key_id);
        return cuda_check(c, "poly_activation");
    }
    if (!(degree == 3 && coeffs[2] == 0.0)) return fail(c, EDL_ERR_ARG, "poly_activation: unsupported schedule");
    if (l < 2) return fail(c, EDL_ERR_LEVEL, "LevelExhausted");
    const double c0 = coeffs[0], c1 = coeffs[1], c3 = coeffs[3];
    const double ql = (double)c->prm.q[l], qlm1 = (double)c->prm.q[l - 1];
    // O13 schedule, scale bookkeeping in the oracle's order
    const double Sy = x->scale;
    const double S2 = (Sy * Sy) / ql;                    // y2 = Rescale(Relin(y*y))
    const double Su = (Sy * ql) / ql;                    // u  = Rescale(y * c3@q_l)
    const double S3 = (Su * S2) / qlm1;                  // v  = Rescale(Relin(u*y2))
    const double p1 = (S3 * ql) / Sy;                    // w  = Rescale(y * c1@p1)
    const double Sw = (Sy * p1) / ql;
    if (!scales_match(S3, Sw)) return fail(c, EDL_ERR_SCALE, "poly_activation: scale drift");
    if (cnt > 0) {
        const size_t wl = ct_words(c, cnt, l - 1);
        const size_t rs = relin_scratch_words(cnt, l, c->logn);
        uint64_t* base = scratch(c, 3 * wl + 2 * (size_t)cnt * 2 * c->N + rs);
        if (!base) return fail(c, EDL_ERR_CUDA, "poly_activation: scratch");
        uint64_t* y2 = base;
        uint64_t* u = y2 + wl;
        uint64_t* w = u + wl;
        uint64_t* r = w + wl;
        uint64_t* rsc = r + (size_t)cnt * 2 * c->N;
        std::vector<int64_t> i3(cnt, const_int(c3, ql)), i1(cnt, const_int(c1, p1)), i0(cnt, const_int(c0, S3));
        const ulonglong2* w3 = upload(c, shoup_consts(c, i3, l));
        if (!w3) return fail(c, EDL_ERR_CAPACITY, "CapacityError: constant table exceeds the staging ring");
        const ulonglong2* w1 = upload(c, shoup_consts(c, i1, l));
        if (!w1) return fail(c, EDL_ERR_CAPACITY, "CapacityError: constant table exceeds the staging ring");
        const uint64_t* k0 = upload(c, residues(c, i0, l - 1));
        if (!k0) return fail(c, EDL_ERR_CAPACITY, "CapacityError: constant table exceeds the staging ring");
        uint64_t* r2 = rsc + rs;   // second INTT output
        // 2.+4. (independent of 1.) run on the side stream, overlapping 1.'s tails and its
        // memory-light phases; 3. joins them
        // (per-kernel profiling keeps one stream so every launch's event pair times it alone)
        const bool side = !c->prof.on;
        Dev d2 = d;
        if (side) {
            d2.st = c->st2;
            cudaEventRecord(c->fork, c->st);
            cudaStreamWaitEvent(c->st2, c->fork, 0);
        }
        launch_rescale_intt(d2, x->data, cnt, l, w3, r, w1, r2);                            // 2.+4. INTT shared
        launch_rescale_ntt(d2, x->data, cnt, l, w3, r, nullptr, u);                         // 2.
        launch_rescale_ntt(d2, x->data, cnt, l, w1, r2, nullptr, w, l - 2);                 // 4. (+ mod_drop)
        if (side) cudaEventRecord(c->join, c->st2);
        relin_split(c, d, x->data, x->data, cnt, l, true, c->d_rlk, c->d_rlk_s, rsc, y2);    // 1.
        if (side) cudaStreamWaitEvent(c->st, c->join, 0);
        // 3. + 5.: out = Rs(Relin(u y2)) + w + c0, the assembly fused into the last kernel
        relin_split(c, d, u, y2, cnt, l - 1, true, c->d_rlk, c->d_rlk_s, rsc, out->data, w, k0);
    }
    set_meta(out, cnt, l - 2, S3, x->key_id);
    return cuda_check(c, "poly_activation");
}

edl_status edl_ntt(edl_ctx* c, uint64_t* limbs, int64_t n_polys, int32_t level, int32_t inverse) {
    if (!c || (!limbs && n_polys > 0) || n_polys < 0 || level < 0 || level > c->L + 1)
        return fail(c, EDL_ERR_ARG, "ntt: bad arguments");
    std::vector<int> pm(level + 1);
    for (int j = 0; j <= level; j++) pm[j] = j;
    // grid.y limit: split very large batches
    for (int64_t b0 = 0; b0 < n_polys; b0 += 65535) {
        const int64_t nb = (n_polys - b0) < 65535 ? (n_polys - b0) : 65535;
        launch_ntt_limbs(c->dev(), limbs + (size_t)b0 * (level + 1) * c->N, nb, level + 1, pm.data(), inverse != 0);
    }
    return cuda_check(c, "ntt");
}

edl_status edl_philox(edl_ctx* c, uint64_t seed, const uint32_t* ctr, int64_t n, uint32_t* out) {
    if (!c || !ctr || !out || n <= 0) return EDL_ERR_ARG;
    uint32_t* d = reinterpret_cast<uint32_t*>(scratch(c, (size_t)n * 4));
    if (!d) return fail(c, EDL_ERR_CUDA, "philox: scratch");
    cudaMemcpyAsync(d, ctr, (size_t)n * 16, cudaMemcpyHostToDevice, c->st);
    launch_philox_words(c->dev(), seed, d, n, d);
    cudaMemcpyAsync(out, d, (size_t)n * 16, cudaMemcpyDeviceToHost, c->st);
    cudaStreamSynchronize(c->st);
    return cuda_check(c, "philox");
}

edl_status edl_bfly_peak(edl_ctx* c, int32_t prime_index, int32_t iters, double* bfly_per_s) {
    if (!c || !bfly_per_s || iters <= 0 || prime_index < 0 || prime_index > c->L + 1) return EDL_ERR_ARG;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    const int blocks = sms * 8;
    uint64_t* sink = scratch(c, 1);
    if (!sink) return fail(c, EDL_ERR_CUDA, "bfly_peak: scratch");
    const ModInfo& m = c->h_mods[prime_index];
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch_bfly_peak(c->dev(), m.q, m.fp == 2, m.tw_fwd + 1, iters, blocks, sink);   // warm-up
    cudaEventRecord(a, c->st);
    launch_bfly_peak(c->dev(), m.q, m.fp == 2, m.tw_fwd + 1, iters, blocks, sink);
    cudaEventRecord(b, c->st);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *bfly_per_s = (double)blocks * 256.0 * 8.0 * (double)iters / (ms * 1e-3);
    return cuda_check(c, "bfly_peak");
}

edl_status edl_modmul_peak(edl_ctx* c, int32_t iters, double* modmul_per_s) {
    if (!c || !modmul_per_s || iters <= 0) return EDL_ERR_ARG;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    const int blocks = sms * 8;
    uint64_t* sink = scratch(c, 1);
    if (!sink) return fail(c, EDL_ERR_CUDA, "modmul_peak: scratch");
    const uint64_t q = c->prm.q[c->L];
    const uint64_t w = q / 3 + 7, ws = host::shoup_companion(w, q);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch_modmul_peak(c->dev(), q, w, ws, iters, blocks, sink);   // warm-up
    cudaEventRecord(a, c->st);
    launch_modmul_peak(c->dev(), q, w, ws, iters, blocks, sink);
    cudaEventRecord(b, c->st);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *modmul_per_s = (double)blocks * 256.0 * 8.0 * (double)iters / (ms * 1e-3);
    return cuda_check(c, "modmul_peak");
}

edl_status edl_pipe_peak(edl_ctx* c, int32_t which, int32_t iters, double* ops_per_s) {
    if (!c || !ops_per_s || iters <= 0 || which < 0 || which > 3) return EDL_ERR_ARG;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    const int blocks = sms * 8;
    uint64_t* sink = scratch(c, 1);
    if (!sink) return fail(c, EDL_ERR_CUDA, "pipe_peak: scratch");
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch_pipe_probe(c->dev(), which, iters, blocks, sink);   // warm-up
    cudaEventRecord(a, c->st);
    launch_pipe_probe(c->dev(), which, iters, blocks, sink);
    cudaEventRecord(b, c->st);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *ops_per_s = (double)blocks * 256.0 * 8.0 * (double)iters / (ms * 1e-3);
    return cuda_check(c, "pipe_peak");
}

edl_status edl_export_galois_key(edl_ctx* c, int32_t steps, uint64_t* host_out, size_t words) {
    if (!c || !host_out) return EDL_ERR_ARG;
    auto it = c->gkeys.find(galois_elt(c, steps));
    if (it == c->gkeys.end()) return fail(c, EDL_ERR_NOKEY, "export_galois_key: no key");
    const size_t need = (size_t)(c->L + 1) * 2 * (c->L + 2) * c->N;
    if (words < need) return fail(c, EDL_ERR_ARG, "export_galois_key: buffer too small");
    cudaMemcpy(host_out, it->second.first, need * 8, cudaMemcpyDeviceToHost);
    return cuda_check(c, "export_galois_key");
}

edl_status edl_export_key(edl_ctx* c, int32_t which, uint64_t* host_out, size_t words) {
    if (!c || !host_out) return EDL_ERR_ARG;
    if (!c->has_key) return fail(c, EDL_ERR_NOKEY, "export_key: no key");
    const size_t N = c->N, nm = c->L + 2;
    const uint64_t* src = nullptr;
    size_t need = 0;
    if (which == 0) {
        src = c->d_s;
        need = nm * N;
    } else if (which == 1) {
        src = c->d_pk;
        need = 2 * (size_t)(c->L + 1) * N;
    } else if (which == 2) {
        src = c->d_rlk;
        need = (size_t)(c->L + 1) * 2 * nm * N;
    } else {
        return fail(c, EDL_ERR_ARG, "export_key: which");
    }
    if (words < need) return fail(c, EDL_ERR_ARG, "export_key: buffer too small");
    cudaMemcpyAsync(host_out, src, need * 8, cudaMemcpyDeviceToHost, c->st);
    cudaStreamSynchronize(c->st);
    return cuda_check(c, "export_key");
}

}  // extern "C"
