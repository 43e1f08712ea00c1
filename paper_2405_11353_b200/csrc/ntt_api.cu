// ntt_api.cu -- implementation of include/ntt_b200.h.
//
// Host-side pieces (field validation, twiddle tables, plans) are native C++;
// every transform runs on the B200.  There is no CPU fallback: with no CUDA
// device every exec returns NTT_E_NO_DEVICE.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <cstdlib>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/ntt_b200.h"
#include "launch.cuh"
#include "multipass.cuh"

using namespace nttb200;
typedef unsigned __int128 u128;

namespace {

thread_local std::string g_last_error;
std::atomic<unsigned long long> g_launches{0};
std::atomic<int> g_counters_enabled{0};
std::mutex g_mu;
std::map<int, unsigned long long*> g_dev_counters;   // device -> 4 counters

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* where) {
    return fail(NTT_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------- field --
// modmath.py:23-45 is_prime (deterministic Miller-Rabin for n < 2^64)
uint64_t mulmod(uint64_t a, uint64_t b, uint64_t m) { return (uint64_t)((u128)a * b % m); }
uint64_t powmod(uint64_t b, uint64_t e, uint64_t m) {
    uint64_t r = 1 % m;
    b %= m;
    while (e) {
        if (e & 1) r = mulmod(r, b, m);
        b = mulmod(b, b, m);
        e >>= 1;
    }
    return r;
}

bool is_prime(uint64_t n) {
    if (n < 2) return false;
    static const uint64_t small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    for (uint64_t s : small)
        if (n % s == 0) return n == s;
    uint64_t d = n - 1;
    int r = 0;
    while ((d & 1) == 0) { d >>= 1; ++r; }
    for (uint64_t a : small) {
        uint64_t x = powmod(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (int i = 0; i < r - 1; ++i) {
            x = mulmod(x, x, n);
            if (x == n - 1) { comp = false; break; }
        }
        if (comp) return false;
    }
    return true;
}

// modmath.py:48-60 prime_factors (trial division; stops early once the
// cofactor is prime -- same factor set, bounded time for 64-bit p-1)
std::vector<uint64_t> prime_factors(uint64_t n) {
    std::vector<uint64_t> f;
    for (uint64_t d = 2; d <= n / d; d += (d == 2 ? 1 : 2)) {
        if (n % d == 0) {
            f.push_back(d);
            while (n % d == 0) n /= d;
            if (n > 1 && is_prime(n)) break;
        }
    }
    if (n > 1) f.push_back(n);
    return f;
}

bool is_generator(uint64_t g, uint64_t p, const std::vector<uint64_t>& fac) {
    for (uint64_t q : fac)
        if (powmod(g, (p - 1) / q, p) == 1) return false;
    return true;
}

int check_field(uint64_t p, uint64_t g, int w) {
    if (!is_prime(p)) return fail(NTT_E_NOT_PRIME, std::to_string(p) + " is not prime");
    // modmath.py:95-96: any width with p < 2^w (w > 64 only changes the host
    // table's Shoup words; the device arithmetic has its own word)
    if (w > 4096) return fail(NTT_E_INVALID, "word width w is unreasonably large");
    if (p == 2 || w < 1 || (w < 64 && p >= (1ull << w)))
        return fail(NTT_E_INVALID, "p must be odd and fit in " + std::to_string(w) + " bits");
    if (!(2 <= g && g < p)) return fail(NTT_E_INVALID, "generator out of range");
    if (!is_generator(g, p, prime_factors(p - 1)))
        return fail(NTT_E_INVALID, std::to_string(g) + " is not a primitive root of " + std::to_string(p));
    return NTT_OK;
}

bool pow2(uint64_t n) { return n >= 1 && (n & (n - 1)) == 0; }
int ilog2(uint64_t n) { int l = 0; while ((1ull << l) < n) ++l; return l; }

uint64_t shoup_word(uint64_t tw, uint64_t p, int w) { return (uint64_t)(((u128)tw << w) / p); }

constexpr uint64_t kGold = 0xFFFFFFFF00000001ull;

int field_kind(uint64_t p, int word_bytes) {
    if (word_bytes == 4) return p < (1ull << 31) ? 0 : 1;
    return p == kGold ? 2 : 3;
}

// ---------------------------------------------------------------- tables --
struct DevTable {
    int device = -1;
    void* tw = nullptr;       // F::Tw[N]: w^i (+ Shoup word)
    void* stw = nullptr;      // F::Tw[N]: per-stage table T[2^(s-1)+k] = w^(k*N/2^s)
    uint64_t bytes = 0;
    uint64_t n_inv = 0, n_inv_dev_shoup = 0;
    ~DevTable() {
        if (tw) {
            int cur = 0;
            cudaGetDevice(&cur);
            cudaSetDevice(device);
            cudaFree(tw);
            if (stw) cudaFree(stw);
            cudaSetDevice(cur);
        }
    }
};

using TableKey = std::tuple<uint64_t, uint64_t, uint64_t, int, int, int>;  // p,g,n,dir,word,device
std::map<TableKey, std::weak_ptr<DevTable>> g_tables;

// Host table per twiddle.py:57-88 (repeated multiplication by omega).
void host_powers(uint64_t p, uint64_t omega, uint64_t n, std::vector<uint64_t>& w_pow) {
    w_pow.resize(n);
    w_pow[0] = 1;
    for (uint64_t i = 1; i < n; ++i) w_pow[i] = mulmod(w_pow[i - 1], omega, p);
}

int get_dev_table(uint64_t p, uint64_t g, uint64_t n, int dir, int word, int device,
                  std::shared_ptr<DevTable>& out) {
    TableKey key{p, g, n, dir, word, device};
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_tables.find(key);
    if (it != g_tables.end()) {
        if (auto sp = it->second.lock()) { out = sp; return NTT_OK; }
    }
    uint64_t omega = powmod(g, (p - 1) / n, p);
    if (dir == NTT_INVERSE) omega = powmod(omega, p - 2, p);
    std::vector<uint64_t> w_pow;
    host_powers(p, omega, n, w_pow);
    const int kind = field_kind(p, word);
    auto t = std::make_shared<DevTable>();
    t->device = device;
    std::vector<unsigned char> buf;
    if (kind == 0 || kind == 1) {
        buf.resize(n * 8);
        uint32_t* d = reinterpret_cast<uint32_t*>(buf.data());
        for (uint64_t i = 0; i < n; ++i) { d[2 * i] = (uint32_t)w_pow[i]; d[2 * i + 1] = (uint32_t)shoup_word(w_pow[i], p, 32); }
    } else if (kind == 2) {
        buf.resize(n * 8);
        memcpy(buf.data(), w_pow.data(), n * 8);
    } else {
        buf.resize(n * 16);
        uint64_t* d = reinterpret_cast<uint64_t*>(buf.data());
        for (uint64_t i = 0; i < n; ++i) { d[2 * i] = w_pow[i]; d[2 * i + 1] = shoup_word(w_pow[i], p, 64); }
    }
    if (dir == NTT_INVERSE) {
        t->n_inv = powmod(n % p, p - 2, p);
        t->n_inv_dev_shoup = shoup_word(t->n_inv, p, word == 4 ? 32 : 64);
    }
    // per-stage reordering of the same entries: index i = 2^(s-1) + k holds
    // w^(k * N/2^s), the twiddle of stage s for k < 2^(s-1)
    const size_t esz = buf.size() / n;
    std::vector<unsigned char> sbuf(buf.size());
    memcpy(sbuf.data(), buf.data(), esz);
    for (uint64_t i = 1; i < n; ++i) {
        int s1 = 0;
        while ((2ull << s1) <= i) ++s1;          // s - 1 = floor(log2 i)
        const uint64_t k = i - (1ull << s1);
        const uint64_t e = k * (n >> (s1 + 1));
        memcpy(sbuf.data() + i * esz, buf.data() + e * esz, esz);
    }
    int cur = 0;
    cudaGetDevice(&cur);
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaMalloc(&t->tw, buf.size());
    if (e == cudaSuccess) e = cudaMemcpy(t->tw, buf.data(), buf.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&t->stw, sbuf.size());
    if (e == cudaSuccess) e = cudaMemcpy(t->stw, sbuf.data(), sbuf.size(), cudaMemcpyHostToDevice);
    cudaSetDevice(cur);
    if (e != cudaSuccess) { t->tw = nullptr; t->stw = nullptr; return cuda_fail(e, "twiddle table upload"); }
    t->bytes = 2 * buf.size();
    g_tables[key] = t;
    out = t;
    return NTT_OK;
}

unsigned long long* dev_counters(int device) {
    if (!g_counters_enabled.load()) return nullptr;
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_dev_counters.find(device);
    if (it != g_dev_counters.end()) return it->second;
    unsigned long long* d = nullptr;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    if (cudaMalloc(&d, C_NCOUNTERS * sizeof(unsigned long long)) != cudaSuccess) d = nullptr;
    else cudaMemset(d, 0, C_NCOUNTERS * sizeof(unsigned long long));
    cudaSetDevice(cur);
    g_dev_counters[device] = d;
    return d;
}

}  // namespace

struct ntt_plan_s {
    uint64_t p, g, n, n1, n2;
    int w, variant, dir, word, device, kind, L;
    std::shared_ptr<DevTable> table, table1, table2;   // main, six-step n1 / n2 sub-tables
    // six-step correction twiddles w^e = cor_hi[e >> cor_lb] * cor_lo[e mod 2^cor_lb] (exact)
    void* cor_lo = nullptr;
    void* cor_hi = nullptr;
    int cor_lb = 0;
    // four-step twist hi table (u32 multi-pass): w^(j * 2^twh_bits) + Shoup word
    void* twh = nullptr;
    int twh_bits = 0;
    // four-step twist table (fourstep.cuh): [k1][n2] = w^(k1*n2) + Shoup word
    void* fst = nullptr;
    void* fst_inv = nullptr;      // Goldilocks inverse plans: fst * n^-1
    int num_sms = 148;
    // workspace for multi-pass plans and host-buffer execution
    // multi-pass workspace, one per CUDA stream: a plan is immutable and may run
    // concurrently on several streams (each stream's passes are stream-ordered)
    std::map<cudaStream_t, std::pair<void*, uint64_t>> ws;
    std::map<cudaStream_t, std::pair<void*, uint64_t>> pw_ws;   // unfused pointwise-inverse products
    // two device buffer sets at FIXED offsets set * hset_bytes (a set never
    // moves while a call that uses it may be in flight); last_chunks / last_bytes
    // remember the chunking of the previous call on each set
    void* hbuf = nullptr;
    uint64_t hbuf_bytes = 0;
    uint64_t hset_bytes = 0;
    uint64_t last_chunks[2] = {0, 0};
    uint64_t last_bytes[2] = {0, 0};
    // host-exec pipeline: hs[0] H2D copies, hs[1] transforms, hs[2] D2H copies,
    // chained per chunk by events (kMaxChunks x {copied-in, transformed})
    static constexpr int kMaxChunks = 64;
    cudaStream_t hs[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t hev[2 * kMaxChunks] = {};
    // NTT_FLAG_HOST_ASYNC: two device buffer sets used by alternate calls;
    // hout[set][chunk] = that chunk's copy-out done (the next call on the set
    // waits for it before overwriting), hend orders the caller's stream
    // after the copy-out
    cudaEvent_t hout[2 * kMaxChunks] = {};
    cudaEvent_t hend = nullptr;
    uint64_t host_seq = 0;
    std::mutex mu;        // guards ws / hbuf / stream + event creation
    std::mutex host_mu;   // serialises ntt_exec_host calls (one host pipeline per plan)
    ~ntt_plan_s() {
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(device);
        for (auto& kv : ws)
            if (kv.second.first) cudaFree(kv.second.first);
        for (auto& kv : pw_ws)
            if (kv.second.first) cudaFree(kv.second.first);
        for (auto st : hs)                 // asynchronous host calls may still be in flight
            if (st) cudaStreamSynchronize(st);
        if (hbuf) cudaFree(hbuf);
        for (auto st : hs)
            if (st) cudaStreamDestroy(st);
        for (auto ev : hev)
            if (ev) cudaEventDestroy(ev);
        for (auto ev : hout)
            if (ev) cudaEventDestroy(ev);
        if (hend) cudaEventDestroy(hend);
        if (cor_lo) cudaFree(cor_lo);
        if (cor_hi) cudaFree(cor_hi);
        if (twh) cudaFree(twh);
        if (fst) cudaFree(fst);
        if (fst_inv) cudaFree(fst_inv);
        cudaSetDevice(cur);
    }
};

namespace {

int grow(void*& ptr, uint64_t& have, uint64_t need) {
    if (have >= need) return NTT_OK;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    have = 0;
    cudaError_t e = cudaMalloc(&ptr, need);
    if (e != cudaSuccess) return cuda_fail(e, "workspace allocation");
    have = need;
    return NTT_OK;
}

cudaError_t launch_mp_kind(int kind, const MultipassReq& r) {
    switch (kind) {
        case 0: return mp_launch_f32s(r);
        case 1: return mp_launch_f32w(r);
        case 2: return mp_launch_gold(r);
        default: return mp_launch_f64(r);
    }
}

int smem_max_log2_word(int word) { return single_pass_max_log2(word); }

// Upload count residues omega^(i*step) (device word) for the two-level
// six-step correction table.
int upload_powers(uint64_t p, uint64_t base, uint64_t count, int word, int device, void** out) {
    std::vector<uint64_t> v(count);
    uint64_t x = 1;
    for (uint64_t i = 0; i < count; ++i) { v[i] = x; x = mulmod(x, base, p); }
    std::vector<unsigned char> buf(count * word);
    if (word == 4) { uint32_t* d = reinterpret_cast<uint32_t*>(buf.data()); for (uint64_t i = 0; i < count; ++i) d[i] = (uint32_t)v[i]; }
    else memcpy(buf.data(), v.data(), count * 8);
    int cur = 0;
    cudaGetDevice(&cur);
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaMalloc(out, buf.size());
    if (e == cudaSuccess) e = cudaMemcpy(*out, buf.data(), buf.size(), cudaMemcpyHostToDevice);
    cudaSetDevice(cur);
    if (e != cudaSuccess) { *out = nullptr; return cuda_fail(e, "correction table upload"); }
    return NTT_OK;
}

}  // namespace

extern "C" {

int ntt_abi_version(void) { return NTT_B200_ABI_VERSION; }
const char* ntt_last_error(void) { return g_last_error.c_str(); }

int ntt_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) { cudaGetLastError(); return 0; }
    return n;
}

int ntt_field_check(uint64_t p, uint64_t g, int w_bits) { return check_field(p, g, w_bits); }

int ntt_find_primitive_root(uint64_t p, uint64_t* g_out) {
    if (!is_prime(p)) return fail(NTT_E_NOT_PRIME, std::to_string(p) + " is not prime");
    if (p == 2) { *g_out = 1; return NTT_OK; }
    auto fac = prime_factors(p - 1);
    for (uint64_t g = 2; g < p; ++g)
        if (is_generator(g, p, fac)) { *g_out = g; return NTT_OK; }
    return fail(NTT_E_NOT_PRIME, "no generator found");
}

int ntt_root_of_unity(uint64_t p, uint64_t g, uint64_t n, uint64_t* omega_out) {
    if (!pow2(n)) return fail(NTT_E_NOT_POWER_OF_TWO, "size " + std::to_string(n) + " is not a power of two");
    if ((p - 1) % n) return fail(NTT_E_SIZE_NOT_SUPPORTED, std::to_string(n) + " does not divide p-1 = " + std::to_string(p - 1));
    *omega_out = powmod(g, (p - 1) / n, p);
    return NTT_OK;
}

int ntt_table_build(uint64_t p, uint64_t g, int w_bits, uint64_t n, int direction, uint64_t* w_pow,
                    uint64_t* w_shoup, uint64_t* n_inv, uint64_t* n_inv_shoup) {
    if (direction != NTT_FORWARD && direction != NTT_INVERSE) return fail(NTT_E_INVALID, "unknown direction");
    uint64_t omega = 0;
    int st = ntt_root_of_unity(p, g, n, &omega);
    if (st) return st;
    if (direction == NTT_INVERSE) omega = powmod(omega, p - 2, p);
    std::vector<uint64_t> wp;
    host_powers(p, omega, n, wp);
    memcpy(w_pow, wp.data(), n * 8);
    // (w > 64: the Shoup words do not fit the u64 output; the host computes them)
    for (uint64_t i = 0; i < n; ++i) w_shoup[i] = w_bits <= 64 ? shoup_word(wp[i], p, w_bits) : 0;
    if (direction == NTT_INVERSE) {
        uint64_t ni = powmod(n % p, p - 2, p);
        if (n_inv) *n_inv = ni;
        if (n_inv_shoup) *n_inv_shoup = w_bits <= 64 ? shoup_word(ni, p, w_bits) : 0;
    }
    return NTT_OK;
}

int ntt_plan_create(uint64_t p, uint64_t g, int w_bits, uint64_t n, int variant, int direction, uint64_t n1,
                    uint64_t n2, int word_bytes, int device, ntt_plan_t* plan_out) {
    if (!plan_out) return fail(NTT_E_INVALID, "plan_out is NULL");
    *plan_out = nullptr;
    if (variant < NTT_NAIVE || variant > NTT_SIXSTEP)
        return fail(NTT_E_UNSUPPORTED_VARIANT, "unknown variant id " + std::to_string(variant));
    if (n < 2 || !pow2(n))
        return fail(NTT_E_NOT_POWER_OF_TWO, "transform size " + std::to_string(n) + " is not a power of two >= 2");
    if (direction != NTT_FORWARD && direction != NTT_INVERSE) return fail(NTT_E_INVALID, "unknown direction");
    int st = check_field(p, g, w_bits);
    if (st) return st;
    if ((p - 1) % n)
        return fail(NTT_E_SIZE_NOT_SUPPORTED, std::to_string(n) + " does not divide p-1 = " + std::to_string(p - 1));
    if (word_bytes != 4 && word_bytes != 8) return fail(NTT_E_INVALID, "word_bytes must be 4 or 8");
    if (word_bytes == 4 && p >= (1ull << 32)) return fail(NTT_E_INVALID, "uint32 storage needs p < 2^32");
    const int L = ilog2(n);
    if (variant == NTT_SIXSTEP) {
        if (n1 == 0 && n2 == 0) { n1 = 1ull << ((L + 1) / 2); n2 = n / n1; }
        else if (n1 == 0) n1 = n2 ? n / n2 : 0;
        else if (n2 == 0) n2 = n / n1;
        if (n1 < 1 || n2 < 1 || (u128)n1 * n2 != n || !pow2(n1) || !pow2(n2))
            return fail(NTT_E_BAD_FACTORIZATION, std::to_string(n1) + " * " + std::to_string(n2) + " != " +
                                                     std::to_string(n) + " (powers of two required)");
    } else {
        n1 = n2 = 0;
    }
    int ndev = ntt_device_count();
    if (ndev <= 0) return fail(NTT_E_NO_DEVICE, "no CUDA device visible: the B200 engine has no CPU fallback");
    if (device < 0 || device >= ndev) return fail(NTT_E_INVALID, "device ordinal out of range");
    if (variant == NTT_NAIVE && L > 16) return fail(NTT_E_SIZE_NOT_SUPPORTED, "naive DFT is limited to N <= 2^16");
    std::unique_ptr<ntt_plan_s> pl(new ntt_plan_s());
    pl->p = p; pl->g = g; pl->n = n; pl->n1 = n1; pl->n2 = n2; pl->w = w_bits; pl->variant = variant;
    pl->dir = direction; pl->word = word_bytes; pl->device = device; pl->kind = field_kind(p, word_bytes);
    pl->L = L;
    if (variant == NTT_SIXSTEP) {
        // the six-step kernels only read the n1 / n2 sub-tables and the
        // two-level correction tables; no size-N table on the device
        pl->table = std::make_shared<DevTable>();
        pl->table->device = device;
        if (direction == NTT_INVERSE) {
            pl->table->n_inv = powmod(n % p, p - 2, p);
            pl->table->n_inv_dev_shoup = shoup_word(pl->table->n_inv, p, word_bytes == 4 ? 32 : 64);
        }
    } else {
        st = get_dev_table(p, g, n, direction, word_bytes, device, pl->table);
        if (st) return st;
    }
    if (variant == NTT_SIXSTEP) {
        // sub-transforms beyond one shared-memory pass run the general six-step (launch.cuh)
        if (n1 > 1 && (st = get_dev_table(p, g, n1, direction, word_bytes, device, pl->table1))) return st;
        if (n2 > 1 && (st = get_dev_table(p, g, n2, direction, word_bytes, device, pl->table2))) return st;
        uint64_t omega = powmod(g, (p - 1) / n, p);
        if (direction == NTT_INVERSE) omega = powmod(omega, p - 2, p);
        pl->cor_lb = (L + 1) / 2;
        if ((st = upload_powers(p, omega, 1ull << pl->cor_lb, word_bytes, device, &pl->cor_lo))) return st;
        if ((st = upload_powers(p, powmod(omega, 1ull << pl->cor_lb, p), 1ull << (L - pl->cor_lb), word_bytes,
                                device, &pl->cor_hi))) return st;
    }
    if (word_bytes == 4 && variant != NTT_NAIVE && variant != NTT_SIXSTEP && L > smem_max_log2_word(4) && L <= 20) {
        // twist hi table for the four-step factorisation of the late pass
        const int th = (L + 1) / 2;
        uint64_t omega = powmod(g, (p - 1) / n, p);
        if (direction == NTT_INVERSE) omega = powmod(omega, p - 2, p);
        const uint64_t step = powmod(omega, 1ull << th, p);
        const uint64_t cnt = 1ull << (L - th);
        std::vector<uint32_t> buf(2 * cnt);
        uint64_t x = 1;
        for (uint64_t j = 0; j < cnt; ++j) {
            buf[2 * j] = (uint32_t)x;
            buf[2 * j + 1] = (uint32_t)shoup_word(x, p, 32);
            x = mulmod(x, step, p);
        }
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(device);
        cudaError_t e = cudaMalloc(&pl->twh, buf.size() * 4);
        if (e == cudaSuccess) e = cudaMemcpy(pl->twh, buf.data(), buf.size() * 4, cudaMemcpyHostToDevice);
        cudaSetDevice(cur);
        if (e != cudaSuccess) { pl->twh = nullptr; return cuda_fail(e, "twist table upload"); }
        pl->twh_bits = th;
    }
    if (fourstep_applies(L, variant, p, word_bytes)) {
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(device);
        cudaError_t e = cudaMalloc(&pl->fst, n * 8);
        if (e == cudaSuccess) e = fourstep_twist_build(pl->table->tw, pl->fst, L, word_bytes, 0);
        if (e == cudaSuccess && pl->kind == 2 && direction == NTT_INVERSE) {      // intt: n^-1 folded into the twist
            e = cudaMalloc(&pl->fst_inv, n * 8);
            if (e == cudaSuccess) e = fourstep_twist_build(pl->table->tw, pl->fst_inv, L, word_bytes, 0);
            if (e == cudaSuccess) e = fourstep_twist_scale_gold(pl->fst_inv, n, pl->table->n_inv, 0);
        }
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        cudaSetDevice(cur);
        if (e != cudaSuccess) { if (pl->fst) cudaFree(pl->fst); pl->fst = nullptr; return cuda_fail(e, "four-step twist table"); }
    }
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) == cudaSuccess && sms > 0)
        pl->num_sms = sms;
    *plan_out = pl.release();
    return NTT_OK;
}

int ntt_plan_destroy(ntt_plan_t plan) {
    delete plan;
    return NTT_OK;
}

int ntt_plan_info(ntt_plan_t plan, ntt_plan_info_t* info) {
    if (!plan || !info) return fail(NTT_E_INVALID, "NULL argument");
    memset(info, 0, sizeof(*info));
    info->p = plan->p; info->g = plan->g; info->n = plan->n; info->n1 = plan->n1; info->n2 = plan->n2;
    info->w_bits = plan->w; info->variant = plan->variant; info->direction = plan->dir;
    info->word_bytes = plan->word; info->device = plan->device; info->field_kind = plan->kind;
    if (plan->variant == NTT_SIXSTEP) info->passes = 2;
    else info->passes = mp_num_passes(plan->L, plan->word, plan->variant, plan->p);
    info->n_inv = plan->table->n_inv;
    info->n_inv_shoup = plan->dir == NTT_INVERSE && plan->w <= 64 ? shoup_word(plan->table->n_inv, plan->p, plan->w) : 0;
    info->device_table_bytes = plan->table->bytes + (plan->table1 ? plan->table1->bytes : 0) +
                               (plan->table2 ? plan->table2->bytes : 0);
    return NTT_OK;
}

uint64_t ntt_plan_workspace_bytes(ntt_plan_t plan, uint64_t batch) {
    if (!plan) return 0;
    if (plan->variant == NTT_SIXSTEP) {
        const bool general = plan->n1 > (1ull << smem_max_log2_word(plan->word)) ||
                             plan->n2 > (1ull << smem_max_log2_word(plan->word));
        return (general ? 4 : 2) * batch * plan->n * plan->word;   // step ping-pong (tiles.cuh) / general path
    }
    return mp_workspace_bytes(plan->L, plan->word, plan->variant, batch, plan->p);
}

static int exec_device(ntt_plan_t plan, const void* d_in, void* d_out, uint64_t batch, unsigned flags,
                       cudaStream_t stream) {
    const bool scale = (flags & NTT_FLAG_SCALE) != 0;
    const bool independent = (flags & NTT_FLAG_INDEPENDENT) != 0;
    if (scale && plan->dir != NTT_INVERSE) return fail(NTT_E_INVALID, "intt requires an inverse-direction table");
    if (batch == 0) return NTT_OK;
    if (!d_in || !d_out) return fail(NTT_E_INVALID, "NULL buffer");
    unsigned long long* ctr = dev_counters(plan->device);
    uint64_t need = ntt_plan_workspace_bytes(plan, batch);
    // the O(N^2) naive DFT reads every input while writing: in place it first
    // copies the input aside (the reference is pure, algorithms.py:52-79)
    const bool naive_inplace = plan->variant == NTT_NAIVE && d_in == d_out;
    if (naive_inplace) need = batch * plan->n * plan->word;
    void* ws = nullptr;
    if (need) {
        std::lock_guard<std::mutex> lk(plan->mu);
        auto& slot = plan->ws[stream];
        int st = grow(slot.first, slot.second, need);
        if (st) return st;
        ws = slot.first;
    }
    if (naive_inplace) {
        cudaError_t ce = cudaMemcpyAsync(ws, d_in, need, cudaMemcpyDeviceToDevice, stream);
        if (ce != cudaSuccess) return cuda_fail(ce, "naive in-place copy");
        d_in = ws;
    }
    int launches = 0;
    MultipassReq r{};
    r.variant = plan->variant; r.L = plan->L; r.in = d_in; r.out = d_out; r.batch = batch;
    r.tw = plan->table->tw; r.stw = plan->table->stw; r.p = plan->p; r.scale = scale;
    r.ninv = plan->table->n_inv; r.ninv_shoup = plan->table->n_inv_dev_shoup;
    r.counters = ctr; r.stream = stream; r.num_sms = plan->num_sms; r.launches = &launches;
    r.ws = ws;
    r.independent = independent ? 1 : 0;
    // launch window (planner.cu): single-pass launches register themselves in the fast
    // kernel's launcher; every other launch on the stream ends the run of deferred waits
    if (plan->variant == NTT_SIXSTEP || plan->variant == NTT_NAIVE ||
        mp_num_passes(plan->L, plan->word, plan->variant, plan->p) != 1)
        window_break(stream);
    r.twh = plan->twh;
    r.twh_bits = plan->twh_bits;
    r.fst = plan->fst;
    r.fst_scaled = plan->fst_inv;
    if (plan->variant == NTT_SIXSTEP) {
        r.n1 = plan->n1; r.n2 = plan->n2;
        r.tw1 = plan->table1 ? plan->table1->tw : nullptr;
        r.tw2 = plan->table2 ? plan->table2->tw : nullptr;
        r.stw1 = plan->table1 ? plan->table1->stw : nullptr;
        r.stw2 = plan->table2 ? plan->table2->stw : nullptr;
        r.cor_lo = plan->cor_lo; r.cor_hi = plan->cor_hi; r.cor_lb = plan->cor_lb;
    }
    cudaError_t e = launch_mp_kind(plan->kind, r);
    g_launches += launches;
    if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
    return NTT_OK;
}

int ntt_exec(ntt_plan_t plan, const void* d_in, void* d_out, uint64_t batch, unsigned flags, void* stream) {
    if (!plan) return fail(NTT_E_INVALID, "NULL plan");
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != plan->device) cudaSetDevice(plan->device);
    int st = exec_device(plan, d_in, d_out, batch, flags, static_cast<cudaStream_t>(stream));
    if (cur != plan->device) cudaSetDevice(cur);
    return st;
}

int ntt_exec_host(ntt_plan_t plan, const void* h_in, void* h_out, uint64_t batch, unsigned flags, void* stream) {
    if (!plan) return fail(NTT_E_INVALID, "NULL plan");
    if (batch == 0) return NTT_OK;
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != plan->device) cudaSetDevice(plan->device);
    const uint64_t row_bytes = plan->n * plan->word;
    const uint64_t bytes = batch * row_bytes;
    int st = NTT_OK;
    const bool async = (flags & NTT_FLAG_HOST_ASYNC) != 0;
    flags &= ~NTT_FLAG_HOST_ASYNC;
    std::lock_guard<std::mutex> host_lk(plan->host_mu);
    const int set = async ? (int)(plan->host_seq++ & 1) : 0;
    {
        std::lock_guard<std::mutex> lk(plan->mu);
        if (bytes > plan->hset_bytes) {    // reallocation: earlier asynchronous calls must be done with it
            for (auto hs : plan->hs)
                if (hs) cudaStreamSynchronize(hs);
            st = grow(plan->hbuf, plan->hbuf_bytes, 2 * bytes);
            plan->hset_bytes = st ? 0 : bytes;
            plan->last_chunks[0] = plan->last_chunks[1] = 0;
        }
        for (auto& hs : plan->hs)
            if (!st && !hs && cudaStreamCreateWithFlags(&hs, cudaStreamNonBlocking) != cudaSuccess)
                st = fail(NTT_E_CUDA, "stream creation failed");
        for (auto& ev : plan->hev)
            if (!st && !ev && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess)
                st = fail(NTT_E_CUDA, "event creation failed");
        for (auto& ev : plan->hout)
            if (!st && !ev && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess)
                st = fail(NTT_E_CUDA, "event creation failed");
        if (!st && !plan->hend && cudaEventCreateWithFlags(&plan->hend, cudaEventDisableTiming) != cudaSuccess)
            st = fail(NTT_E_CUDA, "event creation failed");
    }
    cudaError_t e = cudaSuccess;
    // Shared-memory-resident plans need no workspace, so the batch is cut into
    // chunks: all H2D copies run back to back on one stream, all D2H copies on
    // another, and the transform of chunk c waits only for its own copy-in
    // (events) -- both copy engines stay busy (PCIe is full duplex: 55 GB/s
    // each way alone, 97 GB/s aggregate concurrently; tools/pcie_bw.py).
    // (A zero-copy variant -- the kernel reading and writing the pinned host
    // buffers through UVA -- is bit-exact but measured slower: 1.81 vs 1.69 ms
    // for config 2, tools/pcie_pipe.py.)
    // Multi-pass plans chunk the same way: every chunk's transform runs on the
    // one compute stream, so they take turns on that stream's workspace.
    // (The six-step's single giant row is one chunk.)
    const bool resident = plan->variant != NTT_SIXSTEP && plan->variant != NTT_NAIVE;
    uint64_t chunks = 1;
    // 8 chunks measured best for 64 MiB each way (host-buffer path): every
    // pinned copy costs ~20 us on the copy engines, so more chunks lose more
    // than the shorter pipeline fill/drain gains
    if (resident && bytes >= (16ull << 20)) chunks = bytes >= (64ull << 20) ? 8 : 4;
    // asynchronous calls overlap one call's copy-out with the next call's
    // copy-in, so the within-call pipeline only needs to cover the transform:
    // 2 chunks (config 2: 1.43 ms/step at 1-2 chunks, 1.55 at 8; the PCIe
    // floor with both directions busy is 1.35 ms, tools/e2e_async.py)
    if (async && resident && bytes >= (16ull << 20)) chunks = 2;
    if (chunks > (uint64_t)ntt_plan_s::kMaxChunks) chunks = ntt_plan_s::kMaxChunks;
    if (chunks > batch) chunks = batch;
    char* d = static_cast<char*>(plan->hbuf) + (size_t)set * plan->hset_bytes;
    cudaStream_t sH = plan->hs[0], sC = plan->hs[1], sD = plan->hs[2];
    cudaStream_t user = static_cast<cudaStream_t>(stream);
    cudaEvent_t* hout = plan->hout + set * ntt_plan_s::kMaxChunks;
    // chunk c of this call overwrites exactly chunk c of the previous call on
    // this set only if both calls cut the same bytes into the same chunks;
    // otherwise the first copy-in waits for EVERY copy-out of that call
    const bool same_cut = plan->last_chunks[set] == chunks && plan->last_bytes[set] == bytes;
    if (!st && !same_cut)
        for (uint64_t c = 0; c < plan->last_chunks[set]; ++c)
            if ((e = cudaStreamWaitEvent(sH, hout[c], 0)) != cudaSuccess) { st = cuda_fail(e, "stream wait"); break; }
    plan->last_chunks[set] = chunks;
    plan->last_bytes[set] = bytes;
    // (no wait on `stream` at the start: it carries the previous asynchronous
    // call's completion, and waiting for it would serialise the calls -- h_in
    // must be ready on the host when the call is made)
    auto span = [&](uint64_t c, uint64_t& r0, uint64_t& off, uint64_t& nb) {
        r0 = batch * c / chunks;
        const uint64_t r1 = batch * (c + 1) / chunks;
        off = r0 * row_bytes;
        nb = (r1 - r0) * row_bytes;
        return r1 - r0;
    };
    // enqueue order: every copy-in first (the H2D engine starts at once and
    // never waits on the host), then the transforms, then every copy-out
    uint64_t r0, off, nb;
    for (uint64_t c = 0; !st && c < chunks; ++c) {
        span(c, r0, off, nb);
        // the previous call on this buffer set has copied this chunk out (a
        // never-recorded event is already complete)
        e = cudaStreamWaitEvent(sH, hout[c], 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(d + off, static_cast<const char*>(h_in) + off, nb, cudaMemcpyHostToDevice, sH);
        if (e == cudaSuccess) e = cudaEventRecord(plan->hev[2 * c], sH);
        if (e != cudaSuccess) st = cuda_fail(e, "H2D copy");
    }
    for (uint64_t c = 0; !st && c < chunks; ++c) {
        const uint64_t rows = span(c, r0, off, nb);
        e = cudaStreamWaitEvent(sC, plan->hev[2 * c], 0);
        if (e != cudaSuccess) { st = cuda_fail(e, "stream wait"); break; }
        // (the chunk's input comes from the library's own copy, ordered by an event: independent)
        st = exec_device(plan, d + off, d + off, rows, flags | NTT_FLAG_INDEPENDENT, sC);
        if (!st && (e = cudaEventRecord(plan->hev[2 * c + 1], sC)) != cudaSuccess) st = cuda_fail(e, "event");
    }
    for (uint64_t c = 0; !st && c < chunks; ++c) {
        span(c, r0, off, nb);
        e = cudaStreamWaitEvent(sD, plan->hev[2 * c + 1], 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(static_cast<char*>(h_out) + off, d + off, nb, cudaMemcpyDeviceToHost, sD);
        if (e == cudaSuccess) e = cudaEventRecord(hout[c], sD);
        if (e != cudaSuccess) st = cuda_fail(e, "D2H copy");
    }
    if (async && !st) {                    // the caller's stream continues after the copy-out
        e = cudaEventRecord(plan->hend, sD);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(user, plan->hend, 0);
        if (e != cudaSuccess) st = cuda_fail(e, "stream order");
        if (cur != plan->device) cudaSetDevice(cur);
        return st;
    }
    for (auto hs : plan->hs) {
        cudaError_t e2 = cudaStreamSynchronize(hs);
        if (!st && e2 != cudaSuccess) st = cuda_fail(e2, "host exec");
    }
    if (cur != plan->device) cudaSetDevice(cur);
    return st;
}

int ntt_exec_host_sharded(const ntt_plan_t* plans, int nplans, const void* h_in, void* h_out, uint64_t batch,
                          unsigned flags) {
    if (!plans || nplans < 1) return fail(NTT_E_INVALID, "plans must hold at least one plan");
    for (int i = 0; i < nplans; ++i) {
        if (!plans[i]) return fail(NTT_E_INVALID, "NULL plan in the shard list");
        const ntt_plan_s& a = *plans[0];
        const ntt_plan_s& b = *plans[i];
        if (a.p != b.p || a.g != b.g || a.n != b.n || a.variant != b.variant || a.dir != b.dir ||
            a.word != b.word || a.n1 != b.n1 || a.n2 != b.n2)
            return fail(NTT_E_INVALID, "sharded plans must share field, size, variant, direction and word");
        for (int j = 0; j < i; ++j)
            if (plans[j] == plans[i] || plans[j]->device == plans[i]->device)
                return fail(NTT_E_INVALID, "one plan per device");
    }
    if (batch == 0) return NTT_OK;
    if (!h_in || !h_out) return fail(NTT_E_INVALID, "NULL buffer");
    const uint64_t row_bytes = plans[0]->n * plans[0]->word;
    // enqueue every device's pipeline first (each call returns once its copies
    // and transforms are queued), then wait for all of them
    int st = NTT_OK;
    int queued = 0;
    for (int i = 0; i < nplans && !st; ++i, ++queued) {
        const uint64_t lo = batch * i / nplans, hi = batch * (i + 1) / nplans;
        if (hi == lo) continue;
        st = ntt_exec_host(plans[i], static_cast<const char*>(h_in) + lo * row_bytes,
                           static_cast<char*>(h_out) + lo * row_bytes, hi - lo,
                           (flags & NTT_FLAG_SCALE) | NTT_FLAG_HOST_ASYNC, nullptr);
    }
    const std::string err = st ? g_last_error : std::string();
    int cur = 0;
    cudaGetDevice(&cur);
    for (int i = 0; i < queued; ++i) {
        cudaSetDevice(plans[i]->device);
        std::lock_guard<std::mutex> lk(plans[i]->host_mu);
        for (auto hs : plans[i]->hs) {
            if (!hs) continue;
            cudaError_t e = cudaStreamSynchronize(hs);
            if (!st && e != cudaSuccess) st = cuda_fail(e, "sharded host exec");
        }
    }
    cudaSetDevice(cur);
    if (!err.empty()) g_last_error = err;
    return st;
}

static int dist_step(ntt_plan_t plan, int step, int rank, int world, const void* d_in, void* d_out,
                     void* const* d_peers, void* stream) {
    if (!plan) return fail(NTT_E_INVALID, "NULL plan");
    if (plan->variant != NTT_SIXSTEP) return fail(NTT_E_BAD_FACTORIZATION, "plan is not a six-step plan");
    if (step != 0 && step != 1) return fail(NTT_E_INVALID, "step must be 0 (A) or 1 (B)");
    if (world < 1 || (world & (world - 1)) || (uint64_t)world > plan->n1 || (uint64_t)world > plan->n2 ||
        rank < 0 || rank >= world)
        return fail(NTT_E_INVALID, "world must be a power of two dividing n1 and n2; 0 <= rank < world");
    if (!d_in || (!d_out && !d_peers)) return fail(NTT_E_INVALID, "NULL buffer");
    if (d_peers) {
        if (world > kMaxPeers) return fail(NTT_E_INVALID, "peer pack supports at most 8 ranks");
        for (int h = 0; h < world; ++h)
            if (!d_peers[h]) return fail(NTT_E_INVALID, "NULL peer receive buffer");
    }
    if (plan->kind != 2)
        return fail(NTT_E_SIZE_NOT_SUPPORTED, "distributed four-step is implemented for the Goldilocks field");
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != plan->device) cudaSetDevice(plan->device);
    int launches = 0;
    MultipassReq r{};
    r.variant = plan->variant; r.L = plan->L; r.batch = 1; r.p = plan->p;
    r.n1 = plan->n1; r.n2 = plan->n2;
    r.tw1 = plan->table1 ? plan->table1->tw : nullptr;
    r.tw2 = plan->table2 ? plan->table2->tw : nullptr;
    r.stw1 = plan->table1 ? plan->table1->stw : nullptr;
    r.stw2 = plan->table2 ? plan->table2->stw : nullptr;
    r.cor_lo = plan->cor_lo; r.cor_hi = plan->cor_hi; r.cor_lb = plan->cor_lb;
    r.counters = dev_counters(plan->device);
    r.stream = static_cast<cudaStream_t>(stream); r.num_sms = plan->num_sms; r.launches = &launches;
    {   // per-stream workspace of the long-run passes (2 x n/G residues)
        std::lock_guard<std::mutex> lk(plan->mu);
        auto& slot = plan->ws[r.stream];
        int st = grow(slot.first, slot.second, sixstep_dist_ws_bytes(plan->n, world, plan->word));
        if (st) { if (cur != plan->device) cudaSetDevice(cur); return st; }
        r.ws = slot.first;
    }
    bool ok = false;
    window_break(r.stream);
    cudaError_t e = tile_sixstep_dist_gold(r, step, rank, world, d_in, d_out, &ok, d_peers);
    g_launches += launches;
    if (cur != plan->device) cudaSetDevice(cur);
    if (e != cudaSuccess) return cuda_fail(e, "distributed six-step");
    if (!ok) return fail(NTT_E_SIZE_NOT_SUPPORTED, "no compiled tile shape for this (n1, n2) split");
    return NTT_OK;
}

int ntt_sixstep_dist_step(ntt_plan_t plan, int step, int rank, int world, const void* d_in, void* d_out,
                          void* stream) {
    return dist_step(plan, step, rank, world, d_in, d_out, nullptr, stream);
}

int ntt_sixstep_dist_step_a_peer(ntt_plan_t plan, int rank, int world, const void* d_in, void* const* d_peer_recv,
                                 void* stream) {
    if (!d_peer_recv) return fail(NTT_E_INVALID, "NULL peer table");
    return dist_step(plan, 0, rank, world, d_in, nullptr, d_peer_recv, stream);
}

int ntt_exec_pointwise_inverse(ntt_plan_t plan, const void* d_a, const void* d_b, void* d_out, uint64_t batch,
                               void* stream) {
    if (!plan) return fail(NTT_E_INVALID, "NULL plan");
    if (plan->dir != NTT_INVERSE) return fail(NTT_E_INVALID, "pointwise-inverse requires an inverse-direction plan");
    if (batch == 0) return NTT_OK;
    if (!d_a || !d_b || !d_out) return fail(NTT_E_INVALID, "NULL buffer");
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != plan->device) cudaSetDevice(plan->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int st = NTT_OK;
    bool done = false;
    if (plan->kind == 0 && plan->variant != NTT_NAIVE && plan->variant != NTT_SIXSTEP && plan->variant != NTT_FLAT) {
        // fused: Montgomery product in the first group, n^-1 * 2^32 in the last
        const uint64_t ninv_m = (uint64_t)(((u128)plan->table->n_inv << 32) % plan->p);
        int launches = 0;
        MultipassReq r{};
        r.variant = plan->variant; r.L = plan->L; r.in = d_a; r.out = d_out; r.batch = batch;
        r.tw = plan->table->tw; r.stw = plan->table->stw; r.p = plan->p; r.scale = 1;
        r.ninv = ninv_m; r.ninv_shoup = shoup_word(ninv_m, plan->p, 32);
        r.counters = dev_counters(plan->device); r.stream = s; r.num_sms = plan->num_sms; r.launches = &launches;
        window_break(s);
        cudaError_t e = pointwise_inverse_f32(r, d_b, &done);
        g_launches += launches;
        if (e != cudaSuccess) st = cuda_fail(e, "pointwise-inverse");
    }
    if (!st && !done) {           // pointwise kernel into a per-stream buffer, then intt
        void* tmp = nullptr;
        {
            std::lock_guard<std::mutex> lk(plan->mu);
            auto& slot = plan->pw_ws[s];
            st = grow(slot.first, slot.second, batch * plan->n * plan->word);
            tmp = slot.first;
        }
        if (!st) st = ntt_pointwise_mul(plan, d_a, d_b, tmp, batch * plan->n, stream);
        if (!st) st = exec_device(plan, tmp, d_out, batch, NTT_FLAG_SCALE, s);
    }
    if (cur != plan->device) cudaSetDevice(cur);
    return st;
}

int ntt_pointwise_mul(ntt_plan_t plan, const void* d_a, const void* d_b, void* d_c, uint64_t count, void* stream) {
    if (!plan) return fail(NTT_E_INVALID, "NULL plan");
    int launches = 0;
    window_break(static_cast<cudaStream_t>(stream));
    cudaError_t e = pointwise_launch(plan->kind, plan->p, d_a, d_b, d_c, count,
                                     static_cast<cudaStream_t>(stream), plan->num_sms, &launches);
    g_launches += launches;
    if (e != cudaSuccess) return cuda_fail(e, "pointwise_mul");
    return NTT_OK;
}

int ntt_counters_enable(int enable) {
    g_counters_enabled = enable ? 1 : 0;
    return NTT_OK;
}

int ntt_counters_read(ntt_counters_t* out) {
    if (!out) return fail(NTT_E_INVALID, "NULL argument");
    memset(out, 0, sizeof(*out));
    out->kernel_launches = g_launches.load();
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto& kv : g_dev_counters) {
        if (!kv.second) continue;
        unsigned long long h[C_NCOUNTERS] = {0};
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(kv.first);
        cudaError_t e = cudaMemcpy(h, kv.second, sizeof(h), cudaMemcpyDeviceToHost);
        cudaSetDevice(cur);
        if (e != cudaSuccess) return cuda_fail(e, "counter read");
        out->transforms += h[C_TRANSFORMS];
        out->bitrev_passes += h[C_BITREV];
        out->stage_copies += h[C_COPIES];
        out->hbm_passes += h[C_HBM];
    }
    return NTT_OK;
}

int ntt_counters_reset(void) {
    g_launches = 0;
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto& kv : g_dev_counters) {
        if (!kv.second) continue;
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(kv.first);
        cudaMemset(kv.second, 0, C_NCOUNTERS * sizeof(unsigned long long));
        cudaDeviceSynchronize();
        cudaSetDevice(cur);
    }
    return NTT_OK;
}

}  // extern "C"
