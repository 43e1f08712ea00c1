// Micro-benchmark: butterfly throughput of each arithmetic policy with no
// memory traffic (register-resident, 16 independent values per thread), to
// measure the integer-pipe ceiling that bounds the NTT kernels on B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr
//      -I paper_2405_11353_b200/csrc tools/ubench_bfly.cu -o build/ubench_bfly
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "lazy.cuh"

using namespace nttb200;

// variant of LazyF32 with the two output additions written as 3-input PTX
// adds (IADD3-able) and the quotient product via mul.wide
struct LazyF32b : LazyF32 {
    NTT_D void dit(T& x, T& y, Tw w) const {
        const T xr = umin32(x, x - p2);
        const T q = __umulhi(y, w.y);
        const T t = y * w.x - q * p;
        uint32_t X, Y;
        asm("vadd.u32.u32.u32.add %0, %2, %3, %4;\n\t"
            "sub.u32 %1, %2, %3;\n\t"
            : "=r"(X), "=r"(Y) : "r"(xr), "r"(t), "r"(0u));
        x = X;
        y = Y + p2;
    }
};
struct LazyF32c : LazyF32 {      // q*p folded: t = y*w - q*p via mad with negated p
    NTT_D void dit(T& x, T& y, Tw w) const {
        const T xr = umin32(x, x - p2);
        const T q = __umulhi(y, w.y);
        T t;
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(q), "r"(0u - p), "r"(y * w.x));
        x = xr + t;
        y = xr - t + p2;
    }
};


// quotient q = floor(y*w'/2^32) on the FP64 pipe instead of IMAD.HI:
// fma_rz(2^52 + y, w'/2^32, 2^52 - w'*2^20) = 2^52 + y*w'/2^32 exactly before
// the one rounding, so the low word of the result is Shoup's q bit-for-bit.
struct TwD { uint32_t w, ws; double wd, c; };
struct LazyF32D : LazyF32 {
    using Tw = TwD;
    NTT_D void dit(T& x, T& y, Tw w) const {
        const T xr = umin32(x, x - p2);
        const double qd = __fma_rz(__hiloint2double(0x43300000, (int)y), w.wd, w.c);
        const T q = (T)__double2loint(qd);
        const T t = y * w.w - q * p;
        x = xr + t;
        y = xr - t + p2;
    }
};
// per-butterfly conversion of w' (no precomputed doubles)
struct LazyF32E : LazyF32 {
    NTT_D void dit(T& x, T& y, Tw w) const {
        const T xr = umin32(x, x - p2);
        const double wd = __hiloint2double(0x41300000, (int)w.y) - 1048576.0;
        const double c = __fma_rn(-4503599627370496.0, wd, 4503599627370496.0);
        const double qd = __fma_rz(__hiloint2double(0x43300000, (int)y), wd, c);
        const T q = (T)__double2loint(qd);
        const T t = y * w.x - q * p;
        x = xr + t;
        y = xr - t + p2;
    }
};
// butterflies with bit 1 of the register index on the FP64 pipe, the rest on IMAD.HI
struct LazyF32M : LazyF32D {};
template <class A, class T, class W>
__device__ __forceinline__ void bf(const A& ar, int c, T& x, T& y, W w) { ar.dit(x, y, w); }
template <class T, class W>
__device__ __forceinline__ void bf(const LazyF32M& ar, int c, T& x, T& y, W w) {
    if (c & 2) ar.LazyF32D::dit(x, y, w);
    else {
        const T xr = umin32(x, x - ar.p2);
        const T q = __umulhi(y, w.ws);
        const T t = y * w.w - q * ar.p;
        x = xr + t;
        y = xr - t + ar.p2;
    }
}

template <class A>
__global__ void k_bfly(typename A::T* out, uint64_t p, int iters, typename A::Tw w0, typename A::Tw w1) {
    using T = typename A::T;
    A ar;
    ar.init(p);
    T v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = (T)(threadIdx.x * 16 + i + blockIdx.x);
    typename A::Tw w = w0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                if (c & (1 << j)) continue;
                bf(ar, c, v[c], v[c | (1 << j)], w);
            }
        }
        w = (it & 1) ? w0 : w1;
    }
    T acc = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) acc = (T)(((uint64_t)acc * 3 + v[i] % (T)p) % p);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <class A>
void run(const char* name, uint64_t p, typename A::Tw w0, typename A::Tw w1, int threads) {
    using T = typename A::T;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    T* out;
    cudaMalloc(&out, (size_t)sms * 8 * threads * sizeof(T));
    const int iters = 2000;
    const int blocks = sms * (2048 / threads);
    k_bfly<A><<<blocks, threads>>>(out, p, 10, w0, w1);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_bfly<A><<<blocks, threads>>>(out, p, iters, w0, w1);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    double bfly = (double)blocks * threads * iters * 32;   // 4 stages x 8 butterflies
    const size_t nout = (size_t)blocks * threads;
    T* h = (T*)malloc(nout * sizeof(T));
    cudaMemcpy(h, out, nout * sizeof(T), cudaMemcpyDeviceToHost);
    unsigned long long hs = 1469598103934665603ull;
    for (size_t i = 0; i < nout; ++i) hs = (hs ^ (unsigned long long)h[i]) * 1099511628211ull;
    free(h);
    printf("%-12s threads/blk=%4d  %.3f ms  %.2f Tbfly/s  (%.2f warp-bfly/clk/SM at 1.9GHz)  out-hash %016llx\n", name, threads, ms,
           bfly / ms / 1e9, bfly / 32 / (ms * 1e-3) / sms / 1.9e9, hs);
    cudaFree(out);
}

// the four-mul.wide product (previous default) for comparison
struct FGoldOld : FGoldC {
    NTT_D T mul(T x, Tw w) const { return mul_c(x, w); }
};

// mul_m with u = r2 * EPS on the FMA pipe (IMAD.WIDE) instead of two ALU subtractions
struct FGoldW : FGoldC {
    NTT_D static T mul_w(T a, T b) {
        const uint32_t a0 = lo(a), a1 = hi(a), b0 = lo(b), b1 = hi(b);
        const uint64_t p00 = (uint64_t)a0 * b0;
        const uint64_t t = (uint64_t)a0 * b1 + (p00 >> 32);
        const uint64_t u = (uint64_t)a1 * b0 + (uint32_t)t;
        const uint64_t v = (uint64_t)a1 * b1 + (t >> 32) + (u >> 32);
        const uint32_t r0 = lo(p00), r1 = lo(u), r2 = lo(v), r3 = hi(v);
        const uint64_t ue = (uint64_t)r2 * 0xFFFFFFFFu;          // r2 * EPS (IMAD.WIDE)
        uint32_t t0, t1, m, c, s0, s1, q0, q1, c2;
        asm("sub.cc.u32 %0, %9, %11;\n\t"
            "subc.cc.u32 %1, %10, 0;\n\t"
            "subc.u32 %2, 0, 0;\n\t"
            "sub.cc.u32 %0, %0, %2;\n\t"
            "subc.u32 %1, %1, 0;\n\t"
            "add.cc.u32 %0, %0, %12;\n\t"
            "addc.cc.u32 %1, %1, %13;\n\t"
            "addc.u32 %3, 0, 0;\n\t"
            "neg.s32 %3, %3;\n\t"
            "add.cc.u32 %4, %0, %3;\n\t"
            "addc.u32 %5, %1, 0;\n\t"
            "add.cc.u32 %6, %4, 0xffffffff;\n\t"
            "addc.cc.u32 %7, %5, 0;\n\t"
            "addc.u32 %8, 0, 0;"
            : "=&r"(t0), "=&r"(t1), "=&r"(m), "=&r"(c), "=&r"(s0), "=&r"(s1), "=&r"(q0), "=&r"(q1), "=&r"(c2)
            : "r"(r0), "r"(r1), "r"(r3), "r"(lo(ue)), "r"(hi(ue)));
        (void)m;
        return c2 ? mk(q0, q1) : mk(s0, s1);
    }
    NTT_D T mul(T x, Tw w) const { return mul_w(x, w); }
};

// all-C formulation: 64-bit arithmetic, carries from compares (compiler-chosen SASS)
struct FGoldCC : FGoldC {
    static constexpr uint64_t E = 0xFFFFFFFFull;
    NTT_D static T addcc(T a, T b) {
        const uint64_t s = a + b;
        const bool c1 = s < a;
        const uint64_t t = s + E;
        const bool c2 = t < s;
        return (c1 | c2) ? t : s;
    }
    NTT_D static T subcc(T a, T b) {
        const uint64_t d = a - b;
        return a < b ? d - E : d;
    }
    NTT_D static T mulcc(T a, T b) {
        const uint32_t a0 = lo(a), a1 = hi(a), b0 = lo(b), b1 = hi(b);
        const uint64_t p00 = (uint64_t)a0 * b0;
        const uint64_t t = (uint64_t)a0 * b1 + (p00 >> 32);
        const uint64_t u = (uint64_t)a1 * b0 + (uint32_t)t;
        const uint64_t v = (uint64_t)a1 * b1 + (t >> 32) + (u >> 32);
        const uint64_t lo64 = ((uint64_t)(uint32_t)u << 32) | (uint32_t)p00;
        const uint64_t r2 = (uint32_t)v, r3 = v >> 32;
        uint64_t t0 = lo64 - r3;
        if (lo64 < r3) t0 -= E;
        const uint64_t t1 = (r2 << 32) - r2;
        uint64_t sm = t0 + t1;
        if (sm < t1) sm += E;
        return sm >= P ? sm - P : sm;
    }
    NTT_D T add(T a, T b) const { return addcc(a, b); }
    NTT_D T sub(T a, T b) const { return subcc(a, b); }
    NTT_D T mul(T x, Tw w) const { return mulcc(x, w); }
};
// PTX carry chains for add/sub, all-C multiply
struct FGoldMix : FGoldC {
    NTT_D T mul(T x, Tw w) const { return FGoldCC::mulcc(x, w); }
};
// all-C add/sub, PTX multiply
struct FGoldMix2 : FGoldC {
    NTT_D T add(T a, T b) const { return FGoldCC::addcc(a, b); }
    NTT_D T sub(T a, T b) const { return FGoldCC::subcc(a, b); }
};

// the previous default (mad.wide product, SEL-based corrections)
struct FGoldM : FGoldC {
    NTT_D T add(T a, T b) const { return add_c(a, b); }
    NTT_D T mul(T x, Tw w) const { return mul_m(x, w); }
};
__global__ void k_goldcheck(const uint64_t* a, const uint64_t* b, int n, int* bad) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t x = a[i], y = b[i];
    if (FGoldC::mul_c(x, y) != FGold::reduce128(x * y, __umul64hi(x, y))) atomicAdd(bad, 1);
    if (FGoldC::mul_m(x, y) != FGold::reduce128(x * y, __umul64hi(x, y))) atomicAdd(bad, 1);
    if (FGoldCC::mulcc(x, y) != FGold::reduce128(x * y, __umul64hi(x, y))) atomicAdd(bad, 1);
    if (FGoldW::mul_w(x, y) != FGold::reduce128(x * y, __umul64hi(x, y))) atomicAdd(bad, 1);
    { uint64_t s_ = x + y; if (s_ < x) s_ += FGold::EPS; if (FGoldCC::addcc(x, y) != FGold::canon(s_)) atomicAdd(bad + 1, 1); }
    if (FGoldCC::subcc(x, y) != (x < y ? x - y - FGold::EPS : x - y)) atomicAdd(bad + 2, 1);
    { uint64_t s_ = x + y; if (s_ < x) s_ += FGold::EPS; if (FGoldC::add_c(x, y) != FGold::canon(s_)) atomicAdd(bad + 1, 1); }
    if (FGoldC::sub_c(x, y) != (x < y ? x - y - FGold::EPS : x - y)) atomicAdd(bad + 2, 1);
    // wide-correction forms; lazy operand xl anywhere in [0, 2^64)
    const uint64_t xl = x + (uint64_t)(i & 3) * (0xFFFFFFFFull * 0x55555555ull) ;
    if (FGoldC::mul_w(xl, y) != FGold::reduce128(xl * y, __umul64hi(xl, y))) atomicAdd(bad, 1);
    if (FGoldC::mul_w(x, y) != FGold::reduce128(x * y, __umul64hi(x, y))) atomicAdd(bad, 1);
    if (FGoldC::mul_m(xl, y) != FGold::reduce128(xl * y, __umul64hi(xl, y))) atomicAdd(bad, 1);
    if (FGoldC::canon_s(xl) != (xl >= FGold::P ? xl - FGold::P : xl)) atomicAdd(bad + 1, 1);
    { const uint64_t l = FGoldC::add_lazy_a(xl, y);
      uint64_t s_ = FGold::canon(FGold::canon(xl)) + y; if (s_ < y) s_ += FGold::EPS;
      if (FGoldC::canon_s(l) != FGold::canon(s_)) atomicAdd(bad + 1, 1); }
    { uint64_t s_ = x + y; if (s_ < x) s_ += FGold::EPS; if (FGoldC::add_w(x, y) != FGold::canon(s_)) atomicAdd(bad + 1, 1); }
    { const uint64_t l = FGoldC::add_lazy(xl, y);
      uint64_t s_ = FGold::canon(FGold::canon(xl)) + y; if (s_ < y) s_ += FGold::EPS;
      if (FGoldC::canon_w(l) != FGold::canon(s_)) atomicAdd(bad + 1, 1); }
    if (FGoldC::canon_w(xl) != (xl >= FGold::P ? xl - FGold::P : xl)) atomicAdd(bad + 1, 1);
    { const uint64_t xc = FGold::canon(xl);
      if (FGoldC::canon_w(FGoldC::sub_c(xl, y)) != (xc < y ? xc - y - FGold::EPS : xc - y)) atomicAdd(bad + 2, 1); }
}
void check_gold() {
    const int n = 1 << 22;
    uint64_t *a, *b; int* bad;
    cudaMallocManaged(&a, n * 8); cudaMallocManaged(&b, n * 8); cudaMallocManaged(&bad, 12);
    uint64_t s = 88172645463325252ull;
    const uint64_t P = FGold::P;
    for (int i = 0; i < n; ++i) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17; a[i] = s % P;
        s ^= s << 13; s ^= s >> 7; s ^= s << 17; b[i] = s % P;
        if (i < 64) { a[i] = P - 1 - i; b[i] = (i & 1) ? P - 1 : i; }
    }
    bad[0] = bad[1] = bad[2] = 0;
    k_goldcheck<<<(n + 255) / 256, 256>>>(a, b, n, bad);
    cudaDeviceSynchronize();
    printf("goldcheck mismatches: mul %d add %d sub %d (of %d)\n", bad[0], bad[1], bad[2], n);
}

int main() {
    const uint32_t p = 998244353u;
    uint2 w0 = make_uint2(3, (uint32_t)(((uint64_t)3 << 32) / p));
    uint2 w1 = make_uint2(5, (uint32_t)(((uint64_t)5 << 32) / p));
    run<LazyF32>("lazy-u32", p, w0, w1, 256);
    run<LazyF32>("lazy-u32", p, w0, w1, 512);
    run<LazyF32b>("lazy-vadd", p, w0, w1, 256);
    run<LazyF32c>("lazy-mad", p, w0, w1, 256);
    auto mk = [&](uint2 w) { TwD d; d.w = w.x; d.ws = w.y; d.wd = (double)w.y / 4294967296.0;
                             d.c = 4503599627370496.0 - (double)w.y * 1048576.0; return d; };
    run<LazyF32D>("lazy-fp64q", p, mk(w0), mk(w1), 256);
    run<LazyF32D>("lazy-fp64q", p, mk(w0), mk(w1), 512);
    run<LazyF32E>("lazy-fp64cv", p, w0, w1, 256);
    run<LazyF32M>("lazy-mix", p, mk(w0), mk(w1), 256);
    run<LazyF32M>("lazy-mix", p, mk(w0), mk(w1), 512);
    run<Canon<F32S>>("canon-u32", p, w0, w1, 256);
    const uint64_t G = 0xFFFFFFFF00000001ull;
    run<Canon<FGold>>("goldilocks", G, 7ull, 49ull, 256);
    run<Canon<FGold>>("goldilocks", G, 7ull, 49ull, 512);
    run<Canon<FGoldC>>("gold-carry", G, 7ull, 49ull, 256);
    run<Canon<FGoldC>>("gold-carry", G, 7ull, 49ull, 512);
    run<Canon<FGoldOld>>("gold-mulc", G, 7ull, 49ull, 256);
    run<Canon<FGoldOld>>("gold-mulc", G, 7ull, 49ull, 512);
    run<Canon<FGoldW>>("gold-wideE", G, 7ull, 49ull, 256);
    run<Canon<FGoldW>>("gold-wideE", G, 7ull, 49ull, 512);
    run<Canon<FGoldM>>("gold-mulm", G, 7ull, 49ull, 256);
    run<Canon<FGoldM>>("gold-mulm", G, 7ull, 49ull, 512);
    run<LazyGoldT<0>>("gold-lazy0", G, 7ull, 49ull, 256);
    run<LazyGoldT<0>>("gold-lazy0", G, 7ull, 49ull, 512);
    run<LazyGoldT<1>>("gold-lazy1", G, 7ull, 49ull, 512);
    run<LazyGoldT<2>>("gold-lazy2", G, 7ull, 49ull, 512);
    // exactness check of FGoldC vs FGold on random operands
    check_gold();
    return 0;
}
