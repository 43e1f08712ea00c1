// Does an immediate operand change the FMA-pipe cost of integer multiplies?
// (B300 notes: FFMA with an immediate issues at rt=1 vs 2 for the 3-register
// form.)  Reciprocal throughput per SMSP of IMAD / IMAD.HI / IMAD.WIDE with a
// register vs an immediate multiplier, and of the lazy Shoup butterfly with
// the prime in a register vs baked in as an immediate.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ubench_imm.cu -o build/ubench_imm
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr uint32_t PIMM = 998244353u;

template <int OP>
__global__ void k(uint32_t* out, int iters, uint32_t a_in, uint32_t b_in) {
    uint32_t v[8];
    float f[8];
    // runtime values the compiler cannot fold (register operands)
    const uint32_t a = a_in + (threadIdx.x & 1), b = b_in + (threadIdx.x & 2);
#pragma unroll
    for (int i = 0; i < 8; ++i) { v[i] = threadIdx.x + i * 77; f[i] = (float)(threadIdx.x + i); }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v[i]) : "r"(a), "r"(b));
            if (OP == 1) asm volatile("mad.lo.u32 %0, %0, 998244353, %1;" : "+r"(v[i]) : "r"(b));
            if (OP == 2) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(v[i]) : "r"(a));
            if (OP == 3) asm volatile("mul.hi.u32 %0, %0, 998244353;" : "+r"(v[i]));
            if (OP == 4) asm volatile("{.reg .u64 t; mul.wide.u32 t, %0, %1; cvt.u32.u64 %0, t;}" : "+r"(v[i]) : "r"(a));
            if (OP == 5) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[i]) : "f"(__uint_as_float(a)), "f"(__uint_as_float(b)));
            if (OP == 6) asm volatile("fma.rn.f32 %0, %0, 0f3F800001, %1;" : "+f"(f[i]) : "f"(__uint_as_float(b)));
            if (OP == 7) asm volatile("mul.lo.u32 %0, %0, 998244353;" : "+r"(v[i]));
            if (OP == 8) asm volatile("mul.lo.u32 %0, %0, %1;" : "+r"(v[i]) : "r"(a));
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += v[i] + __float_as_uint(f[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// register-resident lazy Shoup DIT butterflies (LazyF32::dit); IMM: p, 2p, 4p immediates
template <bool IMM>
__global__ void kb(uint32_t* out, int iters, uint32_t p_in, uint32_t w_in, uint32_t ws_in) {
    const uint32_t p = IMM ? PIMM : p_in + (threadIdx.x & 1) * 0;
    const uint32_t p2 = 2 * p, p4 = 4 * p;
    uint32_t x[8], y[8];
    const uint32_t w = w_in + (threadIdx.x & 1), ws = ws_in + (threadIdx.x & 1);
#pragma unroll
    for (int i = 0; i < 8; ++i) { x[i] = (threadIdx.x * 7 + i) % p; y[i] = (threadIdx.x * 13 + i) % p; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            uint32_t xr = min(x[i], x[i] - p2);
            uint32_t q = __umulhi(y[i], ws);
            uint32_t t = y[i] * w - q * p;
            uint32_t nx = min(xr + t, p4);
            uint32_t ny = xr - t + p2;
            x[i] = nx; y[i] = ny;
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += x[i] ^ y[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <class K>
double timeit(K kern, int blocks, int thr, uint32_t* o) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    kern(blocks, thr, o, 10);
    cudaEventRecord(e0);
    kern(blocks, thr, o, 4000);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}

int main() {
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    uint32_t* o;
    cudaMalloc(&o, sms * 4096 * 4);
    const int thr = 512, blocks = sms * 4;
    const double warp_ops = (double)blocks * thr / 32 * 4000 * 32;    // per instruction slot
    auto rep = [&](const char* name, double ms, double per) {
        printf("%-26s %.2f SMSP-cycles per warp-op (%.3f ms)\n", name,
               ms * 1e-3 * clk * 1e3 * sms * 4 / (warp_ops * per), ms);
    };
#define RUN(OP, NAME, PER) rep(NAME, timeit([](int b, int t, uint32_t* o, int it) { k<OP><<<b, t>>>(o, it, 3, 5); }, blocks, thr, o), PER)
    RUN(0, "IMAD reg,reg,reg", 1);
    RUN(1, "IMAD reg,imm,reg", 1);
    RUN(8, "IMUL reg,reg", 1);
    RUN(7, "IMUL reg,imm", 1);
    RUN(2, "IMAD.HI reg,reg", 1);
    RUN(3, "IMAD.HI reg,imm", 1);
    RUN(4, "IMAD.WIDE reg,reg", 1);
    RUN(5, "FFMA reg", 1);
    RUN(6, "FFMA imm", 1);
    double m0 = timeit([](int b, int t, uint32_t* o, int it) { kb<false><<<b, t>>>(o, it, PIMM, 12345, 678); }, blocks, thr, o);
    double m1 = timeit([](int b, int t, uint32_t* o, int it) { kb<true><<<b, t>>>(o, it, PIMM, 12345, 678); }, blocks, thr, o);
    const double bf = (double)blocks * thr * 4000 * 32;
    printf("butterfly p in register   %.3f Tbfly/s (%.3f ms)\n", bf / (m0 * 1e-3) / 1e12, m0);
    printf("butterfly p immediate     %.3f Tbfly/s (%.3f ms)\n", bf / (m1 * 1e-3) / 1e12, m1);
    return 0;
}
