// Reciprocal throughput of the integer / FP64 instructions a lazy Shoup
// butterfly is built from (8 independent chains per thread, 16 warps/SMSP).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ubench_pipes.cu -o build/ubench_pipes
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(uint32_t* out, int iters, uint32_t a, uint32_t b) {
    uint32_t v[8];
    double d[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { v[i] = threadIdx.x + i * 77; d[i] = (double)(threadIdx.x + i); }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) asm volatile("mul.lo.u32 %0, %0, %1;" : "+r"(v[i]) : "r"(a));
            if (OP == 1) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(v[i]) : "r"(a));
            if (OP == 2) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v[i]) : "r"(a), "r"(b));
            if (OP == 3) asm volatile("add.u32 %0, %0, %1;" : "+r"(v[i]) : "r"(a));
            if (OP == 4) asm volatile("{.reg .u32 t; sub.u32 t, %0, %1; min.u32 %0, %0, t;}" : "+r"(v[i]) : "r"(a));
            if (OP == 5) asm volatile("fma.rz.f64 %0, %0, %1, %2;" : "+d"(d[i]) : "d"(1.0000001), "d"(0.5));
            if (OP == 6) asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(v[i]) : "r"(a), "r"(b));
            if (OP == 7) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(v[i]) : "r"(a), "r"(b));
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += v[i] + (uint32_t)d[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int OP>
void run(const char* name, int per) {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* o;
    cudaMalloc(&o, sms * 2048 * 4);
    const int iters = 4000, thr = 512, blocks = sms * 4;
    k<OP><<<blocks, thr>>>(o, 10, 3, 5);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<OP><<<blocks, thr>>>(o, iters, 3, 5);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double warp_instr = (double)blocks * thr / 32 * iters * 32 * per;
    const double smsp_cycles = ms * 1e-3 * clk * 1e3 * sms * 4;
    printf("%-14s %.2f cycles per warp-instruction per SMSP (max clk %d MHz, %.3f ms)\n", name, smsp_cycles / warp_instr,
           clk / 1000, ms);
    cudaFree(o);
}

int main() {
    run<0>("mul.lo", 1);
    run<1>("mul.hi", 1);
    run<2>("mad.lo", 1);
    run<3>("add", 1);
    run<4>("sub+min", 1);
    run<5>("fma.f64", 1);
    run<6>("add+add", 2);
    run<7>("fma.f32", 1);
    return 0;
}
