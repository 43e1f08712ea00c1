// IMAD.WIDE.U32 (both product halves) vs IMAD.HI + IMAD: FMA-pipe cost per
// SMSP.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ubench_wide.cu -o build/ubench_wide
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(uint32_t* out, int iters, uint32_t a_in) {
    const uint32_t a = a_in + (threadIdx.x & 1);
    uint32_t v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = threadIdx.x + i * 77;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) {        // IMAD.WIDE.U32: hi and lo in one instruction
                uint64_t t;
                asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(t) : "r"(v[i]), "r"(a));
                v[i] = (uint32_t)(t >> 32) ^ (uint32_t)t;
            } else if (OP == 1) { // IMAD.HI + IMAD
                uint32_t h, l;
                asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(h) : "r"(v[i]), "r"(a));
                asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(l) : "r"(v[i]), "r"(a));
                v[i] = h ^ l;
            } else if (OP == 2) { // hi only through IMAD.WIDE
                uint64_t t;
                asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(t) : "r"(v[i]), "r"(a));
                v[i] = (uint32_t)(t >> 32) ^ 0x1234u;
            } else {              // IMAD.HI alone
                uint32_t h;
                asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(h) : "r"(v[i]), "r"(a));
                v[i] = h ^ 0x1234u;
            }
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
template <int OP>
void run(const char* name) {
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    uint32_t* o;
    cudaMalloc(&o, sms * 4096 * 4);
    const int thr = 512, blocks = sms * 4, iters = 4000;
    k<OP><<<blocks, thr>>>(o, 10, 3);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<OP><<<blocks, thr>>>(o, iters, 3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)blocks * thr / 32 * iters * 32;
    printf("%-22s %.2f SMSP-cycles per step (%.3f ms)\n", name, ms * 1e-3 * clk * 1e3 * sms * 4 / ops, ms);
    cudaFree(o);
}
int main() {
    run<0>("IMAD.WIDE + LOP3");
    run<1>("IMAD.HI + IMAD + LOP3");
    run<2>("IMAD.WIDE hi + LOP3");
    run<3>("IMAD.HI + LOP3");
    return 0;
}
