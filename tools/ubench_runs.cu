// HBM efficiency vs contiguous run length: each warp reads/writes runs of R
// bytes spread over rows 64 KiB apart (the access shape of a strided NTT
// pass), 4 GiB footprint.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

// element e (uint4 units) of a run-major enumeration: run r, offset o
__global__ void k_runs(const uint4* __restrict__ in, uint4* __restrict__ out, uint64_t n16, int run16, uint64_t nruns_per_row,
                       uint64_t row16, int mode) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x) {
        // consecutive threads: walk the run offset first, then successive ROWS (stride), then the run index
        const uint64_t o = i % run16;
        const uint64_t j = i / run16;
        const uint64_t rows = n16 / row16;
        const uint64_t r = j % rows, c = j / rows;       // row r, column-run c
        const uint64_t a = r * row16 + c * run16 + o;
        if (mode == 0) out[a] = in[a];          // both sides strided
        else if (mode == 1) out[a] = in[i];     // contiguous read, strided write
        else out[i] = in[a];                    // strided read, contiguous write
    }
}

int main(int argc, char** argv) {
    const uint64_t bytes = (argc > 1 ? (uint64_t)atoll(argv[1]) : 4096ull) << 20;   // MiB
    const uint64_t n16 = bytes / 16;
    uint4 *in, *out;
    cudaMalloc(&in, bytes);
    cudaMalloc(&out, bytes);
    cudaMemset(in, 1, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint64_t row16 = (64 << 10) / 16;   // 64 KiB rows
    for (int mode = 0; mode < 3; ++mode)
    for (int runb : {16, 32, 64, 128, 256, 512, 4096}) {
        const int run16 = runb / 16;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        k_runs<<<sms * 8, 256>>>(in, out, n16, run16, row16 / run16, row16, mode);
        cudaEventRecord(a);
        for (int it = 0; it < 3; ++it) k_runs<<<sms * 8, 256>>>(in, out, n16, run16, row16 / run16, row16, mode);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("mode %d (%s) footprint %llu MiB run %5d B: %.1f GB/s (read+write)\n", mode,
               mode == 0 ? "both strided" : (mode == 1 ? "strided write" : "strided read"), (unsigned long long)(bytes >> 20), runb,
               3 * 2.0 * bytes / (ms * 1e-3) / 1e9);
    }
    return 0;
}
