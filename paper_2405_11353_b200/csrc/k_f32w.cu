// Kernel instantiations for field F32W (see launch.cuh / multipass.cuh / engine.cuh).
#include "launch.cuh"
namespace nttb200 {
cudaError_t mp_launch_f32w(const MultipassReq& r) { return launch_field<F32W>(r); }
cudaError_t pointwise_f32w(uint64_t p, const void* a, const void* b, void* c, uint64_t n, cudaStream_t s,
                         int num_sms, int* launches) {
    return pointwise_field<F32W>(p, a, b, c, n, s, num_sms, launches);
}
}  // namespace nttb200
