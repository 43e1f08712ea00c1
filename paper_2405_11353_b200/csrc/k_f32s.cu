// Kernel instantiations for field F32S (see launch.cuh / multipass.cuh / engine.cuh).
#include "launch.cuh"
namespace nttb200 {
cudaError_t mp_launch_f32s(const MultipassReq& r) { return launch_field<F32S>(r); }
cudaError_t pointwise_f32s(uint64_t p, const void* a, const void* b, void* c, uint64_t n, cudaStream_t s,
                         int num_sms, int* launches) {
    return pointwise_field<F32S>(p, a, b, c, n, s, num_sms, launches);
}
}  // namespace nttb200
