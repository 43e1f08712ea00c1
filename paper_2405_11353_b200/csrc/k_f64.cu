// Kernel instantiations for field F64 (see launch.cuh / multipass.cuh / engine.cuh).
#include "launch.cuh"
namespace nttb200 {
cudaError_t mp_launch_f64(const MultipassReq& r) { return launch_field<F64>(r); }
cudaError_t pointwise_f64(uint64_t p, const void* a, const void* b, void* c, uint64_t n, cudaStream_t s,
                         int num_sms, int* launches) {
    return pointwise_field<F64>(p, a, b, c, n, s, num_sms, launches);
}
}  // namespace nttb200
