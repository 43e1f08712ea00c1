// Kernel instantiations for field FGold (see launch.cuh / multipass.cuh / engine.cuh).
#include "launch.cuh"
namespace nttb200 {
cudaError_t mp_launch_gold(const MultipassReq& r) { return launch_field<FGold>(r); }
cudaError_t pointwise_gold(uint64_t p, const void* a, const void* b, void* c, uint64_t n, cudaStream_t s,
                         int num_sms, int* launches) {
    return pointwise_field<FGold>(p, a, b, c, n, s, num_sms, launches);
}
}  // namespace nttb200
