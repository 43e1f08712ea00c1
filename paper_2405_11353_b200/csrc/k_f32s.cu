// Kernel instantiations for field F32S (see launch.cuh / multipass.cuh / engine.cuh).
#include "launch.cuh"
namespace nttb200 {
cudaError_t mp_launch_f32s(const MultipassReq& r) { return launch_field<F32S>(r); }
cudaError_t pointwise_inverse_f32(const MultipassReq& r, const void* in2, bool* ok) {
    *ok = false;
    if (r.p >= (1ull << 30) || r.L < 9 || r.L > 13 || !r.stw) return cudaSuccess;
    if ((reinterpret_cast<uintptr_t>(r.in) | reinterpret_cast<uintptr_t>(in2) | reinterpret_cast<uintptr_t>(r.out)) & 15)
        return cudaSuccess;
    switch (r.variant) {
        case V_DIT: return run_fast_pw<V_DIT>(r, in2, ok);
        case V_DIF: return run_fast_pw<V_DIF>(r, in2, ok);
        case V_PEASE: return run_fast_pw<V_PEASE>(r, in2, ok);
        case V_PEASE_NC: return run_fast_pw<V_PEASE_NC>(r, in2, ok);
        case V_STOCKHAM: return run_fast_pw<V_STOCKHAM>(r, in2, ok);
        default: return cudaSuccess;
    }
}
cudaError_t pointwise_f32s(uint64_t p, const void* a, const void* b, void* c, uint64_t n, cudaStream_t s,
                         int num_sms, int* launches) {
    return pointwise_field<F32S>(p, a, b, c, n, s, num_sms, launches);
}
}  // namespace nttb200
#ifdef NTT_FAST_TIMELINE
extern "C" int ntt_debug_timeline(unsigned long long* out, int n) {
    return (int)cudaMemcpyFromSymbol(out, nttb200::fastk::g_tl, sizeof(unsigned long long) * n);
}
#endif
