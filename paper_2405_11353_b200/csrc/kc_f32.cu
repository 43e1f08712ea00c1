// Cluster single-pass kernels (fastclus.cuh), u32 fields: LazyF32 (p < 2^30)
// here, the canonical policies in kc_f32c.cu; the dispatcher.
#include "kc_impl.cuh"
namespace nttb200 {
cudaError_t fastc_u32_canon(const MultipassReq& r, bool* ok);   // kc_f32c.cu
cudaError_t fastc_f32(const MultipassReq& r, bool* ok) {
    *ok = false;
    if (!clus_applies(r.L, r.variant, r.p, 4) || !r.stw || (reinterpret_cast<uintptr_t>(r.in) & 15)) return cudaSuccess;
    if (r.p < (1ull << 30)) return fastc_policy<LazyF32>(r, ok);
    return fastc_u32_canon(r, ok);
}
}  // namespace nttb200
