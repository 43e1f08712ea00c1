// Cluster single-pass kernels (fastclus.cuh), canonical u32 fields: 2^30 <= p <
// 2^31 (Canon<F32S>) and 2^31 <= p < 2^32 (Canon<F32W>, the reference's DEFAULT_PRIME).
#include "kc_impl.cuh"
namespace nttb200 {
cudaError_t fastc_u32_canon(const MultipassReq& r, bool* ok) {
    if (r.p < (1ull << 31)) return fastc_policy<Canon<F32S>>(r, ok);
    return fastc_policy<Canon<F32W>>(r, ok);
}
}  // namespace nttb200
