// Cluster single-pass kernels (fastclus.cuh), Goldilocks 2^14 .. 2^16 (config 3:
// 2^16 on a cluster of 8 CTAs): lazy sums for DIT-type dataflows, canonical DIF.
#include "kc_impl.cuh"
namespace nttb200 {
cudaError_t fastc_gold(const MultipassReq& r, bool* ok) {
    *ok = false;
    if (!clus_applies(r.L, r.variant, r.p, 8) || !r.stw || (reinterpret_cast<uintptr_t>(r.in) & 15)) return cudaSuccess;
    if (r.variant == V_DIF) return fastc_policy<GoldPolicy<true>>(r, ok);
    return fastc_policy<GoldPolicy<false>>(r, ok);
}
}  // namespace nttb200
