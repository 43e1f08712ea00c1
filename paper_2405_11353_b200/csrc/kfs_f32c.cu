// Four-step instantiation for canonical u32 fields 2^30 <= p < 2^31 (BabyBear, ...).
#include "kfs_impl.cuh"
namespace nttb200 {
cudaError_t fourstep_u32_canon_s(const MultipassReq& r) { return fourstep_u32_policy<Canon<F32S>>(r); }
}  // namespace nttb200
