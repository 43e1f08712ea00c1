// Four-step instantiation for u32 fields 2^31 <= p < 2^32 (the reference's
// DEFAULT_PRIME 3221225473): Shoup with a 33-bit intermediate, canonical.
#include "kfs_impl.cuh"
namespace nttb200 {
cudaError_t fourstep_u32_canon_w(const MultipassReq& r) { return fourstep_u32_policy<Canon<F32W>>(r); }
}  // namespace nttb200
