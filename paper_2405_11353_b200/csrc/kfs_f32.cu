// Four-step two-pass kernels for large u32 N: the LazyF32 instantiation
// (p < 2^30), the dispatcher over the u32 policies, and the twist-table build.
#include "kfs_impl.cuh"
namespace nttb200 {

cudaError_t fourstep_u32_canon_s(const MultipassReq& r);   // kfs_f32c.cu: 2^30 <= p < 2^31
cudaError_t fourstep_u32_canon_w(const MultipassReq& r);   // kfs_f32w.cu: 2^31 <= p < 2^32

cudaError_t fourstep_f32(const MultipassReq& r, bool* ok) {
    *ok = false;
    if (!fourstep_applies(r.L, r.variant, r.p, 4) || !r.fst || !r.stw || !r.ws)
        return cudaSuccess;
    *ok = true;
    if (r.p < (1ull << 30)) return fourstep_u32_policy<LazyF32>(r);
    if (r.p < (1ull << 31)) return fourstep_u32_canon_s(r);
    return fourstep_u32_canon_w(r);
}

cudaError_t fourstep_twist_build(const void* tw, void* out, int L, int word, cudaStream_t s) {
    const int Kr = fourstep_kr(L), Kc = L - Kr;
    if (word == 4)   // (w, Shoup word) pairs
        fstep::k_fs_twist_table<uint2><<<1024, 256, 0, s>>>(static_cast<const uint2*>(tw), static_cast<uint2*>(out), Kr, Kc);
    else             // Goldilocks: values
        fstep::k_fs_twist_table<uint64_t><<<1024, 256, 0, s>>>(static_cast<const uint64_t*>(tw), static_cast<uint64_t*>(out), Kr, Kc);
    return cudaGetLastError();
}

}  // namespace nttb200
#ifdef NTT_FS_TIMELINE
extern "C" int ntt_debug_fs_timeline(unsigned long long* out, int n) {
    return (int)cudaMemcpyFromSymbol(out, nttb200::fstep::g_fstl, sizeof(unsigned long long) * n);
}
#endif
