// Four-step two-pass kernels for large u32 N (fourstep.cuh), LazyF32 fields.
#include <cstdlib>
#include "fourstep.cuh"
#include "multipass.cuh"
#include "lazy.cuh"
namespace nttb200 {

// NTT_FOURSTEP=0 routes these sizes to the stage-faithful tile passes (A/B experiments)
static bool fourstep_enabled() {
    static const bool on = [] { const char* e = getenv("NTT_FOURSTEP"); return !(e && e[0] == '0'); }();
    return on;
}

template <int V>
static cudaError_t fs_run(const MultipassReq& r, int Kr, int Kc) {
    using A = LazyF32;
    fstep::FsArgs<A> a{};
    a.batch = r.batch;
    a.Kr = Kr;
    a.Kc = Kc;
    a.stw = static_cast<const uint2*>(r.stw);
    a.twist = static_cast<const uint2*>(r.fst);
    a.tw_main = static_cast<const uint2*>(r.tw);
    a.p = r.p;
    a.ninv = make_uint2((uint32_t)r.ninv, (uint32_t)r.ninv_shoup);
    a.counters = r.counters;
    // pass A: column sub-transforms + twist -> workspace
    a.in = static_cast<const uint32_t*>(r.in);
    a.out = static_cast<uint32_t*>(r.ws);
    a.scale = 0;
    a.count_bitrev = 1;          // DIT / Pease_nc sub-transforms bit-reverse their inputs
    cudaError_t e = fstep::fs_pass_any<A, V>(Kr, 0, a, r.stream, r.num_sms, r.launches);
    if (e != cudaSuccess) return e;
    // pass B: row sub-transforms -> out[k1 + R*k2]
    a.in = static_cast<const uint32_t*>(r.ws);
    a.out = static_cast<uint32_t*>(r.out);
    a.scale = r.scale;
    a.count_bitrev = 0;
    return fstep::fs_pass_any<A, V>(Kc, 1, a, r.stream, r.num_sms, r.launches);
}

cudaError_t fourstep_f32(const MultipassReq& r, bool* ok) {
    *ok = false;
    if (!fourstep_enabled() || !fourstep_applies(r.L, r.variant, r.p, 4) || !r.fst || !r.stw || !r.ws)
        return cudaSuccess;
    const int Kr = fourstep_kr(r.L), Kc = r.L - Kr;
    *ok = true;
    if (r.variant == V_DIT) return fs_run<V_DIT>(r, Kr, Kc);
    return fs_run<V_PEASE_NC>(r, Kr, Kc);
}

cudaError_t fourstep_twist_build(const void* tw, void* out, int L, cudaStream_t s) {
    const int Kr = fourstep_kr(L), Kc = L - Kr;
    fstep::k_fs_twist_table<uint2><<<1024, 256, 0, s>>>(static_cast<const uint2*>(tw), static_cast<uint2*>(out), Kr, Kc);
    return cudaGetLastError();
}

}  // namespace nttb200
