// Four-step two-pass kernels (fourstep.cuh) for Goldilocks 2^16 = 256 x 256
// (config 3): DIT / DIF / Pease_nc sub-transforms of length 2^8, canonical field.
#include <cstdlib>
#include "fourstep.cuh"
#include "multipass.cuh"
namespace nttb200 {

static bool fourstep_gold_enabled() {
    static const bool on = [] { const char* e = getenv("NTT_FOURSTEP"); return !(e && e[0] == '0'); }();
    return on;
}

template <int V>
static cudaError_t fsg_run(const MultipassReq& r) {
    using A = Canon<FGold>;
    fstep::FsArgs<A> a{};
    a.batch = r.batch;
    a.Kr = 8;
    a.Kc = 8;
    a.stw = static_cast<const uint64_t*>(r.stw);
    a.twist = static_cast<const uint64_t*>(r.fst);
    a.tw_main = static_cast<const uint64_t*>(r.tw);
    a.p = r.p;
    a.ninv = r.ninv;
    a.counters = r.counters;
    a.in = static_cast<const uint64_t*>(r.in);
    a.out = static_cast<uint64_t*>(r.ws);
    a.scale = 0;
    a.count_bitrev = 1;          // every variant here bit-reverses (DIT/Pease on input, DIF on output)
    cudaError_t e = fstep::fs_launch<A, V, 8, 0, 8>(a, r.stream, r.num_sms, r.launches);
    if (e != cudaSuccess) return e;
    a.in = static_cast<const uint64_t*>(r.ws);
    a.out = static_cast<uint64_t*>(r.out);
    a.scale = r.scale;
    a.count_bitrev = 0;
    return fstep::fs_launch<A, V, 8, 1, 8>(a, r.stream, r.num_sms, r.launches);
}

cudaError_t fourstep_gold(const MultipassReq& r, bool* ok) {
    *ok = false;
    if (!fourstep_gold_enabled() || !fourstep_applies(r.L, r.variant, r.p, 8) || !r.fst || !r.stw || !r.ws)
        return cudaSuccess;
    *ok = true;
    if (r.variant == V_DIT) return fsg_run<V_DIT>(r);
    if (r.variant == V_DIF) return fsg_run<V_DIF>(r);
    return fsg_run<V_PEASE_NC>(r);
}

}  // namespace nttb200
