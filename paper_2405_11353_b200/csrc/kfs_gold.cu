// Four-step two-pass kernels (fourstep.cuh) for Goldilocks 2^14..2^18 (config 3:
// 2^16 = 256 x 256): DIT / Flat / DIF / Pease_nc / Stockham sub-transforms, canonical field.
#include <cstdlib>
#include "fourstep.cuh"
#include "multipass.cuh"
namespace nttb200 {


template <int V, int L>
static cudaError_t fsg_run_l(const MultipassReq& r) {
    using A = GoldPolicy<V == V_DIF>;
    constexpr int KR = (L + 1) / 2, KC = L - KR;
    fstep::FsArgs<A> a{};
    a.batch = r.batch;
    a.Kr = KR;
    a.Kc = KC;
    a.stw = static_cast<const uint64_t*>(r.stw);
    a.twist = static_cast<const uint64_t*>(r.fst);
    a.tw_main = static_cast<const uint64_t*>(r.tw);
    a.p = r.p;
    a.ninv = r.ninv;
    a.counters = r.counters;
    // intt: n^-1 rides the twist (a second [k1][n2] table holding w^(k1 n2) * n^-1, built with the
    // inverse plan), so pass B's stores skip their scaling product -- where pass A reads the table
    const bool fold = r.scale && r.fst_scaled && V == V_DIF;
    if (fold) a.twist = static_cast<const uint64_t*>(r.fst_scaled);
    a.in = static_cast<const uint64_t*>(r.in);
    a.out = static_cast<uint64_t*>(r.ws);
    a.scale = 0;
    a.count_bitrev = V == V_STOCKHAM ? 0 : 1;   // Stockham never bit-reverses
    cudaError_t e = fstep::fs_launch<A, V, KR, 0, KC>(a, r.stream, r.num_sms, r.launches);
    if (e != cudaSuccess) return e;
    a.in = static_cast<const uint64_t*>(r.ws);
    a.out = static_cast<uint64_t*>(r.out);
    a.scale = fold ? 0 : r.scale;
    a.count_bitrev = 0;
    return fstep::fs_launch<A, V, KC, 1, KR>(a, r.stream, r.num_sms, r.launches);
}

template <int V>
static cudaError_t fsg_run(const MultipassReq& r) {
    switch (r.L) {
        case 14: return fsg_run_l<V, 14>(r);
        case 15: return fsg_run_l<V, 15>(r);
        case 16: return fsg_run_l<V, 16>(r);
        case 17: return fsg_run_l<V, 17>(r);
        case 18: return fsg_run_l<V, 18>(r);
        default: return cudaErrorInvalidValue;
    }
}

__global__ void k_twist_scale_gold(uint64_t* t, uint64_t n, uint64_t c) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        t[i] = FGoldC::mul_m(t[i], c);
}
// t[i] *= c (the n^-1-carrying copy of the twist table)
cudaError_t fourstep_twist_scale_gold(void* t, uint64_t n, uint64_t c, cudaStream_t s) {
    k_twist_scale_gold<<<1024, 256, 0, s>>>(static_cast<uint64_t*>(t), n, c);
    return cudaGetLastError();
}

cudaError_t fourstep_gold(const MultipassReq& r, bool* ok) {
    *ok = false;
    if (!fourstep_applies(r.L, r.variant, r.p, 8) || !r.fst || !r.stw || !r.ws)
        return cudaSuccess;
    *ok = true;
    // Flat's per-stage states are DIT's: DIT sub-transforms
    if (r.variant == V_DIT || r.variant == V_FLAT) return fsg_run<V_DIT>(r);
    if (r.variant == V_DIF) return fsg_run<V_DIF>(r);
    if (r.variant == V_STOCKHAM) return fsg_run<V_STOCKHAM>(r);
    if (r.variant == V_PEASE) return fsg_run<V_PEASE>(r);
    return fsg_run<V_PEASE_NC>(r);
}

}  // namespace nttb200
