// Host runners of the cluster single-pass kernels (fastclus.cuh), templated on
// the arithmetic policy; instantiated per policy by kc_*.cu.
#pragma once
#include "fastclus.cuh"
#include "launch.cuh"
namespace nttb200 {

template <class A, int V, int L, int CB>
cudaError_t fastc_run_l(const MultipassReq& r, bool* ok) {
    fastk::FastArgs<A> a{};
    a.in = static_cast<const typename A::T*>(r.in);
    a.out = static_cast<typename A::T*>(r.out);
    a.batch = r.batch;
    a.stw = static_cast<const typename A::Tw*>(r.stw);
    a.p = r.p;
    a.scale = r.scale;
    a.ninv = make_tw<typename A::Field>(r.ninv, r.ninv_shoup);
    a.counters = r.counters;
    return fastk::launch_fastc<A, V, L, CB>(a, r.stream, r.launches, ok);
}

// sizes per word: u32 2^15 (2 CTAs), 2^16 (4); u64 2^14 (2), 2^15 (4), 2^16 (8)
template <class A, int V>
cudaError_t fastc_run_v(const MultipassReq& r, bool* ok) {
    *ok = false;
    if constexpr (sizeof(typename A::T) == 4) {
        if (r.L == 15) return fastc_run_l<A, V, 15, 1>(r, ok);
        if (r.L == 16) return fastc_run_l<A, V, 16, 2>(r, ok);
    } else {
        if (r.L == 14) return fastc_run_l<A, V, 14, 1>(r, ok);
        if (r.L == 15) return fastc_run_l<A, V, 15, 2>(r, ok);
        if (r.L == 16) return fastc_run_l<A, V, 16, 3>(r, ok);
    }
    return cudaSuccess;
}

template <class A>
cudaError_t fastc_policy(const MultipassReq& r, bool* ok) {
    // Flat's per-stage states are DIT's (algorithms.py:161-195)
    if (r.variant == V_DIT || r.variant == V_FLAT) return fastc_run_v<A, V_DIT>(r, ok);
    if (r.variant == V_DIF) return fastc_run_v<A, V_DIF>(r, ok);
    if (r.variant == V_PEASE_NC) return fastc_run_v<A, V_PEASE_NC>(r, ok);
    *ok = false;
    return cudaSuccess;
}

}  // namespace nttb200
