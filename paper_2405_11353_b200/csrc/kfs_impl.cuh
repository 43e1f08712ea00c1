// Host runners of the u32 four-step (fourstep.cuh, fourstep_tma.cuh), templated
// on the arithmetic policy; instantiated per field policy by kfs_f32*.cu.
#pragma once
#include <cstdlib>
#include <cstring>
#include <cudaTypedefs.h>
#include "fourstep.cuh"
#include "fourstep_tma.cuh"
#include "multipass.cuh"
#include "lazy.cuh"
namespace nttb200 {

#ifndef NTT_FSA_L2PROMO
#define NTT_FSA_L2PROMO 0     // TMA L2 promotion of the 32-byte box rows: 0 none, 1 64B, 2 128B, 3 256B
#endif

inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// a pass with TMA / bulk-copy tile loads (fourstep_tma.cuh): K = the pass's
// sub-transform length, KO = the other dimension
template <class A, int V, int MODE, int K, int KO>
inline cudaError_t fs_pass_tma_k(const MultipassReq& r, const CUtensorMap& map) {
    using GG = fstep::TmaGeo<V, K>;
    constexpr int Kr = MODE == 0 ? K : KO, Kc = MODE == 0 ? KO : K;
    fstep::FsTmaArgs<A> a{};
    a.in = static_cast<const uint32_t*>(MODE == 0 ? r.in : r.ws);
    a.out = static_cast<uint32_t*>(MODE == 0 ? r.ws : r.out);
    a.batch = r.batch;
    a.Kr = Kr;
    a.Kc = Kc;
    a.stw = static_cast<const uint2*>(r.stw);
    a.twist = static_cast<const uint2*>(r.fst);
    a.tw_main = static_cast<const uint2*>(r.tw);
    a.p = r.p;
    a.scale = MODE == 1 ? r.scale : 0;
    a.ninv = make_uint2((uint32_t)r.ninv, (uint32_t)r.ninv_shoup);
    a.count_bitrev = MODE == 0 ? 1 : 0;
    a.counters = r.counters;
    constexpr size_t smem = fstep::fsa_smem_bytes<V, K, MODE>();
    auto kern = fstep::k_fs_tma<A, V, MODE, K, KO>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 512, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
    const uint64_t ntiles = r.batch << ((MODE == 0 ? Kc : Kr) - GG::LQ);
    uint64_t grid = (uint64_t)r.num_sms * occ;
    if (grid > ntiles) grid = ntiles;
    e = fastk::launch_pdl(kern, dim3((unsigned)grid), dim3(512), smem, r.stream, map, a);
    if (r.launches) ++*r.launches;
    return e != cudaSuccess ? e : cudaGetLastError();
}

// true when the pass ran through the TMA kernel (*err its status)
template <class A, int V, int MODE>
inline bool fs_pass_tma(const MultipassReq& r, int Kr, int Kc, cudaError_t* err) {
    *err = cudaSuccess;
    if constexpr (V == V_DIF || V == V_STOCKHAM) return false;      // the TMA passes carry DIT / Pease_nc geometries
    else {
    const void* src = MODE == 0 ? r.in : r.ws;
    const int K = MODE == 0 ? Kr : Kc;
    if (reinterpret_cast<uintptr_t>(src) & 15) return false;
    if (MODE == 1 && K != 10) return false;
    if (K < 7 || K > 10) return false;
    CUtensorMap map;
    memset(&map, 0, sizeof(map));
    if (MODE == 0) {
        auto enc = tensor_map_encoder();
        if (!enc) return false;
        const int tq = 1 << (13 - K);
        cuuint64_t dims[2] = {(cuuint64_t)1 << Kc, (cuuint64_t)r.batch << Kr};
        cuuint64_t strides[1] = {((cuuint64_t)1 << Kc) * 4};
        cuuint32_t box[2] = {(cuuint32_t)tq, (cuuint32_t)(K >= 8 ? 256 : (1 << K))};
        cuuint32_t es[2] = {1, 1};
        if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(src), dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                NTT_FSA_L2PROMO == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                : NTT_FSA_L2PROMO == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                : NTT_FSA_L2PROMO == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    }
    // (K, other dimension) pairs of 2^14 .. 2^20 (Kr = ceil(L/2), Kc = floor(L/2))
#define NTT_FSTK(KK, KOO) \
    if (K == KK && (MODE == 0 ? Kc : Kr) == KOO) { *err = fs_pass_tma_k<A, V, MODE, KK, KOO>(r, map); return true; }
    if constexpr (MODE == 0) {
        NTT_FSTK(7, 7) NTT_FSTK(8, 7) NTT_FSTK(8, 8) NTT_FSTK(9, 8) NTT_FSTK(9, 9) NTT_FSTK(10, 9) NTT_FSTK(10, 10)
    } else {
        NTT_FSTK(10, 10)
    }
#undef NTT_FSTK
    return false;
    }
}

// (The batch cut into chunks whose pass-A output stays L2-resident until pass B reads it
// measured slower at every chunk size -- 2.81 ms at 96 MiB .. 6.05 ms at 8 MiB against 2.62 ms
// for the whole batch, config 4: each chunk boundary drains and refills the grid, and the
// passes are bound by integer issue, not by DRAM.)
template <class A, int V>
inline cudaError_t fs_run(const MultipassReq& r, int Kr, int Kc) {
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
    a.count_bitrev = V == V_STOCKHAM ? 0 : 1;   // DIT / DIF / Pease_nc sub-transforms bit-reverse; Stockham never
    cudaError_t e = cudaSuccess;
    if (!fs_pass_tma<A, V, 0>(r, Kr, Kc, &e)) e = fstep::fs_pass_any<A, V>(Kr + Kc, 0, a, r.stream, r.num_sms, r.launches);
    if (e != cudaSuccess) return e;
    // pass B: row sub-transforms -> out[k1 + R*k2]
    a.in = static_cast<const uint32_t*>(r.ws);
    a.out = static_cast<uint32_t*>(r.out);
    a.scale = r.scale;
    a.count_bitrev = 0;
    if (fs_pass_tma<A, V, 1>(r, Kr, Kc, &e)) return e;
    return fstep::fs_pass_any<A, V>(Kr + Kc, 1, a, r.stream, r.num_sms, r.launches);
}

// the four-step for one u32 policy (kfs_f32*.cu instantiate it per field)
template <class A>
cudaError_t fourstep_u32_policy(const MultipassReq& r) {
    const int Kr = fourstep_kr(r.L), Kc = r.L - Kr;
    // Flat's per-stage states are DIT's (algorithms.py:161-195): DIT sub-transforms
    if (r.variant == V_DIT || r.variant == V_FLAT) return fs_run<A, V_DIT>(r, Kr, Kc);
    if (r.variant == V_DIF) return fs_run<A, V_DIF>(r, Kr, Kc);
    if (r.variant == V_STOCKHAM) return fs_run<A, V_STOCKHAM>(r, Kr, Kc);
    // Pease: Pease_nc's constant geometry with the stage output copied back (a second work buffer)
    if (r.variant == V_PEASE) return fs_run<A, V_PEASE>(r, Kr, Kc);
    return fs_run<A, V_PEASE_NC>(r, Kr, Kc);
}

}  // namespace nttb200
