// fastclus.cuh -- single-pass transforms too large for one CTA's shared
// memory (u32 2^15 / 2^16, Goldilocks 2^14 .. 2^16): ONE polynomial per
// thread-block CLUSTER of CL = 2^CB CTAs, the exchange between CTAs through
// distributed shared memory (DSMEM), so every residue crosses HBM once (read +
// write) instead of twice for the two-pass four-step.
//
// The dataflows are k_fast's (fast.cuh: DIT, DIF, Pease_nc; Flat runs DIT):
// register groups of <= 4 stages on 16 residues per thread, exchanges through a
// padded shared-memory work buffer.  Each CTA holds N/CL positions: the CB
// "cluster bits" of a position select the CTA, the other L-CB bits are the
// CTA-local index (additive padpos layout over L-CB bits, immediates as in
// k_fast).  The cluster bits must be thread bits (never a register window) in
// every group, so they change exactly once, after group 0 (layout A -> B):
//   * layout A (group 0): natural input index bits [L-4-CB, L-4) = CTA rank --
//     each CTA's share of the input is 16 contiguous runs of 2^(L-4-CB)
//     residues, 16 bulk copies (TMA, mbarrier) into a staging buffer;
//   * layout B (groups 1..G-1): DIT position bits [K0-CB, K0), DIF
//     [L-4, L-4+CB), Pease_nc (rotating frame) the bits that end on output bits
//     [K0-CB, K0); group 0's register index decides the destination CTA of
//     every residue at compile time, so the exchange is ONE round of
//     st.shared::cluster stores (one mapa per destination) between two
//     cluster barriers;
//   * the last group stores straight to HBM (runs of 2^(K0-CB) residues per
//     CTA; the sibling CTAs fill the rest of every sector).
// Stage twiddles: stages <= 13 from a shared-memory copy of the per-stage
// table, later stages through the read-only path (as k_fast at 2^14).
#pragma once
#include <utility>
#include "fast.cuh"

namespace nttb200 {
namespace fastk {

// insert the n low bits of v into x at bit lo / delete bits [lo, lo+n) of x
NTT_HD constexpr uint32_t ins_bits(uint32_t x, uint32_t v, int lo, int n) {
    return ((x >> lo) << (lo + n)) | ((v & ((1u << n) - 1)) << lo) | (x & ((1u << lo) - 1));
}
NTT_HD constexpr uint32_t del_bits(uint32_t x, int lo, int n) {
    return ((x >> (lo + n)) << lo) | (x & ((1u << lo) - 1));
}
NTT_HD constexpr uint32_t brevc(uint32_t x, int n) {
    uint32_t r = 0;
    for (int i = 0; i < n; ++i) r |= ((x >> i) & 1u) << (n - 1 - i);
    return r;
}

template <class F, int... Is>
NTT_D void static_for_(F&& f, std::integer_sequence<int, Is...>) {
    (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, class F>
NTT_D void static_for(F&& f) { static_for_(f, std::make_integer_sequence<int, N>{}); }

NTT_D uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// all threads of all CTAs of the cluster; release / acquire: the DSMEM stores
// issued before it are visible to every CTA after it
NTT_D void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
NTT_D uint32_t mapa_u32(uint32_t a, uint32_t rank) {
    uint32_t o;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(rank));
    return o;
}
template <int OFF>
NTT_D void st_cluster(uint32_t a, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0+%2], %1;" ::"r"(a), "r"(v), "n"(OFF) : "memory");
}
template <int OFF>
NTT_D void st_cluster(uint32_t a, uint64_t v) {
    asm volatile("st.shared::cluster.u64 [%0+%2], %1;" ::"r"(a), "l"(v), "n"(OFF) : "memory");
}

template <class T, int L, int CB>
struct ClusGeo {
    static constexpr int N = 1 << L, CL = 1 << CB;
    static constexpr int LP = L - CB;                  // CTA-local position bits
    static constexpr int TT = 1 << (LP - 4);           // threads per CTA (16 residues each)
    static constexpr int G = (L + 3) / 4, K0 = L - 4 * (G - 1);
    static constexpr int RUN = 1 << (L - 4 - CB);      // contiguous input run per CTA
    static constexpr int LS = L < 13 ? L : 13;         // stages with shared-memory twiddles
    static constexpr int NP = padded_len<T, LP>();
    template <class Tw>
    static constexpr size_t smem() {
        return ((size_t)sizeof(Tw) << LS) + (size_t)(N / CL) * sizeof(T) + (size_t)NP * sizeof(T);
    }
};

template <class A, int V, int L, int CB, bool SC>
__global__ void __launch_bounds__(1 << (L - 4 - CB), 1) k_fastc(FastArgs<A> a) {
    using T = typename A::T;
    using Tw = typename A::Tw;
    using GG = ClusGeo<T, L, CB>;
    constexpr int N = GG::N, LP = GG::LP, TT = GG::TT, G = GG::G, K0 = GG::K0, RUN = GG::RUN, LS = GG::LS;
    constexpr int CL = GG::CL;
    constexpr int CW = lane_bits<T>();
    static_assert(V == V_DIT || V == V_DIF || V == V_PEASE_NC, "cluster dataflows: DIT / DIF / Pease_nc");
    static_assert(CB >= 1 && CB <= K0 && G >= 3, "layout B needs CB <= K0");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t mbar;
    Tw* stw = reinterpret_cast<Tw*>(smem_raw);
    T* S = reinterpret_cast<T*>(smem_raw + ((size_t)sizeof(Tw) << LS));    // staging: [16][RUN]
    T* W = S + N / CL;                                                       // work buffer (local layout)
    const Tw* gstw = a.stw;
    A ar;
    ar.init(a.p);
    const uint32_t t = threadIdx.x;
    const uint32_t rank = cluster_rank();
    const uint64_t cid = blockIdx.x >> CB, ncl = gridDim.x >> CB;

    for (int i = t; i < (1 << LS); i += TT) stw[i] = a.stw[i];
    if (t == 0) { mbar_init(&mbar, 1); fence_mbar_init(); }
    __syncthreads();
    pdl_trigger();
    pdl_wait();
    constexpr uint32_t CTA_BYTES = (uint32_t)(N >> CB) * sizeof(T);
    auto issue = [&](uint64_t poly) {          // this CTA's share: 16 runs of RUN residues
        mbar_expect_tx(&mbar, CTA_BYTES);
        const T* src = a.in + poly * N + ((uint64_t)rank << (L - 4 - CB));
#pragma unroll
        for (int h = 0; h < 16; ++h) tma_load_1d(S + h * RUN, src + ((uint64_t)h << (L - 4)), RUN * sizeof(T), &mbar);
    };
    if (t == 0 && cid < a.batch) issue(cid);
    cluster_sync();                            // every CTA initialised before any DSMEM traffic
    const uint32_t Ws = smem_u32(W);
    uint32_t it = 0;
    for (uint64_t poly = cid; poly < a.batch; poly += ncl, ++it) {
        T v[16];
        T* gout = a.out + poly * N;
        // layout A: natural-index bits [L-4-CB, L-4) of this CTA's residues = rank
        const uint32_t tv = t | (rank << (L - 4 - CB));
        mbar_wait(&mbar, it & 1);
        // ---- group 0 (layout A): gather from the staging runs, butterflies
        uint32_t base_rt;          // runtime part of the layout-B local index of the exchange
        if (V == V_DIT || V == V_PEASE_NC) {
            // bit-reversed gather: natural index brev(c) << (L-4) | tv
#pragma unroll
            for (int c = 0; c < 16; ++c) v[c] = S[(brevc((uint32_t)c, 4) << (L - 4 - CB)) | t];
            if (V == V_DIT) {
                const uint32_t pb0 = brev(tv, L - 4) << 4;
                bitwin_regs<A, L, 0, 0, K0, false, 4, 16, LS>(ar, v, pb0, stw, gstw);
                base_rt = pb0 >> CB;                       // pos = pb0 | c, cluster bits [K0-CB, K0) of c
            } else {
                const uint32_t u0 = brev(tv, L - 4);
                pease_regs<A, L, 0, K0, 4, 16, LS>(ar, v, u0, stw, gstw);
                base_rt = u0 << (4 - K0);                  // wpos = u0 << (4-K0) | n | R << (L-K0)
            }
        } else {
            // DIF: natural order, block [L-4, L) in registers
#pragma unroll
            for (int c = 0; c < 16; ++c) v[c] = S[((uint32_t)c << (L - 4 - CB)) | t];
            bitwin_regs<A, L, L - 4, L - 4, 4, true, 4, 16, LS>(ar, v, tv, stw, gstw);
            base_rt = tv;                                  // pos = tv | c << (L-4)
        }
        // every CTA is past the previous row's last-group reads and this CTA's
        // staging is consumed: prefetch the next row, exchange into layout B
        cluster_sync();
        if (t == 0 && poly + ncl < a.batch) {
            fence_proxy_async();
            issue(poly + ncl);
        }
        {
            uint32_t dst[CL];
#pragma unroll
            for (int d = 0; d < CL; ++d) dst[d] = mapa_u32(Ws + padpos<T>(base_rt) * (uint32_t)sizeof(T), (uint32_t)d);
            static_for<16>([&](auto ic) {
                constexpr int c = decltype(ic)::value;
                constexpr uint32_t uc = (uint32_t)c;
                // destination CTA and the register part of the layout-B local index
                constexpr uint32_t dcta = V == V_DIT ? ((uc >> (K0 - CB)) & (CL - 1))
                                        : V == V_DIF ? (uc & (CL - 1))
                                                     : ((uc & ((1u << K0) - 1)) >> (K0 - CB));
                constexpr uint32_t loc = V == V_DIT ? del_bits(uc, K0 - CB, CB)
                                       : V == V_DIF ? ((uc >> CB) << (L - 4))
                                                    : ((uc >> K0) | ((uc & ((1u << (K0 - CB)) - 1)) << (L - K0)));
                constexpr int off = (int)(padpos<T>(loc) * sizeof(T));
                st_cluster<off>(dst[dcta], v[c]);
            });
        }
        cluster_sync();                        // every residue is in its layout-B CTA
        // ---- groups 1 .. G-1 (layout B, CTA-local)
        static_for<G - 1>([&](auto ig) {
            constexpr int g = decltype(ig)::value + 1;
            constexpr bool last = g == G - 1;
            if constexpr (V == V_DIT) {
                constexpr int B = K0 + 4 * (g - 1), Bl = B - CB;          // window (global / local)
                uint32_t pl;
                if constexpr (last) pl = t;
                else {
                    constexpr Perm PM = plan_lanes(LP, Bl, CW);
                    pl = scatter_bits<LP - 4>(t, PM);
                }
                const uint32_t pbase = ins_bits(pl, rank, K0 - CB, CB);
                T* wb = W + padpos<T>(pl);
#pragma unroll
                for (int c = 0; c < 16; ++c) v[c] = wb[padpos<T>((uint32_t)c << Bl)];
                bitwin_regs<A, L, B, B, 4, false, 4, 16, LS>(ar, v, pbase, stw, gstw);
                if constexpr (!last) {
#pragma unroll
                    for (int c = 0; c < 16; ++c) wb[padpos<T>((uint32_t)c << Bl)] = v[c];
                    __syncthreads();
                } else {
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        T r = ar.fin(v[c]);
                        if (SC) r = ar.mulc(r, a.ninv);
                        gout[pbase | ((uint32_t)c << (L - 4))] = r;
                    }
                }
            } else if constexpr (V == V_DIF) {
                constexpr int B = last ? 0 : L - 4 * (g + 1);              // below the cluster bits
                constexpr int kg = last ? K0 : 4;
                uint32_t pl;
                if constexpr (last) pl = brev(t, LP - 4) << 4;
                else {
                    constexpr Perm PM = plan_lanes(LP, B, CW);
                    pl = scatter_bits<LP - 4>(t, PM);
                }
                const uint32_t pbase = ins_bits(pl, rank, L - 4, CB);
                T* wb = W + padpos<T>(pl);
#pragma unroll
                for (int c = 0; c < 16; ++c) v[c] = wb[padpos<T>((uint32_t)c << B)];
                bitwin_regs<A, L, B, B, kg, true, 4, 16, LS>(ar, v, pbase, stw, gstw);
                if constexpr (!last) {
#pragma unroll
                    for (int c = 0; c < 16; ++c) wb[padpos<T>((uint32_t)c << B)] = v[c];
                    __syncthreads();
                } else {
                    // output index brev_L(pbase | c)
                    const uint32_t ob = brev(pbase, L);
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        T r = ar.fin(v[c]);
                        if (SC) r = ar.mulc(r, a.ninv);
                        gout[ob | (brevc((uint32_t)c, 4) << (L - 4))] = r;
                    }
                }
            } else {   // Pease_nc: constant geometry, rotating frame
                constexpr int sg = K0 + 4 * (g - 1);
                constexpr int ub = L - CB - 4 * (g - 1) - 4;                 // cluster bits in u
                const uint32_t u = ins_bits(t, rank, ub, CB);
                const T* rb = W + padpos<T>(t << 4);
#pragma unroll
                for (int c = 0; c < 16; ++c) v[c] = rb[padpos<T>((uint32_t)c)];
                pease_regs<A, L, sg, 4, 4, 16, LS>(ar, v, u, stw, gstw);
                if constexpr (!last) {
                    __syncthreads();           // every read of the single work buffer done
                    T* wo = W + padpos<T>(t);
#pragma unroll
                    for (int c = 0; c < 16; ++c) wo[padpos<T>((uint32_t)c << (LP - 4))] = v[c];
                    __syncthreads();
                } else {
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        T r = ar.fin(v[c]);
                        if (SC) r = ar.mulc(r, a.ninv);
                        gout[u | ((uint32_t)c << (L - 4))] = r;
                    }
                }
            }
        });
        if (a.counters && t == 0 && rank == 0) {
            atomicAdd(a.counters + C_TRANSFORMS, 1ull);
            atomicAdd(a.counters + C_HBM, 1ull);
            atomicAdd(a.counters + C_BITREV, 1ull);
        }
    }
    cluster_sync();                            // no CTA exits while a sibling may still store into it
}

template <class A, int V, int L, int CB>
cudaError_t launch_fastc(const FastArgs<A>& a, cudaStream_t s, int* launches, bool* ok) {
    using T = typename A::T;
    using GG = ClusGeo<T, L, CB>;
    constexpr size_t smem = GG::template smem<typename A::Tw>();
    auto kern = a.scale ? k_fastc<A, V, L, CB, true> : k_fastc<A, V, L, CB, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(GG::TT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = GG::CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // co-resident clusters (a persistent grid: each cluster loops over rows)
    static int max_clusters = 0;
    if (max_clusters == 0) {
        cfg.gridDim = dim3(GG::CL * 256);
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n < 1) n = 1;
        max_clusters = n;
    }
    cfg.numAttrs = 2;
    const uint64_t nc = a.batch < (uint64_t)max_clusters ? a.batch : (uint64_t)max_clusters;
    *ok = true;
    if (nc == 0) return cudaSuccess;
    cfg.gridDim = dim3((unsigned)(nc * GG::CL));
    e = cudaLaunchKernelEx(&cfg, kern, a);
    if (launches) ++*launches;
    return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace fastk
}  // namespace nttb200
