// fourstep_tma.cuh -- pass A of the four-step (fourstep.cuh) with TMA tile loads.
//
// Pass A gathers TQ = 8 columns x R = 1024 rows: 32-byte runs 4 KiB apart.
// Issued as 4-byte cp.async per residue this is bound by the SM's load path
// (measured: loads alone 1.13 ms per 2 GiB pass vs 0.52 ms for contiguous
// rows).  Here the tile is ONE tensor-map box stream: 4 cp.async.bulk.tensor
// 2-D loads of [256 rows][8 columns] per tile, issued by one thread into a
// dense, double-buffered staging area (the tile after next is in flight
// while the current one computes), completion on an mbarrier.
//
// The first register group reads the dense staging with the tile-major thread
// map (lanes = 8 columns x 4 rows that differ in their low 2 bits: 32 distinct
// banks), the middle group keeps the network-major map, the last group the
// tile-major map again; network stride NP and the in-warp position bits per
// variant were chosen by an exhaustive bank model:
//   DIT (groups 2,4,4):      NP = 1 (mod 32); group 0 lanes -> positions 8,9, last -> 3,4
//   Pease_nc (groups 4,4,2): NP = 2 (mod 32); group 0 lanes -> positions 8,9, last -> 4,5
#pragma once
#include <cuda.h>
#include "fourstep.cuh"

namespace nttb200 {
namespace fstep {

template <class A>
struct FsTmaArgs {
    using T = typename A::T;
    using Tw = typename A::Tw;
    const T* in;               // MODE 1: the workspace rows (MODE 0 reads through the tensor map)
    T* out;
    uint64_t batch;
    int Kr, Kc;                // R = 2^Kr rows, C = 2^Kc columns; the sub-transform is 2^10 long
    int scale;                 // MODE 1: n^-1 (intt)
    Tw ninv;
    const Tw* stw;
    const Tw* twist;           // [k1][n2] = w_N^(k1*n2)
    const Tw* tw_main;         // w_N^i (factored twist)
    uint64_t p;
    int count_bitrev;
    unsigned long long* counters;
};

NTT_D void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            fastk::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(fastk::smem_u32(bar))
        : "memory");
}

// Geometry per (variant, sub-transform length 2^K), NT = 512 threads:
//   TQ = 2^(13-K) networks per tile (every tile holds 8192 residues), AB =
//   in-warp thread bits above the network id.  Group splits: DIT (K0, 4, ...),
//   Pease (4, ..., K0).  NP / in-warp bit placements from the exhaustive bank
//   model:
//     K = 10 (AB = 2): DIT NP = 1, group-0 lanes -> u bits 4,5, last -> 3,4;
//                      Pease NP = 2, group 0 -> 4,5, last -> 0,1;
//     K = 9  (AB = 1): DIT NP = 1 with network base + 8*(q >> 3), group 0 -> u4, last -> u3;
//                      Pease NP = 1, group 0 -> u4, last -> u0;
//     K <= 8 (AB = 0): a warp is 32 networks: NP = 1.
template <int V, int K>
struct TmaGeo {
    static constexpr int TQ = 1 << (13 - K), NT = 512, TT = 1 << (K - 4);
    static constexpr int LQ = 13 - K;
    static constexpr int AB = LQ >= 5 ? 0 : 5 - LQ;
    static constexpr int G = (K + 3) / 4;
    static constexpr int K0 = K - 4 * (G - 1);
    static constexpr int KG0 = (V == V_DIT) ? K0 : 4;
    static constexpr int KGL = (V == V_DIT) ? 4 : K0;
    static constexpr int NPM = (K == 10 && V != V_DIT) ? 2 : 1;       // network stride mod 32
    static constexpr bool NLIN = (K == 9 && V == V_DIT);              // base(q) = q*NP + 8*(q >> 3)
    // (the +8 only where the non-linear base needs it: at K = 10 the 32 words saved per
    // network are what lets a third 512-thread CTA fit the SM's shared memory)
    static constexpr int NP = ((fastk::padded_len<uint32_t, K>() + (NLIN ? 8 : 0) + 31) / 32) * 32 + NPM;
    static constexpr int I0a = 4, I0b = 5;                            // group-0 in-warp -> u bits
    static constexpr int ILa = (V == V_DIT) ? (K == 10 ? 3 : 3) : 0;  // last group
    static constexpr int ILb = (V == V_DIT) ? 4 : 1;
    static NTT_HD constexpr uint32_t base(uint32_t q) { return q * NP + (NLIN ? 8 * (q >> 3) : 0); }
};

// u (K-4 bits) from w = tid >> LQ: w's AB low (in-warp) bits on u bits ia (, ib), the rest in order
template <int UB, int AB, int ia, int ib>
NTT_D uint32_t placeN(uint32_t w) {
    if (AB == 0) return w;
    uint32_t u = (w & 1u) << ia;
    if (AB == 2) u |= ((w >> 1) & 1u) << ib;
    uint32_t rest = w >> AB;
#pragma unroll
    for (int b = 0; b < UB; ++b) {
        if (b == ia || (AB == 2 && b == ib)) continue;
        u |= (rest & 1u) << b;
        rest >>= 1;
    }
    return u;
}

#ifndef NTT_FS_BOUNDED
#define NTT_FS_BOUNDED 1       // DIT first groups: bounded stage-1/2 forms and w^0 butterflies without a multiply
                               // (config 4 DIT 2.59 -> 2.49 ms)
#endif
#ifndef NTT_FSA_TWF
#define NTT_FSA_TWF 1          // factored twist (per-tile [c][t] table in shared memory + one w^(n2 u) per thread)
#endif
// MODE 1 staging rows are skewed by 4 words (tile-major reads: 8 rows x 4 residues hit 32 banks)
constexpr int kStgRow = 1024 + 4;
// staging buffers per CTA: 2 = the tile after next in flight (2 CTAs / SM),
// 1 = the next tile issued once group 0 has read the current one (then 3 CTAs / SM,
// 40 registers): config 4 Pease_nc 2.70 -> 2.56 ms, 2^15..2^20 sweep +3..7 %,
// DIT unchanged (measured A/B, tools/time_case.py / tools/sweep.py)
#ifndef NTT_FSA_STAGES
#define NTT_FSA_STAGES 1
#endif
constexpr int kFsaStages = NTT_FSA_STAGES;
// CTAs per SM the register budget is cut for: 3 (40 registers) or 2 (ptxas takes 48).  Shared
// memory admits 3 everywhere but Pease (two work buffers); measured per geometry (tools/sweep.py,
// tools/time_case.py, 2 x interleaved, r2 session 5), 2 vs 3 CTAs: K <= 8 (2^15, 2^16) -2..-5 % for
// DIT and Pease_nc alike; K = 9: Pease_nc -4 % at 2^17, DIT +1.6 %; K = 10: Pease_nc -3 % on
// config 4 (2^10 x 2^10) but +2.3 % at 2^19 (2^10 x 2^9), DIT flat; Pease -0.5..-1 % everywhere
#ifndef NTT_FSA_MINB
#define NTT_FSA_MINB 0          // 2 / 3: force; 0: the measured table below
#endif
template <int V, int K, int KO>
constexpr int fsa_minb() {
    if (NTT_FSA_MINB) return NTT_FSA_MINB;
    if (kFsaStages != 1 || V == V_PEASE || K <= 8) return 2;
    if (V == V_PEASE_NC) return (K == 9 || KO == 10) ? 2 : 3;
    return 3;
}
template <int V, int K, int MODE>
constexpr size_t fsa_smem_bytes() {
    using GG = TmaGeo<V, K>;
    // (Pease: a second work buffer -- the stage output that is copied back, algorithms.py:242)
    return ((size_t)8 << K) + kFsaStages * (size_t)(MODE == 0 ? 8192 : 8 * kStgRow) * 4 +
           (V == V_PEASE ? 2 : 1) * (size_t)((GG::base(GG::TQ) + 1) & ~1u) * 4 + 8 + 16 * (size_t)GG::TQ * 8;
}

// per-CTA phase clocks (tools/fs_timeline.py; experiment builds only): thread 0 sums clock64()
// deltas between the phase boundaries of every tile it processes
#ifdef NTT_FS_TIMELINE
static __device__ unsigned long long g_fstl[2][1024][8];
#define NTT_FSTL(k)                                            \
    if (tid == 0) {                                            \
        const long long now_ = clock64();                      \
        tl_acc[k] += (unsigned long long)(now_ - tl_last);     \
        tl_last = now_;                                        \
    }
#else
#define NTT_FSTL(k) ((void)0)
#endif

NTT_D void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     fastk::smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(fastk::smem_u32(bar))
                 : "memory");
}

// MODE 0: pass A (columns, tensor-map box loads, twist, rows k1 of the workspace), 7 <= K <= 10
// MODE 1: pass B (rows of the workspace by 1-D bulk copies, out[k1 + R*k2]), K = 10
// KO = log2 of the other dimension (C for MODE 0, R for MODE 1), compile time so
// every strided store / twist offset is an immediate
template <class A, int V, int MODE, int K, int KO>
__global__ void __launch_bounds__(512, fsa_minb<V, K, KO>()) k_fs_tma(const __grid_constant__ CUtensorMap tmap, FsTmaArgs<A> a) {
    using T = typename A::T;
    using Tw = typename A::Tw;
    using GG = TmaGeo<V, K>;
    static_assert(MODE == 0 || K == 10, "bulk-row pass B: 2^10 rows");
    constexpr int TQ = GG::TQ, NT = GG::NT, TT = GG::TT, LQ = GG::LQ, AB = GG::AB, G = GG::G, K0 = GG::K0;
    constexpr int UB = K - 4;
    constexpr int CW = fastk::lane_bits<T>();
    constexpr int kIn = !NTT_FS_BOUNDED ? 0 : MODE == 0 ? 1 : ((NTT_FSA_TWF && A::lazy) ? 2 : 1);   // value range of a pass's input
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t mbar[2];
    Tw* tws = reinterpret_cast<Tw*>(smem_raw);                           // 2^K stage twiddles
    T* stg = reinterpret_cast<T*>(smem_raw + ((size_t)8 << K));          // 2 staging tiles
    constexpr int STG = MODE == 0 ? 8192 : 8 * kStgRow;                  // MODE 0 [2^K][TQ], MODE 1 [8][kStgRow]
    constexpr int NST = kFsaStages;
    T* W = stg + NST * STG;                                              // TQ networks at GG::base(q)
    constexpr uint32_t WLEN = (GG::base(TQ) + 1) & ~1u;
    // Pease: groups write the stage output to W2 and copy it back into W (_stage_copy,
    // algorithms.py:242); Pease_nc writes W itself after a barrier (no copy)
    T* W2 = V == V_PEASE ? W + WLEN : W;
    Tw* twB = reinterpret_cast<Tw*>(W2 + WLEN);                          // factored twist [c][q]
    A ar;
    ar.init(a.p);
    const uint32_t tid = threadIdx.x;
    auto copy_back = [&]() {
        __syncthreads();
        for (uint32_t i = tid; i < WLEN; i += NT) W[i] = W2[i];
    };
    for (uint32_t i = tid; i < (1u << K); i += NT) tws[i] = a.stw[i];
    constexpr int Kr = MODE == 0 ? K : KO, Kc = MODE == 0 ? KO : K;
    constexpr uint64_t N = 1ull << (Kr + Kc);
    constexpr int tpp_log = (MODE == 0 ? Kc : Kr) - LQ;   // tiles per polynomial = (C or R) / TQ
    const uint64_t ntiles = a.batch << tpp_log;
    constexpr uint32_t TILE_BYTES = 8192 * 4;
    constexpr int BROWS = K >= 8 ? 256 : (1 << K);        // rows per tensor box
    auto issue = [&](uint64_t tl, int s) {
        fastk::mbar_expect_tx(&mbar[s], TILE_BYTES);
        if (MODE == 0) {                             // boxes of [BROWS rows][TQ cols]
            const int x = (int)((tl & ((1ull << tpp_log) - 1)) * TQ);
            const int y = (int)((tl >> tpp_log) << K);
#pragma unroll
            for (int j = 0; j < (1 << K) / BROWS; ++j)
                tma_load_2d(stg + s * STG + j * BROWS * TQ, &tmap, x, y + BROWS * j, &mbar[s]);
        } else {                                     // 8 rows of 4 KiB
            const T* src = a.in + (tl >> tpp_log) * N + (((tl & ((1ull << tpp_log) - 1)) * 8) << 10);
#pragma unroll
            for (int j = 0; j < 8; ++j) bulk_load(stg + s * STG + j * kStgRow, src + j * 1024, 4096, &mbar[s]);
        }
    };
    if (tid == 0) {
        fastk::mbar_init(&mbar[0], 1);
        fastk::mbar_init(&mbar[1], 1);
        fastk::fence_mbar_init();
    }
    __syncthreads();
    fastk::pdl_trigger();
    fastk::pdl_wait();                       // the previous launch's output (our input) is visible
    if (tid == 0) {
        if ((uint64_t)blockIdx.x < ntiles) issue(blockIdx.x, 0);
        if (NST == 2 && (uint64_t)blockIdx.x + gridDim.x < ntiles) issue(blockIdx.x + gridDim.x, 1);
    }
    const uint32_t q = tid & (TQ - 1), w = tid >> LQ;
    // output position of last-group register c (natural order): a(u) + b(c)
    auto bpart = [](int c) -> uint32_t {
        if (V == V_DIT) return (uint32_t)c << (K - 4);
        return ((uint32_t)c >> GG::KGL) | (((uint32_t)c & ((1u << GG::KGL) - 1)) << (K - GG::KGL));
    };
    auto apart = [](uint32_t u) -> uint32_t { return V == V_DIT ? u : (u << (4 - GG::KGL)); };
    int it = 0;
#ifdef NTT_FS_TIMELINE
    __shared__ unsigned long long tl_acc[8];
    long long tl_last = clock64();
    if (tid == 0)
        for (int k = 0; k < 8; ++k) tl_acc[k] = 0;
#endif
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int s = NST == 2 ? (it & 1) : 0;
        const T* S = stg + s * STG;
        // staging base of this thread's network (the position part added as an immediate)
        const T* Sq = S + (MODE == 0 ? q : q * kStgRow);
        auto sidx = [&](uint32_t x) -> uint32_t { return MODE == 0 ? x * TQ : x; };
        T v[16];
        // ---- group 0 (tile-major): read the dense staging, write the work buffer
        const uint32_t u0 = placeN<UB, AB, GG::I0a, GG::I0b>(w);
        const uint32_t rb = brev(u0 << 4, K);                 // input index of position u0 << 4
        NTT_FSTL(0);                          // previous tile's stores retired from the issue side
        fastk::mbar_wait(&mbar[s], NST == 2 ? ((it >> 1) & 1) : (it & 1));
        NTT_FSTL(1);                          // tile landed
#pragma unroll
        for (int c = 0; c < 16; ++c) v[c] = Sq[sidx(rb) + sidx(brev((uint32_t)c, 4) << (K - 4))];
        if (V == V_DIT) {
            // block [0,4): positions u0 << 4 | c
            const uint32_t pbase = u0 << 4;
            // (pass A reads caller data: canonical; pass B the lazy twist's outputs in [0,2p))
            ftile::t_bitwin<A, K, 0, 0, GG::KG0, false, false, kIn>(ar, v, pbase, 0u, 0, tws);
            __syncthreads();                  // staging consumed; previous tile's last group done with W
            T* wb = W + GG::base(q) + padpos<T>(pbase);
#pragma unroll
            for (int c = 0; c < 16; ++c) wb[padpos<T>((uint32_t)c)] = v[c];
        } else {
            ftile::t_pease<A, K, 0, GG::KG0, false>(ar, v, u0, 0u, 0, tws);
            __syncthreads();
            T* wbo = W2 + GG::base(q) + padpos<T>(u0 << (4 - GG::KG0));
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                const uint32_t n = c >> GG::KG0, Rb = c & ((1u << GG::KG0) - 1);
                wbo[padpos<T>(n | (Rb << (K - GG::KG0)))] = v[c];
            }
            if (V == V_PEASE) copy_back();
        }
        NTT_FSTL(2);                          // group 0: staging reads, butterflies, barrier, work-buffer writes
        // factored twist of the last group: w^(k1 n2) = w^(n2 a(u)) * w^(n2 b(c)), k1 = a(u) + b(c)
        Tw twA;
        const uint32_t uL = placeN<UB, AB, GG::ILa, GG::ILb>(w);
        if (MODE == 0 && NTT_FSA_TWF) {
            const uint64_t col0 = (tile & ((1ull << tpp_log) - 1)) * TQ;
#pragma unroll
            for (uint32_t i = tid; i < 16 * TQ; i += NT) {
                const uint32_t c = i / TQ, t = i % TQ;
                twB[i] = __ldg(a.tw_main + (col0 + t) * bpart((int)c));
            }
            twA = __ldg(a.tw_main + (col0 + q) * apart(uL));
        }
        if (tid == 0) {                       // staging s is free: the tile NST launches ahead
            const uint64_t nn = tile + NST * (uint64_t)gridDim.x;
            if (nn < ntiles) {
                fastk::fence_proxy_async();
                issue(nn, s);
            }
        }
        __syncthreads();
        NTT_FSTL(3);                          // twist factors, next tile issued, barrier
        // ---- middle groups (network-major)
#pragma unroll
        for (int g = 1; g < G - 1; ++g) {
            const uint32_t t = tid >> (K - 4), u = tid & (TT - 1);
            T* sb = W + GG::base(t);
            if (V == V_DIT) {
                const int B = K0 + 4 * (g - 1);
                uint32_t pbase = 0;
#define NTT_TMAP(BB)                                \
    if (B == BB) {                                  \
        constexpr Perm PM = plan_lanes(K, BB, CW);  \
        pbase = scatter_bits<K - 4>(u, PM);         \
    }
                NTT_TMAP(1) NTT_TMAP(2) NTT_TMAP(3) NTT_TMAP(4) NTT_TMAP(5)
#undef NTT_TMAP
                T* wb = sb + padpos<T>(pbase);
#pragma unroll
                for (int c = 0; c < 16; ++c) v[c] = wb[padpos<T>((uint32_t)c << B)];
#define NTT_TBWM(BB) \
    if (B == BB) ftile::t_bitwin<A, K, BB, BB, 4, false, false>(ar, v, pbase, 0u, 0, tws);
                NTT_TBWM(1) NTT_TBWM(2) NTT_TBWM(3) NTT_TBWM(4) NTT_TBWM(5)
#undef NTT_TBWM
#pragma unroll
                for (int c = 0; c < 16; ++c) wb[padpos<T>((uint32_t)c << B)] = v[c];
            } else {
                const int sg = 4 * g;
                const T* rbp = sb + padpos<T>(u << 4);
#pragma unroll
                for (int c = 0; c < 16; ++c) v[c] = rbp[padpos<T>((uint32_t)c)];
#define NTT_TPEM(SG) \
    if (sg == SG) ftile::t_pease<A, K, SG, 4, false>(ar, v, u, 0u, 0, tws);
                NTT_TPEM(4) NTT_TPEM(8)
#undef NTT_TPEM
                if (V != V_PEASE) __syncthreads();   // every read of the single work buffer done
                T* wbo = (V == V_PEASE ? W2 + GG::base(t) : sb) + padpos<T>(u);
#pragma unroll
                for (int c = 0; c < 16; ++c) wbo[padpos<T>((uint32_t)c << (K - 4))] = v[c];
                if (V == V_PEASE) copy_back();
            }
            __syncthreads();
        }
        NTT_FSTL(4);                          // middle groups
        // ---- last group (tile-major) -> twist -> workspace rows k1 / outputs
        {
            const uint32_t u = uL;
            const T* sb = W + GG::base(q);
            const uint64_t col = (tile & ((1ull << tpp_log) - 1)) * TQ + q;
            if (V == V_DIT) {
                const T* wb = sb + padpos<T>(u);
#pragma unroll
                for (int c = 0; c < 16; ++c) v[c] = wb[padpos<T>((uint32_t)c << (K - 4))];
                ftile::t_bitwin<A, K, K - 4, K - 4, 4, false, false>(ar, v, u, 0u, 0, tws);
            } else {
                const T* rbp = sb + padpos<T>(u << 4);
#pragma unroll
                for (int c = 0; c < 16; ++c) v[c] = rbp[padpos<T>((uint32_t)c)];
                ftile::t_pease<A, K, K - GG::KGL, GG::KGL, false>(ar, v, u, 0u, 0, tws);
            }
            NTT_FSTL(5);                      // last group: reads + butterflies
            const uint32_t au = apart(u);
            T* dst = a.out + (tile >> tpp_log) * N + col;    // MODE 0: column n2; MODE 1: row k1
            if (MODE == 0) {
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    const uint64_t ro = (uint64_t)(au + bpart(c)) << Kc;
                    if (NTT_FSA_TWF) dst[ro] = ar.mull(ar.mull(v[c], ftile::lds_tw(&twB[c * TQ + q])), twA);
                    else dst[ro] = ar.mulc(v[c], __ldg(a.twist + col + ro));
                }
            } else if (a.scale) {
#pragma unroll
                for (int c = 0; c < 16; ++c) dst[(uint64_t)(au + bpart(c)) << Kr] = ar.mulc(v[c], a.ninv);
            } else {
#pragma unroll
                for (int c = 0; c < 16; ++c) dst[(uint64_t)(au + bpart(c)) << Kr] = ar.fin(v[c]);
            }
        }
        NTT_FSTL(6);                          // twist + stores issued
        if (a.counters && tid == 0 && (tile & ((1ull << tpp_log) - 1)) == 0) {
            atomicAdd(a.counters + C_HBM, 1ull);
            if (MODE == 1) atomicAdd(a.counters + C_TRANSFORMS, 1ull);
            if (V == V_PEASE) atomicAdd(a.counters + C_COPIES, (unsigned long long)(G - 1));
            if (a.count_bitrev) atomicAdd(a.counters + C_BITREV, (unsigned long long)a.count_bitrev);
        }
    }
#ifdef NTT_FS_TIMELINE
    if (tid == 0 && blockIdx.x < 1024) {
        for (int k = 0; k < 7; ++k) g_fstl[MODE][blockIdx.x][k] = tl_acc[k];
        g_fstl[MODE][blockIdx.x][7] = (unsigned long long)it;
    }
#endif
}

}  // namespace fstep
}  // namespace nttb200
