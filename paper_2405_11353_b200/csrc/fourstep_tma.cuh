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

template <int V>
struct TmaGeo {
    static constexpr int K = 10, TQ = 8, NT = 512, TT = 64;
    static constexpr int NPM = (V == V_DIT) ? 1 : 2;                  // network stride mod 32
    static constexpr int NP = ((fastk::padded_len<uint32_t, K>() + 31) / 32) * 32 + NPM;
    // group split: DIT (2,4,4), Pease (4,4,2)
    static constexpr int KG0 = (V == V_DIT) ? 2 : 4;
    static constexpr int KGL = (V == V_DIT) ? 4 : 2;
    static constexpr int I0a = 4, I0b = 5;                            // group-0 in-warp bits -> u bits
    static constexpr int ILa = (V == V_DIT) ? 3 : 0, ILb = (V == V_DIT) ? 4 : 1;   // last group
};

// u (6 bits) from w = tid >> 3 with w bits 0,1 (in-warp) on u bits ia, ib
template <int ia, int ib>
NTT_D uint32_t place2(uint32_t w) {
    uint32_t u = ((w & 1u) << ia) | (((w >> 1) & 1u) << ib);
    uint32_t rest = w >> 2;
#pragma unroll
    for (int b = 0; b < 6; ++b) {
        if (b == ia || b == ib) continue;
        u |= (rest & 1u) << b;
        rest >>= 1;
    }
    return u;
}

#ifndef NTT_FSA_TWF
#define NTT_FSA_TWF 1          // factored twist (per-tile [c][t] table in shared memory + one w^(n2 u) per thread)
#endif
// MODE 1 staging rows are skewed by 4 words (tile-major reads: 8 rows x 4 residues hit 32 banks)
constexpr int kStgRow = 1024 + 4;
constexpr size_t fsa_smem_bytes(int NP) {
    return (size_t)8 * 1024 + 2 * (size_t)8 * kStgRow * 4 + (size_t)8 * NP * 4 + 16 * 8 * 8;
}

NTT_D void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     fastk::smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(fastk::smem_u32(bar))
                 : "memory");
}

// MODE 0: pass A (columns, tensor-map box loads, twist, rows k1 of the workspace)
// MODE 1: pass B (rows of the workspace by 1-D bulk copies, out[k1 + R*k2])
// KO = log2 of the other dimension (C for MODE 0, R for MODE 1), compile time so
// every strided store / twist offset is an immediate
template <class A, int V, int MODE, int KO>
__global__ void __launch_bounds__(512, 2) k_fs_tma(const __grid_constant__ CUtensorMap tmap, FsTmaArgs<A> a) {
    using T = typename A::T;
    using Tw = typename A::Tw;
    using GG = TmaGeo<V>;
    constexpr int K = GG::K, TQ = GG::TQ, NT = GG::NT, TT = GG::TT, NP = GG::NP;
    constexpr int CW = fastk::lane_bits<T>();
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t mbar[2];
    Tw* tws = reinterpret_cast<Tw*>(smem_raw);                           // 2^10 stage twiddles
    T* stg = reinterpret_cast<T*>(smem_raw + 8 * 1024);                  // 2 staging tiles
    constexpr int STG = MODE == 0 ? 8 * 1024 : 8 * kStgRow;              // MODE 0 [1024][8], MODE 1 [8][kStgRow]
    T* W = stg + 2 * STG;                                                // [8][NP] work buffer
    Tw* twB = reinterpret_cast<Tw*>(W + 8 * NP);                          // factored twist [c][q] (8 * NP * 4 bytes: 8-aligned)
    A ar;
    ar.init(a.p);
    const uint32_t tid = threadIdx.x;
    for (uint32_t i = tid; i < 1024; i += NT) tws[i] = a.stw[i];
    constexpr int Kr = MODE == 0 ? 10 : KO, Kc = MODE == 0 ? KO : 10;
    constexpr uint64_t N = 1ull << (Kr + Kc);
    constexpr int tpp_log = (MODE == 0 ? Kc : Kr) - 3;   // tiles per polynomial = (C or R) / 8
    const uint64_t ntiles = a.batch << tpp_log;
    constexpr uint32_t TILE_BYTES = 8 * 1024 * 4;
    auto issue = [&](uint64_t tl, int s) {
        fastk::mbar_expect_tx(&mbar[s], TILE_BYTES);
        if (MODE == 0) {                             // 4 boxes of [256 rows][8 cols]
            const int x = (int)((tl & ((1ull << tpp_log) - 1)) * 8);
            const int y = (int)((tl >> tpp_log) << 10);
#pragma unroll
            for (int j = 0; j < 4; ++j) tma_load_2d(stg + s * STG + j * 2048, &tmap, x, y + 256 * j, &mbar[s]);
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
        if ((uint64_t)blockIdx.x + gridDim.x < ntiles) issue(blockIdx.x + gridDim.x, 1);
    }
    const uint32_t q = tid & 7, w = tid >> 3;
    int it = 0;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int s = it & 1;
        const T* S = stg + s * STG;
        // staging element (input index x, network q)
        // staging base of this thread's network (the position part added as an immediate)
        const T* Sq = S + (MODE == 0 ? q : q * kStgRow);
        auto sidx = [&](uint32_t x) -> uint32_t { return MODE == 0 ? x * 8 : x; };
        T v[16];
        // ---- group 0 (tile-major): read the dense staging, write the work buffer
        uint32_t u0;
        if (V == V_DIT) u0 = place2<GG::I0a, GG::I0b>(w);
        else u0 = place2<GG::I0a, GG::I0b>(w);
        fastk::mbar_wait(&mbar[s], (it >> 1) & 1);
        if (V == V_DIT) {
            // block [0,4): positions u0 << 4 | c, input row brev10(position)
            const uint32_t pbase = u0 << 4;
            const uint32_t rb = brev(pbase, K);
#pragma unroll
            for (int c = 0; c < 16; ++c) v[c] = Sq[sidx(rb) + sidx(brev((uint32_t)c, 4) << 6)];
            ftile::t_bitwin<A, K, 0, 0, GG::KG0, false, false>(ar, v, pbase, 0u, 0, tws);
            __syncthreads();                  // staging consumed; previous tile's last group done with W
            T* wb = W + q * NP + padpos<T>(pbase);
#pragma unroll
            for (int c = 0; c < 16; ++c) wb[padpos<T>((uint32_t)c)] = v[c];
        } else {
            const uint32_t rb = brev(u0 << 4, K);
#pragma unroll
            for (int c = 0; c < 16; ++c) v[c] = Sq[sidx(rb) + sidx(brev((uint32_t)c, 4) << 6)];
            ftile::t_pease<A, K, 0, GG::KG0, false>(ar, v, u0, 0u, 0, tws);
            __syncthreads();
            T* wbo = W + q * NP + padpos<T>(u0 << (4 - GG::KG0));
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                const uint32_t n = c >> GG::KG0, Rb = c & ((1u << GG::KG0) - 1);
                wbo[padpos<T>(n | (Rb << (K - GG::KG0)))] = v[c];
            }
        }
        // factored twist of the last group: w^(k1 n2) = w^(n2 * a(u)) * w^(n2 * b(c)), k1 = a(u) + b(c)
        Tw twA;
        if (MODE == 0 && NTT_FSA_TWF) {
            const uint64_t col0 = (tile & ((1ull << tpp_log) - 1)) * 8;
            if (tid < 128) {
                const uint32_t c = tid >> 3, t = tid & 7;
                const uint32_t bc = (V == V_DIT) ? (c << 6) : ((c >> 2) | ((c & 3u) << 8));
                twB[tid] = __ldg(a.tw_main + (col0 + t) * bc);
            }
            const uint32_t uL = place2<GG::ILa, GG::ILb>(w);
            const uint32_t au = (V == V_DIT) ? uL : (uL << 2);
            twA = __ldg(a.tw_main + (col0 + q) * au);
        }
        if (tid == 0) {                       // staging s is free: the tile after next
            const uint64_t nn = tile + 2 * (uint64_t)gridDim.x;
            if (nn < ntiles) {
                fastk::fence_proxy_async();
                issue(nn, s);
            }
        }
        __syncthreads();
        // ---- middle group (network-major)
        {
            const uint32_t t = tid >> 6, u = tid & (TT - 1);
            T* sb = W + t * NP;
            if (V == V_DIT) {
                constexpr int B = 2;
                constexpr Perm PM = plan_lanes(K, B, CW);
                const uint32_t pbase = scatter_bits<K - 4>(u, PM);
                T* wb = sb + padpos<T>(pbase);
#pragma unroll
                for (int c = 0; c < 16; ++c) v[c] = wb[padpos<T>((uint32_t)c << B)];
                ftile::t_bitwin<A, K, B, B, 4, false, false>(ar, v, pbase, 0u, 0, tws);
#pragma unroll
                for (int c = 0; c < 16; ++c) wb[padpos<T>((uint32_t)c << B)] = v[c];
            } else {
                constexpr int sg = 4;
                const T* rb = sb + padpos<T>(u << 4);
#pragma unroll
                for (int c = 0; c < 16; ++c) v[c] = rb[padpos<T>((uint32_t)c)];
                ftile::t_pease<A, K, sg, 4, false>(ar, v, u, 0u, 0, tws);
                __syncthreads();              // every read of the single work buffer done
                T* wbo = sb + padpos<T>(u);
#pragma unroll
                for (int c = 0; c < 16; ++c) wbo[padpos<T>((uint32_t)c << (K - 4))] = v[c];
            }
        }
        __syncthreads();
        // ---- last group (tile-major) -> twist -> workspace rows k1
        {
            const uint32_t u = place2<GG::ILa, GG::ILb>(w);
            const T* sb = W + q * NP;
            // output row of register c
            auto xout = [&](int c) -> uint32_t {
                if (V == V_DIT) return u | ((uint32_t)c << 6);
                return (u << 2) | ((uint32_t)c >> 2) | (((uint32_t)c & 3u) << 8);
            };
            const uint64_t col = (tile & ((1ull << tpp_log) - 1)) * 8 + q;
            if (V == V_DIT) {
                const T* wb = sb + padpos<T>(u);
#pragma unroll
                for (int c = 0; c < 16; ++c) v[c] = wb[padpos<T>((uint32_t)c << 6)];
                ftile::t_bitwin<A, K, 6, 6, 4, false, false>(ar, v, u, 0u, 0, tws);
            } else {
                const T* rb = sb + padpos<T>(u << 4);
#pragma unroll
                for (int c = 0; c < 16; ++c) v[c] = rb[padpos<T>((uint32_t)c)];
                ftile::t_pease<A, K, 8, GG::KGL, false>(ar, v, u, 0u, 0, tws);
            }
            T* dst = a.out + (tile >> tpp_log) * N + col;    // MODE 0: column n2; MODE 1: row k1
            if (MODE == 0) {
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    if (NTT_FSA_TWF) dst[(uint64_t)xout(c) << Kc] = ar.mull(ar.mull(v[c], ftile::lds_tw(&twB[c * 8 + q])), twA);
                    else dst[(uint64_t)xout(c) << Kc] = ar.mulc(v[c], __ldg(a.twist + col + ((uint64_t)xout(c) << Kc)));
                }
            } else if (a.scale) {
#pragma unroll
                for (int c = 0; c < 16; ++c) dst[(uint64_t)xout(c) << Kr] = ar.mulc(v[c], a.ninv);
            } else {
#pragma unroll
                for (int c = 0; c < 16; ++c) dst[(uint64_t)xout(c) << Kr] = ar.fin(v[c]);
            }
        }
        if (a.counters && tid == 0 && (tile & ((1ull << tpp_log) - 1)) == 0) {
            atomicAdd(a.counters + C_HBM, 1ull);
            if (MODE == 1) atomicAdd(a.counters + C_TRANSFORMS, 1ull);
            if (a.count_bitrev) atomicAdd(a.counters + C_BITREV, (unsigned long long)a.count_bitrev);
        }
    }
}

}  // namespace fstep
}  // namespace nttb200
