// fourstep.cuh -- two-pass four-step transform for large u32 N (2^14..2^20).
//
// N = R x C (R = 2^Kr, C = 2^Kc), input x[n1*C + n2] viewed as an R x C
// row-major matrix, output X[k1 + R*k2]:
//   pass A (MODE 0): for every column n2, the length-R sub-transform over n1
//                    -> B[k1][n2], times the twist w_N^(k1*n2) (precomputed
//                    [k1][n2] Shoup table), written row-major to the workspace;
//   pass B (MODE 1): for every row k1, the length-C sub-transform over n2,
//                    written to out[k1 + R*k2].
// X[k1 + R k2] = sum_n2 w_C^(n2 k2) w_N^(n2 k1) sum_n1 w_R^(n1 k1) x[n1 C + n2],
// so the output is the transform of the reference (algorithms.py:402-412) for
// every variant; each sub-transform runs the variant's own dataflow (DIT:
// algorithms.py:82-121; Pease_nc: constant geometry with the buffers swapping
// roles, algorithms.py:203-261) with the sub-transform stage twiddles, which
// are the first 2^K entries of the plan's per-stage table.
//
// One CTA owns a tile of TQ networks (pass A: TQ consecutive columns, pass B:
// TQ consecutive rows) in a padded shared-memory work buffer:
//   * copy-in with 4-byte cp.async straight into the bit-reversed work layout
//     (no staging copy); the next tile's copy-in overlaps the current tile's
//     register groups (two work buffers);
//   * ceil(K/4) register groups of 16 residues per thread; the first groups
//     use the network-major thread map (a warp inside one network), the LAST
//     group the tile-major map (a warp spans the TQ networks), so every global
//     store of the tile is a full 32-byte sector run of TQ residues;
//   * pass A multiplies by the twist, pass B by n^-1 (intt) in that last group.
// Shared-memory maps (all bank-conflict free):
//   network stride NP = 2^AB (mod 32), AB = 5 - log2 TQ = lane bits above q;
//   tile-major lane bits land on position bits with padpos residues 0..AB-1.
#pragma once
#include <cstdint>
#include "fasttile.cuh"

// experiment knobs (defaults = measured best)
#ifndef NTT_FS_DIAG
#define NTT_FS_DIAG 0           // diagnostics only: 1 = skip the butterflies (data movement alone), 3 = also skip the stores, 4 = skip butterflies + copy-in
#endif
#ifndef NTT_FS_TWIST_TAB
#define NTT_FS_TWIST_TAB 1      // pass A twist from the precomputed [k1][n2] table (1) or factored (0):
                                // w^(n2 k1) = w^(n2 u) * w^(n2 c 2^(K-4)), one main-table load per
                                // thread + a 16 x TQ shared table per tile instead of 8 L2 bytes per residue
#endif
#ifndef NTT_FS_TW_EARLY
#define NTT_FS_TW_EARLY 1       // pass A: load the 16 twist factors before the last group's butterflies
#endif

namespace nttb200 {
namespace fstep {

using fastk::padpos;
using fastk::Perm;
using fastk::plan_lanes;
using fastk::scatter_bits;
using ftile::cp_async_commit;
using ftile::cp_async_wait_all;

template <class A>
struct FsArgs {
    using T = typename A::T;
    using Tw = typename A::Tw;
    const T* in;
    T* out;
    uint64_t batch;
    int Kr, Kc;                // R = 2^Kr (pass A length), C = 2^Kc (pass B length)
    const Tw* stw;             // per-stage table: entries [0, 2^K) = the length-2^K sub-transform's
    const Tw* twist;           // [k1][n2] = w_N^(k1*n2) with its Shoup word (pass A, NTT_FS_TWIST_TAB)
    const Tw* tw_main;         // the plan's main table w_N^i, i < N (factored twist)
    uint64_t p;
    int scale;                 // pass B: n^-1 (intt)
    Tw ninv;
    int count_bitrev;
    unsigned long long* counters;
};

template <class T>
NTT_D void cpe(uint32_t smem_addr, const void* g) {      // one residue (4 or 8 bytes)
    if (sizeof(T) == 8) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr), "l"(g) : "memory");
    else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr), "l"(g) : "memory");
}

constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v >> 1); }

template <int K, int TQ>
struct FsGeo {
    static constexpr int TT = 1 << (K - 4);              // threads per network
    static constexpr int NT = TQ * TT;
    static constexpr int G = (K + 3) / 4;
    static constexpr int K0 = K - 4 * (G - 1);
    static constexpr int LQ = ilog2c(TQ);
    static constexpr int AB = LQ >= 5 ? 0 : 5 - LQ;      // lane bits above the network id (tile-major)
};

// (NB tile buffers: two -- the next tile's copy-in lands beside the current one -- and for Pease a third,
// the stage output that is copied back)
// 64-bit residues: ONE tile buffer per CTA (the copy-in of a tile is followed by its own wait; other
// resident CTAs cover it) -- 39 KiB instead of 74 and 64 registers: four CTAs per SM instead of three
#ifndef NTT_FS_U64_SINGLE
#define NTT_FS_U64_SINGLE 1
#endif
template <class T>
constexpr bool fs_single_buf() { return NTT_FS_U64_SINGLE && sizeof(T) == 8; }
template <class T, class TwT, int K, int TQ, int NB = 2>
constexpr size_t fs_smem_bytes() {
    return ((size_t)sizeof(TwT) << K) + (size_t)sizeof(TwT) * 16 * TQ +
           (NB - (fs_single_buf<T>() ? 1 : 0)) * (size_t)TQ * ftile::tile_stride<T, K, TQ>() * sizeof(T);
}

// tile-major last group: sub-network id u from the thread's u' so that the AB
// in-warp bits of u' hit position bits with padpos residues 0..AB-1
//   DIT (positions u | c << (K-4)): identity;
//   Pease (reads u << 4 | c): in-warp bits -> u bits 1..AB (positions 5..)
template <int V, int K, int AB>
NTT_D uint32_t last_u(uint32_t up) {
    if (V == V_DIT || AB == 0) return up;      // DIF / Pease / Stockham read u << 4 | c: in-warp bits -> u bits 1..AB
    constexpr uint32_t m = (1u << AB) - 1;
    return ((up & m) << 1) | ((up >> AB) & 1u) | ((up >> (AB + 1)) << (AB + 1));
}

template <class A, int V, int K, int TQ, int MODE, int KO>
__global__ void __launch_bounds__(FsGeo<K, TQ>::NT, (FsGeo<K, TQ>::NT <= 256 ? (fs_single_buf<typename A::T>() ? 4 : 3) : (FsGeo<K, TQ>::NT <= 512 ? 2 : 1))) k_fs(FsArgs<A> a) {
    using T = typename A::T;
    using Tw = typename A::Tw;
    using GG = FsGeo<K, TQ>;
    constexpr int TT = GG::TT, NT = GG::NT, G = GG::G, K0 = GG::K0, LQ = GG::LQ, AB = GG::AB;
    constexpr int CW = fastk::lane_bits<T>();
    constexpr int NP = ftile::tile_stride<T, K, TQ>();
    constexpr int EPT = 16;                             // residues per thread per tile
    // DIT / Pease gather their input bit-reversed (algorithms.py:119,238,255); DIF
    // reads it in natural order and bit-reverses its output (algorithms.py:158)
    constexpr bool BRIN = (V != V_DIF && V != V_STOCKHAM);   // Stockham never bit-reverses
    constexpr bool TWE = NTT_FS_TW_EARLY && sizeof(T) == 4;
    static_assert(NT * EPT == (TQ << K), "one 16-residue sub-network per thread");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Tw* tws = reinterpret_cast<Tw*>(smem_raw);
    Tw* twB = tws + (1 << K);                           // factored twist: [c][t] = w^(n2_t c 2^(K-4))
    T* buf0 = reinterpret_cast<T*>(twB + 16 * TQ);
    A ar;
    ar.init(a.p);
    const uint32_t tid = threadIdx.x;
    for (uint32_t i = tid; i < (1u << K); i += NT) tws[i] = a.stw[i];

    // KO = log2 of the other dimension, compile time: every strided offset is an immediate
    constexpr int Kr = MODE == 0 ? K : KO, Kc = MODE == 0 ? KO : K;
    constexpr uint64_t N = 1ull << (Kr + Kc);
    constexpr uint32_t tpp_log = (MODE == 0 ? Kc : Kr) - LQ;   // log2 tiles per polynomial
    const uint64_t ntiles = a.batch << tpp_log;

    // ---- copy-in geometry (per thread, constant over tiles)
    // MODE 0 (tile-major): q = tid mod TQ, rest = tid / TQ (K-4 bits);
    //   row r = rest_lo << (K-AB) | rest_hi << 4 | j, placed at brev_K(r)
    // MODE 1 (contiguous): element e = tid + j*NT of the TQ x C tile block
    uint32_t cin_soff;          // shared offset (elements) of register j = 0
    uint64_t cin_goff;          // global offset within the tile's base
    if (MODE == 0) {
        const uint32_t q = tid & (TQ - 1), rest = tid >> LQ;
        const uint32_t rlo = rest & ((1u << AB) - 1), rhi = rest >> AB;
        // bit-reversed placement: the in-warp rest bits on r's top bits (positions 0..AB-1);
        // natural placement (DIF): on r's low bits; the register index j fills the other end
        const uint32_t r0 = BRIN ? ((rlo << (K - AB)) | (rhi << 4)) : (rlo | (rhi << AB));
        cin_soff = q * NP + padpos<T>(BRIN ? brev(r0, K) : r0);
        cin_goff = ((uint64_t)r0 << Kc) + q;
    } else {
        const uint32_t x0 = tid & ((1u << K) - 1), q0 = tid >> K;
        cin_soff = q0 * NP + padpos<T>(BRIN ? brev(x0, K) : x0);
        cin_goff = tid;
    }
    auto tile_gbase = [&](uint64_t tl) -> uint64_t {      // global element of the tile's (q=0, r/x=0)
        const uint64_t b = tl >> tpp_log;
        const uint64_t g = tl & ((1ull << tpp_log) - 1);
        return b * N + (MODE == 0 ? g * TQ : (g * TQ) << Kc);
    };
    auto copy_in = [&](uint64_t tl, T* dst) {
        if (NTT_FS_DIAG == 4) return;
        const T* src = a.in + tile_gbase(tl) + cin_goff;
        const uint32_t sb = fastk::smem_u32(dst + cin_soff);
#pragma unroll
        for (int j = 0; j < EPT; ++j) {
            uint32_t so;
            uint64_t go;
            if (MODE == 0) {
                // j = r bits 0..3 (bit-reversed: positions K-4..K-1) / r bits K-4..K-1 (natural)
                so = padpos<T>(BRIN ? brev((uint32_t)j, K) : ((uint32_t)j << (K - 4)));
                go = (uint64_t)(BRIN ? (uint32_t)j : ((uint32_t)j << (K - 4))) << Kc;
            } else {
                // e = tid + j*NT: x = e mod 2^K, q = e >> K (NT = TQ*2^(K-4))
                constexpr uint32_t NTc = NT;
                const uint32_t ej = (uint32_t)j * NTc;
                so = (ej >> K) * NP + padpos<T>(BRIN ? brev(ej & ((1u << K) - 1), K) : (ej & ((1u << K) - 1)));
                go = ej;
            }
            cpe<T>(sb + so * sizeof(T), src + go);
        }
    };

    __syncthreads();                         // twiddle table in place (before the PDL wait)
    fastk::pdl_trigger();
    fastk::pdl_wait();
    constexpr bool SB = fs_single_buf<T>();
    if (!SB && (uint64_t)blockIdx.x < ntiles) copy_in(blockIdx.x, buf0);
    cp_async_commit();
    int it = 0;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        T* X = SB ? buf0 : buf0 + (it & 1) * (TQ * NP);
        T* Y = buf0 + ((it + 1) & 1) * (TQ * NP);
        T* Z = buf0 + (SB ? 1 : 2) * (TQ * NP);   // Pease only: the stage output before its copy-back
        if (SB) {                            // single buffer: the previous tile's last group is done with it
            __syncthreads();
            copy_in(tile, X);
            cp_async_commit();
        }
        cp_async_wait_all();
        __syncthreads();                     // X landed for every thread; Y free (previous tile done)
        auto prefetch_next = [&]() {
            const uint64_t nxt = tile + gridDim.x;
            if (nxt < ntiles) copy_in(nxt, Y);
            cp_async_commit();
        };
        if (!SB) prefetch_next();          // the next tile's copy-in overlaps this tile's groups
        // factored pass-A twist: the tile's [c][t] table and this thread's w^(n2 u)
        Tw twA;
        if (MODE == 0 && !NTT_FS_TWIST_TAB) {
            const uint64_t col0 = (tile & ((1ull << tpp_log) - 1)) * TQ;
            if (tid < 16 * TQ) {
                const uint32_t c = tid / TQ, t = tid % TQ;
                twB[tid] = __ldg(a.tw_main + (((col0 + t) * c) << (K - 4)));
            }
            twA = __ldg(a.tw_main + (col0 + (tid & (TQ - 1))) * last_u<V, K, AB>(tid >> LQ));
        }
        // ---- register groups 0 .. G-2: network-major thread map
#pragma unroll
        for (int g = 0; g < G - 1; ++g) {
            if (NTT_FS_DIAG >= 1) break;
            T v[16];
            const uint32_t t = tid >> (K - 4), u = tid & (TT - 1);
            T* sb = X + t * NP;
            if (V == V_DIT || V == V_DIF) {
                // DIT: windows from bit 0 up (first short); DIF: from the top bit down (short window last)
                const int B = (V == V_DIT) ? (g == 0 ? 0 : K0 + 4 * (g - 1)) : K - 4 * (g + 1);
                const int kg = (V == V_DIT) ? (g == 0 ? K0 : 4) : 4;
                uint32_t pbase = 0;
#define NTT_FSMAP(BB)                                  \
    if (B == BB) {                                     \
        constexpr Perm PM = plan_lanes(K, BB, CW);     \
        pbase = scatter_bits<K - 4>(u, PM);            \
    }
                NTT_FSMAP(0) NTT_FSMAP(1) NTT_FSMAP(2) NTT_FSMAP(3) NTT_FSMAP(4) NTT_FSMAP(5) NTT_FSMAP(6)
#undef NTT_FSMAP
                T* wb = sb + padpos<T>(pbase);
#pragma unroll
                for (int c = 0; c < 16; ++c) v[c] = wb[padpos<T>((uint32_t)c << B)];
#define NTT_FSBW(BB, kgv) \
    if (B == BB && kg == kgv) ftile::t_bitwin<A, K, BB, BB, kgv, V == V_DIF, false>(ar, v, pbase, 0u, 0, tws);
                if (V == V_DIF) { NTT_FSBW(1, 4) NTT_FSBW(2, 4) NTT_FSBW(3, 4) NTT_FSBW(4, 4) NTT_FSBW(5, 4) NTT_FSBW(6, 4) }
                else if (g == 0) { NTT_FSBW(0, 1) NTT_FSBW(0, 2) NTT_FSBW(0, 3) NTT_FSBW(0, 4) }
                else { NTT_FSBW(1, 4) NTT_FSBW(2, 4) NTT_FSBW(3, 4) NTT_FSBW(4, 4) NTT_FSBW(5, 4) }
#undef NTT_FSBW
#pragma unroll
                for (int c = 0; c < 16; ++c) wb[padpos<T>((uint32_t)c << B)] = v[c];
            } else if (V == V_STOCKHAM) {   // self-sorting: window [lob, lob+kg), one buffer
                const int sg = g == 0 ? 0 : K0 + 4 * (g - 1);
                const int kg = g == 0 ? K0 : 4;
                const int lob = K - sg - kg;
                uint32_t hi, lo;
                if (g == 0) { hi = 0; lo = u; }
                else { lo = u & ((1u << lob) - 1); hi = u >> lob; }
                const T* rb = sb + padpos<T>((hi << (K - sg)) | lo);
#pragma unroll
                for (int c = 0; c < 16; ++c) v[c] = rb[padpos<T>((uint32_t)c << (lob - (4 - kg)))];
#define NTT_FSST(SG, KGV) \
    if (sg == SG && kg == KGV) ftile::t_stockham<A, K, SG, KGV, false>(ar, v, hi, 0u, 0, tws);
                if (g == 0) { NTT_FSST(0, 1) NTT_FSST(0, 2) NTT_FSST(0, 3) NTT_FSST(0, 4) }
                else { NTT_FSST(1, 4) NTT_FSST(2, 4) NTT_FSST(3, 4) NTT_FSST(4, 4) NTT_FSST(5, 4) }
#undef NTT_FSST
                __syncthreads();             // every read of the (single) work buffer done
                T* wbo = sb + padpos<T>((hi << lob) | lo);
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    const uint32_t Rb = (uint32_t)c >> (4 - kg), xx = (uint32_t)c & ((1u << (4 - kg)) - 1);
                    wbo[padpos<T>((Rb << (K - kg)) | (xx << (lob - (4 - kg))))] = v[c];
                }
            } else {   // Pease / Pease_nc: constant geometry, one buffer (roles swap through the registers)
                const int sg = g == 0 ? 0 : K0 + 4 * (g - 1);
                const int kg = g == 0 ? K0 : 4;
                const T* rb = sb + padpos<T>(u << 4);
#pragma unroll
                for (int c = 0; c < 16; ++c) v[c] = rb[padpos<T>((uint32_t)c)];
#define NTT_FSPE(SG, KGV) \
    if (sg == SG && kg == KGV) ftile::t_pease<A, K, SG, KGV, false>(ar, v, u, 0u, 0, tws);
                if (g == 0) { NTT_FSPE(0, 1) NTT_FSPE(0, 2) NTT_FSPE(0, 3) NTT_FSPE(0, 4) }
                else { NTT_FSPE(1, 4) NTT_FSPE(2, 4) NTT_FSPE(3, 4) NTT_FSPE(4, 4) NTT_FSPE(5, 4) }
#undef NTT_FSPE
                if (V != V_PEASE) __syncthreads();   // every read of the (single) work buffer done
                // Pease: the stage output goes to Z and is copied back (_stage_copy, algorithms.py:242)
                T* wbo = (V == V_PEASE ? Z + t * NP : sb) + padpos<T>(u << (4 - kg));
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    const uint32_t n = c >> kg, Rb = c & ((1u << kg) - 1);
                    wbo[padpos<T>(n | (Rb << (K - kg)))] = v[c];
                }
                if (V == V_PEASE) {
                    __syncthreads();
                    for (uint32_t i = tid; i < (uint32_t)(TQ * NP); i += NT) X[i] = Z[i];
                }
            }
            __syncthreads();
        }
        // ---- last group: tile-major thread map, stores straight to HBM
        {
            T v[16];
            const uint32_t t = tid & (TQ - 1);
            const uint32_t u = last_u<V, K, AB>(tid >> LQ);
            const T* sb = X + t * NP;
            constexpr int sgL = K - 4;
            // pass A: the twist factors of this thread's 16 outputs, loaded before the
            // butterflies so their L2 latency overlaps the last group's arithmetic
            // output index of register c: DIT / Pease u | c << (K-4) (natural order);
            // DIF block [0,4) at u << 4, output brev_K(position)
            auto xo = [&](int c) -> uint32_t {
                if (V == V_DIF) return brev((u << 4) | (uint32_t)c, K);
                return u | ((uint32_t)c << (K - 4));
            };
            Tw twv[(MODE == 0 && TWE && NTT_FS_TWIST_TAB) ? 16 : 1];
            if (MODE == 0 && TWE && NTT_FS_TWIST_TAB) {
                const uint64_t col = (tile & ((1ull << tpp_log) - 1)) * TQ + t;
#pragma unroll
                for (int c = 0; c < 16; ++c)
                    twv[(MODE == 0 && TWE && NTT_FS_TWIST_TAB) ? c : 0] = __ldg(a.twist + col + ((uint64_t)xo(c) << Kc));
            }
            if (V == V_DIF) {
                const T* wb = sb + padpos<T>(u << 4);
#pragma unroll
                for (int c = 0; c < 16; ++c) v[c] = wb[padpos<T>((uint32_t)c)];
                if (NTT_FS_DIAG == 0) ftile::t_bitwin<A, K, 0, 0, K0, true, false>(ar, v, u << 4, 0u, 0, tws);   // stages K0..1
            } else if (V == V_DIT) {
                const T* wb = sb + padpos<T>(u);
#pragma unroll
                for (int c = 0; c < 16; ++c) v[c] = wb[padpos<T>((uint32_t)c << sgL)];
                if (NTT_FS_DIAG == 0) ftile::t_bitwin<A, K, sgL, sgL, 4, false, false>(ar, v, u, 0u, 0, tws);
            } else {
                const T* rb = sb + padpos<T>(u << 4);
#pragma unroll
                for (int c = 0; c < 16; ++c) v[c] = rb[padpos<T>((uint32_t)c)];
                // Stockham's last window (lob = 0) reads the same 16 contiguous positions
                if (NTT_FS_DIAG == 0) {
                    if (V == V_STOCKHAM) ftile::t_stockham<A, K, sgL, 4, false>(ar, v, u, 0u, 0, tws);
                    else ftile::t_pease<A, K, sgL, 4, false>(ar, v, u, 0u, 0, tws);
                }
            }
            const uint64_t gb = tile_gbase(tile);
            if (NTT_FS_DIAG == 3) {
                if (a.count_bitrev == 77) a.out[tid] = v[0] ^ v[5] ^ v[15];   // never: keeps the loads
            } else if (MODE == 0) {
                // B[k1][n2] * w_N^(k1 n2) -> ws[k1*C + n2], n2 = tile column t
                const uint64_t col = (tile & ((1ull << tpp_log) - 1)) * TQ + t;
                T* dst = a.out + gb + t;
                if (NTT_FS_TWIST_TAB || V == V_DIF) {
                    // (u32) Shoup with x < 4p < 2^32 is exact and canonicalising: no separate fin
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        const uint64_t ro = (uint64_t)xo(c) << Kc;
                        dst[ro] = ar.mulc(v[c], TWE ? twv[TWE ? c : 0] : __ldg(a.twist + col + ro));
                    }
                } else {
                    // [0,2p) results: pass B's first stage takes lazy inputs
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        const uint64_t ro = (uint64_t)c << (K - 4 + Kc);
                        dst[ro + ((uint64_t)u << Kc)] = ar.mull(ar.mull(v[c], ftile::lds_tw(&twB[c * TQ + t])), twA);
                    }
                }
            } else {
                // out[k1 + R*k2]: k1 = tile row t, k2 = xo(c)
                const uint64_t k1 = (tile & ((1ull << tpp_log) - 1)) * TQ + t;
                T* dst = a.out + (tile >> tpp_log) * N + k1;
                if (a.scale) {
#pragma unroll
                    for (int c = 0; c < 16; ++c) dst[(uint64_t)xo(c) << Kr] = ar.mulc(v[c], a.ninv);
                } else {
#pragma unroll
                    for (int c = 0; c < 16; ++c) dst[(uint64_t)xo(c) << Kr] = ar.fin(v[c]);
                }
            }
        }
        if (a.counters && tid == 0 && (tile & ((1ull << tpp_log) - 1)) == 0) {
            atomicAdd(a.counters + C_HBM, 1ull);
            if (MODE == 1) atomicAdd(a.counters + C_TRANSFORMS, 1ull);
            if (V == V_PEASE) atomicAdd(a.counters + C_COPIES, (unsigned long long)(G - 1));
            if (MODE == 0 && a.count_bitrev) atomicAdd(a.counters + C_BITREV, (unsigned long long)a.count_bitrev);
        }
    }
}

#ifndef NTT_FS_TQ10
#define NTT_FS_TQ10 8
#endif
template <class T, int K>
constexpr int fs_tq() {
    if (sizeof(T) == 8) return K == 8 ? 16 : (K == 9 ? 8 : 32);
    return K == 10 ? NTT_FS_TQ10 : (K == 9 ? 8 : (K == 8 ? 16 : 32));
}

template <class A, int V, int K, int MODE, int KO>
cudaError_t fs_launch(const FsArgs<A>& a, cudaStream_t s, int num_sms, int* launches) {
    using T = typename A::T;
    constexpr int TQ = fs_tq<T, K>();
    constexpr int NT = FsGeo<K, TQ>::NT;
    constexpr size_t smem = fs_smem_bytes<T, typename A::Tw, K, TQ, V == V_PEASE ? 3 : 2>();
    auto kern = k_fs<A, V, K, TQ, MODE, KO>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
    const int lq = ilog2c(TQ);
    const uint64_t ntiles = a.batch << (KO - lq);
    uint64_t grid = (uint64_t)num_sms * occ;
    if (grid > ntiles) grid = ntiles;
    if (grid == 0) return cudaSuccess;
    cudaError_t le = fastk::launch_pdl(kern, dim3((unsigned)grid), dim3(NT), smem, s, a);
    if (launches) ++*launches;
    return le != cudaSuccess ? le : cudaGetLastError();
}

// pass `mode` of a transform of size 2^L (Kr = ceil(L/2), Kc = floor(L/2))
template <class A, int V, int L>
cudaError_t fs_pass_l(int mode, const FsArgs<A>& a, cudaStream_t s, int num_sms, int* launches) {
    constexpr int KR = (L + 1) / 2, KC = L - KR;
    return mode == 0 ? fs_launch<A, V, KR, 0, KC>(a, s, num_sms, launches)
                     : fs_launch<A, V, KC, 1, KR>(a, s, num_sms, launches);
}

template <class A, int V>
cudaError_t fs_pass_any(int L, int mode, const FsArgs<A>& a, cudaStream_t s, int num_sms, int* launches) {
    switch (L) {
        case 14: return fs_pass_l<A, V, 14>(mode, a, s, num_sms, launches);
        case 15: return fs_pass_l<A, V, 15>(mode, a, s, num_sms, launches);
        case 16: return fs_pass_l<A, V, 16>(mode, a, s, num_sms, launches);
        case 17: return fs_pass_l<A, V, 17>(mode, a, s, num_sms, launches);
        case 18: return fs_pass_l<A, V, 18>(mode, a, s, num_sms, launches);
        case 19: return fs_pass_l<A, V, 19>(mode, a, s, num_sms, launches);
        case 20: return fs_pass_l<A, V, 20>(mode, a, s, num_sms, launches);
        default: return cudaErrorInvalidValue;
    }
}

// Builds the pass-A twist table tw4[k1*C + n2] = w^(k1*n2) from the plan's
// main table (w^i with its Shoup word, i < N; k1*n2 < N needs no reduction).
template <class Tw>
__global__ void k_fs_twist_table(const Tw* tw, Tw* out, int Kr, int Kc) {
    const uint64_t n = 1ull << (Kr + Kc);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k1 = i >> Kc, n2 = i & ((1ull << Kc) - 1);
        out[i] = tw[k1 * n2];
    }
}

}  // namespace fstep

}  // namespace nttb200
