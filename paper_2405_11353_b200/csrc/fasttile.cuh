// fasttile.cuh -- compile-time specialised HBM pass kernel for large N.
//
// One pass = K consecutive stages of the variant (index algebra in
// docs/PASS_ALGEBRA.md).  A CTA owns a TILE of TQ networks (2^K residues
// each) in a padded shared-memory layout:
//   1. coalesced 16-byte-vector gather of the tile from HBM (bit reversal of
//      the first DIT / Pease pass fused into the gather addresses),
//   2. ceil(K/4) register groups (16 residues per thread, <= 4 stages each,
//      conflict-free lane maps), twiddles from the per-stage table
//      T[2^(s-1)+k]: the first 2^SMB entries staged in shared memory once per
//      CTA, later stages read through the read-only path (L2-resident table),
//      one 8-byte load per DISTINCT twiddle of a thread's group,
//   3. coalesced 16-byte-vector scatter (final reduction, n_inv scaling,
//      six-step correction twiddles fused).
// Tiles are persistent over the grid.  Stage-faithful: the HBM buffer after a
// pass holds the reference's state after the same stage (congruent; exact
// when the policy is canonical).
#pragma once
#include <cstdint>
#include "fast.cuh"

// staged prefetch for 64-bit tiles: off by default -- the Goldilocks passes are
// integer-bound, and the 32 KiB staging buffer costs them a resident CTA
// (config 3: 0.385 -> 0.399 ms with it)
#ifndef NTT_TILE_PF_U64
#define NTT_TILE_PF_U64 0
#endif

#ifndef NTT_TILE_MINB256
#define NTT_TILE_MINB256 3      // resident CTAs the 256-thread tile kernels are compiled for
#endif

namespace nttb200 {
namespace ftile {

using fastk::padded_len;
using fastk::padpos;
using fastk::Perm;
using fastk::plan_lanes;
using fastk::scatter_bits;

// TL_COLS: a DIT pass over the column index j of an [2^L][2^l1] row-major
// matrix (element (i, j) at i + j*2^l1) for all 2^l1 columns at once; the
// network id is Q = i | Qj << l1, so consecutive networks of a tile are
// consecutive columns and both HBM sides move runs of TQ residues
enum TileLayout { TL_VARIANT = 0, TL_SIX_A = 1, TL_SIX_B = 2, TL_COLS = 3 };
enum TileQ { TQM_LINEAR = 1, TQM_REV = 2, TQM_2D = 3 };
enum TileOrder { TO_C_FAST = 0, TO_T_FAST = 1, TO_TB_FAST = 2 };

template <class A>
struct TileArgs {
    using T = typename A::T;
    using Tw = typename A::Tw;
    const T* in;
    T* out;
    uint64_t batch;
    int L, S0;
    int qmode, TA, la;         // TQM_2D: TQ = TA x TB, la = log2 TA
    int in_order, out_order;
    int vec_in, vec_out;       // 16-byte vector copies valid for this pass
    int rev_in, rev_out;
    int rev_local;             // bit-reverse the K local bits on the gather (six-step sub-DIT input;
                               // Pease pass 1 reading the row-bit-reversed intermediate)
    int out_trb;               // Pease pass 0: write position (x << (L-K)) | rev_{L-K}(Q) (row-bit-reversed
                               // transpose of the stage state) so both HBM sides are 32-byte runs
    int count_row, count_bitrev;
    const Tw* gstw;            // global per-stage table of the (sub-)transform
    int smb;                   // entries [0, 2^smb) are staged in shared memory
    uint64_t p;
    int scale;
    Tw ninv;
    int twist;                 // four-step factorisation of a late pass (docs/PASS_ALGEBRA.md):
                               // 0 none, 1 pre W^(r*rev(x)), 2 pre W^(r*x), 3 post W^(r*rev(x)),
                               // W = w^(N / 2^(S0+K)); r = the network's twiddle-carrying bits:
    int tw_rsel;               //   0: Q mod 2^S0 (DIT/DIF), 1: Q >> (L-K-S0) (Pease qtop / Stockham ghi)
    const Tw* tw_lo;           // w^j, j < 2^th          (the plan's main table prefix)
    const Tw* tw_hi;           // w^(j*2^th), j < 2^(L-th)
    int th;
    int l1, l2;                // six-step: gather stride bits (A: local columns n1/G), row bits (B)
    int qoff;                  // six-step A: global index of local column 0 (distributed: rank*n1/G)
    int pb;                    // six-step A: log2 of the row slice per destination (n2/G); = l2 when G = 1
    uint64_t pblk;             // six-step A: elements per destination block (n1/G * n2/G)
    const T* cor_lo;
    const T* cor_hi;
    int cor_lb;
    int cor_on;                // TL_COLS: multiply by w_N^(i * k2) in the scatter (six-step correction)
    int cor_lgn;               // TL_COLS correction: log2 N when the tile's columns are a slab (0: L + l1)
    unsigned long long* counters;
    // colpass.cuh transposing pass of the distributed step A: output row k2 goes to destination
    // h = k2 >> dist_pb as dist_dst[h][i_local << dist_pb | k2 mod 2^dist_pb] (0: single device)
    int dist_pb = 0;
    T* dist_dst[8] = {};
};

template <class A, int V, int K, int LAY>
NTT_D uint64_t t_gpos_in(const TileArgs<A>& a, uint32_t Q, uint32_t x) {
    if (LAY == TL_SIX_A) return ((uint64_t)x << a.l1) | Q;
    if (LAY == TL_SIX_B) return ((uint64_t)x << a.l2) | Q;
    const int L = a.L, S0 = a.S0;
    if (LAY == TL_COLS) {
        const uint32_t Qj = Q >> a.l1;
        uint64_t g = (Qj & ((1u << S0) - 1)) | ((uint64_t)x << S0) | ((uint64_t)(Qj >> S0) << (S0 + K));
        if (a.rev_in) g = brev((uint32_t)g, L);
        return (Q & ((1u << a.l1) - 1)) | (g << a.l1);
    }
    uint64_t g;
    if (V == V_PEASE || V == V_PEASE_NC) g = ((uint64_t)Q << K) | x;
    else if (V == V_STOCKHAM) {
        const int glob = L - S0 - K;
        g = ((uint64_t)(Q >> glob) << (L - S0)) | ((uint64_t)x << glob) | (Q & ((1u << glob) - 1));
    } else g = (Q & ((1u << S0) - 1)) | ((uint64_t)x << S0) | ((uint64_t)(Q >> S0) << (S0 + K));
    return a.rev_in ? (uint64_t)brev((uint32_t)g, L) : g;
}

template <class A, int V, int K, int LAY>
NTT_D uint64_t t_gpos_out(const TileArgs<A>& a, uint32_t Q, uint32_t x) {
    if (LAY == TL_SIX_A)      // packed for the all-to-all: [dest h][i_local][k2 mod n2/G]
        return (uint64_t)(x >> a.pb) * a.pblk + ((uint64_t)Q << a.pb) + (x & ((1u << a.pb) - 1));
    if (LAY == TL_SIX_B) return ((uint64_t)x << a.l2) | Q;
    const int L = a.L, S0 = a.S0;
    if (LAY == TL_COLS) {
        const uint32_t Qj = Q >> a.l1;
        const uint64_t g = (Qj & ((1u << S0) - 1)) | ((uint64_t)x << S0) | ((uint64_t)(Qj >> S0) << (S0 + K));
        return (Q & ((1u << a.l1) - 1)) | (g << a.l1);
    }
    uint64_t g;
    if (V == V_PEASE || V == V_PEASE_NC || V == V_STOCKHAM) {
        if (a.out_trb) return ((uint64_t)x << (L - K)) | brev(Q, L - K);
        g = Q | ((uint64_t)x << (L - K));
    } else g = (Q & ((1u << S0) - 1)) | ((uint64_t)x << S0) | ((uint64_t)(Q >> S0) << (S0 + K));
    return a.rev_out ? (uint64_t)brev((uint32_t)g, L) : g;
}

// twiddle T[idx]: the group decides (uniformly) whether all its stages are
// covered by the shared-memory copy or must use the read-only path, so the
// loads are unconditional and the compiler can hoist them.
template <class Tw>
struct TwSrc {
    const Tw* p;
    bool global;
};
// explicit shared-space loads (a generic pointer would compile to LD, not LDS)
NTT_D uint2 lds_tw(const uint2* p) {
    uint2 r;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(fastk::smem_u32(p)));
    return r;
}
NTT_D uint64_t lds_tw(const uint64_t* p) {
    uint64_t r;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(r) : "r"(fastk::smem_u32(p)));
    return r;
}
NTT_D ulonglong2 lds_tw(const ulonglong2* p) {
    ulonglong2 r;
    asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(r.x), "=l"(r.y) : "r"(fastk::smem_u32(p)));
    return r;
}
template <bool GL, class Tw>
NTT_D Tw twld(const Tw* p, uint32_t idx) {
    if (GL) return __ldg(p + idx);
    return lds_tw(p + idx);
}

// ---------------------------------------------------------------- DIT/DIF --
// IN (first group of a LOCAL transform only: S0 = 0, qlow = 0, the thread's low position bits
// zero, so a butterfly's twiddle index is the compile-time kc): 1 = canonical inputs (caller data,
// modmath.py:112), 2 = inputs in [0,2p) (a lazy twist's outputs).  Stage 1 / 2 then take the
// bounded forms and every w^0 butterfly skips its multiply, as in the single-pass kernel.
// (The same forms in the Pease first group measured 1.3 % SLOWER on config 4 in three
// interleaved A/Bs -- 2.66-2.68 vs 2.63 ms -- so t_pease keeps the general butterflies.)
template <class A, int K, int B, int b0, int kg, bool DIF, bool GL, int IN = 0>
NTT_D void t_bitwin(const A& ar, typename A::T (&v)[16], uint32_t pbase, uint32_t qlow, int S0,
                    const typename A::Tw* tw) {
    constexpr int off = b0 - B;
    static_assert(IN == 0 || (!DIF && B == 0 && b0 == 0), "bounded first stages: DIT-type first groups");
#pragma unroll
    for (int jj = 0; jj < kg; ++jj) {
        const int j = DIF ? kg - 1 - jj : jj;
        const int sl = b0 + j;                         // local bit = local stage - 1
        const int s = S0 + sl + 1;                     // global stage
        const bool triv = (sl == 0) && (S0 == 0);      // s == 1: every twiddle is w^0
        const uint32_t lmask = (1u << sl) - 1;
        const uint32_t kthr = qlow | ((pbase & lmask) << S0);
        const uint32_t rowi = (1u << (s - 1)) + kthr;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            if (c & (1 << (off + j))) continue;
            const uint32_t kc = ((uint32_t)c << B) & lmask;
            const int hi = c | (1 << (off + j));
            if (IN != 0) {
                const bool one = kc == 0;              // w^0
                if (sl == 0) { if (IN == 1) ar.dit1_c(v[c], v[hi]); else ar.dit1_2p(v[c], v[hi]); }
                else if (sl == 1 && IN == 1) {
                    if (one) ar.dit1_2p(v[c], v[hi]); else ar.dit_2p(v[c], v[hi], twld<GL>(tw, rowi + kc));
                } else if (one) ar.dit1(v[c], v[hi]);
                else ar.dit(v[c], v[hi], twld<GL>(tw, rowi + kc));
            } else if (triv) {
                if (DIF) ar.dif1(v[c], v[hi]); else ar.dit1(v[c], v[hi]);
            } else {
                const typename A::Tw w = twld<GL>(tw, rowi + (kc << S0));
                if (DIF) ar.dif(v[c], v[hi], w); else ar.dit(v[c], v[hi], w);
            }
        }
    }
}

// ------------------------------------------------------------------ Pease --
template <class A, int K, int sg, int kg, bool GL>
NTT_D void t_pease(const A& ar, typename A::T (&v)[16], uint32_t u, uint32_t qtop, int S0,
                   const typename A::Tw* tw) {
    using T = typename A::T;
    constexpr int NB = 16 >> kg;
    constexpr int H = 1 << (kg - 1);
#pragma unroll
    for (int n = 0; n < NB; ++n) {
        const uint32_t q = (u << (4 - kg)) | n;                   // local network id (K-kg bits)
        const uint32_t bprev = sg ? (q >> ((K - kg - sg) > 0 ? (K - kg - sg) : 0)) : 0u;     // output bits of earlier groups
#pragma unroll
        for (int m = 0; m < kg; ++m) {
            const int s = S0 + sg + m + 1;
            const bool triv = (sg + m == 0) && (S0 == 0);
            const uint32_t rowi = (1u << (s - 1)) + ((bprev << S0) | qtop);
            T nv[1 << kg];
#pragma unroll
            for (int i = 0; i < H; ++i) {
                const uint32_t Bg = (2u * i) >> (kg - m);
                T x = v[n * (1 << kg) + 2 * i], y = v[n * (1 << kg) + 2 * i + 1];
                if (triv) ar.dit1(x, y);
                else ar.dit(x, y, twld<GL>(tw, rowi + (Bg << (sg + S0))));
                nv[i] = x;
                nv[i + H] = y;
            }
#pragma unroll
            for (int c = 0; c < (1 << kg); ++c) v[n * (1 << kg) + c] = nv[c];
        }
    }
}

// --------------------------------------------------------------- Stockham --
template <class A, int K, int sg, int kg, bool GL>
NTT_D void t_stockham(const A& ar, typename A::T (&v)[16], uint32_t hi, uint32_t ghi, int S0,
                      const typename A::Tw* tw) {
    using T = typename A::T;
    constexpr int NB = 16 >> kg;
    constexpr int H = 1 << (kg - 1);
#pragma unroll
    for (int x = 0; x < NB; ++x) {
#pragma unroll
        for (int m = 0; m < kg; ++m) {
            const int s = S0 + sg + m;     // 0-based
            const bool triv = (sg + m == 0) && (S0 == 0);
            const uint32_t rowi = (1u << s) + ((hi << S0) | ghi);
            T nv[1 << kg];
#pragma unroll
            for (int i = 0; i < H; ++i) {
                const uint32_t Bv = i & ((1u << m) - 1), crest = (uint32_t)i >> m;
                T a = v[(i << (4 - kg)) | x], b = v[((i + H) << (4 - kg)) | x];
                if (triv) ar.dit1(a, b);
                else ar.dit(a, b, twld<GL>(tw, rowi + (Bv << (sg + S0))));
                nv[(crest << (m + 1)) | Bv] = a;
                nv[(crest << (m + 1)) | (1u << m) | Bv] = b;
            }
#pragma unroll
            for (int c = 0; c < (1 << kg); ++c) v[(c << (4 - kg)) | x] = nv[c];
        }
    }
}

// Network stride in shared memory: the padded length, skewed so that the
// TQ networks of a tile land in different banks for t-fast copies
// (stride = max(1, 32/TQ) mod 32 for u32; max(1, 16/TQ) mod 16 for u64).
template <class T, int K, int TQ>
NTT_HD constexpr int tile_stride() {
    constexpr int NB = sizeof(T) == 4 ? 32 : 16;
    constexpr int want = TQ >= NB ? 1 : NB / TQ;
    int n = padded_len<T, K>();
    while (n % NB != want) ++n;
    return n;
}

// Network base of a tile: t * NP, except the u64 column-layout tiles with 4-8
// threads per network (config 5's 2^6 / 2^7 passes), where a warp spans 4-8
// networks and no linear stride keeps both the vector copies and the DIT
// register groups conflict-free; there base(t) = t * NP + (t >> XS) with the
// NP / XS an exhaustive bank search chose (tools/bankcheck.py replays it).
template <class T, int K, int TQ, int LAY>
NTT_HD constexpr int tile_np() {
    if (sizeof(T) == 8 && LAY == 3 && K == 7 && TQ == 32) return (padded_len<T, K>() + 16 + 15) / 16 * 16 + 4;
    if (sizeof(T) == 8 && LAY == 3 && K == 6 && TQ == 64) return (padded_len<T, K>() + 16 + 15) / 16 * 16 + 2;
    return tile_stride<T, K, TQ>();
}
template <class T, int K, int TQ, int LAY>
NTT_HD constexpr int tile_xs() {
    if (sizeof(T) == 8 && LAY == 3 && K == 7 && TQ == 32) return 2;
    if (sizeof(T) == 8 && LAY == 3 && K == 6 && TQ == 64) return 3;
    return 0;
}
template <class T, int K, int TQ, int LAY>
NTT_HD constexpr uint32_t tile_nbase(uint32_t t) {
    return t * (uint32_t)tile_np<T, K, TQ, LAY>() + (tile_xs<T, K, TQ, LAY>() ? (t >> tile_xs<T, K, TQ, LAY>()) : 0u);
}

template <int K, int TQ>
struct TileGeo {
    static constexpr int TT = 1 << (K - 4);       // threads per network
    static constexpr int G = (K + 3) / 4;
    static constexpr int K0 = K - 4 * (G - 1);
};

// --------------------------------------------------------------- cp.async --
NTT_D void cp_async(void* smem, const void* g, int bytes) {
    const uint32_t d = fastk::smem_u32(smem);
    if (bytes == 16) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(g) : "memory");
    else if (bytes == 8) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(g) : "memory");
    else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(g) : "memory");
}
NTT_D void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
NTT_D void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ----------------------------------------------------------------- kernel --
// per-network twist table shape: w^(r*xr) = lo[xr & 31] * hi[xr >> 5], xr < 2^K
template <int K> constexpr int twc_lo() { return K < 5 ? (1 << K) : 32; }
template <int K> constexpr int twc_hi() { return K > 5 ? (1 << (K - 5)) : 1; }
template <int K> constexpr int tw_row() { return twc_lo<K>() + 1 + twc_hi<K>() + 1; }   // odd-padded rows
constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v >> 1); }

// shared-memory footprint of one k_tile instantiation (bytes)
template <class T, class Tw, int V, int K, int TQ, int NT, int LAY, int SMB, int TWB>
constexpr size_t tile_smem_bytes() {
    constexpr bool PP = (V == V_PEASE || V == V_PEASE_NC || V == V_STOCKHAM);
    constexpr int TT = 1 << (K - 4);
    constexpr bool ONEBUF = (TQ * TT) / NT == 1;
    const size_t bufs = (PP && !ONEBUF ? 2 : 1) * (size_t)tile_nbase<T, K, TQ, LAY>(TQ) * sizeof(T);
    const size_t head = ((size_t)sizeof(Tw) << SMB) + (TWB ? (size_t)sizeof(Tw) * TQ * tw_row<K>() : 0);
    return ((head + bufs + 15) & ~(size_t)15) + ((LAY == 0 && NTT_TILE_PF_U64 >= (int)sizeof(T) - 4) ? ((size_t)TQ << K) * sizeof(T) : 0);
}


template <class A, int V, int K, int TQ, int NT, int LAY, int SMB, int TWB>
__global__ void __launch_bounds__(NT, ((LAY == TL_SIX_A || LAY == TL_SIX_B || NT >= 1024) ? 1 : (NT <= 256 ? NTT_TILE_MINB256 : 2))) k_tile(TileArgs<A> a) {
    using T = typename A::T;
    using Tw = typename A::Tw;
    using GG = TileGeo<K, TQ>;
    constexpr int TT = GG::TT, G = GG::G, K0 = GG::K0;
    constexpr int CW = fastk::lane_bits<T>();
    constexpr int NP = tile_np<T, K, TQ, LAY>();
    auto nb = [](uint32_t t) -> uint32_t { return tile_nbase<T, K, TQ, LAY>(t); };
    constexpr bool PP = (V == V_PEASE || V == V_PEASE_NC || V == V_STOCKHAM);
    constexpr int REP = (TQ * TT) / NT;             // sub-networks per thread per group
    constexpr int VE = 16 / sizeof(T);              // residues per 16-byte vector
    static_assert(REP >= 1 && REP * NT == TQ * TT, "thread count must divide the tile");
    // ping-pong variants keep ONE work buffer when each thread holds its whole
    // sub-network in registers across a barrier (REP == 1), as in the
    // single-pass kernel; the freed space holds the staged NEXT tile
    constexpr bool ONEBUF = (REP == 1);
    // staged prefetch of the next tile (variant passes; the six-step layouts
    // keep whole sub-transform tables in shared memory and gather directly)
    constexpr bool PF = (LAY == TL_VARIANT) && NTT_TILE_PF_U64 >= (int)sizeof(T) - 4;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ uint32_t Qs[TQ];
    __shared__ uint32_t Is[LAY == TL_COLS ? TQ : 1];   // TL_COLS: column index i of each network
    __shared__ uint64_t Rb[TQ];
    // every layout is additive over disjoint bits: gpos(Q, x) = gpos(Q, 0) + gpos(0, x)
    __shared__ uint64_t GinB[2][TQ], Gout[TQ];
    Tw* tws = reinterpret_cast<Tw*>(smem_raw);
    // per-tile twist tables (only when a.twist): network t, j < 32:
    //   twl[t][j] = w^(Q_t * j), twh[t][j] = w^(Q_t * 32 * j)  (rows odd-padded)
    constexpr int TSL = twc_lo<K>() + 1, TSH = twc_hi<K>() + 1;
    Tw* twl = tws + (1 << SMB);
    Tw* twh = twl + TQ * TSL;
    T* bufA = reinterpret_cast<T*>(smem_raw + ((size_t)sizeof(Tw) << SMB) + (TWB ? (size_t)sizeof(Tw) * TQ * tw_row<K>() : 0));
    T* bufB = (PP && !ONEBUF) ? bufA + nb(TQ) : bufA;
    // staging buffer: the next tile's input, raw gather order, filled by
    // cp.async while the current tile runs its register groups
    // (offset rounded at compile time: an integer round trip of the pointer would turn every
    // staging access into a generic LD instead of LDS)
    constexpr size_t kStageOff = (((size_t)sizeof(Tw) << SMB) + (TWB ? (size_t)sizeof(Tw) * TQ * tw_row<K>() : 0) +
                                  ((PP && !ONEBUF) ? 2 : 1) * (size_t)tile_nbase<T, K, TQ, LAY>(TQ) * sizeof(T) + 15) & ~(size_t)15;
    T* stage = !PF ? nullptr : reinterpret_cast<T*>(smem_raw + kStageOff);
    A ar;
    ar.init(a.p);
    const int L = a.L, S0 = a.S0;
    const int M = (LAY == TL_VARIANT) ? L - K : (LAY == TL_SIX_A ? a.l1 : (LAY == TL_SIX_B ? a.l2 : a.l1 + L - K));
    const uint64_t N = 1ull << L;
    const uint64_t RS = (LAY == TL_COLS) ? (1ull << (L + a.l1)) : N;   // row stride of a batch
    constexpr int LTQ = ilog2c(TQ);
    const int ltpr = M - LTQ;                          // log2 tiles per row
    const uint64_t tiles_per_row = 1ull << ltpr;
    const uint64_t ntiles = a.batch << ltpr;
    const int smb = a.smb < SMB ? a.smb : SMB;
    const uint32_t smlim = 1u << smb;
    for (uint32_t i = threadIdx.x; i < smlim; i += NT) tws[i] = a.gstw[i];
    // twiddle source per register group: smem when every stage of the group is < 2^smb
    auto twsrc = [&](int last_stage) -> TwSrc<Tw> {
        return last_stage <= smb ? TwSrc<Tw>{tws, false} : TwSrc<Tw>{a.gstw, true};
    };
    // local mode: six-step sub-transforms, or a late pass factorised into
    // twist + local transform -- stage twiddles from the local table prefix only
    const bool loc = (LAY == TL_SIX_A || LAY == TL_SIX_B) || a.twist;
    const int S0t = loc ? 0 : S0;
    const int Lg = loc ? K : L;
    // twist factor w^(Q_t * xr) = twl[t][xr mod 32] * twh[t][xr >> 5] applied to v
    auto twistr = [&](T v, uint32_t t, uint32_t xr) -> T {     // xr = the exponent's local index
        if (K <= 5) return ar.mulc(v, twl[t * TSL + xr]);
        return ar.mulc(ar.mulc(v, twl[t * TSL + (xr & 31)]), twh[t * TSH + (xr >> 5)]);
    };
    auto twistv = [&](T v, uint32_t t, uint32_t x) -> T {
        return twistr(v, t, (a.twist == 2) ? x : brev(x, K));
    };

    // network ids of a tile (qmode) -- shared by the prefetch and the tile body
    auto tileQ = [&](uint64_t tl, uint32_t t) -> uint32_t {
        const uint32_t tr = (uint32_t)(tl & (tiles_per_row - 1));
        if (a.qmode == TQM_LINEAR) return tr * TQ + t;
        if (a.qmode == TQM_REV) return brev(tr * TQ + t, M);
        const int hb = LTQ - a.la;
        return (brev(tr * a.TA + (t & (a.TA - 1)), M - hb) << hb) | (t >> a.la);
    };
    // issue the cp.async copies of tile tl into the staging buffer (raw order
    // of the gather loops below: vector i -> stage[i*VE], scalar i -> stage[i])
    auto prefetch = [&](uint64_t tl, const uint64_t* Gin) {
        if (a.vec_in && a.in_order == TO_T_FAST) {
            const uint64_t gb = Gin[(threadIdx.x % (TQ / VE)) * VE];
#pragma unroll 4
            for (uint32_t i = threadIdx.x; i < (uint32_t)(TQ << K) / VE; i += NT) {
                const uint32_t x = i / (TQ / VE);
                cp_async(stage + i * VE, a.in + gb + t_gpos_in<A, V, K, LAY>(a, 0u, x), 16);
            }
        } else if (a.vec_in && a.in_order == TO_C_FAST) {
#pragma unroll 4
            for (uint32_t i = threadIdx.x; i < (uint32_t)(TQ << K) / VE; i += NT) {
                const uint32_t t = i / ((1u << K) / VE), x0 = (i % ((1u << K) / VE)) * VE;
                cp_async(stage + i * VE, a.in + Gin[t] + t_gpos_in<A, V, K, LAY>(a, 0u, x0), 16);
            }
        } else {
#pragma unroll 4
            for (uint32_t i = threadIdx.x; i < (uint32_t)(TQ << K); i += NT) {
                uint32_t t, x;
                if (a.in_order == TO_C_FAST) { t = i >> K; x = i & ((1u << K) - 1); }
                else if (a.in_order == TO_T_FAST) { t = i % TQ; x = i / TQ; }
                else { const int lb = LTQ - a.la; const uint32_t tb = i & ((1u << lb) - 1), ta = (i >> lb) & (a.TA - 1); t = ta + (tb << a.la); x = i / TQ; }
                cp_async(stage + i, a.in + Gin[t] + t_gpos_in<A, V, K, LAY>(a, 0u, x), (int)sizeof(T));
            }
        }
    };
    int pbuf = 0;
    if (threadIdx.x < TQ && (uint64_t)blockIdx.x < ntiles) {
        const uint64_t row = (uint64_t)blockIdx.x >> ltpr;
        GinB[0][threadIdx.x] = row * RS + t_gpos_in<A, V, K, LAY>(a, tileQ(blockIdx.x, threadIdx.x), 0);
    }
    __syncthreads();
    fastk::pdl_trigger();                      // PDL: prologue (plan tables, indices) overlapped;
    fastk::pdl_wait();                         // the previous launch's output visible from here on
    if (PF && (uint64_t)blockIdx.x < ntiles) prefetch(blockIdx.x, GinB[0]);
    cp_async_commit();

    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        __syncthreads();                       // previous tile's scatter done with the work buffers
        if (threadIdx.x < TQ) {
            const int t = threadIdx.x;
            const uint64_t row = tile >> ltpr;
            const uint32_t Q = tileQ(tile, t);
            Qs[t] = (LAY == TL_COLS) ? (Q >> a.l1) : Q;      // twiddle-carrying part
            if (LAY == TL_COLS) Is[t] = Q & ((1u << a.l1) - 1);
            Rb[t] = row * RS;
            Gout[t] = row * RS + t_gpos_out<A, V, K, LAY>(a, Q, 0);
        }
        cp_async_wait_all();
        __syncthreads();                       // staged tile landed (all threads' copies); Qs visible
        if (TWB && a.twist) {                 // per-network twist tables from the main table w^i
            const uint64_t nm = N - 1;
            const int sh = L - S0 - K;
            constexpr uint32_t CL = twc_lo<K>(), CH = K > 5 ? twc_hi<K>() : 0;
            for (uint32_t i = threadIdx.x; i < TQ * (CL + CH); i += NT) {
                const uint32_t t = i / (CL + CH), j = i % (CL + CH);
                const uint32_t Q = Qs[t];
                const uint64_t r = a.tw_rsel ? (uint64_t)(Q >> (L - K - S0)) : (uint64_t)(Q & ((1u << S0) - 1));
                if (j < CL) twl[t * TSL + j] = __ldg(a.tw_lo + (((r * j) << sh) & nm));
                else twh[t * TSH + (j - CL)] = __ldg(a.tw_lo + (((r * 32u * (j - CL)) << sh) & nm));
            }
            __syncthreads();
        }
        // ---- gather (16-byte vectors along the contiguous run when valid)
        if (a.vec_in && a.in_order == TO_T_FAST) {
            const uint64_t gb = GinB[pbuf][(threadIdx.x % (TQ / VE)) * VE];
#pragma unroll 4
            for (uint32_t i = threadIdx.x; i < (uint32_t)(TQ << K) / VE; i += NT) {
                const uint32_t t0 = (i % (TQ / VE)) * VE, x = i / (TQ / VE);
                T tmp[VE];
                *reinterpret_cast<uint4*>(tmp) =
                    PF ? *reinterpret_cast<const uint4*>(stage + i * VE)
                       : __ldg(reinterpret_cast<const uint4*>(a.in + gb + t_gpos_in<A, V, K, LAY>(a, 0u, x)));
                // one position per vector: local index, its padded offset and the twist index
                const uint32_t xl = a.rev_local ? brev(x, K) : x;
                const uint32_t xr = (a.twist == 2) ? xl : brev(xl, K);
                T* db = bufA + nb(t0) + padpos<T>(xl);       // t0 + e stays in t0's (t >> XS) class
#pragma unroll
                for (int e = 0; e < VE; ++e) {
                    T v = tmp[e];
                    if (TWB && a.twist && a.twist < 3) v = twistr(v, t0 + e, xr);
                    db[e * NP] = v;
                }
            }
        } else if (a.vec_in && a.in_order == TO_C_FAST) {
#pragma unroll 4
            for (uint32_t i = threadIdx.x; i < (uint32_t)(TQ << K) / VE; i += NT) {
                const uint32_t t = i / ((1u << K) / VE), x0 = (i % ((1u << K) / VE)) * VE;
                T tmp[VE];
                *reinterpret_cast<uint4*>(tmp) =
                    PF ? *reinterpret_cast<const uint4*>(stage + i * VE)
                       : __ldg(reinterpret_cast<const uint4*>(a.in + GinB[pbuf][t] + t_gpos_in<A, V, K, LAY>(a, 0u, x0)));
                // x0 + e and its K-bit reversal brev(x0) | brev(e) << (K-2) split into a
                // per-vector part and a compile-time part (disjoint bits: padpos is additive)
                constexpr int EB = VE == 4 ? 2 : 1;
                const uint32_t nat0 = x0, rev0 = brev(x0, K);
                T* db = bufA + nb(t) + padpos<T>(a.rev_local ? rev0 : nat0);
#pragma unroll
                for (int e = 0; e < VE; ++e) {
                    const uint32_t ce = (uint32_t)e, cr = brev((uint32_t)e, EB) << (K - EB);
                    T v = tmp[e];
                    if (TWB && a.twist && a.twist < 3) {
                        // twist 1: xr = brev(xl); twist 2: xr = xl
                        const bool xr_rev = (a.twist == 2) == (a.rev_local != 0);
                        v = twistr(v, t, xr_rev ? (rev0 | cr) : (nat0 + ce));
                    }
                    db[padpos<T>(a.rev_local ? cr : ce)] = v;
                }
            }
        } else {
#pragma unroll 4
            for (uint32_t i = threadIdx.x; i < (uint32_t)(TQ << K); i += NT) {
                uint32_t t, x;
                if (a.in_order == TO_C_FAST) { t = i >> K; x = i & ((1u << K) - 1); }
                else if (a.in_order == TO_T_FAST) { t = i % TQ; x = i / TQ; }
                else { const int lb = LTQ - a.la; const uint32_t tb = i & ((1u << lb) - 1), ta = (i >> lb) & (a.TA - 1); t = ta + (tb << a.la); x = i / TQ; }
                T v = PF ? stage[i] : __ldg(a.in + GinB[pbuf][t] + t_gpos_in<A, V, K, LAY>(a, 0u, x));
                if (TWB && a.twist && a.twist < 3) v = twistv(v, t, a.rev_local ? brev(x, K) : x);
                bufA[nb(t) + padpos<T>(a.rev_local ? brev(x, K) : x)] = v;
            }
        }
        __syncthreads();                       // staging consumed, tile in the work buffer
        {                                      // prefetch the next tile behind this one's compute
            const uint64_t nxt = tile + gridDim.x;
            if (nxt < ntiles && !PF) {         // direct gather next time: just its bases
                if (threadIdx.x < TQ)
                    GinB[pbuf ^ 1][threadIdx.x] =
                        (nxt >> ltpr) * RS + t_gpos_in<A, V, K, LAY>(a, tileQ(nxt, threadIdx.x), 0);
            } else if (nxt < ntiles) {
                if (threadIdx.x < TQ)
                    GinB[pbuf ^ 1][threadIdx.x] =
                        (nxt >> ltpr) * RS + t_gpos_in<A, V, K, LAY>(a, tileQ(nxt, threadIdx.x), 0);
                __syncthreads();
                prefetch(nxt, GinB[pbuf ^ 1]);
            }
            cp_async_commit();
            pbuf ^= 1;
        }

        // ---- register groups
        T* src = bufA;
        T* dst = bufB;
#pragma unroll
        for (int g = 0; g < G; ++g) {
            T v[16];
#pragma unroll
            for (int r = 0; r < REP; ++r) {
                const uint32_t tid = threadIdx.x + r * NT;
                const uint32_t t = tid / TT, u = tid % TT;
                const uint32_t Q = loc ? 0u : Qs[t];
                T* sb = src + nb(t);
                T* db = dst + nb(t);
                if (V == V_DIT || V == V_DIF) {
                    const int B = (V == V_DIT) ? (g == 0 ? 0 : K0 + 4 * (g - 1)) : (g == G - 1 ? 0 : K - 4 * (g + 1));
                    const int kg = (V == V_DIT) ? (g == 0 ? K0 : 4) : (g == G - 1 ? K0 : 4);
                    uint32_t pbase = 0;
#define NTT_TMAP(BB)                                                   \
    if (B == BB) {                                                     \
        constexpr Perm PM = plan_lanes(K, BB, CW);                     \
        pbase = scatter_bits<K - 4>(u, PM);                            \
    }
                    NTT_TMAP(0) NTT_TMAP(1) NTT_TMAP(2) NTT_TMAP(3) NTT_TMAP(4) NTT_TMAP(5) NTT_TMAP(6)
                    NTT_TMAP(7) NTT_TMAP(8) NTT_TMAP(9)
#undef NTT_TMAP
                    const uint32_t qlow = loc ? 0u : (Q & ((1u << S0t) - 1));
                    const int b0g = (V == V_DIT) ? (g == 0 ? 0 : B) : (g == G - 1 ? 0 : B);
                    const TwSrc<Tw> tw = twsrc(S0t + b0g + kg);
                    T* wb = sb + padpos<T>(pbase);
#pragma unroll
                    for (int c = 0; c < 16; ++c) v[c] = wb[padpos<T>((uint32_t)c << B)];
#define NTT_TBW(BB, b0v, kgv)                                                                        \
    if (B == BB && kg == kgv) {                                                                        \
        if (tw.global) t_bitwin<A, K, BB, b0v, kgv, V == V_DIF, true>(ar, v, pbase, qlow, S0t, tw.p);  \
        else t_bitwin<A, K, BB, b0v, kgv, V == V_DIF, false>(ar, v, pbase, qlow, S0t, tw.p);           \
    }
                    if ((V == V_DIT && g == 0) || (V == V_DIF && g == G - 1)) {
                        NTT_TBW(0, 0, 1) NTT_TBW(0, 0, 2) NTT_TBW(0, 0, 3) NTT_TBW(0, 0, 4)
                    } else {
                        NTT_TBW(1, 1, 4) NTT_TBW(2, 2, 4) NTT_TBW(3, 3, 4) NTT_TBW(4, 4, 4) NTT_TBW(5, 5, 4)
                        NTT_TBW(6, 6, 4) NTT_TBW(7, 7, 4) NTT_TBW(8, 8, 4) NTT_TBW(9, 9, 4)
                    }
#undef NTT_TBW
#pragma unroll
                    for (int c = 0; c < 16; ++c) wb[padpos<T>((uint32_t)c << B)] = v[c];
                } else if (V != V_STOCKHAM) {
                    const int sg = g == 0 ? 0 : K0 + 4 * (g - 1);
                    const int kg = g == 0 ? K0 : 4;
                    const uint32_t qtop = S0t ? (Q >> (Lg - K - S0t)) : 0u;
                    const TwSrc<Tw> tw = twsrc(S0t + sg + kg);
                    const T* rb = sb + padpos<T>(u << 4);
#pragma unroll
                    for (int c = 0; c < 16; ++c) v[c] = rb[padpos<T>((uint32_t)c)];
#define NTT_TPE(SG, KGV) \
    if (sg == SG && kg == KGV) {                                                 \
        if (tw.global) t_pease<A, K, SG, KGV, true>(ar, v, u, qtop, S0t, tw.p);    \
        else t_pease<A, K, SG, KGV, false>(ar, v, u, qtop, S0t, tw.p);             \
    }
                    if (g == 0) { NTT_TPE(0, 1) NTT_TPE(0, 2) NTT_TPE(0, 3) NTT_TPE(0, 4) }
                    else { NTT_TPE(1, 4) NTT_TPE(2, 4) NTT_TPE(3, 4) NTT_TPE(4, 4) NTT_TPE(5, 4) NTT_TPE(6, 4)
                           NTT_TPE(7, 4) NTT_TPE(8, 4) NTT_TPE(9, 4) }
#undef NTT_TPE
                    if (PP && ONEBUF) __syncthreads();      // every read of the (single) buffer done
                    T* wbo = db + padpos<T>(u << (4 - kg));
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        const uint32_t n = c >> kg, R = c & ((1u << kg) - 1);
                        wbo[padpos<T>(n | (R << (K - kg)))] = v[c];
                    }
                } else {
                    const int sg = g == 0 ? 0 : K0 + 4 * (g - 1);
                    const int kg = g == 0 ? K0 : 4;
                    const int lob = K - sg - kg;
                    const int glob = Lg - S0t - K;
                    const uint32_t ghi = (!loc && S0t) ? (Q >> glob) : 0u;
                    const TwSrc<Tw> tw = twsrc(S0t + sg + kg);
                    uint32_t hi, lo;
                    if (g == 0) { hi = 0; lo = u; }
                    else if (g == G - 1) { hi = u; lo = 0; }
                    else { lo = u & ((1u << lob) - 1); hi = u >> lob; }
                    const T* rb = sb + padpos<T>((hi << (K - sg)) | lo);
#pragma unroll
                    for (int c = 0; c < 16; ++c) v[c] = rb[padpos<T>((uint32_t)c << (lob - (4 - kg)))];
#define NTT_TST(SG, KGV) \
    if (sg == SG && kg == KGV) {                                                  \
        if (tw.global) t_stockham<A, K, SG, KGV, true>(ar, v, hi, ghi, S0t, tw.p);  \
        else t_stockham<A, K, SG, KGV, false>(ar, v, hi, ghi, S0t, tw.p);           \
    }
                    if (g == 0) { NTT_TST(0, 1) NTT_TST(0, 2) NTT_TST(0, 3) NTT_TST(0, 4) }
                    else { NTT_TST(1, 4) NTT_TST(2, 4) NTT_TST(3, 4) NTT_TST(4, 4) NTT_TST(5, 4) NTT_TST(6, 4)
                           NTT_TST(7, 4) NTT_TST(8, 4) NTT_TST(9, 4) }
#undef NTT_TST
                    if (PP && ONEBUF) __syncthreads();
                    T* wbo = db + padpos<T>((hi << lob) | lo);
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        const uint32_t R = (uint32_t)c >> (4 - kg), x = (uint32_t)c & ((1u << (4 - kg)) - 1);
                        wbo[padpos<T>((R << (K - kg)) | (x << (lob - (4 - kg))))] = v[c];
                    }
                }
            }
            __syncthreads();
            if (PP) { T* tmp = src; src = dst; dst = tmp; }
        }
        const T* res = src;   // DIT/DIF: in place (bufA); ping-pong: last written buffer

        // ---- scatter (final reduction, n_inv, six-step correction twiddles)
        auto finish = [&](uint32_t t, uint32_t x, T v) -> T {
            if (TWB && a.twist == 3) v = twistv(v, t, x);
            T r = ar.fin(v);
            if (LAY == TL_SIX_A) {
                const uint64_t e = ((uint64_t)(Qs[t] + a.qoff) * x) & (N - 1);
                const T w = ar.mulfull(__ldg(a.cor_hi + (e >> a.cor_lb)), __ldg(a.cor_lo + (e & ((1ull << a.cor_lb) - 1))));
                r = ar.mulfull(r, w);
            }
            if (LAY == TL_COLS && a.cor_on) {   // w_N^(i * k2), k2 = the column output index (natural order)
                const uint32_t Qj = Qs[t];
                const uint64_t k2 = (Qj & ((1u << a.S0) - 1)) | ((uint64_t)x << a.S0) | ((uint64_t)(Qj >> a.S0) << (a.S0 + K));
                // global column i = qoff + local column (distributed slabs); exponent mod N
                const int lgn = a.cor_lgn ? a.cor_lgn : L + a.l1;
                const uint64_t e = ((uint64_t)(Is[t] + a.qoff) * k2) & ((1ull << lgn) - 1);
                const T w = ar.mulfull(__ldg(a.cor_hi + (e >> a.cor_lb)), __ldg(a.cor_lo + (e & ((1ull << a.cor_lb) - 1))));
                r = ar.mulfull(r, w);
            }
            if (a.scale) r = ar.mulc(r, a.ninv);
            return r;
        };
        if (a.vec_out && a.out_order == TO_T_FAST) {
            const uint64_t gb = Gout[(threadIdx.x % (TQ / VE)) * VE];
#pragma unroll 4
            for (uint32_t i = threadIdx.x; i < (uint32_t)(TQ << K) / VE; i += NT) {
                const uint32_t t0 = (i % (TQ / VE)) * VE, x = i / (TQ / VE);
                T tmp[VE];
#pragma unroll
                for (int e = 0; e < VE; ++e) tmp[e] = finish(t0 + e, x, res[nb(t0 + e) + padpos<T>(x)]);
                *reinterpret_cast<uint4*>(a.out + gb + t_gpos_out<A, V, K, LAY>(a, 0u, x)) =
                    *reinterpret_cast<uint4*>(tmp);
            }
        } else if (a.vec_out && a.out_order == TO_C_FAST) {
#pragma unroll 4
            for (uint32_t i = threadIdx.x; i < (uint32_t)(TQ << K) / VE; i += NT) {
                const uint32_t t = i / ((1u << K) / VE), x0 = (i % ((1u << K) / VE)) * VE;
                T tmp[VE];
#pragma unroll
                for (int e = 0; e < VE; ++e) tmp[e] = finish(t, x0 + e, res[nb(t) + padpos<T>(x0 + e)]);
                *reinterpret_cast<uint4*>(a.out + Gout[t] + t_gpos_out<A, V, K, LAY>(a, 0u, x0)) =
                    *reinterpret_cast<uint4*>(tmp);
            }
        } else {
            for (uint32_t i = threadIdx.x; i < (uint32_t)(TQ << K); i += NT) {
                uint32_t t, x;
                if (a.out_order == TO_C_FAST) { t = i >> K; x = i & ((1u << K) - 1); }
                else if (a.out_order == TO_T_FAST) { t = i % TQ; x = i / TQ; }
                else { const int lb = LTQ - a.la; const uint32_t tb = i & ((1u << lb) - 1), ta = (i >> lb) & (a.TA - 1); t = ta + (tb << a.la); x = i / TQ; }
                a.out[Gout[t] + t_gpos_out<A, V, K, LAY>(a, 0u, x)] = finish(t, x, res[nb(t) + padpos<T>(x)]);
            }
        }
        if (a.counters && threadIdx.x == 0 && tile % tiles_per_row == 0) {
            atomicAdd(a.counters + C_HBM, 1ull);
            if (a.count_row) atomicAdd(a.counters + C_TRANSFORMS, 1ull);
            if (a.count_bitrev) atomicAdd(a.counters + C_BITREV, (unsigned long long)a.count_bitrev);
        }
    }
}

template <class A, int V, int K, int TQ, int NT, int LAY, int SMB, int TWB = 0>
cudaError_t launch_tile(const TileArgs<A>& a, cudaStream_t s, int num_sms, int* launches) {
    using T = typename A::T;
    using Tw = typename A::Tw;
    constexpr bool PP = (V == V_PEASE || V == V_PEASE_NC || V == V_STOCKHAM);
    constexpr size_t smem = tile_smem_bytes<T, Tw, V, K, TQ, NT, LAY, SMB, TWB>();
    if (a.twist && K > 10) return cudaErrorInvalidValue;   // twist tables cover xr < 2^10
    auto kern = k_tile<A, V, K, TQ, NT, LAY, SMB, TWB>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
    const int M = LAY == TL_VARIANT ? a.L - K : (LAY == TL_SIX_A ? a.l1 : (LAY == TL_SIX_B ? a.l2 : a.l1 + a.L - K));
    const uint64_t ntiles = a.batch * ((1ull << M) / TQ);
    uint64_t grid = (uint64_t)num_sms * occ;
    if (grid > ntiles) grid = ntiles;
    if (grid == 0) return cudaSuccess;
    cudaError_t le = fastk::launch_pdl(kern, dim3((unsigned)grid), dim3(NT), smem, s, a);
    if (launches) ++*launches;
    return le != cudaSuccess ? le : cudaGetLastError();
}

}  // namespace ftile
}  // namespace nttb200
