// engine.cuh -- stage-faithful NTT pass kernels for every NTTSuite variant.
//
// A PASS applies a contiguous run of K stages of one variant to a whole
// batch.  The L stages of a size-N transform (L = log2 N) are covered by one
// pass when a polynomial fits in shared memory, or by several HBM passes
// otherwise.  In a pass the residues split into NETWORKS of 2^K elements that
// only interact with each other during those K stages; a CTA stages a TILE
// of TQ networks in shared memory, runs the K stages as register-blocked
// GROUPS of <= 4 stages (each thread owns a closed 2^kg-element sub-network,
// runs kg stages in registers, writes it back; one barrier per group), and
// writes the tile out.  Global positions are tracked exactly, so every
// twiddle exponent is the reference's:
//
//   DIT      algorithms.py:82-121   bit reversal fused into the first gather;
//                                   in-place CT stages 1..L over bit windows
//   DIF      algorithms.py:124-158  in-place GS stages L..1; bit reversal fused
//                                   into the final scatter
//   Flat     algorithms.py:161-195  explicit bit-reverse pass, then radix-2
//                                   stages with the flat r -> (lo,hi) index map
//   Pease    algorithms.py:203-243  constant geometry (read 2r,2r+1 / write
//                                   r,r+N/2) + a copy-back after every group/pass
//   Pease_nc algorithms.py:246-261  same stages, buffers swap roles (no copy)
//   Stockham algorithms.py:264-301  self-sorting ping-pong, never bit-reverses
//
// All arithmetic is canonical (arith.cuh): each stage's buffer equals the
// reference's buffer after that stage, bit for bit.
#pragma once
#include <cstdint>
#include "arith.cuh"

namespace nttb200 {

enum Variant { V_NAIVE = 0, V_DIT = 1, V_DIF = 2, V_FLAT = 3, V_PEASE = 4, V_PEASE_NC = 5,
               V_STOCKHAM = 6, V_SIXSTEP = 7 };

enum CounterIdx { C_TRANSFORMS = 0, C_BITREV = 1, C_COPIES = 2, C_HBM = 3, C_NCOUNTERS = 4 };

constexpr int kThreads = 256;
constexpr int kMaxKG = 4;   // register sub-network = 16 residues per thread

// XOR-fold swizzle of a position inside one network: bank bits ^= fold of the
// upper bits.  Linear over GF(2); a bijection on [0, 2^K).
template <class T>
NTT_D uint32_t swz(uint32_t pos) {
    constexpr int CW = sizeof(T) == 4 ? 5 : 4;
    uint32_t u = pos >> CW;
    uint32_t f = u ^ (u >> CW) ^ (u >> (2 * CW));
    return pos ^ (f & ((1u << CW) - 1));
}

NTT_D uint32_t brev(uint32_t x, int L) { return L ? (__brev(x) >> (32 - L)) : 0u; }

template <class Tw>
NTT_D Tw ldtw(const Tw* tw, uint32_t e) { return __ldg(tw + e); }

// Shared-memory slot of element c of tile network t (2^K elements each).
template <class T>
NTT_D uint32_t slot(uint32_t t, uint32_t c, int K) {
    constexpr uint32_t M = sizeof(T) == 4 ? 31u : 15u;
    return (t << K) + (swz<T>(c) ^ ((t & M) & ((1u << K) - 1)));
}

// Where the tile's networks sit in the whole transform.
struct GCtx {
    int L;        // global log2 N
    int K;        // log2 network size in this pass
    int S0;       // DIT/DIF: global bit offset of local bit 0; Pease/Stockham: stages before this pass
    const uint32_t* Q;   // global network id of each tile network (shared memory)
};

// ------------------------------------------------------------- groups ----

// DIT / DIF group over the LOCAL bit window [b0, b0+KG) of each network.
// Global position of local position x of network Q:
//   g = (Q mod 2^S0) | x << S0 | (Q >> S0) << (S0+K);  stage s = S0 + b0 + 1 + j,
//   twiddle exponent (g mod 2^(s-1)) * N/2^s == (g << (L-s)) & (N/2-1)
//   (algorithms.py:97-99, 141-143).
template <class F, int KG, bool DIF>
NTT_D void bitwin_group(const F& f, const typename F::T* src, typename F::T* dst, const GCtx& g, int b0,
                        const typename F::Tw* tw, int TQ, bool rev_in, bool rev_out) {
    using T = typename F::T;
    const int K = g.K, L = g.L;
    const int qb = K - KG;
    const uint32_t emask = (1u << (L - 1)) - 1;
    const int nn = TQ << qb;
    for (int qq = threadIdx.x; qq < nn; qq += blockDim.x) {
        const uint32_t t = qq >> qb, u = qq & ((1u << qb) - 1);
        const uint32_t Q = g.Q ? g.Q[t] : 0u;
        const uint32_t gb = (Q & ((1u << g.S0) - 1)) | ((Q >> g.S0) << (g.S0 + K));
        const uint32_t base = (u & ((1u << b0) - 1)) | ((u >> b0) << (b0 + KG));
        T v[1 << KG];
#pragma unroll
        for (int c = 0; c < (1 << KG); ++c) {
            uint32_t x = base | ((uint32_t)c << b0);
            v[c] = src[slot<T>(t, rev_in ? brev(x, K) : x, K)];
        }
        if (!DIF) {
#pragma unroll
            for (int j = 0; j < KG; ++j) {
                const int s = g.S0 + b0 + 1 + j;
#pragma unroll
                for (int c = 0; c < (1 << KG); ++c) {
                    if (c & (1 << j)) continue;
                    const uint32_t gp = gb | ((base | ((uint32_t)c << b0)) << g.S0);
                    const uint32_t e = (gp << (L - s)) & emask;
                    T tt = f.mul(v[c | (1 << j)], ldtw(tw, e));
                    T a = v[c];
                    v[c] = f.add(a, tt);
                    v[c | (1 << j)] = f.sub(a, tt);
                }
            }
        } else {
#pragma unroll
            for (int j = KG - 1; j >= 0; --j) {
                const int s = g.S0 + b0 + 1 + j;
#pragma unroll
                for (int c = 0; c < (1 << KG); ++c) {
                    if (c & (1 << j)) continue;
                    const uint32_t gp = gb | ((base | ((uint32_t)c << b0)) << g.S0);
                    const uint32_t e = (gp << (L - s)) & emask;
                    T a = v[c], b = v[c | (1 << j)];
                    v[c] = f.add(a, b);
                    v[c | (1 << j)] = f.mul(f.sub(a, b), ldtw(tw, e));
                }
            }
        }
#pragma unroll
        for (int c = 0; c < (1 << KG); ++c) {
            uint32_t x = base | ((uint32_t)c << b0);
            dst[slot<T>(t, rev_out ? brev(x, K) : x, K)] = v[c];
        }
    }
}

// Pease constant-geometry group: local stages sg+1 .. sg+KG of this pass
// (global stages S0+sg+1 ..).  Sub-network u reads the contiguous local block
// u*2^KG + c and writes positions u | R << (K-KG); in registers the same
// constant geometry runs: v[2i], v[2i+1] -> nv[i], nv[i + 2^(KG-1)].
// Global position after m_tot local stages of local position x:
//   g = Q << (K-m_tot) | (x mod 2^(K-m_tot)) | (x >> (K-m_tot)) << (L-m_tot)
// and butterfly r = g >> 1 of stage s uses e = (r >> (L-s)) << (L-s)
// (algorithms.py:216-217).
template <class F, int KG>
NTT_D void pease_group(const F& f, const typename F::T* src, typename F::T* dst, const GCtx& g, int sg,
                       const typename F::Tw* tw, int TQ, bool rev_in) {
    using T = typename F::T;
    const int K = g.K, L = g.L;
    const int qb = K - KG;
    constexpr int H = 1 << (KG - 1);
    const int nn = TQ << qb;
    for (int qq = threadIdx.x; qq < nn; qq += blockDim.x) {
        const uint32_t t = qq >> qb, u = qq & ((1u << qb) - 1);
        const uint32_t Q = g.Q ? g.Q[t] : 0u;
        T v[1 << KG];
#pragma unroll
        for (int c = 0; c < (1 << KG); ++c) {
            uint32_t x = (u << KG) | (uint32_t)c;
            v[c] = src[slot<T>(t, rev_in ? brev(x, K) : x, K)];
        }
#pragma unroll
        for (int m = 0; m < KG; ++m) {
            const int mt = sg + m;                 // local stages done in this pass
            const int s = g.S0 + mt + 1;           // global stage
            T nv[1 << KG];
#pragma unroll
            for (int i = 0; i < H; ++i) {
                const uint32_t R = 2u * i;
                const uint32_t x = (u << (KG - m)) | (R & ((1u << (KG - m)) - 1)) | ((R >> (KG - m)) << (K - m));
                const uint32_t gp = (Q << (K - mt)) | (x & ((1u << (K - mt)) - 1)) | ((x >> (K - mt)) << (L - mt));
                const uint32_t e = (gp >> (L - s + 1)) << (L - s);
                T tt = f.mul(v[2 * i + 1], ldtw(tw, e));
                nv[i] = f.add(v[2 * i], tt);
                nv[i + H] = f.sub(v[2 * i], tt);
            }
#pragma unroll
            for (int c = 0; c < (1 << KG); ++c) v[c] = nv[c];
        }
#pragma unroll
        for (int R = 0; R < (1 << KG); ++R) dst[slot<T>(t, u | ((uint32_t)R << (K - KG)), K)] = v[R];
    }
}

// Stockham group: local stages sg .. sg+KG-1 (0-based; global s = S0 + sg + m).
// Stage s pairs position bit L-s-1 and moves the butterfly's output bit to
// the top, [j | b | i] -> [b | j | i]; twiddle w[j * N/2^(s+1)] with
// j = top s bits of the position (algorithms.py:281-299).  Globally the tile
// network Q = hi (S0 bits) | lo: position = [local top bits | hi | local rest | lo].
template <class F, int KG>
NTT_D void stockham_group(const F& f, const typename F::T* src, typename F::T* dst, const GCtx& g, int sg,
                          const typename F::Tw* tw, int TQ) {
    using T = typename F::T;
    const int K = g.K, L = g.L;
    const int qb = K - KG;
    const int lob = K - sg - KG;               // local low bits below the group's pair bits
    const int glob = L - g.S0 - K;             // global low bits of Q
    constexpr int H = 1 << (KG - 1);
    const int nn = TQ << qb;
    for (int qq = threadIdx.x; qq < nn; qq += blockDim.x) {
        const uint32_t t = qq >> qb, u = qq & ((1u << qb) - 1);
        const uint32_t Q = g.Q ? g.Q[t] : 0u;
        const uint32_t ghi = Q >> glob;
        const uint32_t hi = u >> lob, lo = u & ((1u << lob) - 1);
        T v[1 << KG];
#pragma unroll
        for (int c = 0; c < (1 << KG); ++c)
            v[c] = src[slot<T>(t, (hi << (K - sg)) | ((uint32_t)c << lob) | lo, K)];
#pragma unroll
        for (int m = 0; m < KG; ++m) {
            const int s = g.S0 + sg + m;
            T nv[1 << KG];
#pragma unroll
            for (int i = 0; i < H; ++i) {
                const uint32_t B = i & ((1u << m) - 1), crest = (uint32_t)i >> m;
                const uint32_t jl = (B << sg) | hi;                  // local top (sg+m) bits
                const uint32_t j = (jl << g.S0) | ghi;               // global top s bits
                const uint32_t e = j << (L - s - 1);
                T a = v[i];
                T tt = f.mul(v[i + H], ldtw(tw, e));
                nv[(crest << (m + 1)) | B] = f.add(a, tt);
                nv[(crest << (m + 1)) | (1u << m) | B] = f.sub(a, tt);
            }
#pragma unroll
            for (int c = 0; c < (1 << KG); ++c) v[c] = nv[c];
        }
#pragma unroll
        for (int R = 0; R < (1 << KG); ++R)
            dst[slot<T>(t, ((uint32_t)R << (K - KG)) | (hi << lob) | lo, K)] = v[R];
    }
}

// Flat stage (algorithms.py:176-194): one butterfly per flat index r, over
// local bit b (global stage s = S0 + b + 1), in place.
template <class F>
NTT_D void flat_stage(const F& f, typename F::T* buf, const GCtx& g, int b, const typename F::Tw* tw, int TQ) {
    using T = typename F::T;
    const int K = g.K, L = g.L;
    const int s = g.S0 + b + 1;
    const uint32_t half = 1u << (K - 1);
    const uint32_t kmask = (1u << b) - 1;
    const uint32_t emask = (1u << (L - 1)) - 1;
    for (uint32_t rr = threadIdx.x; rr < (uint32_t)TQ * half; rr += blockDim.x) {
        const uint32_t t = rr >> (K - 1), r = rr & (half - 1);
        const uint32_t Q = g.Q ? g.Q[t] : 0u;
        const uint32_t gb = (Q & ((1u << g.S0) - 1)) | ((Q >> g.S0) << (g.S0 + K));
        const uint32_t k = r & kmask;
        const uint32_t lo = ((r >> b) << (b + 1)) + k, hi = lo + (1u << b);
        const uint32_t gp = gb | (lo << g.S0);
        const uint32_t e = (gp << (L - s)) & emask;      // == stride * k for a whole-row pass
        T tt = f.mul(buf[slot<T>(t, hi, K)], ldtw(tw, e));
        T a = buf[slot<T>(t, lo, K)];
        buf[slot<T>(t, lo, K)] = f.add(a, tt);
        buf[slot<T>(t, hi, K)] = f.sub(a, tt);
    }
}

// Group schedule: K stages in groups of <= kMaxKG, the SHORT group first.
NTT_HD int group_schedule(int K, int* kg) {
    int G = (K + kMaxKG - 1) / kMaxKG;
    kg[0] = K - kMaxKG * (G - 1);
    for (int i = 1; i < G; ++i) kg[i] = kMaxKG;
    return G;
}

template <class F>
NTT_D void dispatch_bitwin(int kg, bool dif, const F& f, const typename F::T* s, typename F::T* d,
                           const GCtx& g, int b0, const typename F::Tw* tw, int TQ, bool ri, bool ro) {
#define NTT_BW(KGV)                                                                       \
    if (dif) bitwin_group<F, KGV, true>(f, s, d, g, b0, tw, TQ, ri, ro);                  \
    else bitwin_group<F, KGV, false>(f, s, d, g, b0, tw, TQ, ri, ro);
    switch (kg) {
        case 1: NTT_BW(1) break;
        case 2: NTT_BW(2) break;
        case 3: NTT_BW(3) break;
        default: NTT_BW(4) break;
    }
#undef NTT_BW
}

template <class F>
NTT_D void dispatch_pease(int kg, const F& f, const typename F::T* s, typename F::T* d, const GCtx& g, int sg,
                          const typename F::Tw* tw, int TQ, bool ri) {
    switch (kg) {
        case 1: pease_group<F, 1>(f, s, d, g, sg, tw, TQ, ri); break;
        case 2: pease_group<F, 2>(f, s, d, g, sg, tw, TQ, ri); break;
        case 3: pease_group<F, 3>(f, s, d, g, sg, tw, TQ, ri); break;
        default: pease_group<F, 4>(f, s, d, g, sg, tw, TQ, ri); break;
    }
}

template <class F>
NTT_D void dispatch_stockham(int kg, const F& f, const typename F::T* s, typename F::T* d, const GCtx& g,
                             int sg, const typename F::Tw* tw, int TQ) {
    switch (kg) {
        case 1: stockham_group<F, 1>(f, s, d, g, sg, tw, TQ); break;
        case 2: stockham_group<F, 2>(f, s, d, g, sg, tw, TQ); break;
        case 3: stockham_group<F, 3>(f, s, d, g, sg, tw, TQ); break;
        default: stockham_group<F, 4>(f, s, d, g, sg, tw, TQ); break;
    }
}

// Runs the K local stages of `V` on the tile held in A (B = second buffer).
// Returns the buffer holding the result; *copies counts Pease copy-backs.
// rev_first: the first group gathers through the bit reversal (single-pass
// DIT / Pease); rev_last: the last group scatters through it (single-pass DIF).
template <class F, int V>
NTT_D typename F::T* tile_stages(const F& f, typename F::T* A, typename F::T* B, const GCtx& g,
                                 const typename F::Tw* tw, int TQ, bool rev_first, bool rev_last,
                                 int* copies) {
    using T = typename F::T;
    int kg[8];
    const int G = group_schedule(g.K, kg);
    const int span = TQ << g.K;
    if (V == V_DIT) {
        int b0 = 0;
        T* res = A;
        for (int i = 0; i < G; ++i) {
            T* src = res;
            T* dst = (i == 0 && rev_first) ? B : res;
            dispatch_bitwin<F>(kg[i], false, f, src, dst, g, b0, tw, TQ, i == 0 && rev_first, false);
            res = dst;
            b0 += kg[i];
            __syncthreads();
        }
        return res;
    } else if (V == V_DIF) {
        int b0 = g.K;
        T* res = A;
        for (int i = G - 1; i >= 0; --i) {
            b0 -= kg[i];
            const bool ro = (i == 0) && rev_last;
            T* dst = ro ? B : res;
            dispatch_bitwin<F>(kg[i], true, f, res, dst, g, b0, tw, TQ, false, ro);
            res = dst;
            __syncthreads();
        }
        return res;
    } else if (V == V_FLAT) {
        T* res = A;
        if (rev_first) {              // bit_reverse_permute as its own pass (algorithms.py:174)
            for (uint32_t i = threadIdx.x; i < (uint32_t)span; i += blockDim.x) {
                const uint32_t t = i >> g.K, x = i & ((1u << g.K) - 1);
                B[slot<T>(t, x, g.K)] = A[slot<T>(t, brev(x, g.K), g.K)];
            }
            __syncthreads();
            res = B;
        }
        for (int b = 0; b < g.K; ++b) {
            flat_stage<F>(f, res, g, b, tw, TQ);
            __syncthreads();
        }
        return res;
    } else if (V == V_PEASE || V == V_PEASE_NC) {
        T* src = A;
        T* dst = B;
        int sg = 0;
        for (int i = 0; i < G; ++i) {
            dispatch_pease<F>(kg[i], f, src, dst, g, sg, tw, TQ, i == 0 && rev_first);
            sg += kg[i];
            __syncthreads();
            if (V == V_PEASE) {           // _stage_copy(cur, nxt)  (algorithms.py:242)
                for (int k = threadIdx.x; k < span; k += blockDim.x) src[k] = dst[k];
                ++*copies;
                __syncthreads();
            } else {                      // src, dst = dst, src    (algorithms.py:260)
                T* tmp = src; src = dst; dst = tmp;
            }
        }
        return src;
    } else {  // V_STOCKHAM
        T* src = A;
        T* dst = B;
        int sg = 0;
        for (int i = 0; i < G; ++i) {
            dispatch_stockham<F>(kg[i], f, src, dst, g, sg, tw, TQ);
            sg += kg[i];
            __syncthreads();
            T* tmp = src; src = dst; dst = tmp;
        }
        return src;
    }
}

}  // namespace nttb200
