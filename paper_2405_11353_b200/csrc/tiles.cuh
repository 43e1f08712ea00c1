// tiles.cuh -- host planner chaining fasttile.cuh passes (multi-pass N and
// the six-step split).  Instantiated in kt_f32.cu / kt_gold.cu.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include "fasttile.cuh"
#include "colpass.cuh"
#include "multipass.cuh"

namespace nttb200 {

template <class F>
inline typename F::Tw make_tw2(uint64_t w, uint64_t ws);
template <> inline uint2 make_tw2<F32S>(uint64_t w, uint64_t ws) { return make_uint2((uint32_t)w, (uint32_t)ws); }
template <> inline uint64_t make_tw2<FGold>(uint64_t w, uint64_t) { return w; }

template <class T>
__global__ void k_copy_rows(const T* src, T* dst, uint64_t n, uint64_t rows, unsigned long long* counters) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0 && (n * sizeof(T)) % 16 == 0) {
        const uint64_t n4 = n * sizeof(T) / 16;
        for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += stride)
            reinterpret_cast<uint4*>(dst)[i] = __ldg(reinterpret_cast<const uint4*>(src) + i);
    } else {                                   // caller buffers only element-aligned
        for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = src[i];
    }
    if (counters && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(counters + C_COPIES, (unsigned long long)rows);
}

namespace ftile {

// Compile-time tile shapes: residues per tile = 2^TE (u32: 2^13, u64: 2^12),
// except u32 K = 10 passes: 2^14 (TQ = 16 networks, one 1024-thread CTA per
// SM) -- the strided HBM side then moves 64-byte runs instead of 32-byte ones
// (a 32-byte-run strided write pass cannot beat 2.2 TB/s).
#ifndef NTT_TILE_E32_K10
#define NTT_TILE_E32_K10 14
#endif
#ifndef NTT_TILE_E64
#define NTT_TILE_E64 12
#endif
constexpr int tile_e_rt(int word, int K) { return word == 4 ? (K == 10 ? NTT_TILE_E32_K10 : 13) : NTT_TILE_E64; }
template <class T, int K>
constexpr int tile_e() { return tile_e_rt((int)sizeof(T), K); }
template <class T, int K>
constexpr int tile_tq() { return 1 << (tile_e<T, K>() - K); }
template <class T, int K>
constexpr int tile_nt() { return (tile_tq<T, K>() << (K - 4)) < 1024 ? (tile_tq<T, K>() << (K - 4)) : 1024; }
constexpr int kSmb = 11;

template <class A, int V, int K>
cudaError_t pass_k(const TileArgs<A>& a, cudaStream_t s, int sms, int* launches) {
    using T = typename A::T;
    constexpr int TWB = sizeof(T) == 4 ? 10 : 0;    // twist tables for the u32 late pass
    return launch_tile<A, V, K, tile_tq<T, K>(), tile_nt<T, K>(), TL_VARIANT, kSmb, TWB>(a, s, sms, launches);
}

template <class A, int V>
cudaError_t pass_any(int K, const TileArgs<A>& a, cudaStream_t s, int sms, int* launches, bool* ok) {
    using T = typename A::T;
    *ok = true;
    if (sizeof(T) == 4) {
        switch (K) {
            case 6: return pass_k<A, V, 6>(a, s, sms, launches);
            case 7: return pass_k<A, V, 7>(a, s, sms, launches);
            case 8: return pass_k<A, V, 8>(a, s, sms, launches);
            case 9: return pass_k<A, V, 9>(a, s, sms, launches);
            case 10: return pass_k<A, V, 10>(a, s, sms, launches);
        }
    } else {
        switch (K) {
            case 6: return pass_k<A, V, 6>(a, s, sms, launches);     // (2^19, 2^20: three passes of 7 / 6 stages)
            case 7: return pass_k<A, V, 7>(a, s, sms, launches);
            case 8: return pass_k<A, V, 8>(a, s, sms, launches);
            case 9: return pass_k<A, V, 9>(a, s, sms, launches);
        }
    }
    *ok = false;
    return cudaSuccess;
}


// Pass plan.  Tiles hold 2^13 (u32) / 2^12 (u64) residues, so a pass of K
// stages has TQ = 2^(13-K) networks and every strided HBM side moves runs of
// TQ residues.  Measured on B200 (profiles/r1/summary.md): a 3-pass 2^20 plan
// with 256 B runs (K = 7,7,6) ran 9-11 ms against 4.6 ms for 2 passes of
// K = 10 with 32 B runs: the TQ >= 32 tiles fit one CTA per SM and their
// 8-thread networks share warps with bank-conflicting strides.  So: fewest
// passes, K <= 10.
inline int tile_plan(int L, int word, int* K) {
    const int kmax = word == 4 ? 10 : 9;
    const int kmin = 6;
    int P = (L + kmax - 1) / kmax;
    if (P < 2) P = 2;
    for (int i = 0; i < P; ++i) K[i] = L / P + (i < L % P ? 1 : 0);
    for (int i = 0; i < P; ++i)
        if (K[i] < kmin || K[i] > 10) return 0;
    return P;
}

template <class A>
TileArgs<A> tile_base(const MultipassReq& r) {
    TileArgs<A> a{};
    a.batch = r.batch;
    a.L = r.L;
    a.gstw = static_cast<const typename A::Tw*>(r.stw);
    a.smb = kSmb;
    a.p = r.p;
    a.ninv = make_tw2<typename A::Field>(r.ninv, r.ninv_shoup);
    a.counters = r.counters;
    a.TA = 1;
    return a;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Multi-pass transform by compile-time tile kernels.  *ok = false when no
// tile shape covers this (L, word): the caller uses the generic engine.
template <class A, int V>
cudaError_t run_tile_passes(const MultipassReq& r, bool* ok) {
    using T = typename A::T;
    *ok = false;
    if (!r.stw || V == V_NAIVE || V == V_SIXSTEP) return cudaSuccess;
    int K[8];
    const int P = tile_plan(r.L, sizeof(T), K);
    if (!P) return cudaSuccess;
    const int L = r.L;
    const uint64_t N = 1ull << L;
    constexpr int VE = 16 / sizeof(T);
    T* ws0 = static_cast<T*>(r.ws);
    T* ws1 = ws0 + r.batch * N;
    const T* cur = static_cast<const T*>(r.in);
    const bool al = aligned16(r.in) && aligned16(r.out) && aligned16(r.ws);
    // four-step factorisation of the later passes (u32): the network-dependent
    // stage twiddles become one per-element twist W^(r*x'), docs/PASS_ALGEBRA.md
    const bool fac = sizeof(T) == 4;
    // Pease with >= 3 passes: the reference's separate bit_reverse_permute pass
    // (algorithms.py:238,255) as a 64x64 transpose, so every Pease pass reads
    // contiguous networks and writes TQ-residue runs; 2-pass Pease fuses the
    // reversal into the first gather and writes a row-bit-reversed transpose
    const bool pease = (V == V_PEASE || V == V_PEASE_NC);
    const bool sep_bitrev = (V == V_FLAT) || (pease && P >= 3);
    cudaError_t e = cudaSuccess;
    if (sep_bitrev) {
        uint64_t blocks = r.batch << (L - 12);
        uint64_t cap = (uint64_t)r.num_sms * 8;
        k_bitrev<T><<<(unsigned)(blocks < cap ? blocks : cap), 256, 0, r.stream>>>(cur, ws1, r.batch, L, r.counters);
        if (r.launches) ++*r.launches;
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        cur = ws1;
    }
    int done = 0;
    for (int i = 0; i < P; ++i) {
        const bool last = (i == P - 1);
        T* dst = last ? static_cast<T*>(r.out) : ((cur == ws0) ? ws1 : ws0);
        if (V == V_PEASE && !last) dst = ws0;
        TileArgs<A> a = tile_base<A>(r);
        a.in = cur;
        a.out = dst;
        a.count_row = last;
        a.scale = last ? r.scale : 0;
        int k = K[i];
        const int tq = 1 << (tile_e_rt((int)sizeof(T), k) - k);
        bool okp = false;
        if (fac) a.tw_lo = static_cast<const typename A::Tw*>(r.tw);     // main table w^i
        if (V == V_DIT || V == V_FLAT) {
            a.S0 = done;
            if (i == 0 && V == V_DIT) {
                a.qmode = TQM_REV; a.rev_in = 1; a.in_order = TO_T_FAST; a.out_order = TO_C_FAST; a.count_bitrev = 1;
            } else if (i == 0) {
                a.qmode = TQM_LINEAR; a.in_order = TO_C_FAST; a.out_order = TO_C_FAST;
            } else {
                a.qmode = TQM_LINEAR; a.in_order = TO_T_FAST; a.out_order = TO_T_FAST;
            }
            a.vec_in = a.vec_out = al && tq >= VE;
            if (fac && i > 0) { a.twist = 1; a.tw_rsel = 0; }
            e = pass_any<A, V_DIT>(k, a, r.stream, r.num_sms, r.launches, &okp);
            done += k;
        } else if (V == V_DIF) {
            k = K[P - 1 - i];
            a.S0 = L - done - k;
            if (last) {
                a.qmode = TQM_REV; a.rev_out = 1; a.in_order = TO_C_FAST; a.out_order = TO_T_FAST; a.count_bitrev = 1;
            } else {
                a.qmode = TQM_LINEAR; a.in_order = TO_T_FAST; a.out_order = TO_T_FAST;
            }
            a.vec_in = a.vec_out = al && (1 << (tile_e_rt((int)sizeof(T), k) - k)) >= VE;
            if (fac && !last) { a.twist = 3; a.tw_rsel = 0; }
            e = pass_any<A, V_DIF>(k, a, r.stream, r.num_sms, r.launches, &okp);
            done += k;
        } else if (pease) {
            a.S0 = done;
            if (sep_bitrev) {
                a.qmode = TQM_LINEAR; a.in_order = TO_C_FAST; a.out_order = TO_T_FAST;
                a.vec_in = al;
                a.vec_out = al && tq >= VE;
                if (i == 0) a.count_bitrev = 0;
                if (fac && i > 0) { a.twist = 1; a.tw_rsel = 1; }
            } else if (i == 0) {
                // P == 2: networks with consecutive rev(Q); the stage state is
                // written row-bit-reversed-transposed (out_trb), pass 1 undoes it
                a.qmode = TQM_REV; a.rev_in = 1; a.out_trb = 1;
                a.in_order = TO_T_FAST; a.out_order = TO_T_FAST; a.count_bitrev = 1;
                a.vec_in = a.vec_out = al && tq >= VE;
            } else {
                a.qmode = TQM_LINEAR; a.in_order = TO_C_FAST; a.out_order = TO_T_FAST;
                a.rev_local = 1;
                a.vec_in = al;
                a.vec_out = al && tq >= VE;
                if (fac) { a.twist = 1; a.tw_rsel = 1; }
            }
            e = pass_any<A, V_PEASE_NC>(k, a, r.stream, r.num_sms, r.launches, &okp);
            done += k;
        } else {  // Stockham
            a.S0 = done;
            a.qmode = TQM_LINEAR;
            const int glob = L - done - k;
            a.in_order = glob > 0 ? TO_T_FAST : TO_C_FAST;
            a.out_order = TO_T_FAST;
            a.vec_in = al && (glob == 0 || (1 << glob) >= VE) && tq >= VE;
            a.vec_out = al && tq >= VE;
            if (fac && i > 0) { a.twist = 2; a.tw_rsel = 1; }
            e = pass_any<A, V_STOCKHAM>(k, a, r.stream, r.num_sms, r.launches, &okp);
            done += k;
        }
        if (e != cudaSuccess) return e;
        if (!okp) return cudaErrorInvalidValue;      // tile_plan guarantees coverage
        if (V == V_PEASE) {                          // _stage_copy per pass (algorithms.py:242)
            k_copy_rows<T><<<r.num_sms * 4, 256, 0, r.stream>>>(dst, ws1, r.batch * N, r.batch, r.counters);
            if (r.launches) ++*r.launches;
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
            dst = ws1;
        }
        cur = dst;
    }
    *ok = true;
    return cudaSuccess;
}

// Six-step split by tile kernels (Goldilocks; algorithms.py:355-389), also
// the rank-local steps of the distributed four-step: rank g of G owns input
// columns i in [g*n1/G, (g+1)*n1/G) as a slab x_local[j][i_local] and, after
// the all-to-all, output columns k2 in [g*n2/G, ...) as out_local[k1][k2_local].
template <int K>
constexpr int six_tq() { return K >= 10 ? 2 : 4; }
template <int K>
constexpr int six_nt() { return (six_tq<K>() << (K - 4)) < 512 ? (six_tq<K>() << (K - 4)) : 512; }

template <class A, int K1, int K2>
cudaError_t sixstep_step_a(const MultipassReq& r, int rank, int world, const void* in, void* out) {
    using T = typename A::T;
    int lg = 0;
    while ((1 << lg) < world) ++lg;
    TileArgs<A> a = tile_base<A>(r);
    a.in = static_cast<const T*>(in);
    a.out = static_cast<T*>(out);
    a.l1 = K1 - lg;                     // local columns n1/G
    a.l2 = K2;
    a.pb = K2 - lg;                     // n2/G per destination
    a.pblk = 1ull << (K1 - lg + K2 - lg);
    a.qoff = (uint32_t)rank << (K1 - lg);
    a.S0 = 0;
    a.gstw = static_cast<const typename A::Tw*>(r.stw2);
    a.smb = K2;
    a.qmode = TQM_LINEAR; a.in_order = TO_T_FAST; a.out_order = TO_C_FAST;
    a.rev_local = 1;                    // bit_reverse_permute(row) (algorithms.py:374)
    a.vec_in = 0;
    a.vec_out = aligned16(out) && lg == 0;
    a.cor_lo = static_cast<const T*>(r.cor_lo);
    a.cor_hi = static_cast<const T*>(r.cor_hi);
    a.cor_lb = r.cor_lb;
    return launch_tile<A, V_DIT, K2, six_tq<K2>(), six_nt<K2>(), TL_SIX_A, K2>(a, r.stream, r.num_sms, r.launches);
}

template <class A, int K1, int K2>
cudaError_t sixstep_step_b(const MultipassReq& r, int world, const void* in, void* out) {
    using T = typename A::T;
    int lg = 0;
    while ((1 << lg) < world) ++lg;
    TileArgs<A> a = tile_base<A>(r);
    a.in = static_cast<const T*>(in);
    a.out = static_cast<T*>(out);
    a.l1 = K1;
    a.l2 = K2 - lg;                     // rows of n2/G columns
    a.S0 = 0;
    a.gstw = static_cast<const typename A::Tw*>(r.stw1);
    a.smb = K1;
    a.qmode = TQM_LINEAR; a.in_order = TO_T_FAST; a.out_order = TO_T_FAST;
    a.rev_local = 1;                    // bit_reverse_permute(col) (algorithms.py:385)
    a.vec_in = a.vec_out = 0;
    a.count_row = 1;
    a.scale = r.scale;
    return launch_tile<A, V_DIT, K1, six_tq<K1>(), six_nt<K1>(), TL_SIX_B, K1>(a, r.stream, r.num_sms, r.launches);
}

template <class A, int K1, int K2>
cudaError_t run_sixstep_tiles_k(const MultipassReq& r) {
    cudaError_t e = sixstep_step_a<A, K1, K2>(r, 0, 1, r.in, r.ws);
    if (e != cudaSuccess) return e;
    return sixstep_step_b<A, K1, K2>(r, 1, r.ws, r.out);
}

// ------------------------------------------------------------------------
// Six-step with long HBM runs (algorithms.py:371-389, x[j*n1 + i]):
//   step A: DIT over j (length n2) of EVERY column at once -- TL_COLS tiles
//           hold TQ consecutive columns i, so both HBM sides move TQ-residue
//           runs (the column-at-a-time layout TL_SIX_A moves 16-byte runs);
//           bit_reverse_permute(col) fused into the first gather, the
//           correction w_N^(i*k2) into the last scatter;
//   the six-step's transpose, as its own 32x32-tiled pass;
//   step B: DIT over i (length n1) for every k2, TL_COLS again (inner k2),
//           whose natural-order output IS out[k1*n2 + k2].
// Each length-2^b step is one pass (b <= 9) or two (b = 12, 13: 6+6, 7+6).
inline int cols_split(int b, int* K, int word = 4) {
    if (b >= 6 && b <= 9) { K[0] = b; return 1; }
    if (word == 8) {       // 64-bit fields (colpass.cuh tiles of 2^5..2^8 rows): every length up to 2^16
        if (b == 10) { K[0] = 5; K[1] = 5; return 2; }
        if (b == 11) { K[0] = 6; K[1] = 5; return 2; }
        if (b >= 14 && b <= 16) { K[0] = (b + 1) / 2; K[1] = b / 2; return 2; }
    }
#ifndef NTT_COLS_SPLIT_SWAP
#define NTT_COLS_SPLIT_SWAP 0
#endif
    if (b == 12 || b == 13) {
        K[0] = NTT_COLS_SPLIT_SWAP ? 6 : b - 6;
        K[1] = NTT_COLS_SPLIT_SWAP ? b - 6 : 6;
        return 2;
    }
    return 0;
}

template <class A, int K>
cudaError_t cols_pass(const TileArgs<A>& a, const MultipassReq& r) {
    using T = typename A::T;
    {   // 64-bit fields: the tensor-box column pass (colpass.cuh) where it applies
        bool ok = false;
        cudaError_t e = cpass::launch_cols<A, K>(a, r.stream, r.num_sms, r.launches, &ok);
        if (e != cudaSuccess || ok) return e;
    }
    constexpr int TQ = 1 << (tile_e<T, K>() - K);
    constexpr int NT = (TQ << (K - 4)) < 1024 ? (TQ << (K - 4)) : 1024;
    return launch_tile<A, V_DIT, K, TQ, NT, TL_COLS, kSmb, 0>(a, r.stream, r.num_sms, r.launches);
}

template <class A>
cudaError_t cols_pass_any(int K, const TileArgs<A>& a, const MultipassReq& r) {
    switch (K) {
        case 5: return cols_pass<A, 5>(a, r);
        case 6: return cols_pass<A, 6>(a, r);
        case 7: return cols_pass<A, 7>(a, r);
        case 8: return cols_pass<A, 8>(a, r);
        case 9: return cols_pass<A, 9>(a, r);
        default: return cudaErrorInvalidValue;
    }
}

template <class A>
cudaError_t run_sixstep_cols(const MultipassReq& r, bool* ok) {
    using T = typename A::T;
    *ok = false;
    int K1 = 0, K2 = 0;
    while ((1ull << K1) < r.n1) ++K1;
    while ((1ull << K2) < r.n2) ++K2;
    int KA[2], KB[2];
    const int PA = cols_split(K2, KA, (int)sizeof(T)), PB = cols_split(K1, KB, (int)sizeof(T));
    if (!PA || !PB || K1 < 5 || K2 < 5) return cudaSuccess;
    *ok = true;
    const uint64_t N = 1ull << (K1 + K2);
    T* ws0 = static_cast<T*>(r.ws);
    T* ws1 = ws0 + r.batch * N;
    const bool al = aligned16(r.in) && aligned16(r.out) && aligned16(r.ws);
    cudaError_t e = cudaSuccess;
    // step A: columns (length n2, inner i)
    const T* cur = static_cast<const T*>(r.in);
    int done = 0;
    bool transposed = false;
    for (int p = 0; p < PA; ++p) {
        TileArgs<A> a = tile_base<A>(r);
        a.L = K2; a.l1 = K1; a.S0 = done;
        a.qmode = TQM_LINEAR; a.in_order = a.out_order = TO_T_FAST;
        a.vec_in = a.vec_out = al;
        a.rev_in = (p == 0);                       // bit_reverse_permute(col) (algorithms.py:374)
        a.gstw = static_cast<const typename A::Tw*>(r.stw2);
        a.smb = K2 < kSmb ? K2 : kSmb;
        a.cor_on = (p == PA - 1);                  // w_N^(i*k2) (algorithms.py:377-379)
        a.cor_lo = static_cast<const T*>(r.cor_lo);
        a.cor_hi = static_cast<const T*>(r.cor_hi);
        a.cor_lb = r.cor_lb;
        a.scale = (p == PA - 1) ? r.scale : 0;     // intt: n^-1 folded into the correction (one product per residue less)
        a.in = cur;
        a.out = (p == PA - 1) ? ws1 : ws0;
        if (p == PA - 1 && PA == 2 && cur == ws0) {
            // the transpose folded into this pass: it writes [n1][n2] itself (colpass.cuh, TR tiles)
            bool ok = false;
            a.out = ws1;
            e = KA[p] == 5   ? cpass::launch_cols<A, 5, true>(a, r.stream, r.num_sms, r.launches, &ok)
                : KA[p] == 6 ? cpass::launch_cols<A, 6, true>(a, r.stream, r.num_sms, r.launches, &ok)
                : KA[p] == 7 ? cpass::launch_cols<A, 7, true>(a, r.stream, r.num_sms, r.launches, &ok)
                             : cudaSuccess;
            if (e != cudaSuccess) return e;
            if (ok) { transposed = true; cur = ws1; done += KA[p]; continue; }
        }
        if ((e = cols_pass_any<A>(KA[p], a, r)) != cudaSuccess) return e;
        cur = a.out;
        done += KA[p];
    }
    // transpose [n2][n1] -> [n1][n2]
    if (!transposed) {
        const uint64_t blocks = r.batch << (K1 + K2 - 10);
        const uint64_t cap = (uint64_t)r.num_sms * 8;
        e = fastk::launch_pdl(k_transpose<T>, dim3((unsigned)(blocks < cap ? blocks : cap)), dim3(256), 0, r.stream,
                              static_cast<const T*>(ws1), ws0, r.batch, K2, K1);
        if (r.launches) ++*r.launches;
        if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess) return e;
    }
    // step B: rows (length n1, inner k2); output = out[k1*n2 + k2]
    cur = transposed ? ws1 : ws0;
    done = 0;
    for (int p = 0; p < PB; ++p) {
        const bool last = (p == PB - 1);
        TileArgs<A> a = tile_base<A>(r);
        a.L = K1; a.l1 = K2; a.S0 = done;
        a.qmode = TQM_LINEAR; a.in_order = a.out_order = TO_T_FAST;
        a.vec_in = a.vec_out = al;
        a.rev_in = (p == 0);                       // bit_reverse_permute(row) (algorithms.py:385)
        a.gstw = static_cast<const typename A::Tw*>(r.stw1);
        a.smb = K1 < kSmb ? K1 : kSmb;
        a.count_row = last;
        a.scale = 0;                               // (step A's correction carried n^-1)
        a.in = cur;
        a.out = last ? static_cast<T*>(r.out) : (cur == ws1 ? ws0 : ws1);
        if ((e = cols_pass_any<A>(KB[p], a, r)) != cudaSuccess) return e;
        cur = a.out;
        done += KB[p];
    }
    return cudaSuccess;
}

// Distributed four-step with the long-run column passes (rank g of G):
//   step A: the slab x_local[j][i_local] (n2 x c, c = n1/G): DIT over j of every
//           local column (TL_COLS passes, inner i_local), correction
//           w_N^((g c + i_local) k2) fused into the last pass, then the pack for
//           the all-to-all as a per-destination transpose: [k2][i_local] ->
//           [h][i_local][k2 mod n2/G] (k_transpose with batch = G);
//   step B: [i][k2_local] (n1 x n2/G, the all-to-all's concatenation) -> DIT
//           over i for every local column k2 (TL_COLS, inner k2_local) ->
//           out_local[k1][k2_local].
// ws: 2 x n/G residues.
template <class A>
cudaError_t run_sixstep_cols_dist(const MultipassReq& r, int step, int rank, int world, const void* in, void* out,
                                  void* wsv, bool* ok, void* const* peers = nullptr) {
    using T = typename A::T;
    *ok = false;
    int K1 = 0, K2 = 0, lg = 0;
    while ((1ull << K1) < r.n1) ++K1;
    while ((1ull << K2) < r.n2) ++K2;
    while ((1 << lg) < world) ++lg;
    int KA[2], KB[2];
    const int PA = cols_split(K2, KA, (int)sizeof(T)), PB = cols_split(K1, KB, (int)sizeof(T));
    const int lc = K1 - lg, lk = K2 - lg;             // local columns (step A), local k2 (step B)
    if (!PA || !PB || lc < 6 || lk < 6 || !wsv) return cudaSuccess;   // TL_COLS tiles span up to 64 columns
    *ok = true;
    const uint64_t nloc = 1ull << (K1 + K2 - lg);
    T* ws0 = static_cast<T*>(wsv);
    T* ws1 = ws0 + nloc;
    const bool al = aligned16(in) && aligned16(out) && aligned16(wsv);
    cudaError_t e = cudaSuccess;
    if (step == 0) {
        const T* cur = static_cast<const T*>(in);
        int done = 0;
        for (int p = 0; p < PA; ++p) {
            TileArgs<A> a = tile_base<A>(r);
            a.batch = 1;
            a.L = K2; a.l1 = lc; a.S0 = done;
            a.qmode = TQM_LINEAR; a.in_order = a.out_order = TO_T_FAST;
            a.vec_in = a.vec_out = al;
            a.rev_in = (p == 0);
            a.gstw = static_cast<const typename A::Tw*>(r.stw2);
            a.smb = K2 < kSmb ? K2 : kSmb;
            a.cor_on = (p == PA - 1);
            a.cor_lo = static_cast<const T*>(r.cor_lo);
            a.cor_hi = static_cast<const T*>(r.cor_hi);
            a.cor_lb = r.cor_lb;
            a.cor_lgn = K1 + K2;
            a.qoff = (uint32_t)rank << lc;
            a.in = cur;
            a.out = (p == PA - 1) ? ws1 : ws0;
            if (p == PA - 1 && PA == 2 && world <= 8) {
                // the pack folded into this pass (colpass.cuh TR tiles): its stores go straight to
                // [h][i_local][k2 mod n2/G] -- the all-to-all's send buffer, or with a peer table every
                // rank's receive buffer (slot = this rank): P2P stores from the compute kernel itself
                bool okp = false;
                a.dist_pb = lk;
                for (int h = 0; h < world; ++h)
                    a.dist_dst[h] = peers ? static_cast<T*>(peers[h]) + ((uint64_t)rank << (lk + lc))
                                          : static_cast<T*>(out) + ((uint64_t)h << (lk + lc));
                a.out = static_cast<T*>(out);       // (alignment check of the launcher; peers: unused)
                if (peers) a.out = static_cast<T*>(peers[0]);
                e = KA[p] == 5   ? cpass::launch_cols<A, 5, true>(a, r.stream, r.num_sms, r.launches, &okp)
                    : KA[p] == 6 ? cpass::launch_cols<A, 6, true>(a, r.stream, r.num_sms, r.launches, &okp)
                    : KA[p] == 7 ? cpass::launch_cols<A, 7, true>(a, r.stream, r.num_sms, r.launches, &okp)
                                 : cudaSuccess;
                if (e != cudaSuccess) return e;
                if (okp) return cudaSuccess;
                a.dist_pb = 0;
                a.out = ws1;
            }
            if ((e = cols_pass_any<A>(KA[p], a, r)) != cudaSuccess) return e;
            cur = a.out;
            done += KA[p];
        }
        // pack: per destination h, [k2_local][i_local] -> [i_local][k2_local]
        const uint64_t blocks = (uint64_t)world << (lk + lc - 10);
        const uint64_t cap = (uint64_t)r.num_sms * 8;
        if (peers) {      // pack straight into every rank's receive buffer (slot = this rank)
            if (world > kMaxPeers) return cudaErrorInvalidValue;
            PeerPtrs<T> pp{};
            for (int h = 0; h < world; ++h) pp.p[h] = static_cast<T*>(peers[h]);
            e = fastk::launch_pdl(k_transpose_peer<T>, dim3((unsigned)(blocks < cap ? blocks : cap)), dim3(256), 0,
                                  r.stream, static_cast<const T*>(ws1), pp, (uint64_t)world, rank, lk, lc);
            if (r.launches) ++*r.launches;
            if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess) return e;
            return cudaSuccess;
        }
        e = fastk::launch_pdl(k_transpose<T>, dim3((unsigned)(blocks < cap ? blocks : cap)), dim3(256), 0, r.stream,
                              static_cast<const T*>(ws1), static_cast<T*>(out), (uint64_t)world, lk, lc);
        if (r.launches) ++*r.launches;
        if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess) return e;
        return cudaSuccess;
    }
    const T* cur = static_cast<const T*>(in);
    int done = 0;
    for (int p = 0; p < PB; ++p) {
        const bool last = (p == PB - 1);
        TileArgs<A> a = tile_base<A>(r);
        a.batch = 1;
        a.L = K1; a.l1 = lk; a.S0 = done;
        a.qmode = TQM_LINEAR; a.in_order = a.out_order = TO_T_FAST;
        a.vec_in = a.vec_out = al;
        a.rev_in = (p == 0);
        a.gstw = static_cast<const typename A::Tw*>(r.stw1);
        a.smb = K1 < kSmb ? K1 : kSmb;
        a.count_row = last;
        a.scale = last ? r.scale : 0;
        a.in = cur;
        a.out = last ? static_cast<T*>(out) : ws0;
        if ((e = cols_pass_any<A>(KB[p], a, r)) != cudaSuccess) return e;
        cur = a.out;
        done += KB[p];
    }
    return cudaSuccess;
}

}  // namespace ftile

// entry points compiled in kt_f32.cu / kt_gold.cu
cudaError_t tile_passes_f32(int variant, bool lazy, const MultipassReq& r, bool* ok);
cudaError_t tile_passes_gold(int variant, const MultipassReq& r, bool* ok);
cudaError_t tile_sixstep_gold(const MultipassReq& r, bool* ok);
// distributed four-step, rank-local steps (step = 0: A, 1: B)
cudaError_t tile_sixstep_dist_gold(const MultipassReq& r, int step, int rank, int world, const void* in, void* out,
                                   bool* ok, void* const* peers = nullptr);
// workspace (bytes) the distributed steps need on one rank
uint64_t sixstep_dist_ws_bytes(uint64_t n, int world, int word);

}  // namespace nttb200
