// colpass.cuh -- column passes of the six-step for 64-bit fields (config 5:
// the 2^13 x 2^13 Goldilocks split), the TL_COLS passes of fasttile.cuh
// rebuilt around TMA tensor boxes.
//
// One pass = K consecutive DIT stages (S0+1 .. S0+K) of the length-2^L
// transforms down EVERY column of a row-major [2^L][2^l1] matrix (element
// (j, i) at j * 2^l1 + i; algorithms.py:371-389 reads x[j*n1 + i] this way).
// A tile is one network id Qj (the position bits outside [S0, S0+K)) times TQ
// consecutive columns: 2^K rows x TQ columns = 2^12 residues = 32 KiB.
//
//  * the tile comes in as ONE 4-D tensor box [1][2^K][1][TQ] (cp.async.bulk.tensor,
//    mbarrier completion), issued as soon as the previous tile's last register
//    group holds its residues, so the load runs under that group's butterflies and
//    stores; outputs go straight from registers to HBM (a warp row = a run of TQ
//    consecutive columns); the bit reversal of a sub-transform's
//    input (pass 1) is a tensor-map view: j = jh * 2^(L-K) + jl puts the rows
//    of a network 2^(L-K) apart, and the box delivers them ordered by
//    jh = brev_K(x);
//  * work layout = the dense box [row][column]: a warp's lanes run along the
//    columns, so every shared-memory access of every register group is
//    conflict-free without padding (the network-major layout of k_tile
//    showed 37-40 % conflicting wavefronts here, profiles/r2);
//  * the stage twiddles of a thread depend on its rows only, never on its
//    column: warp-uniform 8-byte broadcasts from a 2^K-entry table that is
//    rebuilt per tile for the later pass (T[2^(s-1) + qlo + 2^S0 m], 63
//    entries) -- no twiddle ever comes from global memory inside a group;
//  * the six-step correction w_N^(i k2) of a thread's 16 outputs is a
//    geometric sequence in the register index (k2 = k2_0 + c 2^(S0+K-4)): two
//    table look-ups per THREAD (first term, ratio) instead of two per residue;
//  * 64 registers, 34 KiB: four to six 256-thread CTAs per SM overlap one
//    another's tile loads / stores.
//
// Stage-faithful and interchangeable with the k_tile passes: the HBM buffer
// after a pass holds the same (canonical) residues.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include "fasttile.cuh"

#ifndef NTT_COLS_MINB
#define NTT_COLS_MINB 4        // resident CTAs the column-pass kernel is compiled for (64 registers)
#endif

namespace nttb200 {
namespace cpass {

NTT_D void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::
            "r"(fastk::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(fastk::smem_u32(bar))
        : "memory");
}
template <class A>
struct ColArgs {
    using T = typename A::T;
    using Tw = typename A::Tw;
    T* out;
    uint64_t batch;
    int L, S0, l1;             // sub-transform length 2^L, stages done before this pass, log2 columns
    const Tw* gstw;            // per-stage table of the length-2^L transform
    int cor_on;                // multiply by w_N^(i * k2) (the last pass of step A)
    const T* cor_lo;           // w_N^e = cor_hi[e >> cor_lb] * cor_lo[e mod 2^cor_lb]
    const T* cor_hi;
    int cor_lb, cor_lgn;       // log2 N of the correction root
    uint32_t qoff;             // global index of local column 0 (distributed slabs)
    int scale;
    Tw ninv;
    int count_row, count_bitrev;
    unsigned long long* counters;
    uint64_t p;
    // transposing pass of the distributed step A: row k2 -> dist_dst[k2 >> dist_pb] (the pack for the
    // all-to-all, or -- peer exchange -- the receive buffer of rank k2 >> dist_pb itself), 0: out[i][k2]
    int dist_pb;
    T* dist_dst[8];
};

template <int K, int TQ>
constexpr size_t cols_smem_bytes() { return ((size_t)8 << K) * TQ; }

// FIRST: S0 == 0 (stage 1's twiddles are 1, the input rows arrive bit-reversed)
// TR: the pass writes the TRANSPOSED matrix out[i][k2] (the six-step's transpose folded into step A's
// last pass): a tile is then 2^QB consecutive network ids x 2^IB columns, so that the transposed
// side moves runs of 2^QB residues; the box is [1][2^K][2^QB][2^IB] of the same tensor map
template <class A, int K, int TQ, bool FIRST, bool TR = false>
__global__ void __launch_bounds__(256, NTT_COLS_MINB) k_cols(const __grid_constant__ CUtensorMap min, ColArgs<A> a) {
    using T = typename A::T;
    using Tw = typename A::Tw;
    static_assert(sizeof(T) == 8 && sizeof(Tw) == 8, "64-bit residues with bare-power twiddles");
    constexpr int NT = 256, TT = 1 << (K - 4), LTQ = ftile::ilog2c(TQ);
    static_assert(TT * TQ == NT && TQ >= 16, "2^12-residue tiles, lanes along the columns");
    constexpr int G = (K + 3) / 4, K0 = K - 4 * (G - 1);
    static_assert(G >= 2, "two register groups or more");
    static_assert(!TR || !FIRST, "the transposing pass is a later pass (network ids carry low position bits)");
    constexpr int QB = TR ? 4 : 0, IB = LTQ - QB;   // tile columns = 2^QB network ids x 2^IB matrix columns
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // TL[(2^sl + m) << QB | ql]: twiddle of local stage sl + 1, local index m, network qlo0 + ql
    __shared__ Tw TLs[2][(1 << K) << QB];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ T* dstS[8];                    // TR, distributed: the per-destination bases
    if (TR && threadIdx.x < 8) dstS[threadIdx.x] = a.dist_dst[threadIdx.x];
    T* S = reinterpret_cast<T*>(smem_raw);   // (128-byte aligned: the box's destination)
    A ar;
    ar.init(a.p);
    const uint32_t tid = threadIdx.x, t = tid % TQ, u = tid / TQ;
    const int L = a.L, S0 = FIRST ? 0 : a.S0, l1 = a.l1;
    const int ltpr = l1 + L - K - LTQ;                    // log2 tiles per matrix
    const uint64_t ntiles = a.batch << ltpr;
    const int lrest = L - K - S0;                         // bits of the network id above the pass's window
    // tile -> (matrix b, network Qj = qlo | qhi << S0, first column)
    // (qlo = the first of the tile's 2^QB network ids, col0 = the first of its 2^IB columns)
    struct Tile { uint64_t b; uint32_t tr, Qj, col0, qlo, qhi; };
    auto decode = [&](uint64_t tile) {
        Tile d;
        d.b = tile >> ltpr;
        d.tr = (uint32_t)(tile & ((1ull << ltpr) - 1));
        d.Qj = (d.tr >> (l1 - IB)) << QB;
        d.col0 = (d.tr << IB) & ((1u << l1) - 1);
        d.qlo = d.Qj & ((1u << S0) - 1);
        d.qhi = d.Qj >> S0;
        return d;
    };
    auto load_tile = [&](const Tile& d) {                  // one thread: the tile's box into S
        fastk::mbar_expect_tx(&mbar, (uint32_t)(sizeof(T) << K) * TQ);
        if (FIRST) tma_load_4d(S, &min, (int)d.col0, (int)brev(d.Qj, L - K), 0, (int)d.b, &mbar);
        else tma_load_4d(S, &min, (int)d.col0, (int)d.qlo, 0, (int)((d.b << lrest) + d.qhi), &mbar);
    };
    // the later pass's twiddles of a tile: stage S0+sl+1, index qlo + 2^S0 m (63 / 127 / 255 entries
    // per network id)
    auto fill_tl = [&](Tw* TL, uint32_t qlo) {
        for (uint32_t i = tid + (1u << QB); i < ((1u << K) << QB); i += NT) {
            const uint32_t e = i >> QB, ql = i & ((1u << QB) - 1);
            const int sl = 31 - __clz(e);
            TL[i] = __ldg(a.gstw + ((1u << (S0 + sl)) + qlo + ql + ((e - (1u << sl)) << S0)));
        }
    };
    if (FIRST)
        for (uint32_t e = tid; e < (1u << K); e += NT) TLs[0][e] = a.gstw[e];
    else if ((uint64_t)blockIdx.x < ntiles) fill_tl(TLs[0], decode(blockIdx.x).qlo);
    if (tid == 0) {
        fastk::mbar_init(&mbar, 1);
        fastk::fence_mbar_init();
    }
    __syncthreads();
    fastk::pdl_trigger();
    fastk::pdl_wait();                       // the previous pass's output (our input) is visible
    if (tid == 0 && (uint64_t)blockIdx.x < ntiles) load_tile(decode(blockIdx.x));

    uint32_t it = 0;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const Tile d = decode(tile);
        const Tw* TL = FIRST ? TLs[0] : TLs[it & 1];
        T v[16];
        if (!FIRST) __syncthreads();         // this tile's twiddle table (filled during the previous tile) is visible
        fastk::mbar_wait(&mbar, it & 1);
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int B = g == 0 ? 0 : K0 + 4 * (g - 1);          // register block [B, B+4) of the row index
            const int kg = g == 0 ? K0 : 4, b0 = g == 0 ? 0 : B;  // stages b0+1 .. b0+kg (local)
            const uint32_t pbase = (u & ((1u << B) - 1)) | ((u >> B) << (B + 4));
            if (g == 0 && FIRST) {
                // staged row r holds x = brev_K(r); x = u << 4 | c  ->  r = brev4(c) << (K-4) | brev(u)
                const T* sp = S + (size_t)brev(u, K - 4) * TQ + t;
#pragma unroll
                for (int c = 0; c < 16; ++c) v[c] = sp[(size_t)(brev((uint32_t)c, 4) << (K - 4)) * TQ];
                __syncthreads();             // every row read before the rows are rewritten in natural order
            } else {
                const T* sp = S + (size_t)pbase * TQ + t;
#pragma unroll
                for (int c = 0; c < 16; ++c) v[c] = sp[(size_t)((uint32_t)c << B) * TQ];
            }
            if (g == G - 1) {
                // the tile is in registers: its buffer takes the next tile's box while the last
                // group computes and stores (the next tile's twiddles are fetched alongside)
                fastk::fence_proxy_async();  // this tile's generic-proxy accesses before the bulk copy's writes
                __syncthreads();
                const uint64_t nxt = tile + gridDim.x;
                if (nxt < ntiles) {
                    const Tile dn = decode(nxt);
                    if (tid == 0) load_tile(dn);
                    if (!FIRST) fill_tl(TLs[(it + 1) & 1], dn.qlo);
                }
            }
#pragma unroll
            for (int jj = 0; jj < kg; ++jj) {
                const int sl = b0 + jj, j = sl - B;                // local stage bit, its register bit
                const uint32_t lmask = (1u << sl) - 1;
                const Tw* row = TL + (((1u << sl) + (pbase & lmask)) << QB) + (TR ? (t >> IB) : 0u);
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    if (c & (1 << j)) continue;
                    const int hi = c | (1 << j);
                    if (FIRST && sl == 0) ar.dit1(v[c], v[hi]);
                    else ar.dit(v[c], v[hi], ftile::lds_tw(row + ((((uint32_t)c << B) & lmask) << QB)));
                }
            }
            if (g < G - 1) {
                T* dp = S + (size_t)pbase * TQ + t;
#pragma unroll
                for (int c = 0; c < 16; ++c) dp[(size_t)((uint32_t)c << B) * TQ] = v[c];
                __syncthreads();
            } else {
                // ---- outputs: correction / n^-1 / canonical form, straight to HBM (a warp row is a
                // run of TQ consecutive columns: 128..512 contiguous bytes)
                // (TR: out[i][k2] -- lanes along the network ids, runs of 2^QB residues)
                const uint32_t ql = TR ? (t >> IB) : 0u, il = TR ? (t & ((1u << IB) - 1)) : t;
                const uint64_t pos0 =
                    (uint64_t)(d.qlo + ql) | ((uint64_t)pbase << S0) | ((uint64_t)d.qhi << (S0 + K));
                T* gp = TR ? a.out + (((d.b << l1) + d.col0 + il) << L) + pos0
                           : a.out + (((d.b << L) + pos0) << l1) + d.col0 + il;
                const uint64_t gs = 1ull << (B + S0 + (TR ? 0 : l1));   // register c -> row pos0 + (c << (B + S0))
                // distributed step A (TR): the exchange rides this store -- row k2 of column i lands in
                // destination k2 >> pb at [i][k2 mod 2^pb] (a local pack buffer, or the peer's receive
                // buffer over NVLink)
                const int pb = TR ? a.dist_pb : 0;
                auto outp = [&](int c) -> T* {
                    if (TR && pb) {
                        const uint64_t k2 = pos0 + ((uint64_t)c << (B + S0));
                        return dstS[k2 >> pb] + ((uint64_t)(d.col0 + il) << pb) + (k2 & ((1ull << pb) - 1));
                    }
                    return gp + c * gs;
                };
                if (a.cor_on) {
                    // k2(c) = pos0 + (c << (S0 + B));  w_N^(i k2(c)) = f0 * r^c
                    // (four interleaved sequences instead of one chain measured the same: the
                    // pass is bound by the integer pipe, not by the chain's latency)
                    const uint64_t nm = (1ull << a.cor_lgn) - 1, lm = (1ull << a.cor_lb) - 1;
                    const uint64_t i = (uint64_t)a.qoff + d.col0 + il;
                    const uint64_t e0 = (i * pos0) & nm, es = (i << (S0 + B)) & nm;
                    T f = ar.mulfull(__ldg(a.cor_hi + (e0 >> a.cor_lb)), __ldg(a.cor_lo + (e0 & lm)));
                    const T r = ar.mulfull(__ldg(a.cor_hi + (es >> a.cor_lb)), __ldg(a.cor_lo + (es & lm)));
                    if (a.scale) f = ar.mulfull(f, a.ninv);        // intt: n^-1 rides the sequence's first term
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        *outp(c) = ar.mulfull(v[c], f);
                        if (c < 15) f = ar.mulfull(f, r);
                    }
                } else if (a.scale) {
#pragma unroll
                    for (int c = 0; c < 16; ++c) *outp(c) = ar.mulc(v[c], a.ninv);
                } else {
#pragma unroll
                    for (int c = 0; c < 16; ++c) *outp(c) = ar.fin(v[c]);
                }
            }
        }
        if (a.counters && tid == 0 && d.tr == 0) {
            atomicAdd(a.counters + C_HBM, 1ull);
            if (a.count_row) atomicAdd(a.counters + C_TRANSFORMS, 1ull);
            if (a.count_bitrev) atomicAdd(a.counters + C_BITREV, (unsigned long long)a.count_bitrev);
        }
    }
}

inline PFN_cuTensorMapEncodeTiled_v12000 tensor_encoder() {
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

// 4-D view [d3][2^K rows][d1][2^l1 columns] of a matrix, boxes [1][2^K][1][TQ]
// (qb: the box spans 2^qb entries of dimension 1 and TQ / 2^qb columns)
inline bool cols_map(CUtensorMap* m, const void* base, int l1, uint64_t d1, int K, uint64_t d3, int TQ, int qb = 0) {
    auto enc = tensor_encoder();
    if (!enc) return false;
    cuuint64_t dims[4] = {(cuuint64_t)1 << l1, d1, (cuuint64_t)1 << K, d3};
    cuuint64_t strides[3] = {((cuuint64_t)8 << l1), ((cuuint64_t)8 << l1) * d1, (((cuuint64_t)8 << l1) * d1) << K};
    cuuint32_t box[4] = {(cuuint32_t)TQ >> qb, (cuuint32_t)1 << qb, (cuuint32_t)1 << K, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// *ok = false when the pass is not covered (the caller falls back to k_tile);
// TR: write the transposed matrix (later passes with S0 >= 4 only)
template <class A, int K, bool TR = false>
cudaError_t launch_cols(const ftile::TileArgs<A>& ta, cudaStream_t s, int num_sms, int* launches, bool* ok) {
    using T = typename A::T;
    *ok = false;
#ifdef NTT_COLS_OFF                // (study builds: the k_tile column passes instead)
    return cudaSuccess;
#endif
    if constexpr (sizeof(T) != 8 || sizeof(typename A::Tw) != 8 || K < 5 || K > 8 || (TR && K > 7)) return cudaSuccess;
    else {
        constexpr int TQ = 1 << (12 - K);
        const int L = ta.L, S0 = ta.S0, l1 = ta.l1;
        if (l1 < 12 - K || L < K + S0 || (S0 == 0) != (ta.rev_in != 0) || ta.twist) return cudaSuccess;
        if (TR && S0 == 0) return cudaSuccess;
        if ((reinterpret_cast<uintptr_t>(ta.in) | reinterpret_cast<uintptr_t>(ta.out)) & 15) return cudaSuccess;
        constexpr int QB = TR ? 4 : 0;
        if (TR && (S0 < QB || l1 < 12 - K - QB)) return cudaSuccess;
        const int lrest = L - K - S0;
        if ((ta.batch << lrest) >= (1ull << 31)) return cudaSuccess;
        CUtensorMap min;
        // pass 1 reads j = brev_L(pos): rows of a network 2^(L-K) apart, networks by brev(Qj)
        const bool mi = S0 == 0 ? cols_map(&min, ta.in, l1, 1ull << (L - K), K, ta.batch, TQ)
                                : cols_map(&min, ta.in, l1, 1ull << S0, K, ta.batch << lrest, TQ, QB);
        if (!mi) return cudaSuccess;
        ColArgs<A> a{};
        a.out = ta.out; a.batch = ta.batch; a.L = L; a.S0 = S0; a.l1 = l1;
        a.gstw = ta.gstw;
        a.cor_on = ta.cor_on; a.cor_lo = ta.cor_lo; a.cor_hi = ta.cor_hi; a.cor_lb = ta.cor_lb;
        a.cor_lgn = ta.cor_lgn ? ta.cor_lgn : L + l1;
        a.qoff = (uint32_t)ta.qoff;
        a.scale = ta.scale; a.ninv = ta.ninv;
        a.count_row = ta.count_row; a.count_bitrev = ta.count_bitrev; a.counters = ta.counters;
        a.p = ta.p;
        a.dist_pb = TR ? ta.dist_pb : 0;
        for (int h = 0; h < 8; ++h) a.dist_dst[h] = ta.dist_dst[h];
        constexpr size_t smem = cols_smem_bytes<K, TQ>();
        auto launch = [&](auto kern) -> cudaError_t {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            int occ = 0;
            if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem);
            if (e != cudaSuccess) return e;
            if (occ < 1) occ = 1;
            const uint64_t ntiles = ta.batch << (l1 + L - K - (12 - K));
            uint64_t grid = (uint64_t)num_sms * occ;
            if (grid > ntiles) grid = ntiles;
            if (grid == 0) return cudaSuccess;
            e = fastk::launch_pdl(kern, dim3((unsigned)grid), dim3(256), smem, s, min, a);
            if (launches) ++*launches;
            return e != cudaSuccess ? e : cudaGetLastError();
        };
        *ok = true;
        if constexpr (TR) return S0 == 0 ? cudaErrorInvalidValue : launch(k_cols<A, K, TQ, false, true>);
        else return S0 == 0 ? launch(k_cols<A, K, TQ, true>) : launch(k_cols<A, K, TQ, false>);
    }
}

}  // namespace cpass
}  // namespace nttb200
