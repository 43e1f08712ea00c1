// multipass.cuh -- the pass kernel (tile load -> tile_stages -> tile store)
// and the host planners that chain passes for every variant and N.
//
//  * N fits in shared memory: ONE pass, a tile = TQ whole rows (K = L).
//  * larger N (DIT/DIF/Flat/Pease/Pease_nc/Stockham): ceil(L/Kmax) HBM passes,
//    each a contiguous run of the variant's own stages (stage-faithful: the
//    HBM buffer between passes is exactly the reference's state after that
//    stage); tiles are chosen so global reads and writes are >= 32-byte runs.
//  * six-step (algorithms.py:355-389): pass A = n1 strided size-n2 DIT
//    sub-transforms + correction twiddles w^(i*k2) (two-level table, exact);
//    pass B = n2 size-n1 DIT sub-transforms written to out[n2*k1 + k2].
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "engine.cuh"

namespace nttb200 {

// How a pass maps tile networks to global positions.
enum Layout { LAY_VARIANT = 0, LAY_SIX_A = 1, LAY_SIX_B = 2 };
// How tile networks map to global network ids.
enum QMode { QM_ROWS = 0, QM_LINEAR = 1, QM_REV = 2, QM_2D = 3 };
// Copy-loop element order.
enum Order { ORD_C_FAST = 0, ORD_T_FAST = 1, ORD_TB_FAST = 2 };

template <class F>
struct PassArgs {
    using T = typename F::T;
    using Tw = typename F::Tw;
    const T* in;
    T* out;
    uint64_t batch;
    int L, K, S0;          // see GCtx
    int TQ;                // networks per tile
    int qmode, TA;         // QM_2D: TQ = TA x TB, t = ta + TA*tb
    int in_order, out_order;
    int rev_in, rev_out;   // global bit reversal fused into the copy-in / copy-out
    int rev_first, rev_last;   // single-pass: bit reversal fused into the first / last group
    int count_row;         // this pass completes the transform (count it)
    int count_bitrev;      // bit-reverse permutations this pass performs per row
    const Tw* tw;          // table for the stage twiddles
    F f;
    int scale;             // multiply by n_inv on the way out (intt)
    Tw ninv;
    // six-step: n1 = 2^l1 (rows are x[i::n1]), correction twiddles w_N^(i*k2)
    int l1, l2;
    const Tw* tw_main;     // main size-N table (may be null when two-level is used)
    const typename F::T* cor_lo;   // two-level correction table: w^e = hi[e >> lb] * lo[e & (2^lb-1)]
    const typename F::T* cor_hi;
    int cor_lb;
    unsigned long long* counters;
};

template <class F>
NTT_D uint64_t gpos_in(const PassArgs<F>& a, int V, int LAY, uint32_t Q, uint32_t x) {
    const int L = a.L, K = a.K, S0 = a.S0;
    uint64_t g;
    if (LAY == LAY_SIX_A) return ((uint64_t)x << a.l1) | Q;            // x[j*n1 + i], i = Q
    if (LAY == LAY_SIX_B) return ((uint64_t)x << a.l2) | Q;            // rows[i][k2], k2 = Q
    if (V == V_PEASE || V == V_PEASE_NC) g = ((uint64_t)Q << K) | x;
    else if (V == V_STOCKHAM) {
        const int glob = L - S0 - K;
        g = ((uint64_t)(Q >> glob) << (L - S0)) | ((uint64_t)x << glob) | (Q & ((1u << glob) - 1));
    } else g = (Q & ((1u << S0) - 1)) | ((uint64_t)x << S0) | ((uint64_t)(Q >> S0) << (S0 + K));
    return a.rev_in ? (uint64_t)brev((uint32_t)g, L) : g;
}

template <class F>
NTT_D uint64_t gpos_out(const PassArgs<F>& a, int V, int LAY, uint32_t Q, uint32_t x) {
    const int L = a.L, K = a.K, S0 = a.S0;
    uint64_t g;
    if (LAY == LAY_SIX_A) return ((uint64_t)Q << a.l2) | x;            // rows[i][k2]
    if (LAY == LAY_SIX_B) return ((uint64_t)x << a.l2) | Q;            // out[n2*k1 + k2]
    if (V == V_PEASE || V == V_PEASE_NC || V == V_STOCKHAM) g = Q | ((uint64_t)x << (L - K));
    else g = (Q & ((1u << S0) - 1)) | ((uint64_t)x << S0) | ((uint64_t)(Q >> S0) << (S0 + K));
    return a.rev_out ? (uint64_t)brev((uint32_t)g, L) : g;
}

NTT_D void order_decode(int order, int TQ, int TA, int K, uint32_t i, uint32_t& t, uint32_t& x) {
    if (order == ORD_C_FAST) { t = i >> K; x = i & ((1u << K) - 1); }
    else if (order == ORD_T_FAST) { t = i % TQ; x = i / TQ; }
    else { const int TB = TQ / TA; const uint32_t tb = i % TB, ta = (i / TB) % TA; t = ta + TA * tb; x = i / TQ; }
}

template <class F, int V, int LAY>
__global__ void __launch_bounds__(kThreads) k_pass(PassArgs<F> a) {
    using T = typename F::T;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ uint32_t Qs[256];
    __shared__ uint64_t Rb[256];
    const int K = a.K;
    const int TQ = a.TQ;
    const int span = TQ << K;
    T* A = reinterpret_cast<T*>(smem_raw);
    T* B = A + span;
    const int M = (LAY == LAY_VARIANT) ? a.L - K : (LAY == LAY_SIX_A ? a.l1 : a.l2);   // network-id bits
    const uint64_t N = 1ull << a.L;
    const uint64_t tiles_per_row = a.qmode == QM_ROWS ? 1 : ((1ull << M) / TQ);
    const uint64_t ntiles = a.qmode == QM_ROWS ? (a.batch + TQ - 1) / TQ : a.batch * tiles_per_row;
    const F f = a.f;
    GCtx g;
    g.L = (LAY == LAY_VARIANT) ? a.L : K;     // six-step sub-transforms are plain size-2^K DITs
    g.K = K;
    g.S0 = (LAY == LAY_VARIANT) ? a.S0 : 0;
    g.Q = (LAY == LAY_VARIANT && a.qmode != QM_ROWS) ? Qs : nullptr;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        // ---- networks of this tile
        for (int t = threadIdx.x; t < TQ; t += blockDim.x) {
            uint64_t row;
            uint32_t Q = 0;
            if (a.qmode == QM_ROWS) { row = tile * TQ + t; }
            else {
                row = tile / tiles_per_row;
                const uint32_t tr = (uint32_t)(tile % tiles_per_row);
                if (a.qmode == QM_LINEAR) Q = tr * TQ + t;
                else if (a.qmode == QM_REV) Q = brev(tr * TQ + t, M);
                else {
                    const int TB = TQ / a.TA;
                    const int hb = 31 - __clz(TB);
                    const uint32_t ta = t % a.TA, tb = t / a.TA;
                    Q = (brev(tr * a.TA + ta, M - hb) << hb) | tb;
                }
            }
            Qs[t] = Q;
            Rb[t] = row < a.batch ? row * N : ~0ull;
        }
        __syncthreads();
        // ---- gather the tile (coalesced runs; bit reversal fused when rev_in)
        for (uint32_t i = threadIdx.x; i < (uint32_t)span; i += blockDim.x) {
            uint32_t t, x;
            order_decode(a.in_order, TQ, a.TA, K, i, t, x);
            const uint64_t rb = Rb[t];
            T v = 0;
            if (rb != ~0ull) v = a.in[rb + gpos_in<F>(a, V, LAY, Qs[t], x)];
            A[slot<T>(t, x, K)] = v;
        }
        __syncthreads();
        int copies = 0;
        T* res = tile_stages<F, V>(f, A, B, g, a.tw, TQ, a.rev_first, a.rev_last, &copies);
        // ---- six-step correction twiddles: row[k2] *= w_N^(i*k2)  (algorithms.py:376-378)
        if (LAY == LAY_SIX_A) {
            for (uint32_t i = threadIdx.x; i < (uint32_t)span; i += blockDim.x) {
                const uint32_t t = i >> K, x = i & ((1u << K) - 1);
                const uint64_t e = ((uint64_t)Qs[t] * x) & (N - 1);
                T w;
                if (a.tw_main) w = F::tw_value(ldtw(a.tw_main, (uint32_t)e));
                else w = f.mul_full(__ldg(a.cor_hi + (e >> a.cor_lb)), __ldg(a.cor_lo + (e & ((1ull << a.cor_lb) - 1))));
                res[slot<T>(t, x, K)] = f.mul_full(res[slot<T>(t, x, K)], w);
            }
            __syncthreads();
        }
        // ---- scatter the tile
        for (uint32_t i = threadIdx.x; i < (uint32_t)span; i += blockDim.x) {
            uint32_t t, x;
            order_decode(a.out_order, TQ, a.TA, K, i, t, x);
            const uint64_t rb = Rb[t];
            if (rb == ~0ull) continue;
            T v = res[slot<T>(t, x, K)];
            if (a.scale) v = f.mul(v, a.ninv);
            a.out[rb + gpos_out<F>(a, V, LAY, Qs[t], x)] = v;
        }
        if (a.counters && threadIdx.x == 0) {
            unsigned long long rows = 0;
            if (a.qmode == QM_ROWS) {
                const uint64_t r0 = tile * TQ;
                rows = (a.batch - r0) < (uint64_t)TQ ? (a.batch - r0) : (uint64_t)TQ;
            } else if (tile % tiles_per_row == 0) rows = 1;
            if (rows) {
                atomicAdd(a.counters + C_HBM, rows);
                if (a.count_row) atomicAdd(a.counters + C_TRANSFORMS, rows);
                if (a.count_bitrev) atomicAdd(a.counters + C_BITREV, rows * a.count_bitrev);
                if (copies) atomicAdd(a.counters + C_COPIES, rows * copies);
            }
        }
        __syncthreads();
    }
}

// Standalone bit-reverse permutation out[i] = in[rev(i)] (modmath.py:171-177)
// -- the reference's own separate pass (algorithms.py:174,238,255) for the
// multi-pass Flat / Pease / Pease_nc transforms.  64 x 64 tiles through
// shared memory so BOTH sides move 64-residue (>= 256-byte) runs:
// i = [a | m | b] (6-bit a, b), out[[a|m|b]] = in[[rev(b)|rev(m)|rev(a)]].
template <class T>
__global__ void __launch_bounds__(256) k_bitrev(const T* in, T* out, uint64_t batch, int L, unsigned long long* counters) {
    __shared__ T tile[64][65];
    const int mb = L - 12;
    const uint64_t N = 1ull << L;
    const uint64_t per_row = 1ull << mb;
    const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;     // 64 x 4
    for (uint64_t blk = blockIdx.x; blk < batch * per_row; blk += gridDim.x) {
        const uint64_t row = blk >> mb;
        const uint32_t m = (uint32_t)(blk & (per_row - 1));
        const T* src = in + row * N;
        T* dst = out + row * N;
        const uint64_t rm = (uint64_t)brev(m, mb) << 6;
        for (int k = ty; k < 64; k += 4)                        // read in[[k | rev(m) | tx]]
            tile[k][tx] = src[((uint64_t)k << (L - 6)) | rm | tx];
        __syncthreads();
        const uint32_t rb = brev(tx, 6);
        for (int k = ty; k < 64; k += 4)                        // write out[[k | m | tx]] = in[[rev(tx)|rev(m)|rev(k)]]
            dst[((uint64_t)k << (L - 6)) | ((uint64_t)m << 6) | tx] = tile[rb][brev(k, 6)];
        __syncthreads();
        if (counters && threadIdx.x == 0 && m == 0) atomicAdd(counters + C_BITREV, 1ull);
    }
}

// Per-row matrix transpose out[c * R + r] = in[r * C + c] (R = 2^rb rows,
// C = 2^cb columns): the six-step's explicit transpose between its column and
// row steps (the "six" of six-step), 32 x 32 tiles through shared memory so
// both HBM sides move 32-residue runs.  rb, cb >= 5.
template <class T>
__global__ void __launch_bounds__(256) k_transpose(const T* in, T* out, uint64_t batch, int rb, int cb) {
    __shared__ T tile[32][33];
    const uint64_t R = 1ull << rb, C = 1ull << cb;
    const int pb = rb + cb - 10;                                // log2 tiles per matrix
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;     // 32 x 8
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // PDL (no-op without the attribute)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (uint64_t blk = blockIdx.x; blk < (batch << pb); blk += gridDim.x) {
        const uint64_t row = blk >> pb, b = blk & ((1ull << pb) - 1);
        const uint64_t br = (b >> (cb - 5)) << 5, bc = (b & ((C >> 5) - 1)) << 5;
        const T* src = in + (row << (rb + cb));
        T* dst = out + (row << (rb + cb));
        for (int k = ty; k < 32; k += 8) tile[k][tx] = src[(br + k) * C + bc + tx];
        __syncthreads();
        for (int k = ty; k < 32; k += 8) dst[(bc + k) * R + br + tx] = tile[tx][k];
        __syncthreads();
    }
}

// Peer-memory variant of the distributed four-step's pack (step A's last
// store): block h of the per-destination transpose is written straight into
// rank h's receive buffer at this rank's slot, over NVLink (P2P stores through
// pointers the caller mapped, e.g. torch symmetric memory), so the exchange
// rides the pack instead of a separate all-to-all.  dst[h] = peers.p[h] +
// slot * 2^(rb+cb); same 32 x 32 tiling as k_transpose.
constexpr int kMaxPeers = 8;
template <class T>
struct PeerPtrs {
    T* p[kMaxPeers];
};
template <class T>
__global__ void __launch_bounds__(256) k_transpose_peer(const T* in, PeerPtrs<T> peers, uint64_t world, int slot,
                                                        int rb, int cb) {
    __shared__ T tile[32][33];
    const uint64_t R = 1ull << rb, C = 1ull << cb;
    const int pb = rb + cb - 10;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (uint64_t blk = blockIdx.x; blk < (world << pb); blk += gridDim.x) {
        const uint64_t h = blk >> pb, b = blk & ((1ull << pb) - 1);
        const uint64_t br = (b >> (cb - 5)) << 5, bc = (b & ((C >> 5) - 1)) << 5;
        const T* src = in + (h << (rb + cb));
        T* dst = peers.p[h] + ((uint64_t)slot << (rb + cb));
        for (int k = ty; k < 32; k += 8) tile[k][tx] = src[(br + k) * C + bc + tx];
        __syncthreads();
        for (int k = ty; k < 32; k += 8) dst[(bc + k) * R + br + tx] = tile[tx][k];
        __syncthreads();
    }
}

template <class F>
__global__ void k_pointwise(const typename F::T* a, const typename F::T* b, typename F::T* c, uint64_t n, F f) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        c[i] = f.mul_full(a[i], b[i]);
}

// Naive O(N^2) DFT (algorithms.py:52-79) -- exact for every field (the
// reference's numpy version overflows for 64-bit p; this one does not).
template <class F>
__global__ void k_naive(const typename F::T* in, typename F::T* out, uint64_t batch, int L,
                        const typename F::Tw* tw, F f, int scale, typename F::Tw ninv,
                        unsigned long long* counters) {
    using T = typename F::T;
    const uint32_t N = 1u << L;
    const uint64_t total = batch * N;
    for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t row = idx >> L;
        const uint32_t k = idx & (N - 1);
        const T* x = in + row * N;
        T acc = 0;
        for (uint32_t j = 0; j < N; ++j) {
            const uint32_t e = (uint32_t)(((uint64_t)k * j) & (N - 1));
            acc = f.add(acc, f.mul(x[j], ldtw(tw, e)));
        }
        if (scale) acc = f.mul(acc, ninv);
        out[idx] = acc;
    }
    if (counters && blockIdx.x == 0 && threadIdx.x == 0) {
        atomicAdd(counters + C_TRANSFORMS, (unsigned long long)batch);
        atomicAdd(counters + C_HBM, (unsigned long long)batch);
    }
}

// ------------------------------------------------------------ host side --

struct MultipassReq {
    int variant;
    int L;
    const void* in;
    void* out;
    uint64_t batch;
    const void* tw;            // main table F::Tw[N]
    const void* stw;           // per-stage table F::Tw[N]: T[2^(s-1)+k] = w^(k*N/2^s)
    const void* tw1;           // six-step size-n1 table
    const void* tw2;           // six-step size-n2 table
    const void* stw1;          // six-step size-n1 / n2 per-stage tables
    const void* stw2;
    const void* twh;           // four-step twist hi table F::Tw[2^(L-twh_bits)]: w^(j*2^twh_bits)
    int twh_bits;
    const void* cor_lo;        // six-step two-level correction tables (F::T)
    const void* cor_hi;
    int cor_lb;
    uint64_t n1, n2;
    uint64_t p;
    int scale;
    uint64_t ninv, ninv_shoup;
    unsigned long long* counters;
    cudaStream_t stream;
    int num_sms;
    int* launches;
    void* ws;                  // workspace: 2 x batch x N residues
    const void* fst;           // four-step twist table [k1][n2] = w^(k1*n2) (fourstep.cuh), or null
    const void* fst_scaled = nullptr;   // Goldilocks inverse plans: the same table times n^-1 (intt folds its scaling)
    int independent = 0;       // NTT_FLAG_INDEPENDENT: the launch window may defer this call's dependency wait
};

// Launch window (planner.cu): may a fast-kernel launch defer its dependency wait
// to its end?  window_admit registers a launch on the current device's `stream`
// (exclusive: one CTA per SM on every SM); window_break ends the run (any launch
// the window does not model).
bool window_admit(cudaStream_t stream, const void* in, const void* out, uint64_t bytes, bool exclusive);
void window_break(cudaStream_t stream);

// pass count / workspace of a plan (single pass: shared-memory resident, no workspace)
int mp_num_passes(int L, int word, int variant, uint64_t p);
uint64_t mp_workspace_bytes(int L, int word, int variant, uint64_t batch, uint64_t p);
cudaError_t mp_launch_f32s(const MultipassReq& r);
// intt(in .* in2) fused into one fast-kernel launch (u32 p < 2^30, 2^9..2^13); *ok = false otherwise
cudaError_t pointwise_inverse_f32(const MultipassReq& r, const void* in2, bool* ok);
// two-pass four-step for large u32 N (fourstep.cuh, kfs_f32.cu); *ok = false when it does not apply
cudaError_t fourstep_f32(const MultipassReq& r, bool* ok);
cudaError_t fourstep_twist_scale_gold(void* t, uint64_t n, uint64_t c, cudaStream_t s);
// four-step: u32 fields DIT / Flat / DIF / Pease / Pease_nc / Stockham 15 <= L <= 20, Goldilocks 2^14..2^18
// (u32 2^14 is one shared-memory pass: the fast kernel, fast.cuh)
inline bool fourstep_applies(int L, int variant, uint64_t p, int word) {
    if (word == 4)
        return p < (1ull << 32) && L >= 15 && L <= 20 &&
               (variant == V_DIT || variant == V_PEASE_NC || variant == V_DIF || variant == V_FLAT ||
                variant == V_STOCKHAM || variant == V_PEASE);
    // Goldilocks 2^14..2^18 (config 3: 2^16 = 256 x 256)
    return word == 8 && p == 0xFFFFFFFF00000001ull && L >= 14 && L <= 18 &&
           (variant == V_DIT || variant == V_DIF || variant == V_PEASE_NC || variant == V_FLAT ||
            variant == V_STOCKHAM || variant == V_PEASE);
}
inline int fourstep_kr(int L) { return (L + 1) / 2; }
// u32 (p < 2^31) 2^14 outside the four-step (Pease, Stockham): the compile-time tile
// passes (2 x 2^7) instead of the generic shared-memory engine
// (superseded: u32 2^14 now runs every variant in one shared-memory pass)
inline bool tile_2p14_applies(int, int, uint64_t, int) { return false; }
cudaError_t fourstep_twist_build(const void* tw, void* out, int L, int word, cudaStream_t s);
cudaError_t fourstep_gold(const MultipassReq& r, bool* ok);
cudaError_t mp_launch_f32w(const MultipassReq& r);
cudaError_t mp_launch_gold(const MultipassReq& r);
cudaError_t mp_launch_f64(const MultipassReq& r);
cudaError_t pointwise_launch(int kind, uint64_t p, const void* a, const void* b, void* c, uint64_t n,
                             cudaStream_t s, int num_sms, int* launches);

}  // namespace nttb200
