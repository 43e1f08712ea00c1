// launch.cuh -- host-side pass planner and per-field launchers (instantiated
// once per field in k_<field>.cu so the four fields compile in parallel).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <type_traits>
#include "multipass.cuh"
#include "fast.cuh"
#include "tiles.cuh"

namespace nttb200 {

// Residues a tile may hold: two buffers of this many residues = 64 KiB.
template <class T>
constexpr int tile_elems_log2() { return sizeof(T) == 4 ? 13 : 12; }
// Largest log2 N handled by ONE pass (a whole row resident in shared memory).
inline int single_pass_max_log2(int word) { return word == 4 ? 14 : 13; }

template <class F>
inline typename F::Tw make_tw(uint64_t w, uint64_t ws);
template <> inline uint2 make_tw<F32S>(uint64_t w, uint64_t ws) { return make_uint2((uint32_t)w, (uint32_t)ws); }
template <> inline uint2 make_tw<F32W>(uint64_t w, uint64_t ws) { return make_uint2((uint32_t)w, (uint32_t)ws); }
template <> inline uint64_t make_tw<FGold>(uint64_t w, uint64_t) { return w; }
template <> inline ulonglong2 make_tw<F64>(uint64_t w, uint64_t ws) { return make_ulonglong2(w, ws); }

// Pass decomposition of L stages (multi-pass variants): K_i per pass.
inline int plan_passes(int L, int word, int variant, int* K) {
    const int elog = word == 4 ? 13 : 12;
    const int kcap = elog - 3;                 // keep >= 8 networks per tile
    int P = (L + kcap - 1) / kcap;
    if (P < 2) P = 2;
    for (int i = 0; i < P; ++i) K[i] = L / P + (i < L % P ? 1 : 0);
    (void)variant;
    return P;
}

template <class F, int V, int LAY>
cudaError_t run_pass(PassArgs<F>& a, cudaStream_t s, int num_sms, int* launches) {
    using T = typename F::T;
    const size_t smem = 2ull * ((size_t)a.TQ << a.K) * sizeof(T);
    auto kern = k_pass<F, V, LAY>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
    const int M = LAY == LAY_VARIANT ? a.L - a.K : (LAY == LAY_SIX_A ? a.l1 : a.l2);
    const uint64_t ntiles = a.qmode == QM_ROWS ? (a.batch + a.TQ - 1) / a.TQ
                                               : a.batch * ((1ull << M) / a.TQ);
    uint64_t grid = (uint64_t)num_sms * occ;
    if (grid > ntiles) grid = ntiles;
    if (grid == 0) return cudaSuccess;
    kern<<<(unsigned)grid, kThreads, smem, s>>>(a);
    if (launches) ++*launches;
    return cudaGetLastError();
}

template <class F>
PassArgs<F> base_args(const MultipassReq& r) {
    PassArgs<F> a{};
    a.batch = r.batch;
    a.L = r.L;
    a.tw = static_cast<const typename F::Tw*>(r.tw);
    a.f.p = (typename F::T)r.p;
    a.ninv = make_tw<F>(r.ninv, r.ninv_shoup);
    a.counters = r.counters;
    a.TA = 1;
    return a;
}

template <class T>
__global__ void k_copy(const T* src, T* dst, uint64_t n, uint64_t rows, unsigned long long* counters) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
    if (counters && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(counters + C_COPIES, (unsigned long long)rows);
}

template <class A, int V>
cudaError_t run_fast_policy(const MultipassReq& r, bool* ok) {
    fastk::FastArgs<A> a{};
    a.in = static_cast<const typename A::T*>(r.in);
    a.out = static_cast<typename A::T*>(r.out);
    a.batch = r.batch;
    a.stw = static_cast<const typename A::Tw*>(r.stw);
    a.p = r.p;
    a.scale = r.scale;
    a.ninv = make_tw<typename A::Field>(r.ninv, r.ninv_shoup);
    a.counters = r.counters;
    a.defer = r.independent;       // allowed; the launcher's window check decides
    return fastk::launch_fast<A, V>(r.L, a, r.stream, r.num_sms, r.launches, ok);
}

// intt(in .* in2) in one fast-kernel launch (LazyF32, 2^9..2^13): the caller
// passes r.ninv / r.ninv_shoup = n^-1 * 2^32 mod p (the Montgomery factor of
// the fused pointwise product)
template <int V>
cudaError_t run_fast_pw(const MultipassReq& r, const void* in2, bool* ok) {
    fastk::FastArgs<LazyF32> a{};
    a.in = static_cast<const uint32_t*>(r.in);
    a.in2 = static_cast<const uint32_t*>(in2);
    a.out = static_cast<uint32_t*>(r.out);
    a.batch = r.batch;
    a.stw = static_cast<const uint2*>(r.stw);
    a.p = r.p;
    a.scale = 1;
    a.ninv = make_uint2((uint32_t)r.ninv, (uint32_t)r.ninv_shoup);
    a.counters = r.counters;
    return fastk::launch_fast_pw<LazyF32, V>(r.L, a, r.stream, r.num_sms, r.launches, ok);
}

// Specialised single-pass kernels (fast.cuh) where they apply.
template <class F, int V0>
cudaError_t try_fast(const MultipassReq& r, bool* ok) {
    // Flat's per-stage states are DIT's (algorithms.py:161-195; its separate
    // bit_reverse_permute is the gather DIT fuses): the DIT kernel serves it
    constexpr int V = V0 == V_FLAT ? V_DIT : V0;
    *ok = false;
    if (V == V_NAIVE || V == V_SIXSTEP) return cudaSuccess;
    if (r.L < 9 || r.L > (sizeof(typename F::T) == 4 ? 14 : 13) || !r.stw) return cudaSuccess;
    if ((reinterpret_cast<uintptr_t>(r.in) & 15) || (reinterpret_cast<uintptr_t>(r.out) & 15)) return cudaSuccess;
    if constexpr (std::is_same<F, F32S>::value) {
        if (r.p < (1ull << 30)) return run_fast_policy<LazyF32, V>(r, ok);
        return run_fast_policy<Canon<F32S>, V>(r, ok);
    } else if constexpr (std::is_same<F, FGold>::value) {
        return run_fast_policy<GoldPolicy<V == V_DIF>, V>(r, ok);
    } else if constexpr (std::is_same<F, F32W>::value) {
        return run_fast_policy<Canon<F32W>, V>(r, ok);     // 2^31 <= p < 2^32 (DEFAULT_PRIME)
    } else if constexpr (std::is_same<F, F64>::value) {
        return run_fast_policy<Canon<F64>, V>(r, ok);      // generic 64-bit primes (Shoup, 65-bit z)
    } else {
        return cudaSuccess;
    }
}

template <class F, int V>
cudaError_t run_variant(const MultipassReq& r) {
    using T = typename F::T;
    const int L = r.L;
    const uint64_t N = 1ull << L;
    constexpr int elog = tile_elems_log2<T>();
    if constexpr (std::is_same<F, F32S>::value || std::is_same<F, F32W>::value || std::is_same<F, FGold>::value) {
        bool ok = false;                                                             // four-step (fourstep.cuh)
        cudaError_t fe = std::is_same<F, FGold>::value ? fourstep_gold(r, &ok) : fourstep_f32(r, &ok);
        if (fe != cudaSuccess || ok) return fe;
    }
    if constexpr (std::is_same<F, F32S>::value) {
        if (tile_2p14_applies(L, V, r.p, 4) && r.ws) {
            bool ok = false;
            cudaError_t te = tile_passes_f32(V, r.p < (1ull << 30), r, &ok);
            if (te != cudaSuccess || ok) return te;
        }
    }
    if (L <= single_pass_max_log2(sizeof(T))) {
        bool ok = false;
        cudaError_t fe = try_fast<F, V>(r, &ok);
        if (fe != cudaSuccess || ok) return fe;
        // ---- one pass: TQ whole rows per tile, bit reversal fused into the groups
        PassArgs<F> a = base_args<F>(r);
        a.in = static_cast<const T*>(r.in);
        a.out = static_cast<T*>(r.out);
        a.K = L;
        a.S0 = 0;
        int tq = L >= elog ? 1 : (1 << (elog - L));
        a.TQ = tq > 256 ? 256 : tq;
        a.qmode = QM_ROWS;
        a.in_order = a.out_order = ORD_C_FAST;
        a.rev_first = (V == V_DIT || V == V_FLAT || V == V_PEASE || V == V_PEASE_NC);
        a.rev_last = (V == V_DIF);
        a.count_row = 1;
        a.count_bitrev = (V == V_STOCKHAM) ? 0 : 1;
        a.scale = r.scale;
        return run_pass<F, V, LAY_VARIANT>(a, r.stream, r.num_sms, r.launches);
    }
    // ---- multi-pass: compile-time tile kernels where a tile shape exists
    {
        bool ok = false;
        cudaError_t te = cudaSuccess;
        if constexpr (std::is_same<F, F32S>::value) te = tile_passes_f32(V, r.p < (1ull << 30), r, &ok);
        else if constexpr (std::is_same<F, FGold>::value) te = tile_passes_gold(V, r, &ok);
        if (te != cudaSuccess || ok) return te;
    }
    int K[8];
    const int P = plan_passes(L, sizeof(T), V, K);
    T* ws0 = static_cast<T*>(r.ws);
    T* ws1 = ws0 + r.batch * N;
    const T* cur = static_cast<const T*>(r.in);
    cudaError_t e = cudaSuccess;
    if (V == V_FLAT) {                     // bit_reverse_permute as its own HBM pass
        uint64_t blocks = r.batch << (L - 12);
        uint64_t cap = (uint64_t)r.num_sms * 8;
        k_bitrev<T><<<(unsigned)(blocks < cap ? blocks : cap), 256, 0, r.stream>>>(cur, ws1, r.batch, L, r.counters);
        if (r.launches) ++*r.launches;
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        cur = ws1;
    }
    int done = 0;   // stages (or low bits) already applied
    for (int i = 0; i < P; ++i) {
        PassArgs<F> a = base_args<F>(r);
        const bool last = (i == P - 1);
        T* dst = last ? static_cast<T*>(r.out) : ((cur == ws0) ? ws1 : ws0);
        if (V == V_PEASE && !last) dst = ws0;      // Pease: write dst, copy back into src (ws1)
        a.in = cur;
        a.out = dst;
        a.K = K[i];
        a.TQ = 1 << (elog - K[i]);
        if (a.TQ > 256) a.TQ = 256;
        a.count_row = last;
        a.scale = last ? r.scale : 0;
        const int Mq = L - K[i];
        if (V == V_DIT || V == V_FLAT) {
            a.S0 = done;
            if (i == 0 && V == V_DIT) {
                a.qmode = QM_REV; a.rev_in = 1; a.in_order = ORD_T_FAST; a.out_order = ORD_C_FAST;
                a.count_bitrev = 1;
            } else if (i == 0) {
                a.qmode = QM_LINEAR; a.in_order = ORD_C_FAST; a.out_order = ORD_C_FAST;
            } else {
                a.qmode = QM_LINEAR; a.in_order = ORD_T_FAST; a.out_order = ORD_T_FAST;
            }
            e = run_pass<F, V_DIT, LAY_VARIANT>(a, r.stream, r.num_sms, r.launches);
            done += K[i];
        } else if (V == V_DIF) {
            const int Kd = K[P - 1 - i];           // windows from the top bit down
            a.K = Kd;
            a.TQ = 1 << (elog - Kd);
            if (a.TQ > 256) a.TQ = 256;
            a.S0 = L - done - Kd;
            if (last) {
                a.qmode = QM_REV; a.rev_out = 1; a.in_order = ORD_C_FAST; a.out_order = ORD_T_FAST;
                a.count_bitrev = 1;
            } else {
                a.qmode = QM_LINEAR; a.in_order = ORD_T_FAST; a.out_order = ORD_T_FAST;
            }
            e = run_pass<F, V_DIF, LAY_VARIANT>(a, r.stream, r.num_sms, r.launches);
            done += Kd;
        } else if (V == V_PEASE || V == V_PEASE_NC) {
            a.S0 = done;
            if (i == 0) {
                int ta = 1;
                while (ta * ta < a.TQ) ta <<= 1;    // TQ = TA x TB, TA >= TB
                if (ta > (1 << Mq)) ta = 1 << Mq;
                a.TA = ta;
                a.qmode = QM_2D; a.rev_in = 1; a.in_order = ORD_T_FAST; a.out_order = ORD_TB_FAST;
                a.count_bitrev = 1;
            } else {
                a.qmode = QM_LINEAR; a.in_order = ORD_C_FAST; a.out_order = ORD_T_FAST;
            }
            e = run_pass<F, V_PEASE_NC, LAY_VARIANT>(a, r.stream, r.num_sms, r.launches);
            done += K[i];
            if (e == cudaSuccess && V == V_PEASE) {   // _stage_copy per pass (algorithms.py:242)
                uint64_t n = r.batch * N;
                k_copy<T><<<r.num_sms * 4, 256, 0, r.stream>>>(dst, ws1, n, r.batch, r.counters);
                if (r.launches) ++*r.launches;
                e = cudaGetLastError();
                dst = ws1;
            }
        } else {  // V_STOCKHAM
            a.S0 = done;
            a.qmode = QM_LINEAR;
            a.in_order = (L - done - K[i]) > 0 ? ORD_T_FAST : ORD_C_FAST;
            a.out_order = ORD_T_FAST;
            e = run_pass<F, V_STOCKHAM, LAY_VARIANT>(a, r.stream, r.num_sms, r.launches);
            done += K[i];
        }
        if (e != cudaSuccess) return e;
        cur = dst;
    }
    return cudaSuccess;
}

// ---- six-step with any split (algorithms.py:355-389) whose sub-transforms
// exceed one shared-memory pass: the same six steps out of batched pieces --
// transposes, the batched size-n2 / size-n1 DITs through the ordinary
// dispatcher (multi-pass / four-step as their sizes need), and the correction
// w_N^(i*k2) from the plan's two-level table.  Workspace 4 x batch x N.
template <class F>
__global__ void k_transpose_gen(const typename F::T* in, typename F::T* out, uint64_t batch, int rb, int cb,
                                F f, int scale, typename F::T ninv) {
    using T = typename F::T;
    __shared__ T tile[32][33];
    const uint64_t R = 1ull << rb, C = 1ull << cb;
    const uint64_t tr = (R + 31) / 32, tc = (C + 31) / 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (uint64_t blk = blockIdx.x; blk < batch * tr * tc; blk += gridDim.x) {
        const uint64_t b = blk / (tr * tc), rem = blk % (tr * tc);
        const uint64_t br = (rem / tc) * 32, bc = (rem % tc) * 32;
        const T* src = in + b * R * C;
        T* dst = out + b * R * C;
        for (int k = ty; k < 32; k += 8)
            if (br + k < R && bc + tx < C) tile[k][tx] = src[(br + k) * C + bc + tx];
        __syncthreads();
        for (int k = ty; k < 32; k += 8)
            if (bc + k < C && br + tx < R) {
                T v = tile[tx][k];
                if (scale) v = f.mul_full(v, ninv);
                dst[(bc + k) * R + br + tx] = v;
            }
        __syncthreads();
    }
}

template <class F>
__global__ void k_six_correct(typename F::T* a, uint64_t batch, int l1, int l2, const typename F::T* cor_lo,
                              const typename F::T* cor_hi, int cor_lb, F f) {
    const uint64_t n = 1ull << (l1 + l2);
    for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < batch * n;
         idx += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t e0 = idx & (n - 1);
        const uint64_t i = e0 >> l2, k2 = e0 & ((1ull << l2) - 1);
        const uint64_t e = (i * k2) & (n - 1);
        const typename F::T w = f.mul_full(cor_hi[e >> cor_lb], cor_lo[e & ((1ull << cor_lb) - 1)]);
        a[idx] = f.mul_full(a[idx], w);
    }
}

template <class F>
cudaError_t launch_field(const MultipassReq& r);

template <class F>
cudaError_t run_sixstep_general(const MultipassReq& r) {
    using T = typename F::T;
    int l1 = 0, l2 = 0;
    while ((1ull << l1) < r.n1) ++l1;
    while ((1ull << l2) < r.n2) ++l2;
    const uint64_t N = 1ull << (l1 + l2);
    T* w0 = static_cast<T*>(r.ws);
    T* w1 = w0 + r.batch * N;
    T* wsub = w1 + r.batch * N;                 // 2 x batch x N for the sub-transforms' own passes
    F f;
    f.p = (T)r.p;
    const unsigned tgrid = (unsigned)((r.batch * ((N + 1023) / 1024) < (uint64_t)r.num_sms * 8)
                                          ? r.batch * ((N + 1023) / 1024) : (uint64_t)r.num_sms * 8);
    auto sub = [&](const void* tw, const void* stw, int L, uint64_t rows, T* buf) -> cudaError_t {
        MultipassReq q = r;
        q.variant = V_DIT; q.L = L; q.in = buf; q.out = buf; q.batch = rows;
        q.tw = tw; q.stw = stw; q.scale = 0; q.fst = nullptr; q.ws = wsub;
        q.counters = nullptr;                    // the pieces are not transforms of the plan's size
        return L == 0 ? cudaSuccess : launch_field<F>(q);
    };
    cudaError_t e;
    // T1: x[j*n1 + i] -> w0[i][j]
    k_transpose_gen<F><<<tgrid, 256, 0, r.stream>>>(static_cast<const T*>(r.in), w0, r.batch, l2, l1, f, 0, T(0));
    if (r.launches) ++*r.launches;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // D1: size-n2 DIT of every column i (algorithms.py:372-376)
    if ((e = sub(r.tw2, r.stw2, l2, r.batch << l1, w0)) != cudaSuccess) return e;
    // C: w0[i][k2] *= w_N^(i*k2) (algorithms.py:377-379)
    k_six_correct<F><<<(unsigned)r.num_sms * 8, 256, 0, r.stream>>>(w0, r.batch, l1, l2, static_cast<const T*>(r.cor_lo),
                                                                    static_cast<const T*>(r.cor_hi), r.cor_lb, f);
    if (r.launches) ++*r.launches;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // T2: w0[i][k2] -> w1[k2][i]
    k_transpose_gen<F><<<tgrid, 256, 0, r.stream>>>(w0, w1, r.batch, l1, l2, f, 0, T(0));
    if (r.launches) ++*r.launches;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // D2: size-n1 DIT of every row k2 (algorithms.py:381-387)
    if ((e = sub(r.tw1, r.stw1, l1, r.batch << l2, w1)) != cudaSuccess) return e;
    // T3: w1[k2][k1] -> out[k1*n2 + k2] (n^-1 folded in for intt)
    k_transpose_gen<F><<<tgrid, 256, 0, r.stream>>>(w1, static_cast<T*>(r.out), r.batch, l2, l1, f, r.scale,
                                                   (T)r.ninv);
    if (r.launches) ++*r.launches;
    return cudaGetLastError();
}

template <class F>
cudaError_t run_sixstep(const MultipassReq& r) {
    using T = typename F::T;
    if (r.n1 > (1ull << single_pass_max_log2(sizeof(T))) || r.n2 > (1ull << single_pass_max_log2(sizeof(T))))
        return run_sixstep_general<F>(r);
    if constexpr (std::is_same<F, FGold>::value) {
        bool ok = false;
        cudaError_t te = tile_sixstep_gold(r, &ok);
        if (te != cudaSuccess || ok) return te;
    }
    constexpr int elog = tile_elems_log2<T>();
    int l1 = 0, l2 = 0;
    while ((1ull << l1) < r.n1) ++l1;
    while ((1ull << l2) < r.n2) ++l2;
    T* rows = static_cast<T*>(r.ws);
    cudaError_t e;
    // pass A: x[i::n1] -> bitrev + DIT(n2) -> * w^(i*k2) -> rows[i][k2]
    {
        PassArgs<F> a = base_args<F>(r);
        a.in = static_cast<const T*>(r.in);
        a.out = rows;
        a.l1 = l1; a.l2 = l2;
        a.K = l2;
        int tq = l2 >= elog ? 1 : 1 << (elog - l2);
        if (tq > (1 << l1)) tq = 1 << l1;
        a.TQ = tq > 256 ? 256 : tq;
        a.qmode = QM_LINEAR; a.in_order = ORD_T_FAST; a.out_order = ORD_C_FAST;
        a.rev_first = l2 > 0;
        a.count_bitrev = 0;
        a.tw = static_cast<const typename F::Tw*>(r.tw2);
        a.tw_main = r.cor_lo ? nullptr : static_cast<const typename F::Tw*>(r.tw);
        a.cor_lo = static_cast<const T*>(r.cor_lo);
        a.cor_hi = static_cast<const T*>(r.cor_hi);
        a.cor_lb = r.cor_lb;
        if (l2 == 0) { a.K = 0; }
        e = run_pass<F, V_DIT, LAY_SIX_A>(a, r.stream, r.num_sms, r.launches);
        if (e != cudaSuccess) return e;
    }
    // pass B: rows[:, k2] -> bitrev + DIT(n1) -> out[n2*k1 + k2]
    {
        PassArgs<F> a = base_args<F>(r);
        a.in = rows;
        a.out = static_cast<T*>(r.out);
        a.l1 = l1; a.l2 = l2;
        a.K = l1;
        int tq = l1 >= elog ? 1 : 1 << (elog - l1);
        if (tq > (1 << l2)) tq = 1 << l2;
        a.TQ = tq > 256 ? 256 : tq;
        a.qmode = QM_LINEAR; a.in_order = ORD_T_FAST; a.out_order = ORD_T_FAST;
        a.rev_first = l1 > 0;
        a.count_row = 1;
        a.tw = static_cast<const typename F::Tw*>(r.tw1);
        a.scale = r.scale;
        e = run_pass<F, V_DIT, LAY_SIX_B>(a, r.stream, r.num_sms, r.launches);
    }
    return e;
}

template <class F>
cudaError_t launch_field(const MultipassReq& r) {
    using T = typename F::T;
    if (r.batch == 0) return cudaSuccess;
    if (r.variant == V_NAIVE) {
        const uint64_t total = r.batch << r.L;
        const uint64_t blocks = (total + 255) / 256, cap = (uint64_t)r.num_sms * 16;
        F f;
        f.p = (T)r.p;
        k_naive<F><<<(unsigned)(blocks < cap ? blocks : cap), 256, 0, r.stream>>>(
            static_cast<const T*>(r.in), static_cast<T*>(r.out), r.batch, r.L,
            static_cast<const typename F::Tw*>(r.tw), f, r.scale, make_tw<F>(r.ninv, r.ninv_shoup), r.counters);
        if (r.launches) ++*r.launches;
        return cudaGetLastError();
    }
    switch (r.variant) {
        case V_DIT: return run_variant<F, V_DIT>(r);
        case V_DIF: return run_variant<F, V_DIF>(r);
        case V_FLAT: return run_variant<F, V_FLAT>(r);
        case V_PEASE: return run_variant<F, V_PEASE>(r);
        case V_PEASE_NC: return run_variant<F, V_PEASE_NC>(r);
        case V_STOCKHAM: return run_variant<F, V_STOCKHAM>(r);
        case V_SIXSTEP: return run_sixstep<F>(r);
        default: return cudaErrorInvalidValue;
    }
}

template <class F>
cudaError_t pointwise_field(uint64_t p, const void* a, const void* b, void* c, uint64_t n, cudaStream_t s,
                            int num_sms, int* launches) {
    using T = typename F::T;
    F f;
    f.p = (T)p;
    uint64_t blocks = (n + 255) / 256, cap = (uint64_t)num_sms * 8;
    if (n == 0) return cudaSuccess;
    k_pointwise<F><<<(unsigned)(blocks < cap ? blocks : cap), 256, 0, s>>>(
        static_cast<const T*>(a), static_cast<const T*>(b), static_cast<T*>(c), n, f);
    if (launches) ++*launches;
    return cudaGetLastError();
}

}  // namespace nttb200
