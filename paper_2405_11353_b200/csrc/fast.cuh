// fast.cuh -- specialised single-pass kernels (whole polynomial in shared
// memory) for 2^9 <= N <= 2^13: DIT, DIF, Pease, Pease_nc, Stockham.
//
// Same stage-faithful dataflows as engine.cuh, specialised at compile time:
//  * a TEAM of N/16 threads owns one polynomial at a time; each thread holds a
//    closed 16-element sub-network in registers per group of <= 4 stages;
//    several teams per CTA share one shared-memory twiddle table; teams sync
//    with named barriers (bar.sync id, N/16);
//  * the next polynomial is prefetched by ONE elected thread with a TMA bulk
//    copy (cp.async.bulk ... mbarrier::complete_tx) into the team's staging
//    buffer while the current one is being transformed;
//  * the bit reversal of DIT / Pease is fused into the first group's gather
//    from the staging buffer, DIF's into the last group's scatter to HBM;
//    every global store is a coalesced 128-byte warp row;
//  * stage twiddles come from the per-stage table T[2^(s-1) + k] = w^(k*N/2^s)
//    (the reference's w_pow entries, reordered) in shared memory -- one
//    8-byte LDS per DISTINCT twiddle of a thread's group, immediate offsets;
//  * exchange buffers use a GF(2)-linear XOR swizzle, and each group's
//    thread->sub-network map is chosen so warp accesses are bank-conflict free.
#pragma once
#include <cstdint>
#include <cstdlib>
#include <utility>
#include "engine.cuh"
#include "lazy.cuh"

#ifndef NTT_FAST_EARLY_LOAD
#define NTT_FAST_EARLY_LOAD 1   // deferred-wait launches issue their first rows before the table copy
#endif

namespace nttb200 {
// launch window (planner.cu): may this fast-kernel launch defer its dependency wait?
bool window_admit(cudaStream_t stream, const void* in, const void* out, uint64_t bytes, bool exclusive);
namespace fastk {

NTT_D uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

NTT_D void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
NTT_D void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
NTT_D void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
NTT_D void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
NTT_D void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
NTT_D void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
// programmatic dependent launch (PDL): griddepcontrol is a no-op without the
// launch attribute, so every kernel that calls these stays correct when
// launched plainly
NTT_D void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
NTT_D void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// launch with the programmatic-stream-serialization (PDL) attribute
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// per-SM phase timestamps (tools/fast_timeline.py; experiment builds only)
#ifdef NTT_FAST_TIMELINE
static __device__ unsigned long long g_tl[256 * 64];
NTT_D unsigned smid() { unsigned sm; asm volatile("mov.u32 %0, %%smid;" : "=r"(sm)); return sm; }
NTT_D unsigned long long gtime() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
#define NTT_TL(team, k) g_tl[fastk::smid() * 64 + (team) * 8 + (k)] = fastk::gtime()
#else
#define NTT_TL(team, k) ((void)0)
#endif

NTT_D void team_sync(int id, int nthreads) {
    if (nthreads == 32) __syncwarp();
    else asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <class T>
NTT_HD constexpr int lane_bits() { return sizeof(T) == 4 ? 5 : 4; }

// first-group source: the TMA staging buffer (shared) or HBM directly
template <bool STAGED, class T>
NTT_D T ldsrc(const T* p) {
    if constexpr (STAGED) return *p;
    else return __ldg(p);
}

// Additive padded layout of the exchange buffers: one pad slot per 2^CW
// (and per 2^(2CW), ...) slots, so bit b of a position moves the bank by
// 2^(b mod CW) -- the same conflict-freedom as an XOR fold, but ADDITIVE for
// positions split into disjoint thread / register bits: address =
// padpos(thread part) + padpos(register part) with the second term a
// compile-time immediate offset.
template <class T>
NTT_HD constexpr uint32_t padpos(uint32_t pos) {
    return sizeof(T) == 4 ? pos + (pos >> 5) + (pos >> 10)
                          : pos + (pos >> 4) + (pos >> 8) + (pos >> 12);
}
template <class T, int L>
NTT_HD constexpr int padded_len() { return ((int)padpos<T>((1u << L) - 1) + 1 + 3) & ~3; }

// Bit permutation of a thread id onto the free position bits of a group
// (everything outside the 4-bit register block [B, B+4)).  The first
// lane_bits() thread bits go to free bits with pairwise distinct residues
// mod CW, so a warp's accesses hit distinct banks under the XOR-fold swizzle.
struct Perm {
    int bit[16];
};
NTT_HD constexpr Perm plan_lanes(int L, int B, int CW) {
    Perm P{};
    int fr[16] = {};
    int nf = 0;
    for (int b = 0; b < L; ++b)
        if (b < B || b >= B + 4) fr[nf++] = b;
    bool used[16] = {};
    bool res[8] = {};
    int k = 0;
    for (int i = 0; i < nf && k < CW; ++i) {
        const int r = fr[i] % CW;
        if (!res[r]) { res[r] = true; used[i] = true; P.bit[k++] = fr[i]; }
    }
    for (int i = 0; i < nf; ++i)
        if (!used[i]) P.bit[k++] = fr[i];
    return P;
}

template <int NBITS>
NTT_D uint32_t scatter_bits(uint32_t t, const Perm& P) {
    uint32_t r = 0;
#pragma unroll
    for (int j = 0; j < NBITS; ++j) r |= ((t >> j) & 1u) << P.bit[j];
    return r;
}

// RB = register-block bits: each thread holds 2^RB residues (a closed
// sub-network of <= RB stages).  RB = 4 for every size; RB = 6 for u32 sizes
// of two groups (2^11, 2^12): one shared-memory exchange per polynomial
// instead of two, and a third fewer LDS/STS per butterfly.
template <int L, int RB = 4>
struct Geo {
    static constexpr int N = 1 << L;
    static constexpr int R = 1 << RB;            // residues per thread
    static constexpr int TT = 1 << (L - RB);     // threads per team
    static constexpr int G = (L + RB - 1) / RB;  // register groups
    static constexpr int K0 = L - RB * (G - 1);  // short group (first; DIF: last)
};

template <class A>
struct FastArgs {
    using T = typename A::T;
    const T* in2 = nullptr;   // PW kernels: the second operand (the product in*in2 is transformed)
    using Tw = typename A::Tw;
    const T* in;
    T* out;
    uint64_t batch;
    const Tw* stw;         // stage table, N entries (index 0 unused)
    uint64_t p;
    int scale;
    Tw ninv;
    unsigned long long* counters;
    int defer = 0;         // dependency wait at the kernel's end (see k_fast)
};

// Stage twiddles: stages s <= LS read the shared-memory copy of the per-stage
// table, later stages (only the last stage of 2^14 u32 transforms, whose
// 2^13-entry row would not fit beside the polynomial and its staging buffer)
// read the plan's global copy through the read-only path (L1-resident).
template <class Tw>
NTT_D Tw twld(const Tw* p, bool global) { return global ? __ldg(p) : *p; }
template <class Tw>
NTT_D const Tw* twrow(const Tw* stw, const Tw* gstw, int s, int LS) { return s > LS ? gstw : stw; }
// shared-memory-resident stages of a single-pass L-stage transform
template <class T, int L>
NTT_HD constexpr int fast_smem_stages() { return (sizeof(T) == 4 && L >= 14) ? L - 1 : L; }
// first-group input through a TMA-prefetched staging buffer (else straight from HBM)
template <int V, int L, int RB>
NTT_HD constexpr bool fast_staged() { return RB == 4 && !(V == V_PEASE && L >= 14); }

// DIT-type butterfly of global stage s (1-based) of a single-pass transform:
// stage 1 sees canonical inputs, stage 2 inputs in [0,2p) (lazy bounds)
// (s is a compile-time constant after the callers' loops unroll)
template <class A>
NTT_D void dit_stage_bf(const A& ar, int s, typename A::T& x, typename A::T& y, const typename A::Tw* w, bool triv,
                        bool g = false) {
    if (s == 1) ar.dit1_c(x, y);
    else if (s == 2) { if (triv) ar.dit1_2p(x, y); else ar.dit_2p(x, y, twld(w, g)); }
    else { if (triv) ar.dit1(x, y); else ar.dit(x, y, twld(w, g)); }
}

// ---------------------------------------------------------------- DIT/DIF --
// In-place window [b0, b0+kg) of a register block [B, B+4); pbase = position
// of register 0.  DIT: stages b0+1.. ascending; DIF: descending.
template <class A, int L, int B, int b0, int kg, bool DIF, int RB, int RN, int LS = L>
NTT_D void bitwin_regs(const A& ar, typename A::T (&v)[RN], uint32_t pbase, const typename A::Tw* stw,
                       const typename A::Tw* gstw = nullptr) {
    // (instantiated for every macro-listed geometry; only valid windows emit code)
    if constexpr (b0 >= B && b0 + kg <= B + RB) {
    constexpr int off = b0 - B;
    // block [0,4): pbase has zero low bits, so k = kc is a compile-time constant
    // and every w^0 butterfly skips its multiply
#pragma unroll
    for (int jj = 0; jj < kg; ++jj) {
        const int j = DIF ? kg - 1 - jj : jj;
        const int s = b0 + 1 + j;
        const uint32_t kmask = (1u << (s - 1)) - 1;
        const bool g = s > LS;
        const typename A::Tw* row = twrow(stw, gstw, s, LS) + (1u << (s - 1)) + (pbase & kmask);
#pragma unroll
        for (int c = 0; c < RN; ++c) {
            if (c & (1 << (off + j))) continue;
            const uint32_t kc = ((uint32_t)c << B) & kmask;      // compile-time part of k
            const int hi = c | (1 << (off + j));
            const bool triv = (s == 1 || (B == 0 && kc == 0));      // w^0 = 1
            if (DIF) {
                if (triv) ar.dif1(v[c], v[hi]);
                else ar.dif(v[c], v[hi], twld(row + kc, g));
            } else if (B == 0) {
                dit_stage_bf(ar, s, v[c], v[hi], row + kc, triv, g);
            } else {
                if (triv) ar.dit1(v[c], v[hi]);
                else ar.dit(v[c], v[hi], twld(row + kc, g));
            }
        }
    }
}
}

// -------------------------------------------------------------- Pease -----
// Networks of 2^kg contiguous positions; a thread holds NB = 16/2^kg of them
// (network n = registers [n*2^kg, (n+1)*2^kg)).  Constant geometry inside the
// registers; twiddle k = (B << sg) | (q >> (L - kg - sg)) for butterfly with
// output-bit prefix B (algorithms.py:216-217 in the rotated frame).
template <class A, int L, int sg, int kg, int RB, int RN, int LS = L>
NTT_D void pease_regs(const A& ar, typename A::T (&v)[RN], uint32_t ubase, const typename A::Tw* stw,
                      const typename A::Tw* gstw = nullptr) {
    using T = typename A::T;
    if constexpr (kg <= RB && sg + kg <= L) {        // (only valid windows emit code)
    constexpr int NB = RN >> kg;
    constexpr int H = 1 << (kg - 1);
#pragma unroll
    for (int n = 0; n < NB; ++n) {
        const uint32_t q = (ubase << (RB - kg)) | n;           // network id (L-kg bits)
        const uint32_t qtop = sg ? (q >> ((L - kg - sg) & 31)) : 0u;   // top sg bits of q
#pragma unroll
        for (int m = 0; m < kg; ++m) {
            const int s = sg + m + 1;
            T nv[1 << kg];
#pragma unroll
            for (int i = 0; i < H; ++i) {
                const uint32_t R = 2u * i;
                const uint32_t Bp = R >> (kg - m);               // output bits so far (m bits)
                T x = v[n * (1 << kg) + 2 * i], y = v[n * (1 << kg) + 2 * i + 1];
                const bool triv = (s == 1 || (sg == 0 && Bp == 0));     // w^0 (k = Bp when sg == 0)
                const bool g = s > LS;
                const typename A::Tw* wp = twrow(stw, gstw, s, LS) + (1u << (s - 1)) + ((Bp << sg) | qtop);
                if (sg == 0) dit_stage_bf(ar, s, x, y, wp, triv, g);
                else if (triv) ar.dit1(x, y);
                else ar.dit(x, y, twld(wp, g));
                nv[i] = x;
                nv[i + H] = y;
            }
#pragma unroll
            for (int c = 0; c < (1 << kg); ++c) v[n * (1 << kg) + c] = nv[c];
        }
    }
    }
}

// ------------------------------------------------------------ Stockham ----
// Window of kg pair bits at [lob, lob+kg) of the position (lob = L-sg-kg);
// registers c = (w << (4-kg)) | x, x = extra bits just below the window (first
// group only).  Stage s = sg+m pairs the window's top remaining bit; the
// output bit is inserted above the previous ones ([c_rest | B] layout);
// twiddle k = j = (B << sg) | hi (algorithms.py:281-299).
template <class A, int L, int sg, int kg, int RB, int RN, int LS = L>
NTT_D void stockham_regs(const A& ar, typename A::T (&v)[RN], uint32_t hi, const typename A::Tw* stw,
                         const typename A::Tw* gstw = nullptr) {
    using T = typename A::T;
    if constexpr (kg <= RB && sg + kg <= L) {        // (only valid windows emit code)
    constexpr int NB = RN >> kg;
    constexpr int H = 1 << (kg - 1);
#pragma unroll
    for (int x = 0; x < NB; ++x) {
#pragma unroll
        for (int m = 0; m < kg; ++m) {
            const int s = sg + m;   // 0-based stage
            T nv[1 << kg];
#pragma unroll
            for (int i = 0; i < H; ++i) {
                const uint32_t Bv = i & ((1u << m) - 1), crest = (uint32_t)i >> m;
                T a = v[(i << (RB - kg)) | x], b = v[((i + H) << (RB - kg)) | x];
                const bool triv = (s == 0 || (sg == 0 && Bv == 0));     // w^0 (j = Bv when sg == 0)
                const bool g = s + 1 > LS;
                const typename A::Tw* wp = twrow(stw, gstw, s + 1, LS) + (1u << s) + ((Bv << sg) | hi);
                if (sg == 0) dit_stage_bf(ar, s + 1, a, b, wp, triv, g);
                else if (triv) ar.dit1(a, b);
                else ar.dit(a, b, twld(wp, g));
                nv[(crest << (m + 1)) | Bv] = a;
                nv[(crest << (m + 1)) | (1u << m) | Bv] = b;
            }
#pragma unroll
            for (int c = 0; c < (1 << kg); ++c) v[(c << (RB - kg)) | x] = nv[c];
        }
    }
    }
}

// -------------------------------------------------------------- kernel ----
// SC: n^-1 scaling compiled in (a runtime flag would leave the predicated-off
// multiply in the store loop: 5 issue slots per residue)
template <class A, int V, int L, int TEAMS, bool SC, int RB, bool DS, bool PW = false>
__global__ void __launch_bounds__(TEAMS*(1 << (L - RB)), 1) k_fast(FastArgs<A> a) {
    using T = typename A::T;
    using Tw = typename A::Tw;
    using GG = Geo<L, RB>;
    constexpr int N = GG::N, TT = GG::TT, G = GG::G, K0 = GG::K0, RV = GG::R;
    static_assert(RB == 4 || G <= 2, "wide register blocks: first/last groups only");
    constexpr int CW = lane_bits<T>();
    // Pease keeps two work buffers + the copy-back (algorithms.py:242); Pease_nc
    // and Stockham swap "buffers" through the registers: every thread holds its
    // whole sub-network, so after a team barrier the group writes the same
    // buffer (no copy, one buffer less => one more team per CTA)
    constexpr bool TWO = (V == V_PEASE);
    // RB = 4: TMA-prefetched staging buffer per team (one row ahead).  RB = 6:
    // no staging -- the first group loads its 64 residues per thread straight
    // from HBM (coalesced 128 B warp rows); the smem saved buys twice the teams,
    // whose interleaved load / compute phases hide the latency instead.
    // (Pease 2^14: its two work buffers leave no room for staging -- direct loads)
    constexpr bool STG_ = fast_staged<V, L, RB>();
    constexpr int NBUF = TWO ? 3 : 2;      // staging + work (+ second work buffer for Pease)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // DS: two staging buffers per team, the polynomial after next in flight
    // PW: the two staging buffers hold the two operands of a pointwise product
    // that is taken as the first group reads its input (polymul.py:61-63 fused)
    constexpr int NSTG = STG_ ? ((DS || PW) ? 2 : 1) : 0;
    static_assert(!PW || (STG_ && !DS), "pointwise-fused kernels stage both operands");
    __shared__ uint64_t mbar[TEAMS * 2];
    constexpr int LS = fast_smem_stages<T, L>();     // stages with shared-memory twiddles
    constexpr int NTS = 1 << LS;                     // table entries held in shared memory

    Tw* stw = reinterpret_cast<Tw*>(smem_raw);
    const Tw* gstw = a.stw;
    const int team = threadIdx.x / TT;
    const uint32_t t = threadIdx.x % TT;
    constexpr int NP = padded_len<T, L>();
    T* S = reinterpret_cast<T*>(smem_raw + (size_t)NTS * sizeof(Tw)) + (size_t)team * (NSTG * N + (NBUF - 1) * NP);
    T* W0 = S + NSTG * N;
    T* W1 = TWO ? W0 + NP : W0;
    A ar;
    ar.init(a.p);

#ifdef NTT_FAST_TIMELINE
    if (t == 0) { g_tl[smid() * 64 + team * 8 + 7] = g_tl[smid() * 64 + team * 8 + 5]; NTT_TL(team, 0); }
#endif
    const uint64_t stride = (uint64_t)gridDim.x * TEAMS;
    uint64_t poly = (uint64_t)blockIdx.x * TEAMS + team;
    const uint32_t bytes = N * sizeof(T);
    auto first_loads = [&]() {          // this team's first row (and the one after it)
        if (STG_ && t == 0 && poly < a.batch) {
            mbar_expect_tx(&mbar[2 * team], PW ? 2 * bytes : bytes);
            tma_load_1d(S, a.in + poly * N, bytes, &mbar[2 * team]);
            if (PW) tma_load_1d(S + N, a.in2 + poly * N, bytes, &mbar[2 * team]);
            if (DS && poly + stride < a.batch) {
                mbar_expect_tx(&mbar[2 * team + 1], bytes);
                tma_load_1d(S + N, a.in + (poly + stride) * N, bytes, &mbar[2 * team + 1]);
            }
        }
    };
    if (t == 0) { mbar_init(&mbar[2 * team], 1); mbar_init(&mbar[2 * team + 1], 1); }
    fence_mbar_init();
    // Programmatic dependent launch.  a.defer (host-checked, ntt_api.cu launch_window: this
    // launch's buffers are disjoint from those of every launch on the stream that may still
    // be running): the rows start loading at once, under the previous launch's tail, and the
    // dependency wait moves to the kernel's end (a grid never completes before its
    // predecessor, so stream order holds for whatever follows).  Otherwise the prologue
    // (plan-owned tables only) overlaps the previous launch's tail, the wait precedes the
    // first input read and the trigger follows the wait (a dependent of a waiting launch
    // never overlaps the launch before it).
    if (a.defer) {
        pdl_trigger();
        if (NTT_FAST_EARLY_LOAD) first_loads();
    }
    // twiddle table once per CTA (a thread loop: a bulk async copy measured the same)
    for (int i = threadIdx.x; i < NTS; i += blockDim.x) stw[i] = a.stw[i];
    __syncthreads();
    if (t == 0) NTT_TL(team, 1);
    if (!a.defer) {
        pdl_wait();
        pdl_trigger();
    }
    if (t == 0) NTT_TL(team, 2);
    if (!a.defer || !NTT_FAST_EARLY_LOAD) first_loads();
    uint32_t it = 0;
    int copies = 0;
    const int bar_id = 1 + team;

    for (; poly < a.batch; poly += stride) {
        T v[RV];
        const uint32_t sb_ = DS ? (it & 1) : 0;     // staging buffer of this polynomial
        if (STG_) mbar_wait(&mbar[2 * team + sb_], DS ? ((it >> 1) & 1) : (it & 1));
        if (it == 0 && t == 0) NTT_TL(team, 3);
        ++it;
        T* Sb = S + sb_ * N;
        const T* S0 = STG_ ? Sb : a.in + poly * N;   // first-group source
        // first-group load (PW: the pointwise product of the two staged operands)
        auto ld0 = [&](uint32_t idx) -> T {
            if constexpr (PW) return ar.pwmul(S0[idx], S0[N + idx]);
            else return ldsrc<STG_>(S0 + idx);
        };
        T* gout = a.out + poly * N;
        const uint64_t next = poly + (DS ? 2 : 1) * stride;   // the polynomial this buffer loads next

        if (V == V_DIT || V == V_DIF) {
#pragma unroll
            for (int g = 0; g < G; ++g) {
                // ---- geometry of group g (compile time after unrolling)
                const int B = (V == V_DIT) ? (g == 0 ? 0 : K0 + RB * (g - 1)) : (g == G - 1 ? 0 : L - RB * (g + 1));
                const int kg = (V == V_DIT) ? (g == 0 ? K0 : RB) : (g == G - 1 ? K0 : RB);
                const bool first = g == 0, last = g == G - 1;
                uint32_t pbase;
                if ((V == V_DIT && first) || (V == V_DIF && last)) pbase = brev(t, L - RB) << RB;   // block [0,RB)
                else if ((V == V_DIT && last) || (V == V_DIF && first)) pbase = t;                 // block [L-4,L)
                else {
                    // middle groups: lane-planned map (compile-time permutation)
                    pbase = 0;
#define NTT_MID(BB)                                                           \
    if (B == BB) {                                                            \
        constexpr Perm PM = plan_lanes(L, BB, CW);                            \
        pbase = scatter_bits<L - 4>(t, PM);                                   \
    }
                    NTT_MID(1) NTT_MID(2) NTT_MID(3) NTT_MID(4) NTT_MID(5) NTT_MID(6) NTT_MID(7)
                    NTT_MID(8) NTT_MID(9)
#undef NTT_MID
                }
                // ---- gather
                T* wb = W0 + padpos<T>(pbase);
#pragma unroll
                for (int c = 0; c < RV; ++c) {
                    const uint32_t pos = pbase | ((uint32_t)c << B);
                    // DIT: pbase = brev(t) << 4, so brev(pos) = brev(c) << (L-4) | t (no per-residue BREV)
                    if (first) v[c] = ld0(V == V_DIT ? ((brev((uint32_t)c, RB) << (L - RB)) | t) : pos);
                    else v[c] = wb[padpos<T>((uint32_t)c << B)];
                }
                if (first) {
                    if (STG_) team_sync(bar_id, TT);      // staging consumed: prefetch the next row
                    if (STG_ && t == 0 && next < a.batch) {
                        fence_proxy_async();
                        mbar_expect_tx(&mbar[2 * team + sb_], PW ? 2 * bytes : bytes);
                        tma_load_1d(Sb, a.in + next * N, bytes, &mbar[2 * team + sb_]);
                        if (PW) tma_load_1d(Sb + N, a.in2 + next * N, bytes, &mbar[2 * team + sb_]);
                    }
                }
                // ---- stages
#define NTT_BW(BB, b0v, kgv)                                                                \
    if (B == BB && kg == kgv) bitwin_regs<A, L, BB, b0v, kgv, V == V_DIF, RB, RV, LS>(ar, v, pbase, stw, gstw);
                if (V == V_DIT) {
                    if (g == 0) {
                        NTT_BW(0, 0, 1) NTT_BW(0, 0, 2) NTT_BW(0, 0, 3) NTT_BW(0, 0, 4) NTT_BW(0, 0, 5)
                        NTT_BW(0, 0, 6)
                    } else if (RB == 4) {
                        NTT_BW(1, 1, 4) NTT_BW(2, 2, 4) NTT_BW(3, 3, 4) NTT_BW(4, 4, 4) NTT_BW(5, 5, 4)
                        NTT_BW(6, 6, 4) NTT_BW(7, 7, 4) NTT_BW(8, 8, 4) NTT_BW(9, 9, 4)
                        NTT_BW(10, 10, 4)
                    } else {
                        NTT_BW(5, 5, 6) NTT_BW(6, 6, 6)
                    }
                } else {
                    if (g == G - 1) {
                        NTT_BW(0, 0, 1) NTT_BW(0, 0, 2) NTT_BW(0, 0, 3) NTT_BW(0, 0, 4) NTT_BW(0, 0, 5)
                        NTT_BW(0, 0, 6)
                    } else if (RB == 4) {
                        NTT_BW(1, 1, 4) NTT_BW(2, 2, 4) NTT_BW(3, 3, 4) NTT_BW(4, 4, 4) NTT_BW(5, 5, 4)
                        NTT_BW(6, 6, 4) NTT_BW(7, 7, 4) NTT_BW(8, 8, 4) NTT_BW(9, 9, 4)
                        NTT_BW(10, 10, 4)
                    } else {
                        NTT_BW(5, 5, 6) NTT_BW(6, 6, 6)
                    }
                }
#undef NTT_BW
                // ---- scatter
                if (!last) {
#pragma unroll
                    for (int c = 0; c < RV; ++c) wb[padpos<T>((uint32_t)c << B)] = v[c];
                    team_sync(bar_id, TT);
                } else {
#pragma unroll
                    for (int c = 0; c < RV; ++c) {
                        const uint32_t pos = pbase | ((uint32_t)c << B);
                        T r = ar.fin(v[c]);
                        if (SC) r = ar.mulc(r, a.ninv);
                        gout[V == V_DIF ? ((brev((uint32_t)c, RB) << (L - RB)) | t) : pos] = r;
                    }
                }
            }
        } else {
            // Pease / Pease_nc / Stockham: ping-pong W0 <-> W1 (Pease: + copy back)
            T* src = W0;
            T* dst = W1;
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const int sg = g == 0 ? 0 : K0 + RB * (g - 1);
                const int kg = g == 0 ? K0 : RB;
                const bool first = g == 0, last = g == G - 1;
                if (V != V_STOCKHAM) {
                    // sub-networks: 2^RB contiguous positions (u << RB) | c
                    const uint32_t u = first ? brev(t, L - RB) : t;
                    const T* sb = src + padpos<T>(u << RB);
#pragma unroll
                    for (int c = 0; c < RV; ++c) {
                        v[c] = first ? ld0((brev((uint32_t)c, RB) << (L - RB)) | t) : sb[padpos<T>((uint32_t)c)];   // u = brev(t)
                    }
                    if (first) {
                        if (STG_) team_sync(bar_id, TT);
                        if (STG_ && t == 0 && next < a.batch) {
                            fence_proxy_async();
                            mbar_expect_tx(&mbar[2 * team + sb_], PW ? 2 * bytes : bytes);
                            tma_load_1d(Sb, a.in + next * N, bytes, &mbar[2 * team + sb_]);
                            if (PW) tma_load_1d(Sb + N, a.in2 + next * N, bytes, &mbar[2 * team + sb_]);
                        }
                    }
#define NTT_PE(SG, KGV) \
    if (sg == SG && kg == KGV) pease_regs<A, L, SG, KGV, RB, RV, LS>(ar, v, u, stw, gstw);
                    if (g == 0) { NTT_PE(0, 1) NTT_PE(0, 2) NTT_PE(0, 3) NTT_PE(0, 4) NTT_PE(0, 5) NTT_PE(0, 6) }
                    else if (RB == 4) { NTT_PE(1, 4) NTT_PE(2, 4) NTT_PE(3, 4) NTT_PE(4, 4) NTT_PE(5, 4) NTT_PE(6, 4)
                           NTT_PE(7, 4) NTT_PE(8, 4) NTT_PE(9, 4) NTT_PE(10, 4) }
                    else { NTT_PE(5, 6) NTT_PE(6, 6) }
#undef NTT_PE
                    if (!TWO && !first && !last) team_sync(bar_id, TT);   // all reads of W0 done
                    // outputs: network n = (u << (4-kg)) | n writes q | R << (L-kg)
                    T* db = dst + padpos<T>(u << (RB - kg));
#pragma unroll
                    for (int c = 0; c < RV; ++c) {
                        const uint32_t n = c >> kg, R = c & ((1u << kg) - 1);
                        const uint32_t pos = (((u << (RB - kg)) | n)) | (R << (L - kg));
                        if (last) {
                            T r = ar.fin(v[c]);
                            if (SC) r = ar.mulc(r, a.ninv);
                            gout[pos] = r;
                        } else db[padpos<T>(n | (R << (L - kg)))] = v[c];
                    }
                } else {
                    // Stockham: window [lob, lob+kg); first group: block [L-RB, L)
                    const int lob = L - sg - kg;
                    uint32_t hi, lo;
                    if (first) { hi = 0; lo = t; }
                    else if (last) { hi = t; lo = 0; }
                    else { lo = t & ((1u << lob) - 1); hi = t >> lob; }
                    const T* sb = src + padpos<T>((hi << (L - sg)) | lo);
#pragma unroll
                    for (int c = 0; c < RV; ++c) {
                        // register c = (w << (RB-kg)) | x; position = hi | w | x | lo
                        const uint32_t pos = (hi << (L - sg)) | ((uint32_t)c << (lob - (RB - kg))) | lo;
                        v[c] = first ? ld0(pos) : sb[padpos<T>((uint32_t)c << (lob - (RB - kg)))];
                    }
                    if (first) {
                        if (STG_) team_sync(bar_id, TT);
                        if (STG_ && t == 0 && next < a.batch) {
                            fence_proxy_async();
                            mbar_expect_tx(&mbar[2 * team + sb_], PW ? 2 * bytes : bytes);
                            tma_load_1d(Sb, a.in + next * N, bytes, &mbar[2 * team + sb_]);
                            if (PW) tma_load_1d(Sb + N, a.in2 + next * N, bytes, &mbar[2 * team + sb_]);
                        }
                    }
#define NTT_ST(SG, KGV) \
    if (sg == SG && kg == KGV) stockham_regs<A, L, SG, KGV, RB, RV, LS>(ar, v, hi, stw, gstw);
                    if (g == 0) { NTT_ST(0, 1) NTT_ST(0, 2) NTT_ST(0, 3) NTT_ST(0, 4) NTT_ST(0, 5) NTT_ST(0, 6) }
                    else if (RB == 4) { NTT_ST(1, 4) NTT_ST(2, 4) NTT_ST(3, 4) NTT_ST(4, 4) NTT_ST(5, 4) NTT_ST(6, 4)
                           NTT_ST(7, 4) NTT_ST(8, 4) NTT_ST(9, 4) NTT_ST(10, 4) }
                    else { NTT_ST(5, 6) NTT_ST(6, 6) }
#undef NTT_ST
                    if (!TWO && !first && !last) team_sync(bar_id, TT);   // all reads of W0 done
                    T* db = dst + padpos<T>((hi << lob) | lo);
#pragma unroll
                    for (int c = 0; c < RV; ++c) {
                        // output position = R << (L-kg) | hi << lob | x | lo  with R = window bits
                        const uint32_t R = (uint32_t)c >> (RB - kg), x = (uint32_t)c & ((1u << (RB - kg)) - 1);
                        const uint32_t pos = (R << (L - kg)) | (hi << lob) | (x << (lob - (RB - kg))) | lo;
                        if (last) {
                            T r = ar.fin(v[c]);
                            if (SC) r = ar.mulc(r, a.ninv);
                            gout[pos] = r;
                        } else db[padpos<T>((R << (L - kg)) | (x << (lob - (RB - kg))))] = v[c];
                    }
                }
                if (!last) {
                    team_sync(bar_id, TT);
                    if (V == V_PEASE) {       // _stage_copy(cur, nxt)  (algorithms.py:242)
                        for (int i = t; i < NP; i += TT) src[i] = dst[i];
                        ++copies;
                        team_sync(bar_id, TT);
                    }                         // Pease_nc / Stockham: roles swap in place
                }
            }
        }
        // work buffers free for the next row: with a staging buffer the next
        // row's "staging consumed" barrier (after its first gather, before its
        // first scatter) already orders every read of this row's last group
        if (it == 1 && t == 0) NTT_TL(team, 4);
        if (!STG_) team_sync(bar_id, TT);
        if (a.counters && t == 0) {
            atomicAdd(a.counters + C_TRANSFORMS, 1ull);
            atomicAdd(a.counters + C_HBM, 1ull);
            if (V != V_STOCKHAM) atomicAdd(a.counters + C_BITREV, 1ull);
            if (V == V_PEASE) { atomicAdd(a.counters + C_COPIES, (unsigned long long)copies); copies = 0; }
        }
    }
    if (t == 0) NTT_TL(team, 5);
    if (a.defer && threadIdx.x == 0) pdl_wait();
}

// ------------------------------------------------------------- launcher --
#ifndef NTT_FAST_MAX_THREADS
#define NTT_FAST_MAX_THREADS 1024
#endif
constexpr int kFastMaxThreads = NTT_FAST_MAX_THREADS;
// 64 residues per thread (RB = 6) for 2^11 / 2^12 cuts instructions per
// butterfly from 10.3 to 7.8 but caps a CTA at 512 threads (128 registers):
// measured 48 us vs 38 us for RB = 4 on config 2 (4 warps/SMSP cannot hide the
// dependency latency; profiles/r1/summary.md).  Kept selectable for study.
#ifndef NTT_FAST_DS
#define NTT_FAST_DS 1     // double staging where the shared memory allows it without losing a team
#endif
#ifndef NTT_FAST_WIDE_RB
#define NTT_FAST_WIDE_RB 4
#endif

template <class A, int V, int L, bool PW = false>
struct FastCfg {
    using T = typename A::T;
    using Tw = typename A::Tw;
    static constexpr int N = 1 << L;
    // register-block bits (NTT_FAST_WIDE_RB = 6 only where two groups cover the transform)
    static constexpr int RB = (sizeof(T) == 4 && (L == 11 || L == 12)) ? NTT_FAST_WIDE_RB : 4;
    static constexpr int TT = 1 << (L - RB);
    static constexpr int NBUF = (V == V_PEASE) ? 3 : 2;
    // opt-in limit per block (227 KiB, static shared memory included) minus the mbarriers
    static constexpr long kSmemCap = 227 * 1024 - 256;
    static constexpr long table = (long)(1 << fast_smem_stages<T, L>()) * sizeof(Tw);
    static constexpr long team_bytes_n(int nstg) {
        return ((fast_staged<V, L, RB>() ? (long)N * nstg : 0L) + (long)(NBUF - 1) * padded_len<T, L>()) * sizeof(T);
    }
    static constexpr int teams_n(int nstg) {
        const int by_smem = (int)((kSmemCap - table) / team_bytes_n(nstg));
        const int by_thr = kFastMaxThreads / TT;
        const int t0 = by_smem < by_thr ? by_smem : by_thr;
        return t0 > 8 ? 8 : (t0 < 0 ? 0 : t0);
    }
    // double staging (two polynomials in flight per team) where it costs no team
    static constexpr bool DS = !PW && NTT_FAST_DS && fast_staged<V, L, RB>() && teams_n(2) == teams_n(1);
    static constexpr int TEAMS = (PW && RB != 4) ? 0 : teams_n((DS || PW) ? 2 : 1);
    static constexpr long team_bytes = team_bytes_n((DS || PW) ? 2 : 1);
    static constexpr long smem = table + (long)TEAMS * team_bytes;
};

constexpr long kMinFastSmem = 40 * 1024;     // smallest shared-memory footprint of a k_fast CTA (2^9, u32)
template <class A, int L>
constexpr uint64_t N_BYTES() { return (uint64_t)sizeof(typename A::T) << L; }
template <class A, int V, int L>
cudaError_t launch_fast_L(const FastArgs<A>& a, cudaStream_t s, int num_sms, int* launches, bool* ok) {
    using C = FastCfg<A, V, L>;
    if constexpr (C::TEAMS < 1) {
        *ok = false;
        return cudaSuccess;
    } else {
        auto kern = a.scale ? k_fast<A, V, L, C::TEAMS, true, C::RB, C::DS> : k_fast<A, V, L, C::TEAMS, false, C::RB, C::DS>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem);
        if (e != cudaSuccess) return e;
        int occ = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::TEAMS * C::TT, C::smem) != cudaSuccess || occ < 1)
            occ = 1;
        uint64_t ctas = (a.batch + C::TEAMS - 1) / C::TEAMS;
        const uint64_t cap = (uint64_t)num_sms * occ;
        uint64_t grid = ctas < cap ? ctas : cap;
        *ok = true;
        if (grid == 0) return cudaSuccess;
        // launch window (planner.cu): defer the dependency wait when the buffers are disjoint from
        // every launch that may still run; a launch of one CTA per SM on every SM is exclusive
        FastArgs<A> al = a;
        // (every launch registers its spans; only calls flagged NTT_FLAG_INDEPENDENT -- a.defer preset --
        // may defer: a foreign kernel on the stream could have produced this call's input)
        // exclusive: one CTA on EVERY SM whose footprint leaves no room for a CTA of any other
        // single-pass launch (each takes at least kMinFastSmem), so once all of this launch's CTAs
        // have started, every older launch has left every SM
        static_assert(C::smem >= kMinFastSmem, "the launch window assumes this lower bound");
        const bool admit = nttb200::window_admit(s, a.in, a.out, a.batch * N_BYTES<A, L>(),
                                                 occ == 1 && C::smem + kMinFastSmem > 227 * 1024 &&
                                                     grid == (uint64_t)num_sms);
        al.defer = (a.defer && admit) ? 1 : 0;
        cudaError_t le = launch_pdl(kern, dim3((unsigned)grid), dim3(C::TEAMS * C::TT), C::smem, s, al);
        if (launches) ++*launches;
        return le != cudaSuccess ? le : cudaGetLastError();
    }
}

// d_out = intt(in .* in2): pointwise product fused into the first group's
// loads, n^-1 (times the Montgomery factor) into the last group's stores
template <class A, int V, int L>
cudaError_t launch_fast_pw_L(const FastArgs<A>& a, cudaStream_t s, int num_sms, int* launches, bool* ok) {
    using C = FastCfg<A, V, L, true>;
    if constexpr (C::TEAMS < 1) {
        *ok = false;
        return cudaSuccess;
    } else {
        auto kern = k_fast<A, V, L, C::TEAMS, true, C::RB, false, true>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem);
        if (e != cudaSuccess) return e;
        uint64_t ctas = (a.batch + C::TEAMS - 1) / C::TEAMS;
        uint64_t grid = ctas < (uint64_t)num_sms ? ctas : (uint64_t)num_sms;
        *ok = true;
        if (grid == 0) return cudaSuccess;
        cudaError_t le = launch_pdl(kern, dim3((unsigned)grid), dim3(C::TEAMS * C::TT), C::smem, s, a);
        if (launches) ++*launches;
        return le != cudaSuccess ? le : cudaGetLastError();
    }
}

template <class A, int V>
cudaError_t launch_fast_pw(int L, const FastArgs<A>& a, cudaStream_t s, int num_sms, int* launches, bool* ok) {
    *ok = false;
    switch (L) {
        case 9: return launch_fast_pw_L<A, V, 9>(a, s, num_sms, launches, ok);
        case 10: return launch_fast_pw_L<A, V, 10>(a, s, num_sms, launches, ok);
        case 11: return launch_fast_pw_L<A, V, 11>(a, s, num_sms, launches, ok);
        case 12: return launch_fast_pw_L<A, V, 12>(a, s, num_sms, launches, ok);
        case 13: return launch_fast_pw_L<A, V, 13>(a, s, num_sms, launches, ok);
        default: return cudaSuccess;
    }
}

template <class A, int V>
cudaError_t launch_fast(int L, const FastArgs<A>& a, cudaStream_t s, int num_sms, int* launches, bool* ok) {
    *ok = false;
    switch (L) {
        case 9: return launch_fast_L<A, V, 9>(a, s, num_sms, launches, ok);
        case 10: return launch_fast_L<A, V, 10>(a, s, num_sms, launches, ok);
        case 11: return launch_fast_L<A, V, 11>(a, s, num_sms, launches, ok);
        case 12: return launch_fast_L<A, V, 12>(a, s, num_sms, launches, ok);
        case 13: return launch_fast_L<A, V, 13>(a, s, num_sms, launches, ok);
        case 14: return launch_fast_L<A, V, 14>(a, s, num_sms, launches, ok);
        default: return cudaSuccess;
    }
}

}  // namespace fastk
}  // namespace nttb200
