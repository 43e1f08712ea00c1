// lazy.cuh -- butterfly policies for the fast kernels.
//
// LazyF32 (p < 2^30): Harvey-style lazy Shoup butterflies.  DIT-type values
// live in [0,4p) between stages and DIF-type values in [0,2p); one final
// reduction makes them canonical, so the transform OUTPUT is bit-identical
// to the reference (intermediate stage values are congruent mod p, not
// canonical).  7 integer ops per DIT butterfly instead of 9.
// Canon<F>: the canonical field ops of arith.cuh behind the same interface
// (every stage canonical, exactly like the reference).
#pragma once
#include "arith.cuh"
#include <type_traits>

namespace nttb200 {

struct LazyF32 {
    using T = uint32_t;
    using Tw = uint2;
    using Field = F32S;
    static constexpr bool lazy = true;
    uint32_t p, p2, p4;
    uint32_t pinv;            // -p^-1 mod 2^32 (Montgomery, pointwise products)
    NTT_D void init(uint64_t pp) {
        p = (uint32_t)pp; p2 = 2u * (uint32_t)pp; p4 = 4u * (uint32_t)pp;
        uint32_t x = p;                        // p * p == 1 (mod 8) for odd p; Newton doubles the bits
        for (int i = 0; i < 4; ++i) x *= 2u - p * x;
        pinv = 0u - x;
    }
    // Montgomery product a * b * 2^-32 mod p of two canonical residues, canonical
    // (a*b + m*p < 2^62 + 2^62: no overflow); the 2^32 is folded into n^-1
    NTT_D T pwmul(T a, T b) const {
        const uint64_t t = (uint64_t)a * b;
        const uint32_t m = (uint32_t)t * pinv;
        const T r = (T)((t + (uint64_t)m * p) >> 32);
        return umin32(r, r - p);
    }
    // x + t written as min(x + t, 4p) (an identity: x + t < 4p): one VIADDMNMX on
    // the ALU pipe, so ptxas cannot move the add onto the FMA pipe (IMAD.IADD),
    // which IMAD.HI + 2 IMAD already saturate (tools/ubench_pipes.cu: IMAD 2,
    // IMAD.HI 4 cycles per warp instruction)
    NTT_D T add4(T a, T b) const { return umin32(a + b, p4); }
    // DIT / Pease / Stockham butterfly: (x, y) -> (x + w*y, x - w*y); in/out [0,4p)
    NTT_D void dit(T& x, T& y, Tw w) const {
        const T xr = umin32(x, x - p2);
        const T q = __umulhi(y, w.y);
        const T t = y * w.x - q * p;          // [0,2p)
        x = add4(xr, t);
        y = xr - t + p2;
    }
    // butterfly with twiddle 1: t = y mod 2p
    NTT_D void dit1(T& x, T& y) const {
        const T xr = umin32(x, x - p2);
        const T t = umin32(y, y - p2);
        x = add4(xr, t);
        y = xr - t + p2;
    }
    // stage 1 of a single-pass transform: canonical inputs (the reference's
    // precondition, modmath.py:112), twiddle 1 -> outputs in [0,2p)
    NTT_D void dit1_c(T& x, T& y) const {
        const T a = x;
        x = a + y;
        y = a - y + p;
    }
    // stage 2: inputs in [0,2p) need no reduction before the butterfly
    NTT_D void dit_2p(T& x, T& y, Tw w) const {
        const T q = __umulhi(y, w.y);
        const T t = y * w.x - q * p;
        const T a = x;
        x = add4(a, t);
        y = a - t + p2;
    }
    NTT_D void dit1_2p(T& x, T& y) const {
        const T a = x;
        x = a + y;
        y = a - y + p2;
    }
    // DIF butterfly: (x, y) -> (x + y, w*(x - y)); in/out [0,2p)
    NTT_D void dif(T& x, T& y, Tw w) const {
        const T s = x + y;
        const T d = x - y + p2;
        x = umin32(s, s - p2);
        const T q = __umulhi(d, w.y);
        y = d * w.x - q * p;
    }
    NTT_D void dif1(T& x, T& y) const {
        const T s = x + y;
        const T d = x - y + p2;
        x = umin32(s, s - p2);
        y = umin32(d, d - p2);
    }
    NTT_D T fin(T x) const {
        x = umin32(x, x - p2);
        return umin32(x, x - p);
    }
    NTT_D T mulc(T x, Tw w) const {           // canonical x*w (x canonical)
        const T q = __umulhi(x, w.y);
        const T z = x * w.x - q * p;
        return umin32(z, z - p);
    }
    NTT_D T mulfull(T a, T b) const { return (T)(((uint64_t)a * b) % p); }
    NTT_D T mull(T x, Tw w) const {           // lazy x*w in [0,2p) for any x < 2^32
        const T q = __umulhi(x, w.y);
        return x * w.x - q * p;
    }
};

// LazyGold: Goldilocks DIT-type butterflies with lazy sums.  Values live in
// [0, 2^64) between stages (congruent mod p, not canonical); products are
// canonical, so x + t (t < p) wraps 2^64 at most once and x - t (t < p)
// borrows at most once; fin() canonicalises at the stores.  Per butterfly
// 19 ALU-pipe instructions instead of 29 (the canonical kernels are ALU-bound).
// DIF-type butterflies canonicalise the y input only (one canon per butterfly
// instead of canonical sums).  Bit-exact, but measured slower on config 3
// (four-step DIF 322 vs 314 us/step, ncu: 118 M instructions in pass A at the
// same 62 % issue-active), so DIF plans keep Canon<FGold> unless built with
// NTT_GOLD_LAZY_DIF=1.
template <int AW>
struct LazyGoldT {
    NTT_D static uint64_t addl(uint64_t a, uint64_t b) { return AW ? FGoldC::add_lazy(a, b) : FGoldC::add_lazy_a(a, b); }
    NTT_D static uint64_t canon(uint64_t s) { return AW == 2 ? FGoldC::canon_w(s) : FGoldC::canon_s(s); }
    NTT_D static uint64_t mul(uint64_t a, uint64_t b) { return AW == 2 ? FGoldC::mul_w(a, b) : FGoldC::mul_m(a, b); }
    NTT_D static uint64_t add(uint64_t a, uint64_t b) { return AW == 2 ? FGoldC::add_w(a, b) : FGoldC::add_c(a, b); }
    using T = uint64_t;
    using Tw = uint64_t;
    using Field = FGold;
    static constexpr bool lazy = true;
    NTT_D void init(uint64_t) {}
    NTT_D void dit(T& x, T& y, Tw w) const {
        const T t = mul(y, w);
        const T a = x;
        x = addl(a, t);
        y = FGoldC::sub_c(a, t);
    }
    NTT_D void dit1(T& x, T& y) const {
        const T t = canon(y);
        const T a = x;
        x = addl(a, t);
        y = FGoldC::sub_c(a, t);
    }
    NTT_D void dit1_c(T& x, T& y) const { dit1(x, y); }
    NTT_D void dit_2p(T& x, T& y, Tw w) const { dit(x, y, w); }
    NTT_D void dit1_2p(T& x, T& y) const { dit1(x, y); }
    // DIF: only y is canonicalised -- x + b (x < 2^64, b < p) wraps at most once
    // and x - b borrows at most once, exactly the DIT forms; the sum stays lazy,
    // the product is canonical
    NTT_D void dif(T& x, T& y, Tw w) const {
        const T a = x, b = canon(y);
        x = addl(a, b);
        y = mul(FGoldC::sub_c(a, b), w);
    }
    NTT_D void dif1(T& x, T& y) const {
        const T a = x, b = canon(y);
        x = addl(a, b);
        y = FGoldC::sub_c(a, b);
    }
    NTT_D T fin(T x) const { return canon(x); }
    NTT_D T mulc(T x, Tw w) const { return mul(x, w); }
    NTT_D T mull(T x, Tw w) const { return mul(x, w); }
    NTT_D T mulfull(T a, T b) const { return mul(a, b); }
};
#ifndef NTT_GOLD_LAZY_AW
#define NTT_GOLD_LAZY_AW 0
#endif
using LazyGold = LazyGoldT<NTT_GOLD_LAZY_AW>;

template <class F>
struct Canon {
    using T = typename F::T;
    using Tw = typename F::Tw;
    using Field = F;
    static constexpr bool lazy = false;
    F f;
    NTT_D void init(uint64_t pp) { f.p = (T)pp; }
    NTT_D void dit(T& x, T& y, Tw w) const {
        const T t = f.mul(y, w);
        const T a = x;
        x = f.add(a, t);
        y = f.sub(a, t);
    }
    NTT_D void dit1(T& x, T& y) const {
        const T a = x;
        x = f.add(a, y);
        y = f.sub(a, y);
    }
    // canonical policies: the bounded first-stage forms are the plain ones
    NTT_D void dit1_c(T& x, T& y) const { dit1(x, y); }
    NTT_D void dit_2p(T& x, T& y, Tw w) const { dit(x, y, w); }
    NTT_D void dit1_2p(T& x, T& y) const { dit1(x, y); }
    NTT_D void dif(T& x, T& y, Tw w) const {
        const T a = x, b = y;
        x = f.add(a, b);
        y = f.mul(f.sub(a, b), w);
    }
    NTT_D void dif1(T& x, T& y) const {
        const T a = x, b = y;
        x = f.add(a, b);
        y = f.sub(a, b);
    }
    NTT_D T fin(T x) const { return x; }
    NTT_D T mulc(T x, Tw w) const { return f.mul(x, w); }
    NTT_D T mull(T x, Tw w) const { return f.mul(x, w); }
    NTT_D T mulfull(T a, T b) const { return f.mul_full(a, b); }
};

#ifndef NTT_GOLD_LAZY
#define NTT_GOLD_LAZY 1      // 0: every Goldilocks plan on Canon<FGold>
#endif
// Goldilocks policy of a plan: lazy sums for the DIT-type dataflows (DIT,
// Flat, Pease, Pease_nc, Stockham, six-step), canonical for DIF
#ifndef NTT_GOLD_LAZY_DIF
#define NTT_GOLD_LAZY_DIF 0
#endif
template <bool DIF_TYPE>
using GoldPolicy =
    typename std::conditional<(DIF_TYPE && !NTT_GOLD_LAZY_DIF) || !NTT_GOLD_LAZY, Canon<FGold>, LazyGold>::type;

}  // namespace nttb200
