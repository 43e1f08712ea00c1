// arith.cuh -- Z_p arithmetic for the B200 butterfly kernels.
//
// Replaces the reference's inlined butterfly arithmetic
// (modmath.py:110-145 mod_add / mod_sub / shoup_mul, inlined in
// algorithms.py:104-113, 148-157, 185-194, 218-227, 290-299).  Every field
// returns CANONICAL residues in [0,p) from every operation, so each stage of
// each kernel leaves exactly the values the reference's stage leaves (the
// per-stage buffers are bit-identical, not merely congruent).
//
// Field policies (the device word is 32-bit for p < 2^32, 64-bit otherwise):
//   F32S  p < 2^31        u32 Shoup with w=32 (umulhi); branch-free min() fixups
//   F32W  2^31 <= p < 2^32  u32 storage, carry-safe: Shoup z in [0,2p) needs 33 bits
//   FGold p = 2^64-2^32+1 u64, special reduction 2^64 = 2^32-1 (mod p); twiddle = w only
//   F64   any p < 2^64    u64 Shoup with w=64 (__umul64hi), 65-bit z kept exactly
//
// Twiddles are stored per field as F::Tw: (w, floor(w*2^W/p)) pairs for the
// Shoup fields (W = 32 / 64: the reference's own w_shoup when the plan's w
// equals the word width), the bare power for Goldilocks.
#pragma once
#include <cstdint>

#define NTT_HD __host__ __device__ __forceinline__
#define NTT_D __device__ __forceinline__
// Goldilocks multiply: mad.wide product chain (1) or four mul.wide + carry adds (0)
#ifndef NTT_GOLD_W
#define NTT_GOLD_W 0      // 1: Goldilocks wrap corrections as IMAD.WIDE (FGoldC::madw) -- slower, FMA-pipe bound
#endif
#ifndef NTT_GOLD_MULM
#define NTT_GOLD_MULM 1
#endif

namespace nttb200 {

NTT_D uint32_t umin32(uint32_t a, uint32_t b) { return a < b ? a : b; }

struct F32S {
    using T = uint32_t;
    using Tw = uint2;          // {w, w_shoup}
    static constexpr int kind = 0;
    uint32_t p;
    NTT_D T add(T a, T b) const { T s = a + b; return umin32(s, s - p); }
    NTT_D T sub(T a, T b) const { T d = a - b; return umin32(d, d + p); }
    // shoup_mul (modmath.py:135-145): q = (x*wq)>>32; z = x*w - q*p in [0,2p) < 2^32.
    NTT_D T mul(T x, Tw w) const {
        T q = __umulhi(x, w.y);
        T z = x * w.x - q * p;
        return umin32(z, z - p);
    }
    NTT_D T mulw(T x, Tw w) const { return mul(x, w); }
    NTT_D T mul_full(T a, T b) const { return (T)(((uint64_t)a * b) % p); }
    NTT_D static T tw_value(Tw w) { return w.x; }
};

struct F32W {
    using T = uint32_t;
    using Tw = uint2;
    static constexpr int kind = 1;
    uint32_t p;
    NTT_D T add(T a, T b) const {
        T s = a + b;
        return (s < a || s >= p) ? s - p : s;
    }
    NTT_D T sub(T a, T b) const { T d = a - b; return a < b ? d + p : d; }
    NTT_D T mul(T x, Tw w) const {
        T q = __umulhi(x, w.y);
        uint64_t z = (uint64_t)x * w.x - (uint64_t)q * p;   // [0, 2p) needs 33 bits
        return (T)(z >= p ? z - p : z);
    }
    NTT_D T mul_full(T a, T b) const { return (T)(((uint64_t)a * b) % p); }
    NTT_D static T tw_value(Tw w) { return w.x; }
};

// Goldilocks with explicit 32-bit carry chains (PTX add.cc / addc / mad.wide).
// Same canonical results as FGold (every op returns a value in [0,p)), but
// the compiler's 64-bit compare+select sequences are replaced by carry flags:
//   add: s = a+b; t = s + EPS; result = (carry(s) | carry(t)) ? t : s
//        (a,b < p: s >= p  <=>  s + EPS overflows)
//   sub: d = a-b; result = borrow ? d - EPS : d
//   mul: 128-bit product from 4 mul.wide.u32, reduction 2^64 = EPS, 2^96 = -1.
// the carry-chain asm blocks below produce temporaries the compiler sees as "set but never used"
#pragma nv_diag_suppress 550
struct FGoldC {
    using T = uint64_t;
    using Tw = uint64_t;
    static constexpr int kind = 2;
    static constexpr uint64_t P = 0xFFFFFFFF00000001ull;
    uint64_t p;
    NTT_D static uint32_t lo(uint64_t x) { return (uint32_t)x; }
    NTT_D static uint32_t hi(uint64_t x) { return (uint32_t)(x >> 32); }
    NTT_D static uint64_t mk(uint32_t l, uint32_t h) { return ((uint64_t)h << 32) | l; }
    NTT_D static T add_c(T a, T b) {
        uint32_t s0, s1, t0, t1, c;
        asm("add.cc.u32 %0, %5, %7;\n\t"
            "addc.cc.u32 %1, %6, %8;\n\t"
            "addc.u32 %4, 0, 0;\n\t"
            "add.cc.u32 %2, %0, 0xffffffff;\n\t"
            "addc.cc.u32 %3, %1, 0;\n\t"
            "addc.u32 %4, %4, 0;"
            : "=r"(s0), "=r"(s1), "=r"(t0), "=r"(t1), "=r"(c)
            : "r"(lo(a)), "r"(hi(a)), "r"(lo(b)), "r"(hi(b)));
        return c ? mk(t0, t1) : mk(s0, s1);
    }
    NTT_D static T sub_c(T a, T b) {
        uint32_t d0, d1, m;
        asm("sub.cc.u32 %0, %3, %5;\n\t"
            "subc.cc.u32 %1, %4, %6;\n\t"
            "subc.u32 %2, 0, 0;\n\t"          // m = 0 or 0xffffffff (= EPS on borrow)
            "sub.cc.u32 %0, %0, %2;\n\t"
            "subc.u32 %1, %1, 0;"
            : "=r"(d0), "=r"(d1), "=r"(m)
            : "r"(lo(a)), "r"(hi(a)), "r"(lo(b)), "r"(hi(b)));
        (void)m;
        return mk(d0, d1);
    }
    NTT_D static T mul_c(T a, T b) {
        uint32_t r0 = lo((uint64_t)lo(a) * lo(b)), r1 = hi((uint64_t)lo(a) * lo(b));
        uint32_t r2 = lo((uint64_t)hi(a) * hi(b)), r3 = hi((uint64_t)hi(a) * hi(b));
        // 128-bit product r3:r2:r1:r0 from four 32x32->64 partial products
        const uint64_t p01 = (uint64_t)lo(a) * hi(b), p10 = (uint64_t)hi(a) * lo(b);
        asm("add.cc.u32 %1, %1, %4;\n\t"
            "addc.cc.u32 %2, %2, %5;\n\t"
            "addc.u32 %3, %3, 0;\n\t"
            "add.cc.u32 %1, %1, %6;\n\t"
            "addc.cc.u32 %2, %2, %7;\n\t"
            "addc.u32 %3, %3, 0;"
            : "+r"(r0), "+r"(r1), "+r"(r2), "+r"(r3)
            : "r"(lo(p01)), "r"(hi(p01)), "r"(lo(p10)), "r"(hi(p10)));
        // x = r1:r0 + r2 * 2^64 + r3 * 2^96 == (r1:r0) - r3 + r2 * (2^32 - 1)
        uint32_t t0, t1, m, u0, u1, c;
        asm("sub.cc.u32 %0, %6, %9;\n\t"          // t = lo64 - r3
            "subc.cc.u32 %1, %7, 0;\n\t"
            "subc.u32 %2, 0, 0;\n\t"              // m = borrow ? EPS : 0
            "sub.cc.u32 %0, %0, %2;\n\t"          // t -= EPS on borrow (cannot underflow)
            "subc.u32 %1, %1, 0;\n\t"
            "sub.cc.u32 %3, 0, %8;\n\t"           // u = r2 * EPS = (r2 << 32) - r2
            "subc.u32 %4, %8, 0;\n\t"
            "add.cc.u32 %0, %0, %3;\n\t"          // t += u, carry c
            "addc.cc.u32 %1, %1, %4;\n\t"
            "addc.u32 %5, 0, 0;"
            : "=r"(t0), "=r"(t1), "=r"(m), "=r"(u0), "=r"(u1), "=r"(c)
            : "r"(r0), "r"(r1), "r"(r2), "r"(r3));
        // on carry add EPS (2^64 = EPS, cannot overflow again); then canonicalise
        // with the +EPS overflow test (s >= p  <=>  s + EPS >= 2^64)
        uint32_t s0, s1, q0, q1, c2, mneg;
        asm("neg.s32 %5, %6;\n\t"                  // 0 / 0xffffffff
            "add.cc.u32 %0, %7, %5;\n\t"
            "addc.u32 %1, %8, 0;\n\t"
            "add.cc.u32 %2, %0, 0xffffffff;\n\t"
            "addc.cc.u32 %3, %1, 0;\n\t"
            "addc.u32 %4, 0, 0;"
            : "=r"(s0), "=r"(s1), "=r"(q0), "=r"(q1), "=r"(c2), "=r"(mneg)
            : "r"(c), "r"(t0), "r"(t1));
        (void)m; (void)u0; (void)u1;
        return c2 ? mk(q0, q1) : mk(s0, s1);
    }
    // 128-bit product by a mad.wide chain (each partial sum fits 64 bits:
    // (2^32-1)^2 + 2(2^32-1) = 2^64-1), r2 * EPS as one IMAD.WIDE (FMA pipe: the
    // Goldilocks kernels are ALU-bound), then the reduction 2^64 = EPS, 2^96 = -1
    NTT_D static T mul_m(T a, T b) {
        const uint32_t a0 = lo(a), a1 = hi(a), b0 = lo(b), b1 = hi(b);
        const uint64_t p00 = (uint64_t)a0 * b0;
        const uint64_t t = (uint64_t)a0 * b1 + (p00 >> 32);
        const uint64_t u = (uint64_t)a1 * b0 + (uint32_t)t;
        const uint64_t v = (uint64_t)a1 * b1 + (t >> 32) + (u >> 32);
        const uint32_t r0 = lo(p00), r1 = lo(u), r2 = lo(v), r3 = hi(v);
        const uint64_t ue = (uint64_t)r2 * 0xFFFFFFFFu;          // r2 * EPS
        // x = r1:r0 - r3 + r2 * EPS
        uint32_t t0, t1, m, c, s0, s1, q0, q1, c2;
        asm("sub.cc.u32 %0, %9, %11;\n\t"          // t = lo64 - r3
            "subc.cc.u32 %1, %10, 0;\n\t"
            "subc.u32 %2, 0, 0;\n\t"                // m = borrow ? EPS : 0
            "sub.cc.u32 %0, %0, %2;\n\t"            // t -= EPS on borrow (no underflow)
            "subc.u32 %1, %1, 0;\n\t"
            "add.cc.u32 %0, %0, %12;\n\t"           // t += r2 * EPS, carry c
            "addc.cc.u32 %1, %1, %13;\n\t"
            "addc.u32 %3, 0, 0;\n\t"
            "neg.s32 %3, %3;\n\t"                   // carry: + EPS (cannot overflow again)
            "add.cc.u32 %4, %0, %3;\n\t"
            "addc.u32 %5, %1, 0;\n\t"
            "add.cc.u32 %6, %4, 0xffffffff;\n\t"     // canonical: s >= p <=> s + EPS overflows
            "addc.cc.u32 %7, %5, 0;\n\t"
            "addc.u32 %8, 0, 0;"
            : "=&r"(t0), "=&r"(t1), "=&r"(m), "=&r"(c), "=&r"(s0), "=&r"(s1), "=&r"(q0), "=&r"(q1), "=&r"(c2)
            : "r"(r0), "r"(r1), "r"(r3), "r"(lo(ue)), "r"(hi(ue)));
        (void)m;
        return c2 ? mk(q0, q1) : mk(s0, s1);
    }
    // ---- wrap corrections as c * EPS + s (one IMAD.WIDE.U32 on the FMA pipe)
    // instead of compare / SEL pairs on the ALU pipe, which the Goldilocks
    // kernels saturate.  c is a carry bit; the 64-bit sum wraps mod 2^64, so
    // s + EPS - 2^64 = s - p comes out of the same instruction.
    NTT_D static T madw(uint32_t c, T s) {
        T r;
        asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(c), "r"(0xffffffffu), "l"(s));
        return r;
    }
    // carry of s + EPS (s >= p  <=>  s + EPS >= 2^64)
    NTT_D static uint32_t ge_p(T s) {
        uint32_t c;
        asm("add.cc.u32 %0, %1, 0xffffffff;\n\t"
            "addc.cc.u32 %0, %2, 0;\n\t"
            "addc.u32 %0, 0, 0;"
            : "=&r"(c) : "r"(lo(s)), "r"(hi(s)));
        return c;
    }
    NTT_D static T canon_w(T s) { return madw(ge_p(s), s); }
    // a + b reduced once: for any a < 2^64 and b < p the result is < 2^64 and
    // congruent to a + b (a + b - 2^64 <= p - 2, so + EPS cannot wrap again)
    NTT_D static T add_lazy(T a, T b) {
        uint32_t s0, s1, c;
        asm("add.cc.u32 %0, %3, %5;\n\t"
            "addc.cc.u32 %1, %4, %6;\n\t"
            "addc.u32 %2, 0, 0;"
            : "=r"(s0), "=r"(s1), "=r"(c)
            : "r"(lo(a)), "r"(hi(a)), "r"(lo(b)), "r"(hi(b)));
        return madw(c, mk(s0, s1));
    }
    NTT_D static T add_w(T a, T b) { return canon_w(add_lazy(a, b)); }   // a, b < p
    // the same lazy sum with the correction on the ALU pipe
    NTT_D static T add_lazy_a(T a, T b) {
        uint32_t s0, s1, c;
        asm("add.cc.u32 %0, %3, %5;\n\t"
            "addc.cc.u32 %1, %4, %6;\n\t"
            "addc.u32 %2, 0, 0;\n\t"
            "neg.s32 %2, %2;\n\t"                 // carry: + EPS
            "add.cc.u32 %0, %0, %2;\n\t"
            "addc.u32 %1, %1, 0;"
            : "=&r"(s0), "=&r"(s1), "=&r"(c)
            : "r"(lo(a)), "r"(hi(a)), "r"(lo(b)), "r"(hi(b)));
        return mk(s0, s1);
    }
    // canonical by compare / select (s + EPS overflows  <=>  s >= p)
    NTT_D static T canon_s(T s) {
        uint32_t q0, q1, c;
        asm("add.cc.u32 %0, %3, 0xffffffff;\n\t"
            "addc.cc.u32 %1, %4, 0;\n\t"
            "addc.u32 %2, 0, 0;"
            : "=&r"(q0), "=&r"(q1), "=&r"(c) : "r"(lo(s)), "r"(hi(s)));
        return c ? mk(q0, q1) : s;
    }
    // mul_m with both corrections as IMAD.WIDE; canonical for any a < 2^64, b < 2^64
    NTT_D static T mul_w(T a, T b) {
        const uint32_t a0 = lo(a), a1 = hi(a), b0 = lo(b), b1 = hi(b);
        const uint64_t p00 = (uint64_t)a0 * b0;
        const uint64_t t = (uint64_t)a0 * b1 + (p00 >> 32);
        const uint64_t u = (uint64_t)a1 * b0 + (uint32_t)t;
        const uint64_t v = (uint64_t)a1 * b1 + (t >> 32) + (u >> 32);
        const uint32_t r0 = lo(p00), r1 = lo(u), r2 = lo(v), r3 = hi(v);
        const uint64_t ue = (uint64_t)r2 * 0xFFFFFFFFu;          // r2 * EPS
        uint32_t t0, t1, m, c;
        asm("sub.cc.u32 %0, %4, %6;\n\t"          // t = lo64 - r3
            "subc.cc.u32 %1, %5, 0;\n\t"
            "subc.u32 %2, 0, 0;\n\t"                // m = borrow ? EPS : 0
            "sub.cc.u32 %0, %0, %2;\n\t"            // t -= EPS on borrow (no underflow)
            "subc.u32 %1, %1, 0;\n\t"
            "add.cc.u32 %0, %0, %7;\n\t"           // t += r2 * EPS, carry c
            "addc.cc.u32 %1, %1, %8;\n\t"
            "addc.u32 %3, 0, 0;"
            : "=&r"(t0), "=&r"(t1), "=&r"(m), "=&r"(c)
            : "r"(r0), "r"(r1), "r"(r3), "r"(lo(ue)), "r"(hi(ue)));
        (void)m;
        return canon_w(madw(c, mk(t0, t1)));       // carry: + EPS (cannot wrap again)
    }
    NTT_D T add(T a, T b) const { return NTT_GOLD_W ? add_w(a, b) : add_c(a, b); }
    NTT_D T sub(T a, T b) const { return sub_c(a, b); }
    NTT_D T mul(T x, Tw w) const { return NTT_GOLD_W ? mul_w(x, w) : NTT_GOLD_MULM ? mul_m(x, w) : mul_c(x, w); }
    NTT_D T mul_full(T a, T b) const { return NTT_GOLD_W ? mul_w(a, b) : NTT_GOLD_MULM ? mul_m(a, b) : mul_c(a, b); }
    NTT_D static T tw_value(Tw w) { return w; }
};
#pragma nv_diag_default 550


// Goldilocks p = 2^64 - 2^32 + 1.  Reduction of a 128-bit product uses
// 2^64 = 2^32 - 1 and 2^96 = -1 (mod p) -- the published Goldilocks
// reduction; every result is canonicalised.
struct FGold {
    using T = uint64_t;
    using Tw = uint64_t;
    static constexpr int kind = 2;
    static constexpr uint64_t P = 0xFFFFFFFF00000001ull;
    static constexpr uint64_t EPS = 0xFFFFFFFFull;   // 2^64 mod p
    uint64_t p;
    NTT_D static T canon(T x) { return x >= P ? x - P : x; }
    // the kernels use the carry-chain forms (FGoldC, bit-identical results,
    // ~15% more butterflies/s); reduce128/canon stay for reference
    NTT_D T add(T a, T b) const { return NTT_GOLD_W ? FGoldC::add_w(a, b) : FGoldC::add_c(a, b); }
    NTT_D T sub(T a, T b) const { return FGoldC::sub_c(a, b); }
    NTT_D static T reduce128(uint64_t lo, uint64_t hi) {
        uint64_t hh = hi >> 32, hl = hi & EPS;
        uint64_t t0 = lo - hh;
        if (lo < hh) t0 -= EPS;        // borrow: add p == subtract EPS
        uint64_t t1 = hl * EPS;        // < 2^64
        uint64_t t2 = t0 + t1;
        if (t2 < t1) t2 += EPS;        // carry: 2^64 == EPS
        return canon(t2);
    }
    NTT_D T mul_full(T a, T b) const { return FGoldC().mul_full(a, b); }
    NTT_D T mul(T x, Tw w) const { return FGoldC().mul(x, w); }
    NTT_D static T tw_value(Tw w) { return w; }
};

struct F64 {
    using T = uint64_t;
    using Tw = ulonglong2;     // {w, floor(w*2^64/p)}
    static constexpr int kind = 3;
    uint64_t p;
    NTT_D T add(T a, T b) const {
        T s = a + b;
        return (s < a || s >= p) ? s - p : s;
    }
    NTT_D T sub(T a, T b) const { T d = a - b; return a < b ? d + p : d; }
    // Shoup with w=64; z = x*w - q*p in [0,2p) can need 65 bits.
    NTT_D T mul(T x, Tw w) const {
        uint64_t q = __umul64hi(x, w.y);
        uint64_t lo1 = x * w.x, hi1 = __umul64hi(x, w.x);
        uint64_t lo2 = q * p, hi2 = __umul64hi(q, p);
        uint64_t zlo = lo1 - lo2;
        uint64_t zhi = hi1 - hi2 - (lo1 < lo2 ? 1 : 0);
        return (zhi || zlo >= p) ? zlo - p : zlo;
    }
    // exact (a*b) mod p via 128-bit long division by shifting (table-free path)
    NTT_D T mul_full(T a, T b) const {
        uint64_t lo = a * b, hi = __umul64hi(a, b);
        // reduce hi:lo mod p bit by bit (only used off the hot path)
        uint64_t r = hi % p;
        for (int i = 63; i >= 0; --i) {
            uint64_t top = r >> 63;
            r = (r << 1) | ((lo >> i) & 1);
            if (top || r >= p) r -= p;
        }
        return r;
    }
    NTT_D static T tw_value(Tw w) { return w.x; }
};

}  // namespace nttb200

