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
    NTT_D T add(T a, T b) const {
        T s = a + b;
        T c = (s < a) ? EPS : 0;       // wrapped: s + 2^64 - p == s + EPS
        s += c;
        return canon(s);               // a,b < p => no second wrap
    }
    NTT_D T sub(T a, T b) const {
        T d = a - b;
        return (a < b) ? d - EPS : d;  // d + p (mod 2^64) == d - EPS
    }
    NTT_D static T reduce128(uint64_t lo, uint64_t hi) {
        uint64_t hh = hi >> 32, hl = hi & EPS;
        uint64_t t0 = lo - hh;
        if (lo < hh) t0 -= EPS;        // borrow: add p == subtract EPS
        uint64_t t1 = hl * EPS;        // < 2^64
        uint64_t t2 = t0 + t1;
        if (t2 < t1) t2 += EPS;        // carry: 2^64 == EPS
        return canon(t2);
    }
    NTT_D T mul_full(T a, T b) const { return reduce128(a * b, __umul64hi(a, b)); }
    NTT_D T mul(T x, Tw w) const { return mul_full(x, w); }
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
