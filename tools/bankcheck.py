"""Design-time shared-memory bank-conflict predictor for the tile kernel
(csrc/fasttile.cuh), in the spirit of the reference's bankmodel.py (SURVEY
sec.8(f) row 4: per-stage address traces -> bank schedule), but for B200's
32 four-byte banks and OUR layouts: it replays every warp-wide shared-memory
access of one tile (gather stores, register-group loads/stores, scatter
loads) for a candidate network stride NP and counts wavefronts.

usage: python tools/bankcheck.py [--u64] [K TQ]       (default: the u32 shapes)
prints, per variant class, wavefronts / ideal for each NP in the window and
the best NP (what tile_stride<T,K,TQ>() should return)."""
import sys

CW32 = 5


def padpos(pos, word=4):
    return pos + (pos >> 5) + (pos >> 10) if word == 4 else pos + (pos >> 4) + (pos >> 8) + (pos >> 12)


def padded_len(K, word=4):
    return (padpos((1 << K) - 1, word) + 1 + 3) & ~3


def plan_lanes(L, B, CW):
    fr = [b for b in range(L) if b < B or b >= B + 4]
    used, res, bits = set(), set(), []
    for i, b in enumerate(fr):
        if len(bits) >= CW:
            break
        if b % CW not in res:
            res.add(b % CW); used.add(i); bits.append(b)
    bits += [b for i, b in enumerate(fr) if i not in used]
    return bits


def scatter_bits(u, bits):
    r = 0
    for j, b in enumerate(bits):
        r |= ((u >> j) & 1) << b
    return r


def brev(x, n):
    return int(format(x, f"0{n}b")[::-1], 2) if n else 0


def wavefronts(addrs, word):
    """addrs: word addresses (in units of `word` bytes) of the 32 lanes.
    4-byte accesses: one pass over the warp, a wavefront per distinct word of the worst bank.
    8-byte accesses: the hardware serves the two HALF-warps one after the other (measured on
    B200, ncu source counters of k_tile's u64 column passes: 4 wavefronts per access where a
    whole-warp model promised 2), so the count is the sum of the two halves' worst banks."""
    def worst(lanes):
        banks = {}
        for a in lanes:
            if a is None:
                continue
            for k in range(word // 4):
                byte_word = a * (word // 4) + k
                banks.setdefault(byte_word % 32, set()).add(byte_word)
        return max((len(v) for v in banks.values()), default=0)
    if word == 8 and len(addrs) == 32:
        return worst(addrs[:16]) + worst(addrs[16:])
    return worst(addrs)


def geo(K):
    G = (K + 3) // 4
    return 1 << (K - 4), G, K - 4 * (G - 1)


def tile_trace(V, K, TQ, NT, NP, word, in_order, out_order, vec_in, vec_out, rev_local=False):
    """yield (kind, [addr per lane]) for every warp instruction of one tile."""
    VE = 16 // word
    TT, G, K0 = geo(K)
    nthreads = NT
    # gather stores
    if vec_in and in_order == "T":
        n = (TQ << K) // VE
        for w0 in range(0, nthreads, 32):
            for it in range(w0, n, nthreads):
                for e in range(VE):
                    lanes = []
                    for i in range(it, it + 32):
                        if i >= n:
                            lanes.append(None); continue
                        t0, x = (i % (TQ // VE)) * VE, i // (TQ // VE)
                        xl = brev(x, K) if rev_local else x
                        lanes.append((t0 + e) * NP + padpos(xl, word))
                    yield "gather", lanes
    elif vec_in and in_order == "C":
        n = (TQ << K) // VE
        for w0 in range(0, nthreads, 32):
            for it in range(w0, n, nthreads):
                for e in range(VE):
                    lanes = []
                    for i in range(it, it + 32):
                        t, x0 = i // ((1 << K) // VE), (i % ((1 << K) // VE)) * VE
                        xl = brev(x0 + e, K) if rev_local else x0 + e
                        lanes.append(t * NP + padpos(xl, word))
                    yield "gather", lanes
    # register groups
    for g in range(G):
        kg = K0 if g == 0 else 4
        for w0 in range(0, TQ * TT, 32):
            tids = list(range(w0, w0 + 32))
            if V in ("dit", "dif"):
                if V == "dit":
                    B = 0 if g == 0 else K0 + 4 * (g - 1)
                else:
                    B = 0 if g == G - 1 else K - 4 * (g + 1)
                bits = plan_lanes(K, B, CW32 if word == 4 else 4)
                rd = []
                for c in range(16):
                    rd.append([(tid // TT) * NP + padpos(scatter_bits(tid % TT, bits) | (c << B), word) for tid in tids])
                for lanes in rd:
                    yield "group_ld", lanes
                for lanes in rd:
                    yield "group_st", lanes
            elif V == "pease":
                for c in range(16):
                    yield "group_ld", [(tid // TT) * NP + padpos(((tid % TT) << 4) | c, word) for tid in tids]
                for c in range(16):
                    n_, R = c >> kg, c & ((1 << kg) - 1)
                    yield "group_st", [(tid // TT) * NP + padpos(((tid % TT) << (4 - kg)) | n_ | (R << (K - kg)), word) for tid in tids]
            else:  # stockham
                sg = 0 if g == 0 else K0 + 4 * (g - 1)
                lob = K - sg - kg
                def hilo(u):
                    if g == 0:
                        return 0, u
                    if g == G - 1:
                        return u, 0
                    return u >> lob, u & ((1 << lob) - 1)
                for c in range(16):
                    lanes = []
                    for tid in tids:
                        hi, lo = hilo(tid % TT)
                        lanes.append((tid // TT) * NP + padpos((hi << (K - sg)) | lo | (c << (lob - (4 - kg))), word))
                    yield "group_ld", lanes
                for c in range(16):
                    R, x = c >> (4 - kg), c & ((1 << (4 - kg)) - 1)
                    lanes = []
                    for tid in tids:
                        hi, lo = hilo(tid % TT)
                        lanes.append((tid // TT) * NP + padpos((hi << lob) | lo | (R << (K - kg)) | (x << (lob - (4 - kg))), word))
                    yield "group_st", lanes
    # scatter loads
    if vec_out and out_order == "T":
        n = (TQ << K) // VE
        for w0 in range(0, nthreads, 32):
            for it in range(w0, n, nthreads):
                for e in range(VE):
                    lanes = []
                    for i in range(it, it + 32):
                        t0, x = (i % (TQ // VE)) * VE, i // (TQ // VE)
                        lanes.append((t0 + e) * NP + padpos(x, word))
                    yield "scatter", lanes
    elif vec_out and out_order == "C":
        n = (TQ << K) // VE
        for w0 in range(0, nthreads, 32):
            for it in range(w0, n, nthreads):
                for e in range(VE):
                    lanes = []
                    for i in range(it, it + 32):
                        t, x0 = i // ((1 << K) // VE), (i % ((1 << K) // VE)) * VE
                        lanes.append(t * NP + padpos(x0 + e, word))
                    yield "scatter", lanes


def score(V, K, TQ, NT, NP, word, passes):
    tot, ideal = 0, 0
    for (io, oo, vi, vo, rl) in passes:
        for kind, lanes in tile_trace(V, K, TQ, NT, NP, word, io, oo, vi, vo, rl):
            wf = wavefronts(lanes, word)
            tot += wf
            ideal += max(1, word // 4 * 32 * 4 // 128) if word == 8 else 1
    return tot, ideal


def tile_nt(K, TQ):
    return min(TQ << (K - 4), 512)


# pass shapes used by run_tile_passes (in_order, out_order, vec_in, vec_out, rev_local)
SHAPES = {
    "dit": [("T", "C", True, True, False), ("T", "T", True, True, False)],
    "dif": [("T", "T", True, True, False), ("C", "T", True, True, False)],
    "pease": [("C", "T", True, True, False), ("T", "T", True, True, False)],
    "stockham": [("T", "T", True, True, False), ("C", "T", True, True, False)],
}


def main():
    word = 8 if "--u64" in sys.argv else 4
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    E = 13 if word == 4 else 12
    shapes = [(int(args[0]), int(args[1]))] if args else [(K, 1 << (E - K)) for K in range(6, 11 if word == 4 else 10)]
    for K, TQ in shapes:
        NT = tile_nt(K, TQ)
        base = padded_len(K, word)
        print(f"K={K} TQ={TQ} NT={NT} padded_len={base}")
        for V, passes in SHAPES.items():
            vec = [(a, b, c and TQ >= 16 // word if a == "T" else c, d and TQ >= 16 // word if b == "T" else d, e)
                   for (a, b, c, d, e) in passes]
            res = []
            for NP in range(base, base + 33):
                t, i = score(V, K, TQ, NT, NP, word, vec)
                res.append((t / i, NP))
            best = min(res)
            cur = [r for r in res if (r[1] % 32) == (1 if TQ >= 32 else 32 // TQ)]
            print(f"   {V:9s} best NP={best[1]} ({best[1] % 32} mod 32) ratio {best[0]:.2f}; "
                  f"current rule NP={cur[0][1] if cur else '-'} ratio {cur[0][0] if cur else float('nan'):.2f}")


if __name__ == "__main__":
    main()


def breakdown(V, K, TQ, NP, word=4, passes=None):
    NT = tile_nt(K, TQ)
    passes = passes or SHAPES[V]
    out = {}
    for p in passes:
        for kind, lanes in tile_trace(V, K, TQ, NT, NP, word, *p):
            key = (p[0] + p[1], kind)
            a = out.setdefault(key, [0, 0])
            a[0] += wavefronts(lanes, word)
            a[1] += 1
    return {k: round(v[0] / v[1], 2) for k, v in out.items()}


# ---- u64 column-layout tiles (config 5's 2^6 / 2^7 passes): non-linear network base
def cols_u64_nbase(K, TQ):
    """csrc/fasttile.cuh tile_nbase<uint64_t, K, TQ, TL_COLS>: (NP, XS)"""
    npb = (padded_len(K, 8) + 16 + 15) // 16 * 16
    return {(7, 32): (npb + 4, 2), (6, 64): (npb + 2, 3)}[(K, TQ)]


def cols_u64_worst(K, TQ, NP, XS):
    """worst wavefronts per warp access (2 = ideal for 8-byte lanes) of the T-fast
    vector copies and the DIT register groups (plan_lanes maps) of one tile"""
    base = lambda t: t * NP + (t >> XS if XS else 0)
    TT, G, K0 = geo(K)
    worst = 0
    for e in range(2):                                   # 16-byte vector copies, lane i -> (t0 + e, x)
        for x in range(4):
            lanes = [base((i % (TQ // 2)) * 2 + e) + padpos(i // (TQ // 2) + x * (32 // (TQ // 2)), 8) for i in range(32)]
            worst = max(worst, wavefronts(lanes, 8))
    for g in range(G):
        B = 0 if g == 0 else K0 + 4 * (g - 1)
        bits = plan_lanes(K, B, 4)
        for w0 in range(0, TQ * TT, 32):
            for c in range(16):
                lanes = [base(tid // TT) + padpos(scatter_bits(tid % TT, bits) | (c << B), 8) for tid in range(w0, w0 + 32)]
                worst = max(worst, wavefronts(lanes, 8))
    return worst
