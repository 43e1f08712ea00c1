"""Prototype (pure Python, small N) of the four-step factorisation of a late
pass: K consecutive stages of DIT / Pease / Stockham (second pass) or DIF
(first pass) == per-element twist + a LOCAL size-2^K transform of the same
variant using only local twiddles.  Verifies the twist exponents used by
csrc/fasttile.cuh against the oracle's per-stage replay.
"""
import random

P = 998244353
G = 3


def rev(x, b):
    return int(format(x, f"0{b}b")[::-1], 2) if b else 0


def tables(L):
    n = 1 << L
    w = pow(G, (P - 1) // n, P)
    return n, w, [pow(w, i, P) for i in range(n)]


def dit_stage(a, s, L, wp):
    n = 1 << L
    m, half, stride = 1 << s, 1 << (s - 1), n >> s
    for j in range(0, n, m):
        for k in range(half):
            lo, hi = j + k, j + k + half
            t = a[hi] * wp[k * stride] % P
            a[lo], a[hi] = (a[lo] + t) % P, (a[lo] - t) % P


def dif_stage(a, s, L, wp):
    n = 1 << L
    m, half, stride = 1 << s, 1 << (s - 1), n >> s
    for j in range(0, n, m):
        for k in range(half):
            lo, hi = j + k, j + k + half
            f1, f2 = a[lo], a[hi]
            a[lo] = (f1 + f2) % P
            a[hi] = (f1 - f2) * wp[k * stride] % P


def pease_stage(src, s, L, wp):
    n = 1 << L
    dst = [0] * n
    low = L - s
    for r in range(n // 2):
        e = (r >> low) << low
        t = src[2 * r + 1] * wp[e] % P
        dst[r] = (src[2 * r] + t) % P
        dst[r + n // 2] = (src[2 * r] - t) % P
    return dst


def stockham_stage(cur, s, L, wp):
    n = 1 << L
    nxt = [0] * n
    span, stride = 1 << s, n >> (s + 1)
    for j in range(span):
        e = j * stride
        for i in range(stride):
            a, b = cur[2 * j * stride + i], cur[2 * j * stride + stride + i] * wp[e] % P
            nxt[j * stride + i] = (a + b) % P
            nxt[j * stride + i + n // 2] = (a - b) % P
    return nxt


def check(L, K0):
    """2-pass split L = K0 + K1 for each variant."""
    n, w, wp = tables(L)
    K1 = L - K0
    x = [random.randrange(P) for _ in range(n)]
    ok = {}
    # ---------------- DIT: pass 2 (window [K0, L)) = twist + local DIT (size 2^K1)
    a = [x[rev(i, L)] for i in range(n)]
    for s in range(1, K0 + 1):
        dit_stage(a, s, L, wp)
    ref = list(a)
    for s in range(K0 + 1, L + 1):
        dit_stage(ref, s, L, wp)
    M = 1 << K1
    _, wl, wpl = tables(K1)            # local table (size-2^K1 root = w^(N/M))
    assert wl == pow(w, n // M, P)
    out = [0] * n
    for r in range(1 << K0):           # network = low K0 bits
        v = [a[r + (xx << K0)] for xx in range(M)]               # local position xx = block
        v = [v[xx] * pow(w, r * rev(xx, K1), P) % P for xx in range(M)]   # twist W^(r*rev(x)), W = w
        for s in range(1, K1 + 1):
            dit_stage(v, s, K1, wpl)
        for xx in range(M):
            out[r + (xx << K0)] = v[xx]
    ok["dit"] = out == ref
    # ---------------- Pease: pass 2 = twist + local Pease
    b = [x[rev(i, L)] for i in range(n)]
    for s in range(1, K0 + 1):
        b = pease_stage(b, s, L, wp)
    ref = list(b)
    for s in range(K0 + 1, L + 1):
        ref = pease_stage(ref, s, L, wp)
    out = [0] * n
    for Q in range(1 << K0):           # network Q reads Q*2^K1 + x, writes Q | R << K0
        v = [b[(Q << K1) + xx] for xx in range(M)]
        v = [v[xx] * pow(w, Q * rev(xx, K1), P) % P for xx in range(M)]
        for s in range(1, K1 + 1):
            v = pease_stage(v, s, K1, wpl)
        for R in range(M):
            out[Q | (R << K0)] = v[R]
    ok["pease"] = out == ref
    # ---------------- Stockham: pass 2 = twist + local Stockham
    c = list(x)
    for s in range(K0):
        c = stockham_stage(c, s, L, wp)
    ref = list(c)
    for s in range(K0, L):
        ref = stockham_stage(ref, s, L, wp)
    out = [0] * n
    glob = L - K0 - K1                # = 0 here: Q = ghi (top K0 bits)
    for Q in range(1 << K0):
        v = [c[(Q << K1) + xx] for xx in range(M)]      # position ghi << (L-S0) | x
        v = [v[xx] * pow(w, Q * xx, P) % P for xx in range(M)]   # Stockham twist: natural x
        for s in range(K1):
            v = stockham_stage(v, s, K1, wpl)
        for R in range(M):
            out[(R << K0) | Q] = v[R]
    ok["stockham"] = out == ref
    # ---------------- DIF: pass 1 (window [K0, L), top) = local DIF + post-twist
    d = list(x)
    ref = list(d)
    for s in range(L, K0, -1):
        dif_stage(ref, s, L, wp)
    out = [0] * n
    for r in range(1 << K0):           # network = low K0 bits, local x at bits [K0, L)
        v = [d[r + (xx << K0)] for xx in range(M)]
        for s in range(K1, 0, -1):
            dif_stage(v, s, K1, wpl)
        v = [v[xx] * pow(w, r * rev(xx, K1), P) % P for xx in range(M)]   # post-twist
        for xx in range(M):
            out[r + (xx << K0)] = v[xx]
    ok["dif"] = out == ref
    return ok


if __name__ == "__main__":
    random.seed(1)
    for L, K0 in ((6, 3), (7, 3), (7, 4), (8, 4), (9, 5)):
        print(L, K0, check(L, K0))


def check3(L, a, b):
    """3-pass split (a, b, c) for DIT and Pease: the middle pass (S0=a, K=b)
    and last pass as twist + local transform, twist W^(r * rev_K(x)) with
    W = w^(N / 2^(S0+K)) and r = the network part that enters the twiddles."""
    n, w, wp = tables(L)
    c = L - a - b
    x = [random.randrange(P) for _ in range(n)]
    ok = {}
    # ---- DIT
    d = [x[rev(i, L)] for i in range(n)]
    ref = list(d)
    for s in range(1, L + 1):
        dit_stage(ref, s, L, wp)
    cur = list(d)
    for s in range(1, a + 1):
        dit_stage(cur, s, L, wp)
    for (S0, K) in ((a, b), (a + b, c)):
        W = pow(w, n >> (S0 + K), P)
        _, _, wpl = tables(K)
        out = list(cur)
        for Q in range(1 << (L - K)):
            low, high = Q & ((1 << S0) - 1), Q >> S0
            pos = [low | (xx << S0) | (high << (S0 + K)) for xx in range(1 << K)]
            v = [cur[pp] * pow(W, low * rev(xx, K), P) % P for xx, pp in enumerate(pos)]
            for s in range(1, K + 1):
                dit_stage(v, s, K, wpl)
            for xx, pp in enumerate(pos):
                out[pp] = v[xx]
        cur = out
    ok["dit"] = cur == ref
    # ---- Pease: network Q, local x at Q*2^K + x; enters via qtop = Q >> (L-K-S0)
    e = [x[rev(i, L)] for i in range(n)]
    ref = list(e)
    for s in range(1, L + 1):
        ref = pease_stage(ref, s, L, wp)
    cur = list(e)
    for s in range(1, a + 1):
        cur = pease_stage(cur, s, L, wp)
    for (S0, K) in ((a, b), (a + b, c)):
        W = pow(w, n >> (S0 + K), P)
        _, _, wpl = tables(K)
        out = [0] * n
        for Q in range(1 << (L - K)):
            qtop = Q >> (L - K - S0)
            v = [cur[(Q << K) + xx] * pow(W, qtop * rev(xx, K), P) % P for xx in range(1 << K)]
            for s in range(1, K + 1):
                v = pease_stage(v, s, K, wpl)
            for R in range(1 << K):
                out[Q | (R << (L - K))] = v[R]
        cur = out
    ok["pease"] = cur == ref
    return ok


if __name__ == "__main__":
    for L, a, b in ((6, 2, 2), (7, 3, 2), (8, 3, 3), (9, 3, 3), (10, 4, 3)):
        print("3-pass", L, a, b, check3(L, a, b))


def check3b(L, a, b):
    """3-pass DIF (windows from the top) and Stockham with the generalised twist."""
    n, w, wp = tables(L)
    c = L - a - b
    x = [random.randrange(P) for _ in range(n)]
    ok = {}
    # ---- DIF: windows [L-a, L), [L-a-b, L-a), [0, c); post-twist W^(r*rev(x)), r = low S0 bits
    ref = list(x)
    for s in range(L, 0, -1):
        dif_stage(ref, s, L, wp)
    cur = list(x)
    for (S0, K) in ((L - a, a), (c, b)):
        W = pow(w, n >> (S0 + K), P)
        _, _, wpl = tables(K)
        out = list(cur)
        for Q in range(1 << (L - K)):
            low, high = Q & ((1 << S0) - 1), Q >> S0
            pos = [low | (xx << S0) | (high << (S0 + K)) for xx in range(1 << K)]
            v = [cur[pp] for pp in pos]
            for s in range(K, 0, -1):
                dif_stage(v, s, K, wpl)
            v = [v[xx] * pow(W, low * rev(xx, K), P) % P for xx in range(1 << K)]
            for xx, pp in enumerate(pos):
                out[pp] = v[xx]
        cur = out
    for s in range(c, 0, -1):          # last window [0, c): local twiddles only
        dif_stage(cur, s, L, wp)
    ok["dif"] = cur == ref
    # ---- Stockham: passes (0..a-1), (a..a+b-1), (a+b..L-1); twist W^(ghi * x), natural x
    ref = list(x)
    for s in range(L):
        ref = stockham_stage(ref, s, L, wp)
    cur = list(x)
    for s in range(a):
        cur = stockham_stage(cur, s, L, wp)
    for (S0, K) in ((a, b), (a + b, c)):
        W = pow(w, n >> (S0 + K), P)
        _, _, wpl = tables(K)
        glob = L - S0 - K
        out = [0] * n
        for Q in range(1 << (L - K)):
            ghi, glo = Q >> glob, Q & ((1 << glob) - 1)
            pos = [(ghi << (L - S0)) | (xx << glob) | glo for xx in range(1 << K)]
            v = [cur[pp] * pow(W, ghi * xx, P) % P for xx, pp in enumerate(pos)]
            for s in range(K):
                v = stockham_stage(v, s, K, wpl)
            for R in range(1 << K):
                out[(R << (L - K)) | Q] = v[R]
        cur = out
    ok["stockham"] = cur == ref
    return ok


if __name__ == "__main__":
    for L, a, b in ((6, 2, 2), (7, 3, 2), (8, 3, 3), (9, 3, 3), (10, 4, 3)):
        print("3-pass b", L, a, b, check3b(L, a, b))
