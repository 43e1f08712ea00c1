"""Shared-memory bank model of the TMA four-step column pass
(csrc/fourstep_tma.cuh k_fs_tma, MODE 0): replays, for one tile, every warp's
accesses of the tile-major groups -- group 0 reading the dense TMA staging
[2^K rows][TQ columns] and writing the padded work buffer, and the last group
reading it -- and returns the worst n-way bank conflict (1 = conflict free).
The middle groups use the network-major map of the tile kernels (bankcheck.py).

The geometry below restates TmaGeo<V, K> (NP, network base, in-warp bit
placements); `search()` is the exhaustive search that chose them."""
from collections import defaultdict
import itertools


def padpos(p):
    return p + (p >> 5) + (p >> 10)


def padded_len(K):
    return (padpos((1 << K) - 1) + 1 + 3) & ~3


def brev(x, n):
    return int(format(x, "0%db" % n)[::-1], 2) if n else 0


def geometry(V, K):
    """TmaGeo<V, K> of fourstep_tma.cuh"""
    TQ = 1 << (13 - K)
    LQ = 13 - K
    AB = 0 if LQ >= 5 else 5 - LQ
    G = (K + 3) // 4
    K0 = K - 4 * (G - 1)
    KG0 = K0 if V == "dit" else 4
    KGL = 4 if V == "dit" else K0
    NPM = 2 if (K == 10 and V != "dit") else 1
    nlin = (K == 9 and V == "dit")
    NP = ((padded_len(K) + (8 if nlin else 0) + 31) // 32) * 32 + NPM
    I0 = (4, 5)
    IL = (3, 4) if V == "dit" else (0, 1)
    return dict(TQ=TQ, LQ=LQ, AB=AB, KG0=KG0, KGL=KGL, NP=NP, nlin=nlin, I0=I0, IL=IL,
                base=lambda q: q * NP + (8 * (q >> 3) if nlin else 0))


def place(w, AB, bits, UB):
    if AB == 0:
        return w
    u = 0
    for i in range(AB):
        u |= ((w >> i) & 1) << bits[i]
    rest = w >> AB
    for b in range(UB):
        if b in bits[:AB]:
            continue
        u |= (rest & 1) << b
        rest >>= 1
    return u


def _worst(addrs):
    banks = defaultdict(set)
    for a in addrs:
        banks[a % 32].add(a)
    return max(len(s) for s in banks.values())


def worst_conflict(V, K, geo=None):
    g = geo or geometry(V, K)
    TQ, LQ, AB, UB = g["TQ"], g["LQ"], g["AB"], K - 4
    worst = 1
    nwarps = 512 // 32
    for warp in range(nwarps):
        lanes = range(warp * 32, warp * 32 + 32)
        for c in range(16):
            rd, wr, last = [], [], []
            for tid in lanes:
                q, w = tid & (TQ - 1), tid >> LQ
                u0 = place(w, AB, g["I0"], UB)
                pos = (u0 << 4) | c
                rd.append(brev(pos, K) * TQ + q)                   # dense staging [r][q]
                if V == "dit":
                    wpos = pos
                else:
                    kg = g["KG0"]
                    wpos = ((u0 << (4 - kg)) | (c >> kg)) | ((c & ((1 << kg) - 1)) << (K - kg))
                wr.append(g["base"](q) + padpos(wpos))
                uL = place(w, AB, g["IL"], UB)
                lpos = (uL | (c << (K - 4))) if V == "dit" else ((uL << 4) | c)
                last.append(g["base"](q) + padpos(lpos))
            worst = max(worst, _worst(rd), _worst(wr), _worst(last))
    return worst


def search(V, K):
    """every (NP mod 32, group-0 bits, last-group bits) with a conflict-free tile (linear base)"""
    g0 = geometry(V, K)
    sols = []
    UB = K - 4
    for npm in range(32):
        NP = ((padded_len(K) + 31) // 32) * 32 + npm
        for i0 in itertools.permutations(range(UB), 2):
            for il in itertools.permutations(range(UB), 2):
                g = dict(g0, NP=NP, I0=i0, IL=il, base=lambda q, NP=NP: q * NP)
                if worst_conflict(V, K, g) == 1:
                    sols.append((npm, i0, il))
    return sols


if __name__ == "__main__":
    for V in ("dit", "pease"):
        for K in (7, 8, 9, 10):
            print(V, K, "worst n-way:", worst_conflict(V, K))
