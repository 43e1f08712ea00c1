"""One small launch of every kernel family, each checked against the oracle (61 cases, ~7 s on
a B200):  python tools/family_smoke.py [GROUP ...]
Groups: fast, gold, fs, tile, six, host, poly.  (Written as the workload for compute-sanitizer;
that tool is closed on this GPU pool, so it serves as the quick all-families check.)"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_11353_b200 as P
from oracle import oracle as O

GOLD = (1 << 64) - (1 << 32) + 1
dev = torch.device("cuda", 0)


def to_dev(x):
    if x.dtype == np.uint32:
        return torch.from_numpy(x.view(np.int32)).view(torch.uint32).to(dev)
    return torch.from_numpy(x.view(np.int64)).view(torch.uint64).to(dev)


def to_host(t):
    if t.dtype == torch.uint32:
        return t.cpu().view(torch.int32).numpy().view(np.uint32)
    return t.cpu().view(torch.int64).numpy().view(np.uint64)


def case(p, g, w, dt, B, L, variant, inverse=False, n1=None):
    x = np.random.default_rng(L * 131 + B).integers(0, p, size=(B, 1 << L), dtype=np.uint64).astype(dt)
    params = P.FieldParams(p, g, w)
    n = 1 << L
    if variant == "sixstep":
        plan = P.make_plan(params, "sixstep", n, P.FORWARD, n1=n1)
        got = to_host(P.ntt_sixstep(to_dev(x), plan))
        want = O.ntt(x, p, g, w, "sixstep", n1=n1)
    else:
        table = P.build_table(params, n, P.INVERSE if inverse else P.FORWARD)
        got = to_host(P.intt(to_dev(x), table, variant) if inverse else P.ntt(to_dev(x), table, variant))
        want = O.ntt(x, p, g, w, variant, inverse=inverse, scale=inverse)
    ok = np.array_equal(got, want)
    print(f"{'ok ' if ok else 'BAD'} p={p} B={B} 2^{L} {variant}{' inv' if inverse else ''}", flush=True)
    return ok


def main():
    groups = set(sys.argv[1:]) or {"fast", "gold", "fs", "tile", "six", "host", "poly"}
    ok = True
    P32, BB, DEF = (998244353, 3, 32, np.uint32), (2013265921, 31, 32, np.uint32), (3221225473, 5, 32, np.uint32)
    G64 = (GOLD, 7, 64, np.uint64)
    if "fast" in groups:      # k_fast: single pass, every dataflow, lazy and canonical u32
        for L in (9, 12, 13, 14):
            for v in ("dit", "dif", "pease", "pease_nc", "stockham", "flat"):
                ok &= case(*P32, 5, L, v)
        ok &= case(*P32, 5, 12, "pease_nc", inverse=True)
        ok &= case(*BB, 3, 12, "dit")
        ok &= case(*DEF, 3, 12, "pease_nc")
        ok &= case(*P32, 3, 6, "dit")          # generic shared-memory engine
    if "gold" in groups:      # Goldilocks single pass + four-step
        for v in ("dit", "dif", "pease_nc", "stockham"):
            ok &= case(*G64, 3, 12, v)
            ok &= case(*G64, 2, 16, v)
        ok &= case(*G64, 2, 16, "dif", inverse=True)
    if "fs" in groups:        # four-step: TMA passes (K = 7..10) and the cp.async passes
        for L in (15, 17, 18, 20):
            for v in ("pease_nc", "dit", "pease", "dif"):
                ok &= case(*P32, 2 if L < 20 else 1, L, v)
        ok &= case(*BB, 1, 16, "pease_nc")
    if "tile" in groups:      # multi-pass tile kernels beyond the four-step
        ok &= case(*P32, 1, 21, "pease_nc")
        ok &= case(*G64, 1, 19, "dit")
    if "six" in groups:       # six-step: k_cols column passes with the folded transpose
        ok &= case(*G64, 1, 16, "sixstep", n1=256)
        ok &= case(*G64, 1, 20, "sixstep", n1=1024)
        ok &= case(*P32, 1, 16, "sixstep", n1=256)
    if "host" in groups:      # host-buffer path (chunked copies on three streams)
        x = np.random.default_rng(7).integers(0, P32[0], size=(64, 4096), dtype=np.uint64).astype(np.uint32)
        table = P.build_table(P.FieldParams(*P32[:3]), 4096)
        got = np.array([P.ntt([int(t) for t in row], table, "pease_nc") for row in x[:2]], dtype=np.uint32)
        okh = np.array_equal(got, O.ntt(x[:2], *P32[:3], "pease_nc"))
        print("ok " if okh else "BAD", "list API (host path) 2 x 2^12", flush=True)
        ok &= okh
    if "poly" in groups:      # fused pointwise-inverse
        rng = np.random.default_rng(11)
        a = rng.integers(0, P32[0], size=(4, 4096), dtype=np.uint64).astype(np.uint32)
        b = rng.integers(0, P32[0], size=(4, 4096), dtype=np.uint64).astype(np.uint32)
        params = P.FieldParams(*P32[:3])
        got = to_host(P.cyclic_mul_ntt(to_dev(a), to_dev(b), params))
        fa, fb = O.ntt(a, *P32[:3], "dit"), O.ntt(b, *P32[:3], "dit")
        prod = ((fa.astype(np.uint64) * fb.astype(np.uint64)) % P32[0]).astype(np.uint32)
        want = O.ntt(prod, *P32[:3], "dit", inverse=True, scale=True)
        okp = np.array_equal(got, want)
        print("ok " if okp else "BAD", "cyclic_mul_ntt 4 x 2^12", flush=True)
        ok &= okp
    torch.cuda.synchronize()
    print("ALL OK" if ok else "FAILURES", flush=True)
    sys.exit(0 if ok else 1)


main()
