"""Randomised parity sweep against the CPU oracle: field x variant x size x
batch x direction x in-place x alignment (seeded).  python tools/fuzz_parity.py [cases] [seed]"""
import os, random, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_11353_b200 as P
from oracle import oracle as O

GOLD = (1 << 64) - (1 << 32) + 1


def generic64():
    for c in range((1 << 32) - 2, 1 << 31, -1):
        p = c * (1 << 32) + 1
        if p != GOLD and P.is_prime(p):
            return p, P.find_primitive_root(p)


g64 = generic64()
FIELDS = [(998244353, 3, 32, 4, 20), (3221225473, 5, 32, 4, 20), (2013265921, 31, 32, 4, 20),
          (GOLD, 7, 64, 8, 21), (g64[0], g64[1], 64, 8, 12), (998244353, 3, 64, 8, 12)]
VARIANTS = ("dit", "dif", "flat", "pease", "pease_nc", "stockham", "sixstep", "naive")
cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
fails = 0
t0 = time.time()
for k in range(cases):
    p, g, w, word, lmax = rng.choice(FIELDS)
    variant = rng.choice(VARIANTS)
    L = rng.randint(1, lmax)
    if variant == "sixstep" and L < 2:
        L = 2
    if variant == "naive":
        L = min(L, 10)
    if rng.random() < 0.1 and L <= 14:             # polymul: intt(ntt(a) . ntt(b)) vs the oracle's
        va = rng.choice(("dit", "dif", "pease_nc", "stockham", "flat", "pease"))
        params = P.FieldParams(p, g, w)
        a = np.random.default_rng(10 * k).integers(0, p, size=(2, 1 << L), dtype=np.uint64).astype(np.uint32 if word == 4 else np.uint64)
        b = np.random.default_rng(10 * k + 1).integers(0, p, size=(2, 1 << L), dtype=np.uint64).astype(a.dtype)
        fa, fb = O.ntt(a, p, g, w, va), O.ntt(b, p, g, w, va)
        prod = np.array([[int(u) * int(v) % p for u, v in zip(ra, rb)] for ra, rb in zip(fa, fb)], dtype=a.dtype) \
            if word == 8 else ((fa.astype(np.uint64) * fb.astype(np.uint64)) % p).astype(np.uint32)
        want = O.ntt(prod, p, g, w, va, inverse=True, scale=True)
        vdt = np.int32 if word == 4 else np.int64
        tdt = torch.uint32 if word == 4 else torch.uint64
        ta = torch.from_numpy(a.view(vdt)).view(tdt).cuda()
        tb = torch.from_numpy(b.view(vdt)).view(tdt).cuda()
        got = P.cyclic_mul_ntt(ta, tb, params, va).cpu().view(torch.int32 if word == 4 else torch.int64).numpy().view(a.dtype)
        if not np.array_equal(got, want):
            fails += 1
            print(f"FAIL case {k}: POLYMUL p={p} word={word} {va} L={L}", flush=True)
        continue
    B = rng.randint(1, 4) if L <= 16 else 1
    mode = rng.choice(("fwd", "inv", "intt"))
    inplace = rng.random() < 0.3
    misalign = word == 4 and rng.random() < 0.2
    x = np.random.default_rng(k).integers(0, p, size=(B, 1 << L), dtype=np.uint64).astype(np.uint32 if word == 4 else np.uint64)
    inverse, scale = mode != "fwd", mode == "intt"
    n1 = None
    if variant == "sixstep" and rng.random() < 0.5:
        n1 = 1 << rng.randint(1, L - 1)            # explicit split (make_plan n1)
    want = O.ntt(x, p, g, w, variant, inverse=inverse, scale=scale, n1=n1) if n1 else \
        O.ntt(x, p, g, w, variant, inverse=inverse, scale=scale)
    params = P.FieldParams(p, g, w)
    plan = P.make_plan(params, variant, 1 << L, P.INVERSE if inverse else P.FORWARD, n1=n1)
    dp = P.algorithms.device_plan_for(plan, word, 0)
    if rng.random() < 0.15:                        # host-buffer path (ntt_exec_host)
        src = np.ascontiguousarray(x)
        out_h = np.empty_like(src)
        if os.environ.get("FUZZ_VERBOSE"):
            print(f"case {k}: HOST p={p} word={word} {variant} L={L} B={B} {mode} n1={n1}", flush=True)
        dp.exec_host(src.ctypes.data, out_h.ctypes.data, B, scale)
        if not np.array_equal(out_h, want):
            fails += 1
            print(f"FAIL case {k}: HOST p={p} w={w} word={word} {variant} L={L} B={B} {mode} n1={n1}", flush=True)
        continue
    tdt, vdt = (torch.int32, np.int32) if word == 4 else (torch.int64, np.int64)
    flat = torch.from_numpy(x.view(vdt).reshape(-1)).cuda()
    off = 1 if misalign else 0
    buf = torch.zeros(flat.numel() + off, dtype=tdt, device="cuda")
    buf[off:] = flat
    out = buf if inplace else torch.zeros_like(buf)
    es = word
    if os.environ.get("FUZZ_VERBOSE"):
        print(f"case {k}: p={p} word={word} {variant} L={L} B={B} {mode} inplace={inplace} misalign={misalign}", flush=True)
    dp.exec_device(buf.data_ptr() + off * es, out.data_ptr() + off * es, B, scale, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    got = out[off:].cpu().numpy().view(np.uint32 if word == 4 else np.uint64).reshape(B, -1)
    ok = np.array_equal(got, want)
    if not ok:
        fails += 1
        print(f"FAIL case {k}: p={p} w={w} word={word} {variant} L={L} B={B} {mode} inplace={inplace} misalign={misalign}", flush=True)
print(f"{cases - fails}/{cases} cases bit-exact ({time.time() - t0:.0f} s)")
sys.exit(1 if fails else 0)
