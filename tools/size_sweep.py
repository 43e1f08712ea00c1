"""Every (field, variant, log2 N) once, batch 1, forward (and intt for odd L) against the CPU
oracle: finds sizes that fall between the planners' ranges.  python tools/size_sweep.py [Lmax32] [Lmax64]"""
import os, sys, time
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
l32 = int(sys.argv[1]) if len(sys.argv) > 1 else 23
l64 = int(sys.argv[2]) if len(sys.argv) > 2 else 22
lmin = int(sys.argv[3]) if len(sys.argv) > 3 else 1
FIELDS = [("p998", 998244353, 3, 32, np.uint32, l32), ("default", 3221225473, 5, 32, np.uint32, l32),
          ("babybear", 2013265921, 31, 32, np.uint32, l32), ("goldilocks", GOLD, 7, 64, np.uint64, l64),
          ("generic64", g64[0], g64[1], 64, np.uint64, min(l64, 20)), ("p998_u64", 998244353, 3, 64, np.uint64, min(l64, 20))]
VARIANTS = ("dit", "dif", "flat", "pease", "pease_nc", "stockham", "sixstep")
bad, n, t0 = [], 0, time.time()
for name, p, g, w, dt, lmax in FIELDS:
    params = P.FieldParams(p, g, w)
    adic = ((p - 1) & -(p - 1)).bit_length() - 1          # the field has 2^L-th roots for L <= adic
    for L in range(lmin, min(lmax, adic) + 1):
        x = np.random.default_rng(1000 + L).integers(0, p, size=(1, 1 << L), dtype=np.uint64).astype(dt)
        xd = torch.from_numpy(x.view(np.int32 if dt == np.uint32 else np.int64)).view(torch.uint32 if dt == np.uint32 else torch.uint64).cuda()
        want = {}
        for v in VARIANTS:
            if v == "sixstep" and L < 2:
                continue
            for inv in ((False, True) if L % 2 else (False,)):
                n += 1
                try:
                    key = inv
                    if key not in want:          # every variant has the same output
                        want[key] = O.ntt(x, p, g, w, "dit", inverse=inv, scale=inv)
                    if v == "sixstep":
                        plan = P.make_plan(params, "sixstep", 1 << L, P.INVERSE if inv else P.FORWARD)
                        got = P.run_plan(plan, xd) if inv else P.ntt_sixstep(xd, plan)
                    else:
                        table = P.build_table(params, 1 << L, P.INVERSE if inv else P.FORWARD)
                        got = P.intt(xd, table, v) if inv else P.ntt(xd, table, v)
                    gh = got.cpu().view(torch.int32 if dt == np.uint32 else torch.int64).numpy().view(dt)
                    if not np.array_equal(gh, want[key]):
                        bad.append((name, v, L, inv, "MISMATCH"))
                except Exception as e:          # noqa: BLE001
                    bad.append((name, v, L, inv, repr(e)[:120]))
    print(f"{name}: done to 2^{lmax} ({time.time() - t0:.0f} s, {len(bad)} bad so far)", flush=True)
print(f"{n - len(bad)}/{n} cases bit-exact")
for b in bad:
    print("BAD", b)
