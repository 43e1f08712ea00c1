"""Generate golden fixtures by importing the REFERENCE package (nttkit).

Run in the build container (the reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports /root/reference/pkg/src/nttkit read-only and records, for several
fields and sizes, seeded inputs and the reference's own outputs of every
variant (forward, unscaled inverse via ``ntt(x, inv_table)``, and ``intt``),
the twiddle tables, six-step plans with explicit splits, the Pease per-stage
states, the structural copy counts, and the CLI bench checksum.  The output
(``reference_vectors.json``) is committed; tests/test_oracle_pins.py checks the
CPU oracle against it, tests/test_gpu_parity.py checks the B200 kernels.

Goldilocks is generated with ``FieldParams(P, 7, w=64)`` through the butterfly
variants only: the reference's ``naive_dft`` overflows uint64 for 64-bit p
(algorithms.py:61-62), so its "naive" output is recorded
separately under ``naive_ref_overflow`` to document the defect.
"""

from __future__ import annotations

import json
import os
import random
import sys

REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

import nttkit  # noqa: E402
from nttkit import algorithms  # noqa: E402
from nttkit.cli import bench_input  # noqa: E402
from nttkit.twiddle import FORWARD, INVERSE, build_table  # noqa: E402

GOLD = 2**64 - 2**32 + 1
FIELDS = [
    ("p17", 17, 3, 32, 4),
    ("default", nttkit.DEFAULT_PRIME, 5, 32, 10),
    ("p998", 998244353, 3, 32, 11),
    ("goldilocks", GOLD, 7, 64, 9),
]
BUTTERFLY = ("dit", "dif", "flat", "pease", "pease_nc", "stockham", "sixstep")


def main() -> None:
    out = {"generator": "tests/golden/make_golden.py", "reference": "nttkit " + nttkit.__version__,
           "fields": {}, "cases": [], "sixstep": [], "pease_stages": [], "structural": {},
           "bench_checksum": {}}
    for name, p, g, w, max_log in FIELDS:
        params = nttkit.FieldParams(p, g, w=w)
        tabs = {}
        for log in (1, 2, 3, 4):
            n = 1 << log
            if (p - 1) % n:
                continue
            f = build_table(params, n, FORWARD)
            i = build_table(params, n, INVERSE)
            tabs[str(n)] = {"fwd_w_pow": f.w_pow, "fwd_w_shoup": f.w_shoup,
                            "inv_w_pow": i.w_pow, "inv_w_shoup": i.w_shoup,
                            "n_inv": i.n_inv, "n_inv_shoup": i.n_inv_shoup}
        out["fields"][name] = {"p": p, "g": g, "w": w, "tables": tabs}
        for log in range(1, max_log + 1):
            n = 1 << log
            if (p - 1) % n:
                continue
            fwd = build_table(params, n, FORWARD)
            inv = build_table(params, n, INVERSE)
            reps = 3 if log <= 6 else 1
            rng = random.Random(f"golden-{name}-{log}")
            for r in range(reps):
                x = [rng.randrange(p) for _ in range(n)]
                y = algorithms.ntt(x, fwd, "dit")
                for v in BUTTERFLY:
                    assert algorithms.ntt(x, fwd, v) == y, (name, n, v)
                case = {"field": name, "n": n, "rep": r, "x": x, "fwd": y,
                        "inv_unscaled": algorithms.ntt(x, inv, "dit"),
                        "intt": algorithms.intt(x, inv, "dit"),
                        "variants_checked": list(BUTTERFLY)}
                for v in BUTTERFLY:
                    assert algorithms.ntt(x, inv, v) == case["inv_unscaled"]
                    assert algorithms.intt(x, inv, v) == case["intt"]
                if p < 2**32:
                    assert algorithms.naive_dft(x, fwd) == y
                    case["variants_checked"].append("naive")
                elif log <= 6:
                    case["naive_ref_overflow"] = algorithms.naive_dft(x, fwd)
                out["cases"].append(case)
    # six-step with explicit splits (algorithms.py:322-389)
    for name, p, g, w, _ in FIELDS[1:]:
        params = nttkit.FieldParams(p, g, w=w)
        for n, n1 in ((16, 1), (16, 16), (64, 2), (64, 32), (256, 4), (1024, 8), (1024, 128)):
            plan = algorithms.make_plan(params, "sixstep", n, FORWARD, n1=n1)
            rng = random.Random(f"sixstep-{name}-{n}-{n1}")
            x = [rng.randrange(p) for _ in range(n)]
            out["sixstep"].append({"field": name, "n": n, "n1": n1, "n2": n // n1, "x": x,
                                   "fwd": algorithms.ntt_sixstep(x, plan)})
    # Pease per-stage states (algorithms.py:203-227), for pass-level debugging
    for name, p, g, w, _ in FIELDS[1:3]:
        params = nttkit.FieldParams(p, g, w=w)
        n, log = 64, 6
        tab = build_table(params, n, FORWARD)
        rng = random.Random(f"stages-{name}")
        x = [rng.randrange(p) for _ in range(n)]
        cur = nttkit.bit_reverse_permute(list(x))
        states = [list(cur)]
        for s in range(1, log + 1):
            nxt = [0] * n
            algorithms._pease_stage(cur, nxt, s, log, tab)
            cur = nxt
            states.append(list(cur))
        out["pease_stages"].append({"field": name, "n": n, "x": x, "states": states})
    # structural facts the reference tests assert (test_algorithms.py:116-141)
    calls = []
    real = algorithms._stage_copy
    algorithms._stage_copy = lambda d, s: (calls.append(1), real(d, s))
    try:
        params = nttkit.FieldParams(nttkit.DEFAULT_PRIME, 5)
        tab = build_table(params, 64, FORWARD)
        x = [random.Random(9).randrange(params.p) for _ in range(64)]
        algorithms.ntt_pease(x, tab)
        pease_copies = len(calls)
        calls.clear()
        algorithms.ntt_pease_nc(x, tab)
        pease_nc_copies = len(calls)
    finally:
        algorithms._stage_copy = real
    out["structural"] = {"n": 64, "pease_copies": pease_copies, "pease_nc_copies": pease_nc_copies}
    # cli bench known answer (cli.py:39-42,133): checksum = out[0]
    for n in (1024, 4096):
        x = bench_input(n, 998244353, 42)
        params = nttkit.FieldParams(998244353, 3)
        tab = build_table(params, n, FORWARD)
        out["bench_checksum"][str(n)] = {"seed": 42, "prime": 998244353, "x": x,
                                         "checksum": algorithms.ntt(x, tab, "stockham")[0]}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_vectors.json")
    with open(path, "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print(f"wrote {path}: {len(out['cases'])} cases, {len(out['sixstep'])} six-step cases")


if __name__ == "__main__":
    main()
