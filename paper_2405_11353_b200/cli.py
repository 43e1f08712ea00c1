"""Command-line front end (nttkit/cli.py): ``verify`` and ``bench`` on the B200.

    python -m paper_2405_11353_b200.cli verify [--max-log 10] [--prime P] [--vectors 5]
    python -m paper_2405_11353_b200.cli bench  [--algo A ...] [--size N ...] [--batch B] [--reps R] [--csv F]
    python -m paper_2405_11353_b200.cli banks  --algo A --log-n L [--interleave M | --blocksize B | --banks K --search
                                                | --units U] [--ports 2] [--unroll 1] [--csv F]

``bench`` keeps the reference CSV schema (cli.py:24) and seeding (cli.py:39-42)
and appends GPU columns (batch, device time, NTT/s, Gbutterfly/s, algorithmic
GB/s).  ``verify`` checks every variant against the exact naive DFT on the
device, the round trip, and the convolution theorem against the schoolbook
product -- and imports INVERSE, which the reference's verify forgets
(cli.py:21 vs :71).  Exit codes: 0 pass, 1 failure, 2 usage.
"""

from __future__ import annotations

import argparse
import csv
import random
import statistics
import sys

import numpy as np

from . import bankmodel
from .algorithms import VARIANTS, intt, make_plan, naive_dft, ntt
from .errors import InvalidSize, NttError
from .modmath import DEFAULT_PRIME, FieldParams, find_primitive_root
from .polymul import cyclic_mul_ntt, schoolbook_cyclic
from .twiddle import FORWARD, INVERSE, build_table

BENCH_VARIANTS = tuple(v for v in VARIANTS if v != "naive")
BENCH_CSV_FIELDS = ("algo", "n", "prime", "reps", "mean_ns", "median_ns", "min_ns", "checksum",
                    "device", "batch", "device_ms", "ntt_per_s", "gbfly_per_s", "alg_gbs")


def bench_input(n: int, prime: int, seed: int) -> list[int]:
    """Same deterministic residues as the reference (cli.py:39-42)."""
    rng = random.Random(f"{seed}-{n}-{prime}")
    return [rng.randrange(prime) for _ in range(n)]


def _field(prime: int) -> FieldParams:
    return FieldParams(prime, find_primitive_root(prime), 32 if prime < (1 << 32) else 64)


def verify_run(max_log: int, seed: int, prime: int, vectors: int = 5, echo=print):
    params = _field(prime)
    rng = random.Random(seed)
    failures = []
    for log in range(1, max_log + 1):
        n = 1 << log
        if (prime - 1) % n:
            break
        fwd = build_table(params, n, FORWARD)
        inv = build_table(params, n, INVERSE)
        xs = [[rng.randrange(prime) for _ in range(n)] for _ in range(vectors)]
        want = [naive_dft(x, fwd) for x in xs]
        for algo in BENCH_VARIANTS:
            ok_o = all(ntt(x, fwd, algo) == w for x, w in zip(xs, want))
            ok_r = all(intt(ntt(x, fwd, algo), inv, algo) == x for x in xs)
            if not ok_o:
                failures.append(("oracle", algo, n))
            if not ok_r:
                failures.append(("roundtrip", algo, n))
            if log <= 9:
                a, b = xs[0], xs[-1]
                if cyclic_mul_ntt(a, b, params, algo) != schoolbook_cyclic(a, b, prime):
                    failures.append(("polymul", algo, n))
        echo(f"n={n:<6} {'ok' if not [f for f in failures if f[2] == n] else 'FAIL'}")
    return failures


def bench_run(algos, sizes, reps: int, prime: int, seed: int, batch: int = 1024):
    import time

    import torch
    params = _field(prime)
    word = 4 if prime < (1 << 32) else 8
    tdt, view = (torch.uint32, np.int32) if word == 4 else (torch.uint64, np.int64)
    dev = torch.device("cuda", torch.cuda.current_device())
    records = []
    for n in sizes:
        if n < 2 or n & (n - 1) or (prime - 1) % n:
            raise InvalidSize(f"size {n} unusable with prime {prime}")
        x = bench_input(n, prime, seed)
        xb = np.tile(np.asarray(x, dtype=np.uint64).astype(np.uint32 if word == 4 else np.uint64), (batch, 1))
        xd = torch.from_numpy(np.ascontiguousarray(xb).view(view)).view(tdt).to(dev)
        for algo in algos:
            plan = make_plan(params, algo, n, FORWARD)
            table = plan.table
            checksum = ntt(x, table, algo)[0]
            y = ntt(xd, table, algo)
            torch.cuda.synchronize()
            timings = []
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for _ in range(reps):
                t0 = time.perf_counter_ns()
                ev0.record()
                y = ntt(xd, table, algo)
                ev1.record()
                ev1.synchronize()
                timings.append(time.perf_counter_ns() - t0)
            dev_ms = ev0.elapsed_time(ev1)
            first = int(y[0, 0].cpu().view(torch.int32 if word == 4 else torch.int64).item()) % (1 << (8 * word))
            assert first == checksum
            log = n.bit_length() - 1
            records.append({"algo": algo, "n": n, "prime": prime, "reps": reps,
                            "mean_ns": int(statistics.fmean(timings)), "median_ns": int(statistics.median(timings)),
                            "min_ns": int(min(timings)), "checksum": checksum, "device": torch.cuda.get_device_name(),
                            "batch": batch, "device_ms": dev_ms, "ntt_per_s": batch / (dev_ms * 1e-3),
                            "gbfly_per_s": batch * (n // 2) * log / (dev_ms * 1e-3) / 1e9,
                            "alg_gbs": batch * 2 * n * word / (dev_ms * 1e-3) / 1e9})
    return records


def write_bench_csv(records, path) -> None:
    try:
        empty = not open(path, "rb").read(1)
    except FileNotFoundError:
        empty = True
    with open(path, "a", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=BENCH_CSV_FIELDS)
        if empty:
            w.writeheader()
        for r in records:
            w.writerow({k: r[k] for k in BENCH_CSV_FIELDS})


def banks_run(args) -> int:
    """``banks``: the bank-conflict model (nttkit/cli.py:181-241, same output)."""
    if args.units is not None:
        if args.algo != "pease_nc":
            print("error: --units applies to the pease_nc swap-safety check")
            return 1
        rep = bankmodel.pease_nc_partition_check(args.log_n, args.units, args.ports)
    else:
        trace = bankmodel.gen_trace(args.algo, args.log_n)
        if args.search:
            if args.banks is None:
                print("error: --search requires --banks")
                return 1
            part = bankmodel.feasible_partition(trace, args.banks, ports=args.ports, unroll=args.unroll)
            if part is None:
                print(f"infeasible: no II=1 partition with {args.banks} bank(s) per array")
                return 0
            for arr, m in sorted(part.items()):
                desc = (" ".join(f"{a}->{b}" for a, b in enumerate(m.table)) if m.kind == "explicit"
                        else f"{m.kind}={m.param}")
                print(f"array {arr}: {desc}")
            print("feasible: II=1")
            return 0
        mapping = bankmodel.blocksize(args.blocksize) if args.blocksize is not None else \
            bankmodel.interleave(args.interleave)
        rep = bankmodel.schedule(trace, bankmodel.BankConfig(mapping, ports=args.ports, unroll=args.unroll))
    print(bankmodel.report_text(rep))
    if args.csv:
        row = dict(algo=args.algo, log_n=args.log_n, ports=args.ports, unroll=args.unroll,
                   **bankmodel.report_csv_row(rep))
        fields = ["algo", "log_n", "ports", "unroll", "achieved_ii", "target_ii", "feasible", "conflicts",
                  "swap_safe"]
        try:
            empty = not open(args.csv, "rb").read(1)
        except FileNotFoundError:
            empty = True
        with open(args.csv, "a", newline="") as fh:
            w = csv.DictWriter(fh, fieldnames=fields)
            if empty:
                w.writeheader()
            w.writerow(row)
        print(f"wrote report to {args.csv}")
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2405_11353_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    v = sub.add_parser("verify")
    v.add_argument("--max-log", type=int, default=10)
    v.add_argument("--seed", type=int, default=0)
    v.add_argument("--prime", type=int, default=DEFAULT_PRIME)
    v.add_argument("--vectors", type=int, default=5)
    b = sub.add_parser("bench")
    b.add_argument("--algo", action="append", choices=BENCH_VARIANTS)
    b.add_argument("--size", action="append", type=int)
    b.add_argument("--reps", type=int, default=10)
    b.add_argument("--batch", type=int, default=1024)
    b.add_argument("--seed", type=int, default=42)
    b.add_argument("--prime", type=int, default=DEFAULT_PRIME)
    b.add_argument("--csv")
    k = sub.add_parser("banks")
    k.add_argument("--algo", required=True, choices=bankmodel.TRACE_VARIANTS)
    k.add_argument("--log-n", type=int, required=True)
    k.add_argument("--interleave", type=int, default=1)
    k.add_argument("--blocksize", type=int)
    k.add_argument("--banks", type=int)
    k.add_argument("--ports", type=int, default=2)
    k.add_argument("--unroll", type=int, default=1)
    k.add_argument("--units", type=int)
    k.add_argument("--search", action="store_true")
    k.add_argument("--csv")
    return ap


def main(argv=None) -> int:
    try:
        args = build_parser().parse_args(argv)
    except SystemExit as e:
        return 2 if e.code else 0
    if args.cmd == "banks" and not 1 <= args.log_n <= 16:
        print("error: --log-n must be in [1, 16]", file=sys.stderr)
        return 2
    try:
        if args.cmd == "banks":
            return banks_run(args)
        if args.cmd == "verify":
            fails = verify_run(args.max_log, args.seed, args.prime, args.vectors)
            for f in fails:
                print("FAIL", *f)
            return 1 if fails else 0
        recs = bench_run(args.algo or list(BENCH_VARIANTS), args.size or [1024, 4096, 16384], args.reps,
                         args.prime, args.seed, args.batch)
        print(f"{'algo':<10}{'n':>8}{'batch':>7}{'dev_ms':>10}{'NTT/s':>14}{'Gbfly/s':>10}  checksum")
        for r in recs:
            print(f"{r['algo']:<10}{r['n']:>8}{r['batch']:>7}{r['device_ms']:>10.4f}{r['ntt_per_s']:>14.4g}"
                  f"{r['gbfly_per_s']:>10.1f}  {r['checksum']}")
        if args.csv:
            write_bench_csv(recs, args.csv)
        return 0
    except (NttError, ValueError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
