#!/usr/bin/env python
"""Benchmark of the B200 batched NTT engine (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Headline workload = BASELINE.json configs[1] (config 2): 4096 independent
polynomials of N=2^12 over P=998244353, uint32 residues, Pease_nc forward
(the paper's no-copy variant); DIT on the same batch is reported alongside.
A STEP is one batched forward transform of the whole batch (one kernel
launch).  Inputs are seeded uniform residues, resident in
HBM before the timed region; input/output buffers rotate over a footprint
> 2x L2 so every step streams from HBM ("l2_policy" in the line).

Multi-GPU (independent polynomials, NO collective):
``--gpus N`` with WORLD_SIZE unset re-launches this script under
torch.distributed.run with N ranks (one process per GPU; it fails loudly if
fewer than N GPUs are visible).  Headline = weak scaling: rank r transforms
rows [r*4096, (r+1)*4096) of ONE global seeded batch of N*4096 rows (rank 0's
rows are exactly config 2's input, checked against the reference's SHA-256;
every rank checks intt(ntt(x)) == x on its own rows).  ``configs`` adds
fixed-batch (strong-scaling) runs of configs 2, 3 and 4: the global batch is
split by ``shard_rows``, timed from a common barrier to the last rank's
completion (max over ranks of CUDA-event time), and the rows are gathered
outside the timed region for the full-output SHA-256 of the reference.
`e2e` is the same metric through the C-ABI host-buffer call (ntt_exec_host:
pinned H2D + transform + D2H every step).

--impl reference times the reference algorithm on the host cores: the
reference (nttkit) is pure Python, so its CPU restatement
oracle/libntt_oracle.so (pinned bit-exact to the reference,
tests/test_oracle_pins.py) runs the same workload with every host thread.
The b200 arm's ``cpu_baseline`` also times the reference's OWN Python
(baseline/_ref/nttkit, when installed): serially (the reference's batch path,
estimator.py:61-65) and with a process pool over all host cores.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _ncu_traffic(key: str):
    """DRAM bytes per launch of the dominant kernel: the steady-state ranged
    capture (profiles/<latest round>/traffic_steady.json, tools/traffic_all.sh)
    when present, else the single-launch ncu summary (which under-reads writes
    still in L2)."""
    for rnd in ("r2", "r1"):
        try:
            with open(os.path.join(ROOT, "profiles", rnd, "traffic_steady.json")) as fh:
                d = json.load(fh).get(key)
            if d:
                return d["dram_bytes_per_step"] / d.get("launches_per_step", 1)
        except Exception:
            pass
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(key, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the GPU is loaded."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sms.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        loaded = [s for s in sms if mx and s > 0.5 * mx] or sms
        med = float(np.median(loaded)) if loaded else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sms)}


def plan_passes_of(dp) -> int | None:
    try:
        return int(dp.info.passes)
    except Exception:
        return None


def cpu_oracle_rate(w, variant: str, seconds: float, rows_cap: int | None = None):
    """Rows/s of the CPU restatement on all host threads (bounded sample)."""
    from oracle import oracle as O
    cores = len(os.sched_getaffinity(0))
    rows = min(w.batch, rows_cap or w.batch)
    from paper_2405_11353_b200.configs import seeded_input
    x = seeded_input(w, rows)
    plan = O.OraclePlan(w.p, w.g, w.w, w.n, variant, False, w.n1, None)
    plan.run(x[: max(1, min(rows, cores))], nthreads=cores)   # warm
    done, t0 = 0, time.perf_counter()
    while True:
        plan.run(x, nthreads=cores)
        done += rows
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return done / el, cores, f"{done} rows of {w.batch}x2^{w.log2n} ({rows}-row chunks, {el:.1f} s wall)"


HEADLINE_METRIC = "batched NTTs/s (N=2^12, P=998244353, pease_nc forward)"


def headline_config(world: int) -> dict:
    """The config dict BOTH arms print (byte-identical, so the driver can match them)."""
    return {"workload": "config2: 4096 x 2^12 polys per GPU, P=998244353, pease_nc forward",
            "global_batch": world * 4096, "n": 4096, "parallelism": f"batch-sharded x{world} (weak, no collective)"}


def _nttkit_worker(args):
    """One process of the reference-Python pool leg: transforms rows with nttkit.ntt."""
    rows, p, g, n, variant = args
    import nttkit
    table = nttkit.build_table(nttkit.FieldParams(p, g), n, nttkit.FORWARD)
    for r in rows:
        nttkit.ntt(r, table, variant)
    return len(rows)


def nttkit_leg(variant: str, seconds: float) -> dict:
    """The reference's OWN Python (baseline/_ref/nttkit) on the host cores:
    serial (its batch path, estimator.py:61-65) and a process pool
    (SURVEY.md sec.8d).  Runs in a child process without CUDA (see main)."""
    import multiprocessing as mp
    ref = os.path.join(ROOT, "baseline", "_ref")
    sys.path.insert(0, ref)
    import nttkit
    from paper_2405_11353_b200.configs import CONFIGS, seeded_input
    w = CONFIGS[2]
    x = [[int(v) for v in row] for row in seeded_input(w, 512)]
    table = nttkit.build_table(nttkit.FieldParams(w.p, w.g), w.n, nttkit.FORWARD)
    nttkit.ntt(x[0], table, variant)
    done, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds / 2:
        nttkit.ntt(x[done % len(x)], table, variant)
        done += 1
    serial = done / (time.perf_counter() - t0)
    cores = len(os.sched_getaffinity(0))
    per = 8                                         # rows per task
    with mp.get_context("fork").Pool(cores) as pool:
        pool.map(_nttkit_worker, [(x[:1], w.p, w.g, w.n, variant)] * cores)      # warm (import + table)
        done, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < seconds / 2:
            tasks = [(x[(i * per) % len(x):(i * per) % len(x) + per], w.p, w.g, w.n, variant) for i in range(2 * cores)]
            done += sum(pool.map(_nttkit_worker, tasks))
        pooled = done / (time.perf_counter() - t0)
    cpu = ""
    try:
        with open("/proc/cpuinfo") as fh:
            cpu = next(l.split(":", 1)[1].strip() for l in fh if l.startswith("model name"))
    except Exception:
        pass
    src = "baseline/_ref/nttkit (the reference package, pip-installed unmodified)"
    return {"serial": {"value": serial, "unit": "NTT/s", "cores": 1, "kind": "reference",
                       "sample": f"nttkit.ntt per row of config 2 for {seconds / 2:.0f} s; {src}"},
            "pool": {"value": pooled, "unit": "NTT/s", "cores": cores, "kind": "reference",
                     "sample": f"multiprocessing.Pool({cores}) over rows of config 2 for {seconds / 2:.0f} s; {src}"},
            "cpu_model": cpu}


def run_nttkit_leg_subprocess(variant: str, seconds: float):
    if not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "nttkit")):
        return {"unavailable": "baseline/_ref/nttkit not installed"}
    try:
        res = subprocess.run([sys.executable, os.path.abspath(__file__), "--nttkit-leg", "--variant", variant,
                              "--nttkit-seconds", str(seconds)], capture_output=True, text=True, timeout=600)
        return json.loads(res.stdout.strip().splitlines()[-1])
    except Exception as exc:
        return {"unavailable": repr(exc)[:200]}


def run_reference(args, rank: int, world: int) -> None:
    from paper_2405_11353_b200.configs import CONFIGS
    if rank != 0:
        return
    w = CONFIGS[2]
    rates = []
    for _ in range(args.warmup):
        cpu_oracle_rate(w, args.variant, 0.2)
    sample = ""
    cores = 1
    per_step = max(0.05, min(0.5, 60.0 / max(1, args.steps)))   # whole run ~1 min of CPU work
    for _ in range(args.steps):
        r, cores, sample = cpu_oracle_rate(w, args.variant, per_step, 1024 if args.steps > 100 else None)
        rates.append(r)
    val = float(np.median(rates))
    line = {
        "impl": "reference", "metric": HEADLINE_METRIC,
        "value": val, "unit": "NTT/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * w.batch / val, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (np.random.default_rng(2) uniform residues)",
        "config": headline_config(world),
        "cpu_baseline": {"value": val, "unit": "NTT/s", "cores": cores, "kind": "port",
                         "sample": sample + "; oracle/libntt_oracle.so (C restatement of nttkit, pinned bit-exact)"},
        "e2e": {"value": val, "unit": "NTT/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def spawn_ranks(args) -> int:
    """--gpus N without WORLD_SIZE: re-launch under torch.distributed.run with N ranks."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} requested but only {have} CUDA device(s) are visible"}),
              flush=True)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--variant", default="pease_nc")
    ap.add_argument("--no-extra", action="store_true", help="skip the other BASELINE configs")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-sweep", action="store_true", help="skip the N = 2^9..2^20 u32 sweep")
    ap.add_argument("--peer-exchange", action="store_true",
                    help="N>1: also time config 5's four-step with the exchange fused into step A's pack "
                         "(P2P stores into symmetric memory) -- off by default: not yet run on >1 GPU")
    ap.add_argument("--nttkit-leg", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--nttkit-seconds", type=float, default=16.0, help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.nttkit_leg:          # child process of the cpu_baseline leg (no CUDA)
        print(json.dumps(nttkit_leg(args.variant, args.nttkit_seconds)), flush=True)
        return

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        if args.impl == "reference":
            os.environ["WORLD_SIZE"] = str(args.gpus)    # host-only arm: rank 0 alone runs
        else:
            sys.exit(spawn_ranks(args))

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), flush=True)
        sys.exit(2)

    # the reference-Python CPU leg first, in a child process (CPU only, before
    # this process initialises CUDA: its pool forks)
    ref_leg = None
    if rank == 0 and world == 1 and not args.no_cpu:
        ref_leg = run_nttkit_leg_subprocess(args.variant, 16.0)

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local_rank)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    import paper_2405_11353_b200 as P
    from paper_2405_11353_b200 import _lib
    from paper_2405_11353_b200.configs import CONFIGS, GOLDEN, seeded_input, seeded_rows
    from paper_2405_11353_b200.distributed import shard_rows

    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.Stream(dev)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    peak, peak_src = _peaks()

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local_rank])
        torch.cuda.synchronize(dev)

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def all_ranks(flag) -> bool | None:
        """True iff every rank's check passed (None if no rank checked)."""
        v = -1.0 if flag is None else float(bool(flag))
        if world == 1:
            return None if flag is None else bool(flag)
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        mn = t.clone()
        dist.all_reduce(mn, op=dist.ReduceOp.MIN)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if t.item() < 0:
            return None
        return bool(mn.item() >= 1) if mn.item() >= 0 else None

    sdt_of = lambda word: torch.int32 if word == 4 else torch.int64

    def to_dev(x_host, word):
        tdt = torch.uint32 if word == 4 else torch.uint64
        return torch.from_numpy(x_host.view(np.int32 if word == 4 else np.int64)).view(tdt).to(dev)

    def sha_gathered(y, rows_per_rank: int, word: int) -> str | None:
        """Full-output SHA-256 of the row blocks of every rank, in rank order (rank 0)."""
        flat = y.view(sdt_of(word)).reshape(-1)
        if world > 1:
            full = torch.empty(world * flat.numel(), dtype=flat.dtype, device=dev)
            dist.all_gather_into_tensor(full, flat.contiguous())
            flat = full
        if rank != 0:
            return None
        return hashlib.sha256(flat.cpu().numpy().astype("<u4" if word == 4 else "<u8").tobytes()).hexdigest()

    def measure(w, variant, steps, warmup, inverse=False, sampler=None, check=True, rows=None, golden_rows=None):
        """Device-resident timing of `steps` batched transforms of this rank's rows.
        rows = (lo, hi) of the config's seeded stream (default: the whole batch).
        golden_rows: the rows whose gathered output must hash to the reference's
        SHA-256 (strong scaling: every rank's block of the config's batch)."""
        params = P.FieldParams(w.p, w.g, w.w)
        plan = P.make_plan(params, variant, w.n, P.INVERSE if inverse else P.FORWARD, n1=w.n1)
        dp = P.algorithms.device_plan_for(plan, w.word, local_rank)
        lo, hi = rows if rows is not None else (0, w.batch)
        B = hi - lo
        x_host = seeded_rows(w, lo, hi)
        nbytes = x_host.nbytes
        # rotating in/out buffer sets: footprint >= 2 x L2 so steps stream from HBM
        nset = max(2, min(64, int(np.ceil(2 * l2 / (2 * nbytes))) + 1))
        xs = [to_dev(x_host, w.word)]
        for _ in range(nset - 1):
            xs.append(xs[0].clone())
        ys = [torch.empty_like(xs[0]) for _ in range(nset)]
        sp = stream.cuda_stream
        parity = None
        roundtrip = None
        if check and not inverse:
            dp.exec_device(xs[0].data_ptr(), ys[0].data_ptr(), B, False, sp)
            torch.cuda.synchronize(dev)
            if golden_rows and w.cfg in GOLDEN:
                # full-output SHA-256 vs the hash the reference itself produced
                h = sha_gathered(ys[0], B, w.word)
                parity = None if rank != 0 else h == GOLDEN[w.cfg][1]
            # every rank: intt(ntt(x)) == x on its own rows
            iplan = P.make_plan(params, variant, w.n, P.INVERSE, n1=w.n1)
            idp = P.algorithms.device_plan_for(iplan, w.word, local_rank)
            idp.exec_device(ys[0].data_ptr(), ys[1].data_ptr(), B, True, sp)
            torch.cuda.synchronize(dev)
            roundtrip = bool(torch.equal(ys[1].view(sdt_of(w.word)), xs[0].view(sdt_of(w.word))))
        if check and inverse:
            # no reference hash for the inverse: intt(ntt(x)) == x on the seeded input
            fplan = P.make_plan(params, variant, w.n, P.FORWARD, n1=w.n1)
            fdp = P.algorithms.device_plan_for(fplan, w.word, local_rank)
            fdp.exec_device(xs[0].data_ptr(), ys[0].data_ptr(), B, False, sp)
            dp.exec_device(ys[0].data_ptr(), ys[1].data_ptr(), B, True, sp)
            torch.cuda.synchronize(dev)
            roundtrip = bool(torch.equal(ys[1].view(sdt_of(w.word)), xs[0].view(sdt_of(w.word))))
        if world > 1:
            parity = all_ranks(parity) if rank == 0 else all_ranks(None)
            roundtrip = all_ranks(roundtrip)
        with torch.cuda.stream(stream):
            for i in range(warmup):
                dp.exec_device(xs[i % nset].data_ptr(), ys[i % nset].data_ptr(), B, inverse, sp, independent=True)
            if sampler is not None:     # sustained load while clocks are sampled
                sampler.start()
                t_end = time.perf_counter() + 1.0
                i = 0
                while time.perf_counter() < t_end:
                    for _ in range(20):
                        dp.exec_device(xs[i % nset].data_ptr(), ys[i % nset].data_ptr(), B, inverse, sp, independent=True)
                        i += 1
                    stream.synchronize()
            # the K timed steps are captured once into a CUDA graph and replayed:
            # back-to-back kernels with no host launch gaps between them (an
            # eager Python loop adds ~3 us per step, per-step events ~5 us more)
            _lib.counters_reset()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                for i in range(steps):
                    dp.exec_device(xs[i % nset].data_ptr(), ys[i % nset].data_ptr(), B, inverse, sp, independent=True)
            launches = _lib.counters_read()["kernel_launches"]     # kernels inside the graph
            graph.replay()                                         # one untimed replay
            stream.synchronize()
            barrier()
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            graph.replay()
            ev1.record(stream)
            stream.synchronize()
            torch.cuda.synchronize(dev)
            barrier()
        clocks = sampler.stop() if sampler is not None else None
        total_ms = max_over_ranks(ev0.elapsed_time(ev1))
        per_launch_ms = total_ms / steps       # one step = one ntt_exec call
        del xs, ys, graph
        torch.cuda.empty_cache()
        return {"total_ms": total_ms, "per_step_ms": per_launch_ms, "launches": launches, "parity": parity,
                "roundtrip": roundtrip, "clocks": clocks, "nset": nset, "footprint_bytes": 2 * nset * nbytes,
                "rows": B, "dp": dp}

    def e2e(w, variant, steps, rows, asynchronous=True):
        """Through the C-ABI host-buffer call: pinned H2D + transform + D2H per step.
        asynchronous: NTT_FLAG_HOST_ASYNC -- each call enqueues its step and
        returns, so step i's copy-out overlaps step i+1's copy-in; one stream
        synchronise after the K steps, inside the timed region.  Otherwise the
        synchronous call (the reference's list-in / list-out contract)."""
        params = P.FieldParams(w.p, w.g, w.w)
        plan = P.make_plan(params, variant, w.n, P.FORWARD, n1=w.n1)
        dp = P.algorithms.device_plan_for(plan, w.word, local_rank)
        lo, hi = rows
        x_host = seeded_rows(w, lo, hi)
        hin = torch.from_numpy(x_host.view(np.int32 if w.word == 4 else np.int64)).pin_memory()
        hout = torch.empty_like(hin).pin_memory()
        sp = stream.cuda_stream
        for _ in range(2):
            dp.exec_host(hin.data_ptr(), hout.data_ptr(), hi - lo, False, sp, asynchronous)
        stream.synchronize()
        barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            dp.exec_host(hin.data_ptr(), hout.data_ptr(), hi - lo, False, sp, asynchronous)
        stream.synchronize()
        el = max_over_ranks(time.perf_counter() - t0)
        return world * (hi - lo) * steps / el, x_host.nbytes

    _lib.counters_enable(False)     # device-side structural counters off; host launch count stays on
    w = CONFIGS[2]
    mine = (rank * w.batch, (rank + 1) * w.batch)       # weak scaling: this rank's rows of the global batch
    sampler = ClockSampler(local_rank)
    m = measure(w, args.variant, args.steps, args.warmup, sampler=sampler, rows=mine, golden_rows=(rank == 0))
    step_s = m["total_ms"] / 1e3 / args.steps
    value = world * w.batch / step_s
    alg_bytes = w.algorithmic_bytes()
    achieved = alg_bytes / (m["per_step_ms"] / 1e3) / 1e9
    e2e_val, io_bytes = e2e(w, args.variant, max(3, min(args.steps, 20)), mine)
    e2e_sync, _ = e2e(w, args.variant, max(3, min(args.steps, 20)), mine, asynchronous=False)
    dit = measure(w, "dit", args.steps, args.warmup, rows=mine, golden_rows=(rank == 0))

    extra = {}
    if not args.no_extra:
        # fixed global batch split over the ranks (strong scaling, no collective);
        # rows gathered outside the timed region for the reference's full-output SHA-256
        ext_steps, ext_warm = max(3, min(args.steps, 10)), 3
        for cfg, var, inv in ((2, args.variant, False), (3, "dif", False), (3, "dif", True),
                              (4, "pease_nc", False), (5, "sixstep", False)):
            wc = CONFIGS[cfg]
            if cfg == 2 and world == 1:
                continue                  # identical to the headline at one GPU
            if cfg == 5 and world > 1:
                continue                  # one transform: the distributed four-step below
            try:
                lo, hi = shard_rows(wc.batch, rank, world)
                r = measure(wc, var, ext_steps, ext_warm, inverse=inv, rows=(lo, hi), golden_rows=True)
                t = r["total_ms"] / 1e3 / ext_steps
                ab = wc.algorithmic_bytes()
                key = f"config{cfg}_{var}_{'inv' if inv else 'fwd'}" + ("_strong" if cfg == 2 else "")
                extra[key] = {
                    "ntt_per_s": wc.batch / t, "ms_per_step": 1e3 * t,
                    "gbfly_per_s": wc.butterflies() / t / 1e9,
                    "hbm_alg_gbs": ab / t / 1e9,
                    "roofline_frac": ab / t / 1e9 / (world * peak),
                    "launches_per_step": r["launches"] / ext_steps, "sha256_parity": r["parity"],
                    "roundtrip_parity": r["roundtrip"], "scaling": "strong", "ranks": world,
                    "rows_per_rank": hi - lo,
                    "workload": f"{wc.batch} x 2^{wc.log2n}, p={wc.p} (fixed batch, shard_rows)"}
            except Exception as exc:  # report, do not hide
                extra[f"config{cfg}_{var}"] = {"error": repr(exc)[:300]}

    if not args.no_extra:
        # polymul.cyclic_mul_ntt on config 2's shape: 4096 products
        # c = a * b mod (x^4096 - 1): forward of both operands in one launch, then
        # ntt_exec_pointwise_inverse (product fused into the inverse's first group)
        try:
            p, L, B = 998244353, 12, 4096
            n = 1 << L
            pf = P.algorithms._device_plan(P.FieldParams(p, 3), n, args.variant, P.FORWARD, None, None, 4, local_rank)
            pi = P.algorithms._device_plan(P.FieldParams(p, 3), n, args.variant, P.INVERSE, None, None, 4, local_rank)
            nset = 4
            ab = torch.randint(0, p, (nset, 2, B, n), dtype=torch.int64, device=dev).to(torch.int32).view(torch.uint32)
            spec = torch.empty_like(ab[0])
            cc = torch.empty_like(ab[:, 0])
            sp = stream.cuda_stream
            reps = max(3, min(args.steps, 20))
            def pm(i):
                pf.exec_device(ab[i % nset].data_ptr(), spec.data_ptr(), 2 * B, False, sp, independent=True)
                pi.pointwise_inverse(spec[0].data_ptr(), spec[1].data_ptr(), cc[i % nset].data_ptr(), B, sp)
            with torch.cuda.stream(stream):
                for i in range(3):
                    pm(i)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    for i in range(reps):
                        pm(i)
                g.replay()
                barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                g.replay()
                e1.record(stream)
                stream.synchronize()
            t = max_over_ranks(e0.elapsed_time(e1)) / 1e3 / reps
            extra["polymul_4096x2^12"] = {
                "products_per_s": world * B / t, "ms_per_step": 1e3 * t, "launches_per_step": 2,
                "hbm_alg_gbs": 3 * B * n * 4 / t / 1e9, "roofline_frac": 3 * B * n * 4 / t / 1e9 / peak,
                "workload": "4096 cyclic products of N=2^12, P=998244353 (forward x2 in one launch + fused pointwise-inverse)"}
            del ab, spec, cc, g
            torch.cuda.empty_cache()
        except Exception as exc:
            extra["polymul_4096x2^12"] = {"error": repr(exc)[:300]}

    sweep = {}
    if not args.no_extra and not args.no_sweep:
        # batched u32 transforms N = 2^9 .. 2^20 at 256 MiB of residues per step (P = 998244353,
        # pease_nc): the N range BASELINE.json's metric names; graph replay, CUDA events
        p = 998244353
        for L in range(9, 21):
            n = 1 << L
            B = (1 << 26) // n
            try:
                plan = P.make_plan(P.FieldParams(p, 3), args.variant, n)
                dp = P.algorithms.device_plan_for(plan, 4, local_rank)
                xa = torch.randint(0, p, (2, B, n), dtype=torch.int64, device=dev).to(torch.int32).view(torch.uint32)
                ya = torch.empty_like(xa)
                sp = stream.cuda_stream
                reps = 6
                with torch.cuda.stream(stream):
                    for i in range(3):
                        dp.exec_device(xa[i % 2].data_ptr(), ya[i % 2].data_ptr(), B, False, sp, independent=True)
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=stream):
                        for i in range(reps):
                            dp.exec_device(xa[i % 2].data_ptr(), ya[i % 2].data_ptr(), B, False, sp, independent=True)
                    g.replay()
                    barrier()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    g.replay()
                    e1.record(stream)
                    stream.synchronize()
                t = max_over_ranks(e0.elapsed_time(e1)) / 1e3 / reps
                gbs = 2 * B * n * 4 / t / 1e9
                sweep[f"2^{L}"] = {"batch": B, "ms": round(1e3 * t, 4), "ntt_per_s": world * B / t,
                                   "gbfly_per_s": round(world * B * (n // 2) * L / t / 1e9, 1),
                                   "roofline_frac": round(gbs / peak, 3),
                                   "passes": plan_passes_of(dp)}
                del xa, ya, g
                torch.cuda.empty_cache()
            except Exception as exc:
                sweep[f"2^{L}"] = {"error": repr(exc)[:200]}

    if world > 1 and not args.no_extra:
        # config 5 as ONE transform split four-step across the ranks (strong
        # scaling, one NCCL all-to-all per step); slab layout per distributed.py
        try:
            from paper_2405_11353_b200.distributed import DistributedSixStep, column_slab
            wc = CONFIGS[5]
            params = P.FieldParams(wc.p, wc.g, wc.w)
            ds = DistributedSixStep(params, wc.n, n1=wc.n1, n2=wc.n // wc.n1)
            xh = seeded_input(wc)[0]
            slab = torch.from_numpy(column_slab(xh, rank, world, ds.n1, ds.n2).view(np.int64)).view(torch.uint64).to(dev)
            out5 = torch.empty((ds.n1, ds.kcols), dtype=slab.dtype, device=dev)
            with torch.cuda.stream(stream):
                for _ in range(3):
                    ds.run(slab, out=out5)
                barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                nst = max(3, min(args.steps, 10))
                e0.record(stream)
                for _ in range(nst):
                    ds.run(slab, out=out5)
                e1.record(stream)
                stream.synchronize()
            barrier()
            t = max_over_ranks(e0.elapsed_time(e1)) / 1e3 / nst
            # every rank's output column block, gathered outside the timed region:
            # the reference's full-output SHA-256 of config 5
            from paper_2405_11353_b200.distributed import assemble_output
            full = torch.empty(world * out5.numel(), dtype=torch.int64, device=dev)
            dist.all_gather_into_tensor(full, out5.view(torch.int64).reshape(-1))
            par5 = None
            if rank == 0:
                blocks = full.cpu().numpy().view(np.uint64).reshape(world, -1)
                got = assemble_output([b for b in blocks], ds.n1, ds.n2)
                par5 = hashlib.sha256(got.astype("<u8").tobytes()).hexdigest() == GOLDEN[5][1]
            extra["config5_sixstep_distributed"] = {
                "sha256_parity": par5,
                "ntt_per_s": 1.0 / t, "ms_per_step": 1e3 * t, "scaling": "strong", "ranks": world,
                "gbfly_per_s": wc.butterflies() / t / 1e9,
                "alltoall_bytes_per_rank": (world - 1) * (wc.n // world // world) * 8,
                "workload": "1 x 2^26 Goldilocks, four-step 2^13 x 2^13, one NCCL all_to_all_single"}
        except Exception as exc:
            extra["config5_sixstep_distributed"] = {"error": repr(exc)[:300]}
        if args.peer_exchange:
            try:
                dsp = DistributedSixStep(params, wc.n, n1=wc.n1, n2=wc.n // wc.n1, exchange="peer")
                with torch.cuda.stream(stream):
                    for _ in range(3):
                        dsp.run(slab, out=out5)
                    barrier()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    for _ in range(nst):
                        dsp.run(slab, out=out5)
                    e1.record(stream)
                    stream.synchronize()
                barrier()
                t = max_over_ranks(e0.elapsed_time(e1)) / 1e3 / nst
                extra["config5_sixstep_distributed_peer"] = {
                    "ntt_per_s": 1.0 / t, "ms_per_step": 1e3 * t, "scaling": "strong", "ranks": world,
                    "workload": "1 x 2^26 Goldilocks, four-step, exchange fused into step A's pack (P2P stores)"}
            except Exception as exc:
                extra["config5_sixstep_distributed_peer"] = {"error": repr(exc)[:300]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rate, cores, sample = cpu_oracle_rate(w, args.variant, 10.0)
        cpu = {"value": rate, "unit": "NTT/s", "cores": cores, "kind": "port",
               "sample": sample + "; oracle/libntt_oracle.so = C restatement of nttkit, pinned bit-exact",
               # the reference's own Python on the same host: serial + process pool
               "reference_python": ref_leg}

    if rank == 0:
        line = {
            "metric": HEADLINE_METRIC,
            "value": value, "unit": "NTT/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": m["total_ms"] / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic (np.random.default_rng(2) uniform residues)",
            "config": headline_config(world),
            "l2_policy": f"rotating {m['nset']} in/out buffer sets, footprint "
                         f"{m['footprint_bytes'] >> 20} MiB > 2 x L2 {l2 >> 20} MiB",
            "api": "ntt_exec on resident device buffers, NTT_FLAG_INDEPENDENT (consecutive steps use disjoint "
                   "buffer sets: the launch window may overlap them; NTT_PDL_DEFER=0 times the plain ordering)",
            "roundtrip_parity_all_ranks": m["roundtrip"],
            "gbutterfly_per_s": world * w.butterflies() / step_s / 1e9,
            "sha256_parity": m["parity"],
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": _ncu_traffic("config2_pease_nc"),
                         "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": alg_bytes},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": "NTT/s", "h2d_bytes_per_step": io_bytes,
                    "d2h_bytes_per_step": io_bytes, "api": "ntt_exec_host, NTT_FLAG_HOST_ASYNC (steps pipelined)",
                    "synchronous_value": e2e_sync},
            "gpu_launches": m["launches"],
            "clocks": m["clocks"],
            "dit": {"ntt_per_s": world * w.batch / (dit["total_ms"] / 1e3 / args.steps),
                    "roofline_frac": alg_bytes / (dit["per_step_ms"] / 1e3) / 1e9 / peak,
                    "sha256_parity": dit["parity"], "roundtrip_parity_all_ranks": dit["roundtrip"]},
            "configs": extra,
            "sweep_u32_pease_nc": sweep,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
