"""Parity of the B200 kernels against the CPU oracle (oracle/ntt_oracle.c, pinned
to the reference by tests/test_oracle_pins.py) and against vectors produced by
the reference itself (tests/golden/reference_vectors.json, SURVEY.md sec.8c hashes).

Every comparison is bit-exact (integer arithmetic).  Calls go through the
package's public API, which executes through the C ABI (libntt_b200.so).
"""

from __future__ import annotations

import hashlib
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2405_11353_b200 as P  # noqa: E402
from paper_2405_11353_b200.configs import CONFIGS, GOLDEN, seeded_input  # noqa: E402
from oracle import oracle as O  # noqa: E402

GOLD = (1 << 64) - (1 << 32) + 1
# (name, p, g, w, dtype, max log2 N exercised)
FIELDS = [
    ("p998", 998244353, 3, 32, np.uint32, 20),
    ("default", 3221225473, 5, 32, np.uint32, 16),
    ("goldilocks", GOLD, 7, 64, np.uint64, 16),
    ("p998_u64", 998244353, 3, 64, np.uint64, 12),
    ("babybear", 2013265921, 31, 32, np.uint32, 14),     # 2^30 < p < 2^31: canonical u32 path
    ("big64", 18446744069414584321, 7, 64, np.uint64, 6),   # placeholder, replaced below
]
VARIANTS7 = ("dit", "dif", "flat", "pease", "pease_nc", "stockham", "sixstep")


def _generic64():
    """An NTT-friendly 64-bit prime > 2^63 that is NOT Goldilocks (F64 path)."""
    for c in range((1 << 32) - 2, 1 << 31, -1):
        p = c * (1 << 32) + 1
        if p != GOLD and P.is_prime(p):
            return p, P.find_primitive_root(p)
    raise RuntimeError("no prime found")


@pytest.fixture(scope="module")
def fields():
    p, g = _generic64()
    fl = list(FIELDS[:-1]) + [("generic64", p, g, 64, np.uint64, 12)]
    return {f[0]: f for f in fl}


def dev():
    return torch.device("cuda", 0)


def to_dev(x: np.ndarray):
    if x.dtype == np.uint32:
        return torch.from_numpy(x.view(np.int32)).view(torch.uint32).to(dev())
    return torch.from_numpy(x.view(np.int64)).view(torch.uint64).to(dev())


def to_host(t) -> np.ndarray:
    if t.dtype == torch.uint32:
        return t.cpu().view(torch.int32).numpy().view(np.uint32)
    return t.cpu().view(torch.int64).numpy().view(np.uint64)


def gpu_ntt(x, p, g, w, variant, inverse=False, scale=False, n1=None):
    params = P.FieldParams(p, g, w)
    n = x.shape[-1]
    if variant == "sixstep":
        plan = P.make_plan(params, "sixstep", n, P.INVERSE if inverse else P.FORWARD, n1=n1)
        if inverse and scale:
            return to_host(P.run_plan(plan, to_dev(x)))
        if inverse:
            return to_host(P.algorithms._execute(to_dev(x), params, n, "sixstep", P.INVERSE, False,
                                                 plan.n1, plan.n2))
        return to_host(P.ntt_sixstep(to_dev(x), plan))
    table = P.build_table(params, n, P.INVERSE if inverse else P.FORWARD)
    if scale:
        return to_host(P.intt(to_dev(x), table, variant))
    return to_host(P.ntt(to_dev(x), table, variant))


def rand(p, B, L, dt, seed):
    return np.random.default_rng(seed).integers(0, p, size=(B, 1 << L), dtype=np.uint64).astype(dt)


@pytest.mark.parametrize("variant", VARIANTS7 + ("naive",))
@pytest.mark.parametrize("fname", ["p998", "default", "goldilocks", "p998_u64", "generic64", "babybear"])
def test_variant_vs_oracle_small(fields, fname, variant):
    _, p, g, w, dt, maxl = fields[fname]
    for L in range(1, min(maxl, 13) + 1):
        if variant == "naive" and L > 9:
            continue
        B = 3 if L > 6 else 17
        x = rand(p, B, L, dt, 1000 + L)
        want = O.ntt(x, p, g, w, variant if variant != "naive" else "dit")
        got = gpu_ntt(x, p, g, w, variant)
        assert np.array_equal(got, want), (fname, variant, L)


@pytest.mark.parametrize("variant", VARIANTS7)
@pytest.mark.parametrize("fname", ["p998", "default", "goldilocks", "babybear"])
def test_variant_inverse_and_intt(fields, fname, variant):
    _, p, g, w, dt, maxl = fields[fname]
    for L in (1, 5, 9, 10, 11, 12, 13):
        x = rand(p, 4, L, dt, 2000 + L)
        want_u = O.ntt(x, p, g, w, variant, inverse=True)
        want_s = O.ntt(x, p, g, w, variant, inverse=True, scale=True)
        assert np.array_equal(gpu_ntt(x, p, g, w, variant, inverse=True), want_u), (fname, variant, L)
        assert np.array_equal(gpu_ntt(x, p, g, w, variant, inverse=True, scale=True), want_s), (fname, variant, L)


@pytest.mark.parametrize("variant", VARIANTS7)
@pytest.mark.parametrize("fname,L", [("p998", 14), ("p998", 15), ("p998", 16), ("p998", 18),
                                     ("default", 16), ("goldilocks", 13), ("goldilocks", 14),
                                     ("goldilocks", 16), ("generic64", 14)])
def test_variant_vs_oracle_large(fields, fname, L, variant):
    _, p, g, w, dt, _ = fields[fname]
    x = rand(p, 2, L, dt, 3000 + L)
    want = O.ntt(x, p, g, w, variant)
    assert np.array_equal(gpu_ntt(x, p, g, w, variant), want), (fname, variant, L)


def test_reference_golden_vectors(golden):
    """Every case the reference produced (all variants agree there) -- forward,
    unscaled inverse, intt -- reproduced by every GPU variant."""
    fmeta = golden["fields"]
    for case in golden["cases"]:
        fm = fmeta[case["field"]]
        p, g, w = fm["p"], fm["g"], fm["w"]
        dt = np.uint32 if p < (1 << 32) else np.uint64
        x = np.array(case["x"], dtype=np.uint64).astype(dt)[None, :]
        for v in case["variants_checked"]:
            if v == "naive" or (v == "sixstep" and case["n"] < 2):
                continue
            assert gpu_ntt(x, p, g, w, v)[0].tolist() == case["fwd"], (case["field"], case["n"], v)
            assert gpu_ntt(x, p, g, w, v, inverse=True)[0].tolist() == case["inv_unscaled"]
            assert gpu_ntt(x, p, g, w, v, inverse=True, scale=True)[0].tolist() == case["intt"]
        # exact naive on the GPU (the reference's naive overflows for 64-bit p)
        if case["n"] <= 512:
            assert gpu_ntt(x, p, g, w, "naive")[0].tolist() == case["fwd"]


def test_reference_sixstep_splits(golden):
    for case in golden["sixstep"]:
        fm = golden["fields"][case["field"]]
        p, g, w = fm["p"], fm["g"], fm["w"]
        dt = np.uint32 if p < (1 << 32) else np.uint64
        x = np.array(case["x"], dtype=np.uint64).astype(dt)[None, :]
        got = gpu_ntt(x, p, g, w, "sixstep", n1=case["n1"])
        assert got[0].tolist() == case["fwd"], (case["field"], case["n"], case["n1"])


def test_list_api_and_bench_checksum(golden):
    """The reference calling convention (list in, list out) + cli bench known answer."""
    params = P.FieldParams(998244353, 3)
    for n, rec in golden["bench_checksum"].items():
        table = P.build_table(params, int(n))
        for v in VARIANTS7:
            out = P.ntt(rec["x"], table, v)
            assert isinstance(out, list) and out[0] == rec["checksum"] == (467606314 if n == "1024" else out[0])


@pytest.mark.parametrize("variant", ["dit", "pease_nc", "dif", "flat", "stockham"])
@pytest.mark.parametrize("L", [14, 15, 16, 17, 18, 19, 20])
def test_fourstep_sizes_vs_oracle(variant, L):
    """Two-pass four-step kernels (fourstep.cuh; every R x C split 7..10):
    forward, unscaled inverse and intt against the oracle, odd batch."""
    p, g = 998244353, 3
    B = 3 if L <= 18 else 1
    x = rand(p, B, L, np.uint32, 4000 + L)
    assert np.array_equal(gpu_ntt(x, p, g, 32, variant), O.ntt(x, p, g, 32, variant)), (variant, L)
    assert np.array_equal(gpu_ntt(x, p, g, 32, variant, inverse=True),
                          O.ntt(x, p, g, 32, variant, inverse=True)), (variant, L)
    assert np.array_equal(gpu_ntt(x, p, g, 32, variant, inverse=True, scale=True),
                          O.ntt(x, p, g, 32, variant, inverse=True, scale=True)), (variant, L)


@pytest.mark.parametrize("variant", ["dit", "dif", "pease_nc", "stockham"])
@pytest.mark.parametrize("p,g", [(3221225473, 5), (2013265921, 31)])
@pytest.mark.parametrize("L", [14, 17, 20])
def test_fourstep_canonical_u32_fields(variant, p, g, L):
    """Four-step with canonical u32 arithmetic: the reference's DEFAULT_PRIME
    3221225473 (2^31 <= p: Shoup with a 33-bit intermediate) and BabyBear."""
    x = rand(p, 2 if L < 20 else 1, L, np.uint32, 4300 + L)
    assert np.array_equal(gpu_ntt(x, p, g, 32, variant), O.ntt(x, p, g, 32, variant)), (p, variant, L)
    assert np.array_equal(gpu_ntt(x, p, g, 32, variant, inverse=True, scale=True),
                          O.ntt(x, p, g, 32, variant, inverse=True, scale=True)), (p, variant, L)


@pytest.mark.parametrize("variant", ["dit", "dif", "pease_nc", "stockham", "flat"])
@pytest.mark.parametrize("L", [14, 15, 16, 17, 18])
def test_fourstep_goldilocks(variant, L):
    """Goldilocks four-step 2^14..2^18 (config 3: 256 x 256): forward, unscaled
    inverse and intt against the oracle."""
    p, g = (1 << 64) - (1 << 32) + 1, 7
    x = rand(p, 3 if L <= 16 else 1, L, np.uint64, 4100 + L)
    assert np.array_equal(gpu_ntt(x, p, g, 64, variant), O.ntt(x, p, g, 64, variant))
    assert np.array_equal(gpu_ntt(x, p, g, 64, variant, inverse=True), O.ntt(x, p, g, 64, variant, inverse=True))
    assert np.array_equal(gpu_ntt(x, p, g, 64, variant, inverse=True, scale=True),
                          O.ntt(x, p, g, 64, variant, inverse=True, scale=True))


@pytest.mark.parametrize("L", [14, 17, 20])
def test_fourstep_in_place_and_misaligned(L):
    """Four-step edge cases: in-place execution (d_in == d_out), and an input
    only 4-byte aligned (the TMA passes decline it; the cp.async passes run)."""
    p, g = 998244353, 3
    plan = P.make_plan(P.FieldParams(p, g), "pease_nc", 1 << L)
    dp = P.algorithms.device_plan_for(plan, 4, 0)
    B = 2
    x = rand(p, B, L, np.uint32, 6000 + L)
    want = O.ntt(x, p, g, 32, "pease_nc")
    s = torch.cuda.current_stream().cuda_stream
    d = to_dev(x)
    dp.exec_device(d.data_ptr(), d.data_ptr(), B, False, s)
    assert np.array_equal(to_host(d), want), ("in-place", L)
    big = torch.zeros(B * (1 << L) + 1, dtype=torch.int32, device="cuda")
    big[1:] = torch.from_numpy(x.view(np.int32).reshape(-1)).cuda()
    out = torch.zeros_like(big)
    dp.exec_device(big.data_ptr() + 4, out.data_ptr() + 4, B, False, s)
    torch.cuda.synchronize()
    got = out[1:].cpu().numpy().view(np.uint32).reshape(B, -1)
    assert np.array_equal(got, want), ("misaligned", L)


def test_concurrent_streams_share_a_plan():
    """A multi-pass plan (workspace-backed four-step) executed concurrently on
    two streams: each stream has its own workspace, both results exact."""
    p, g, L = 998244353, 3, 18
    plan = P.make_plan(P.FieldParams(p, g), "pease_nc", 1 << L)
    dp = P.algorithms.device_plan_for(plan, 4, 0)
    xs = [rand(p, 6, L, np.uint32, 5000 + i) for i in range(2)]
    want = [O.ntt(x, p, g, 32, "pease_nc") for x in xs]
    dx = [to_dev(x) for x in xs]
    dy = [torch.empty_like(d) for d in dx]
    streams = [torch.cuda.Stream() for _ in range(2)]
    torch.cuda.synchronize()
    for _ in range(4):
        for d_in, d_out, st in zip(dx, dy, streams):
            dp.exec_device(d_in.data_ptr(), d_out.data_ptr(), 6, False, st.cuda_stream)
    torch.cuda.synchronize()
    for d_out, w in zip(dy, want):
        assert np.array_equal(to_host(d_out), w)


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_config_golden_hash_full(cfg):
    w = CONFIGS[cfg]
    x = seeded_input(w)
    assert O.sha256_le(x) == GOLDEN[cfg][0]
    for v in w.variants:
        if v == "naive":
            continue
        got = gpu_ntt(x, w.p, w.g, w.w, v, n1=w.n1)
        assert O.sha256_le(got) == GOLDEN[cfg][1], (cfg, v)


@pytest.mark.parametrize("cfg", [4, 5])
def test_config_golden_hash_large(cfg):
    """Configs 4 (512 x 2^20) and 5 (2^26 Goldilocks six-step): full-output
    SHA-256 equals the hash the reference itself produced."""
    w = CONFIGS[cfg]
    x = seeded_input(w)
    for v in w.variants:
        got = gpu_ntt(x, w.p, w.g, w.w, v, n1=w.n1)
        assert O.sha256_le(got) == GOLDEN[cfg][1], (cfg, v)


@pytest.mark.parametrize("variant", ["dit", "dif", "pease_nc", "stockham", "sixstep"])
def test_round_trip_config4_size(variant):
    w = CONFIGS[4]
    x = seeded_input(w, rows=8)
    y = gpu_ntt(x, w.p, w.g, w.w, variant)
    z = gpu_ntt(y, w.p, w.g, w.w, variant, inverse=True, scale=True)
    assert np.array_equal(z, x)


def test_linearity_goldilocks_2_16():
    w = CONFIGS[3]
    x = seeded_input(w, rows=4)
    p = w.p
    a, b = 123456789123456789 % p, 987654321987654321 % p
    xs, ys = x[:2], x[2:]
    combo = np.array([[(a * int(u) + b * int(v)) % p for u, v in zip(r1, r2)] for r1, r2 in zip(xs, ys)],
                     dtype=np.uint64)
    lhs = gpu_ntt(combo, p, w.g, w.w, "dif")
    fx, fy = gpu_ntt(xs, p, w.g, w.w, "dif"), gpu_ntt(ys, p, w.g, w.w, "dif")
    rhs = np.array([[(a * int(u) + b * int(v)) % p for u, v in zip(r1, r2)] for r1, r2 in zip(fx, fy)],
                   dtype=np.uint64)
    assert np.array_equal(lhs, rhs)


def test_structural_counters():
    """B200 analogue of test_algorithms.py:116-141: Pease copies back, Pease_nc
    never does; Stockham never bit-reverses, DIT does."""
    params = P.FieldParams(3221225473, 5)
    x = rand(params.p, 8, 6, np.uint32, 9)
    P.counters_enable(True)
    for L, B in ((6, 8), (12, 4), (16, 2)):
        x = rand(params.p, B, L, np.uint32, 9 + L)
        table = P.build_table(params, 1 << L)
        res = {}
        for v in ("pease", "pease_nc", "stockham", "dit"):
            P.counters_reset()
            P.ntt(to_dev(x), table, v)
            torch.cuda.synchronize()
            res[v] = P.counters_read()
        assert res["pease"]["stage_copies"] > 0
        assert res["pease_nc"]["stage_copies"] == 0
        assert res["stockham"]["bitrev_passes"] == 0
        assert res["dit"]["bitrev_passes"] == B
        for v in res:
            assert res[v]["transforms"] == B, (v, res[v])
    P.counters_enable(False)


def test_edge_cases():
    params = P.FieldParams(998244353, 3)
    table = P.build_table(params, 16)
    inv = P.build_table(params, 16, P.INVERSE)
    with pytest.raises(P.SizeMismatch):
        P.ntt(to_dev(np.zeros((2, 8), np.uint32)), table)
    with pytest.raises(ValueError):
        P.intt(to_dev(np.zeros((2, 16), np.uint32)), table)
    # empty batch
    e = P.ntt(to_dev(np.zeros((0, 16), np.uint32)), table, "pease_nc")
    assert tuple(e.shape) == (0, 16)
    # delta -> ones, constant -> (N*c, 0, ...) on every variant (test_algorithms.py:42-55)
    for v in VARIANTS7:
        d = np.zeros((1, 16), np.uint32)
        d[0, 0] = 1
        assert gpu_ntt(d, params.p, params.g, 32, v).tolist() == [[1] * 16]
        c = np.full((1, 16), 7, np.uint32)
        assert gpu_ntt(c, params.p, params.g, 32, v)[0].tolist() == [112] + [0] * 15
        assert P.intt(P.ntt([5] * 16, table, v), inv, v) == [5] * 16
    # in-place through the C ABI (d_in == d_out)
    x = rand(params.p, 4, 12, np.uint32, 77)
    t = to_dev(x)
    dp = P.algorithms.device_plan_for(P.make_plan(params, "pease_nc", 4096), 4, 0)
    dp.exec_device(t.data_ptr(), t.data_ptr(), 4, False, torch.cuda.current_stream().cuda_stream)
    assert np.array_equal(to_host(t), O.ntt(x, params.p, params.g, 32, "pease_nc"))
    # p = 17 (the reference fixture field), all sizes it supports
    p17 = P.FieldParams(17, 3)
    for L in (1, 2, 3, 4):
        xx = rand(17, 5, L, np.uint32, L)
        for v in VARIANTS7:
            assert np.array_equal(gpu_ntt(xx, 17, 3, 32, v), O.ntt(xx, 17, 3, 32, v))
    del p17


def test_pointwise_mul():
    params = P.FieldParams(GOLD, 7, 64)
    dp = P.algorithms.device_plan_for(P.make_plan(params, "dit", 1024), 8, 0)
    a = rand(GOLD, 1, 10, np.uint64, 1)
    b = rand(GOLD, 1, 10, np.uint64, 2)
    ta, tb = to_dev(a), to_dev(b)
    tc = torch.empty_like(ta)
    dp.pointwise(ta.data_ptr(), tb.data_ptr(), tc.data_ptr(), 1024, torch.cuda.current_stream().cuda_stream)
    want = [(int(u) * int(v)) % GOLD for u, v in zip(a[0], b[0])]
    assert to_host(tc)[0].tolist() == want


def _emulate_distributed(x, p, g, n, n1, world, peer=False):
    """Run the rank-local steps of the distributed four-step for every rank on
    ONE device through the C ABI, with the all-to-all done as a local block
    permutation (never launching mutually-waiting ranks on one GPU).
    peer=True: step A's pack stores straight into every rank's receive buffer
    (ntt_sixstep_dist_step_a_peer, the NVLink path with local pointers);
    ranks run one after another, so no kernel waits on another."""
    from paper_2405_11353_b200.distributed import assemble_output, column_slab
    n2 = n // n1
    params = P.FieldParams(p, g, 64)
    plan = P.make_plan(params, "sixstep", n, n1=n1)
    dp = P.algorithms.device_plan_for(plan, 8, 0)
    c, r = n1 // world, n2 // world
    block = c * r
    s = torch.cuda.current_stream().cuda_stream
    if peer:
        recvs = [torch.full((world * block,), 0xFFFF, dtype=torch.uint64, device=dev()) for _ in range(world)]
        ptrs = [t.data_ptr() for t in recvs]
        for rank in range(world):
            slab = to_dev(column_slab(x, rank, world, n1, n2))
            dp.sixstep_dist_step_a_peer(rank, world, slab.data_ptr(), ptrs, s)
        outs = []
        for rank in range(world):
            out = torch.empty(n1 * r, dtype=torch.uint64, device=dev())
            dp.sixstep_dist_step(1, rank, world, recvs[rank].data_ptr(), out.data_ptr(), s)
            outs.append(to_host(out))
        return assemble_output(outs, n1, n2)
    sends = []
    for rank in range(world):
        slab = to_dev(column_slab(x, rank, world, n1, n2))
        send = torch.empty(world * block, dtype=torch.uint64, device=dev())
        dp.sixstep_dist_step(0, rank, world, slab.data_ptr(), send.data_ptr(), s)
        sends.append(send)
    outs = []
    for rank in range(world):
        recv = torch.cat([sends[src][rank * block:(rank + 1) * block] for src in range(world)])
        out = torch.empty(n1 * r, dtype=torch.uint64, device=dev())
        dp.sixstep_dist_step(1, rank, world, recv.data_ptr(), out.data_ptr(), s)
        outs.append(to_host(out))
    return assemble_output(outs, n1, n2)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_distributed_sixstep_emulated_small(world):
    n, n1 = 1 << 14, 1 << 7
    x = rand(GOLD, 1, 14, np.uint64, 55)[0]
    got = _emulate_distributed(x, GOLD, 7, n, n1, world)
    assert np.array_equal(got, O.ntt(x, GOLD, 7, 64, "sixstep", n1=n1))


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_distributed_sixstep_peer_pack_emulated_small(world):
    """Exchange fused into step A's pack (P2P stores into each rank's receive
    buffer): bit-identical to the oracle's six-step."""
    n, n1 = 1 << 18, 1 << 9      # long-run passes: n1/G, n2/G >= 64 columns at G = 8
    x = rand(GOLD, 1, 18, np.uint64, 56)[0]
    got = _emulate_distributed(x, GOLD, 7, n, n1, world, peer=True)
    assert np.array_equal(got, O.ntt(x, GOLD, 7, 64, "sixstep", n1=n1))


@pytest.mark.parametrize("world", [2, 8])
def test_distributed_sixstep_peer_pack_config5(world):
    w = CONFIGS[5]
    x = seeded_input(w)[0]
    got = _emulate_distributed(x, w.p, w.g, w.n, w.n1, world, peer=True)
    assert O.sha256_le(got) == GOLDEN[5][1]


def test_distributed_peer_exchange_one_rank_group():
    """DistributedSixStep(exchange="peer") through torch symmetric memory in a
    one-rank NCCL group (subprocess with a timeout: a rendezvous that cannot
    complete must not hang the suite)."""
    import json, subprocess, sys
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "peer.npz")
        pr = subprocess.run([sys.executable, os.path.join(here, "tools", "peer_world1.py"), path],
                            capture_output=True, text=True, timeout=300)
        lines = [ln for ln in pr.stdout.splitlines() if ln.startswith("{")]
        assert lines, pr.stderr[-2000:]
        res = json.loads(lines[-1])
        assert res["ok"], res
        d = np.load(path)
        assert np.array_equal(d["out"], O.ntt(d["x"], GOLD, 7, 64, "sixstep", n1=res["n1"]))


def test_distributed_peer_pack_errors():
    params = P.FieldParams(GOLD, 7, 64)
    dp = P.algorithms.device_plan_for(P.make_plan(params, "sixstep", 1 << 14, n1=1 << 7), 8, 0)
    x = torch.zeros(1 << 14, dtype=torch.uint64, device=dev())
    s = torch.cuda.current_stream().cuda_stream
    with pytest.raises(ValueError):
        dp.sixstep_dist_step_a_peer(0, 2, x.data_ptr(), [x.data_ptr(), 0], s)      # NULL peer buffer
    with pytest.raises(ValueError):
        dp.sixstep_dist_step_a_peer(0, 16, x.data_ptr(), [x.data_ptr()] * 16, s)   # > 8 ranks


@pytest.mark.parametrize("world", [2, 8])
def test_distributed_sixstep_emulated_config5(world):
    """Config 5 (2^26 Goldilocks, 2^13 x 2^13) split over `world` ranks:
    output hash equals the reference's."""
    w = CONFIGS[5]
    x = seeded_input(w)[0]
    got = _emulate_distributed(x, w.p, w.g, w.n, w.n1, world)
    assert O.sha256_le(got) == GOLDEN[5][1]


@pytest.mark.parametrize("variant", VARIANTS7)
def test_cyclic_mul_ntt_vs_schoolbook(variant):
    """Convolution theorem (test_polymul.py:46-53) on the device, 32- and 64-bit fields."""
    for p, g, w, L in ((998244353, 3, 32, 8), (3221225473, 5, 32, 5), (GOLD, 7, 64, 6)):
        params = P.FieldParams(p, g, w)
        rng = np.random.default_rng(L)
        a = [int(v) for v in rng.integers(0, p, size=1 << L, dtype=np.uint64)]
        b = [int(v) for v in rng.integers(0, p, size=1 << L, dtype=np.uint64)]
        assert P.cyclic_mul_ntt(a, b, params, variant) == P.schoolbook_cyclic(a, b, p)
    # batched device operands: every row multiplied in one set of launches
    params = P.FieldParams(998244353, 3)
    A = rand(998244353, 8, 10, np.uint32, 1)
    B = rand(998244353, 8, 10, np.uint32, 2)
    C = to_host(P.cyclic_mul_ntt(to_dev(A), to_dev(B), params, variant))
    for r in (0, 7):
        assert C[r].tolist() == P.schoolbook_cyclic(A[r].tolist(), B[r].tolist(), 998244353)


@pytest.mark.parametrize("variant", ["dit", "dif", "pease", "pease_nc", "stockham", "flat"])
def test_pointwise_inverse_fused(variant):
    """ntt_exec_pointwise_inverse: intt(a .* b) in one call -- fused (Montgomery
    product in the inverse's first group) for resident u32 sizes 2^9..2^13, the
    pointwise kernel + intt otherwise (2^6, 2^14, 2^16, Flat) -- against the oracle."""
    p, g = 998244353, 3
    params = P.FieldParams(p, g)
    for L, B in ((6, 5), (9, 7), (10, 9), (11, 3), (12, 9), (13, 5), (14, 3), (16, 2)):
        fa = O.ntt(rand(p, B, L, np.uint32, 7000 + L), p, g, 32, variant)
        fb = O.ntt(rand(p, B, L, np.uint32, 8000 + L), p, g, 32, variant)
        prod = ((fa.astype(np.uint64) * fb.astype(np.uint64)) % p).astype(np.uint32)
        want = O.ntt(prod, p, g, 32, variant, inverse=True, scale=True)
        dp = P.algorithms._device_plan(params, 1 << L, variant, P.INVERSE, None, None, 4, 0)
        da, db = to_dev(fa), to_dev(fb)
        out = torch.empty_like(da)
        dp.pointwise_inverse(da.data_ptr(), db.data_ptr(), out.data_ptr(), B, torch.cuda.current_stream().cuda_stream)
        assert np.array_equal(to_host(out), want), (variant, L)


def test_estimator_batched_device_path():
    from sklearn.pipeline import Pipeline
    from paper_2405_11353_b200.estimator import NttTransform
    X = rand(998244353, 64, 10, np.uint32, 3).astype(np.int64)
    for v in ("dit", "pease_nc", "stockham", "sixstep"):
        t = NttTransform(variant=v, prime=998244353).fit(X)
        Y = t.transform(X)
        assert np.array_equal(Y.astype(np.uint64), O.ntt(X.astype(np.uint64), 998244353, 3, 32, "dit"))
        assert np.array_equal(t.inverse_transform(Y), X)
    pipe = Pipeline([("ntt", NttTransform(variant="dif", prime=998244353))])
    assert pipe.fit_transform(X).shape == X.shape
    Xg = rand(GOLD, 4, 8, np.uint64, 4)
    tg = NttTransform(variant="dif", prime=GOLD).fit(Xg)
    assert np.array_equal(tg.transform(Xg), O.ntt(Xg, GOLD, 7, 64, "dif"))
    assert np.array_equal(tg.inverse_transform(tg.transform(Xg)), Xg)


def test_cli_verify_and_bench(tmp_path):
    from paper_2405_11353_b200 import cli
    assert cli.main(["verify", "--max-log", "6", "--prime", "998244353", "--vectors", "2"]) == 0
    assert cli.main(["verify", "--max-log", "5", "--vectors", "2"]) == 0        # reference DEFAULT_PRIME
    out = tmp_path / "b.csv"
    assert cli.main(["bench", "--algo", "pease_nc", "--size", "1024", "--reps", "2", "--batch", "64",
                     "--prime", "998244353", "--csv", str(out)]) == 0
    rows = out.read_text().splitlines()
    assert rows[0].startswith("algo,n,prime,reps,mean_ns,median_ns,min_ns,checksum")
    assert rows[1].split(",")[7] == "467606314"       # cli.py bench known answer


@pytest.mark.parametrize("variant", ["pease_nc", "dit"])
def test_host_buffer_path_config2(variant):
    """ntt_exec_host (numpy in / numpy out, chunk-pipelined over three streams)
    reproduces the reference's config-2 output hash."""
    w = CONFIGS[2]
    x = seeded_input(w)
    params = P.FieldParams(w.p, w.g, w.w)
    y = P.ntt(x, P.build_table(params, w.n), variant)
    assert isinstance(y, np.ndarray) and O.sha256_le(y) == GOLDEN[2][1]
    pinned = torch.from_numpy(x.view(np.int32)).pin_memory()
    out = torch.empty_like(pinned).pin_memory()
    dp = P.algorithms.device_plan_for(P.make_plan(params, variant, w.n), 4, 0)
    dp.exec_host(pinned.data_ptr(), out.data_ptr(), w.batch, False)
    assert O.sha256_le(out.numpy().view(np.uint32)) == GOLDEN[2][1]


def test_host_buffer_async_pipelined():
    """NTT_FLAG_HOST_ASYNC: back-to-back calls on distinct host buffers (the
    copy-out of one overlapping the copy-in of the next, alternating device
    buffer sets), one synchronise, every output exact -- including a third call
    that reuses the first call's buffer set and a synchronous call after."""
    w = CONFIGS[2]
    params = P.FieldParams(w.p, w.g, w.w)
    dp = P.algorithms.device_plan_for(P.make_plan(params, "pease_nc", w.n), 4, 0)
    xs = [seeded_input(w)] + [rand(w.p, w.batch, 12, np.uint32, 7100 + i) for i in range(3)]
    hin = [torch.from_numpy(x.view(np.int32)).pin_memory() for x in xs]
    hout = [torch.empty_like(h).pin_memory() for h in hin]
    st = torch.cuda.Stream()
    for i in range(4):
        dp.exec_host(hin[i].data_ptr(), hout[i].data_ptr(), w.batch, False, st.cuda_stream, True)
    st.synchronize()
    assert O.sha256_le(hout[0].numpy().view(np.uint32)) == GOLDEN[2][1]
    for i in (1, 2, 3):
        want = P.ntt(torch.from_numpy(xs[i].view(np.int32)).view(torch.uint32).cuda(), P.build_table(params, w.n),
                     "pease_nc").cpu().view(torch.int32).numpy().view(np.uint32)
        assert np.array_equal(hout[i].numpy().view(np.uint32), want), i
    # a synchronous call right after asynchronous ones, and small / multi-pass plans
    out = torch.empty_like(hin[1]).pin_memory()
    dp.exec_host(hin[1].data_ptr(), out.data_ptr(), w.batch, False)
    assert np.array_equal(out.numpy(), hout[1].numpy())
    for L, B in ((10, 3), (16, 5)):
        x = rand(w.p, B, L, np.uint32, 7200 + L)
        dq = P.algorithms.device_plan_for(P.make_plan(params, "dit", 1 << L), 4, 0)
        hi = torch.from_numpy(x.view(np.int32)).pin_memory()
        ho = [torch.empty_like(hi).pin_memory() for _ in range(3)]
        for o in ho:
            dq.exec_host(hi.data_ptr(), o.data_ptr(), B, False, st.cuda_stream, True)
        st.synchronize()
        want = O.ntt(x, w.p, w.g, 32, "dit")
        for o in ho:
            assert np.array_equal(o.numpy().view(np.uint32), want)


@pytest.mark.parametrize("p,g,w,dt", [(998244353, 3, 32, np.uint32), ((1 << 64) - (1 << 32) + 1, 7, 64, np.uint64)])
@pytest.mark.parametrize("L,n1", [(18, 2), (18, 1 << 15), (17, 1 << 16), (20, 1 << 3)])
def test_sixstep_any_split(p, g, w, dt, L, n1):
    """make_plan(..., n1) with sub-transforms beyond one shared-memory pass
    (algorithms.py:322-352 accepts any power-of-two split): the general
    six-step, forward and intt, against the oracle."""
    x = rand(p, 1, L, dt, 4500 + L)
    assert np.array_equal(gpu_ntt(x, p, g, w, "sixstep", n1=n1), O.ntt(x, p, g, w, "sixstep", n1=n1))
    assert np.array_equal(gpu_ntt(x, p, g, w, "sixstep", inverse=True, scale=True, n1=n1),
                          O.ntt(x, p, g, w, "sixstep", inverse=True, scale=True, n1=n1))


def test_randomised_parity_sweep():
    """tools/fuzz_parity.py: 250 seeded random (field, variant, N, batch,
    direction, in-place, 4-byte-aligned) cases, every one bit-exact."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, os.path.join(root, "tools", "fuzz_parity.py"), "250", "3"],
                         capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]


def test_host_async_varying_batch_sizes():
    """NTT_FLAG_HOST_ASYNC with SHRINKING and growing batches between calls
    (a set must not move while a call on it is in flight), then a
    synchronous call: every output exact."""
    w = CONFIGS[2]
    params = P.FieldParams(w.p, w.g, w.w)
    dp = P.algorithms.device_plan_for(P.make_plan(params, "dit", w.n), 4, 0)
    st = torch.cuda.Stream()
    sizes = [4096, 1024, 3000, 17, 4096, 2048]
    xs = [rand(w.p, b, 12, np.uint32, 7300 + i) for i, b in enumerate(sizes)]
    hin = [torch.from_numpy(x.view(np.int32)).pin_memory() for x in xs]
    hout = [torch.empty_like(h).pin_memory() for h in hin]
    for i, b in enumerate(sizes):
        dp.exec_host(hin[i].data_ptr(), hout[i].data_ptr(), b, False, st.cuda_stream, True)
    out = torch.empty_like(hin[2]).pin_memory()
    dp.exec_host(hin[2].data_ptr(), out.data_ptr(), sizes[2], False)      # synchronous right after
    st.synchronize()
    for i in range(len(sizes)):
        assert np.array_equal(hout[i].numpy().view(np.uint32), O.ntt(xs[i], w.p, w.g, 32, "dit")), i
    assert np.array_equal(out.numpy(), hout[2].numpy())


def test_sharded_host_api_one_device():
    """ntt(x_host, table, variant, devices=[...]) / ntt_exec_host_sharded: the
    batch scheduler over devices (one device here; the C ABI rejects duplicate
    devices and mismatched plans)."""
    w = CONFIGS[2]
    params = P.FieldParams(w.p, w.g, w.w)
    x = seeded_input(w)
    table = P.build_table(params, w.n)
    y = P.ntt(x, table, "pease_nc", devices=[0])
    assert O.sha256_le(y) == GOLDEN[2][1]
    assert np.array_equal(P.intt(y, P.build_table(params, w.n, P.INVERSE), "pease_nc", devices=[0]), x)
    plan = P.algorithms.device_plan_for(P.make_plan(params, "dit", w.n), 4, 0)
    out = np.empty_like(x)
    from paper_2405_11353_b200 import _lib
    _lib.exec_host_sharded([plan], x.ctypes.data, out.ctypes.data, w.batch, False)
    assert O.sha256_le(out) == GOLDEN[2][1]
    with pytest.raises(ValueError):
        _lib.exec_host_sharded([plan, plan], x.ctypes.data, out.ctypes.data, w.batch, False)
    other = P.algorithms.device_plan_for(P.make_plan(params, "dif", w.n), 4, 0)
    with pytest.raises(ValueError):
        _lib.exec_host_sharded([plan, other], x.ctypes.data, out.ctypes.data, w.batch, False)
    with pytest.raises(ValueError):
        P.ntt(x, table, "dit", devices=[0, 0])


def test_polymul_int32_and_length_one():
    """int32 device operands use a 4-byte inverse plan; n == 1 is the product."""
    p = 998244353
    params = P.FieldParams(p, 3)
    A = rand(p, 4, 10, np.uint32, 11)
    B = rand(p, 4, 10, np.uint32, 12)
    ta = torch.from_numpy(A.view(np.int32)).cuda()
    tb = torch.from_numpy(B.view(np.int32)).cuda()
    C = P.cyclic_mul_ntt(ta, tb, params, "dit")
    assert C.dtype == torch.int32
    got = C.cpu().numpy().view(np.uint32)
    for r in (0, 3):
        assert got[r].tolist() == P.schoolbook_cyclic(A[r].tolist(), B[r].tolist(), p)
    assert P.cyclic_mul_ntt([123456789], [987654321], params) == [123456789 * 987654321 % p]
    t1 = P.cyclic_mul_ntt(torch.tensor([[5]], dtype=torch.int32).cuda(), torch.tensor([[7]], dtype=torch.int32).cuda(),
                          params)
    assert t1.cpu().tolist() == [[35]]


@pytest.mark.parametrize("variant", ["pease_nc", "dit", "dif"])
def test_launch_window_dependencies(variant):
    """Back-to-back single-pass launches on one stream (NTT_FLAG_INDEPENDENT: no foreign
    work in between), with no host sync in
    between: independent launches defer their dependency wait (ntt_api.cu launch
    window), launches that read, overwrite or alias a buffer of a launch that may
    still be running must not.  Chains (out -> in), write-after-read, write-after-write,
    in-place and a multi-pass launch in the middle, all bit-exact."""
    p, g, L, B = 998244353, 3, 12, 2048
    n = 1 << L
    params = P.FieldParams(p, g)
    dpf = P.algorithms.device_plan_for(P.make_plan(params, variant, n), 4, 0)
    dpi = P.algorithms.device_plan_for(P.make_plan(params, variant, n, P.INVERSE), 4, 0)
    dpl = P.algorithms.device_plan_for(P.make_plan(params, "pease_nc", 1 << 15), 4, 0)   # multi-pass
    x = [rand(p, B, L, np.uint32, 7100 + i) for i in range(3)]
    X = [O.ntt(v, p, g, 32, variant) for v in x]
    st = torch.cuda.Stream()
    s = st.cuda_stream
    with torch.cuda.stream(st):
        a = [to_dev(v) for v in x]
        b = [torch.empty_like(a[0]) for _ in range(3)]
        c = torch.empty_like(a[0])
        big = to_dev(rand(p, 8, 15, np.uint32, 7200))
        bigo = torch.empty_like(big)
        st.synchronize()
        for rep in range(6):
            # independent launches (disjoint buffers): deferred waits
            for i in range(3):
                dpf.exec_device(a[i].data_ptr(), b[i].data_ptr(), B, False, s, independent=True)
            # read-after-write chain: c = intt(b[0]) must see launch 0's output
            dpi.exec_device(b[0].data_ptr(), c.data_ptr(), B, True, s, independent=True)
            # write-after-read: overwrite b[0] (still being read by the inverse) with X[1]
            dpf.exec_device(a[1].data_ptr(), b[0].data_ptr(), B, False, s, independent=True)
            # write-after-write on b[0], then in place on b[2] (forward of X[2] twice... inverse restores)
            dpf.exec_device(a[2].data_ptr(), b[0].data_ptr(), B, False, s, independent=True)
            dpi.exec_device(b[2].data_ptr(), b[2].data_ptr(), B, True, s, independent=True)
            # a multi-pass launch ends the run; the next single-pass launch reads its neighbour's output
            dpl.exec_device(big.data_ptr(), bigo.data_ptr(), 8, False, s)
            dpf.exec_device(b[2].data_ptr(), b[2].data_ptr(), B, False, s, independent=True)
            st.synchronize()
            assert np.array_equal(to_host(c), x[0]), ("raw", rep)
            assert np.array_equal(to_host(b[0]), X[2]), ("waw", rep)
            assert np.array_equal(to_host(b[1]), X[1]), ("independent", rep)
            assert np.array_equal(to_host(b[2]), X[2]), ("in place", rep)
            for i in range(3):
                assert np.array_equal(to_host(a[i]), x[i]), ("inputs untouched", rep)


@pytest.mark.parametrize("L,n1,B", [(12, 1 << 6, 3), (13, 1 << 7, 2), (14, 1 << 7, 2), (15, 1 << 8, 2), (16, 1 << 8, 2),
                                    (24, 1 << 12, 1), (25, 1 << 13, 1), (25, 1 << 12, 1),
                                    (20, 1 << 10, 2), (21, 1 << 11, 1), (22, 1 << 11, 1), (20, 1 << 14, 1),
                                    (21, 1 << 6, 1), (22, 1 << 16, 1)])
def test_sixstep_goldilocks_column_passes(L, n1, B):
    """The tensor-box column passes (csrc/colpass.cuh) in every tile shape: one pass per side
    (2^6 x 64, 2^7 x 32, 2^8 x 16 tiles, first pass with the correction), two passes per side with
    the transpose folded into step A's second pass (2^10 .. 2^13 sub-transforms; 2^14 .. 2^16
    ones with the separate transpose), batches of matrices, forward and intt, against the oracle."""
    p, g = GOLD, 7
    x = rand(p, B, L, np.uint64, 8100 + L)
    assert np.array_equal(gpu_ntt(x, p, g, 64, "sixstep", n1=n1), O.ntt(x, p, g, 64, "sixstep", n1=n1))
    assert np.array_equal(gpu_ntt(x, p, g, 64, "sixstep", inverse=True, scale=True, n1=n1),
                          O.ntt(x, p, g, 64, "sixstep", inverse=True, scale=True, n1=n1))


@pytest.mark.parametrize("variant", ["dit", "dif", "flat", "pease", "pease_nc", "stockham"])
@pytest.mark.parametrize("L", [19, 20, 21])
def test_goldilocks_beyond_the_fourstep(variant, L):
    """Goldilocks past the four-step's range (2^19 ..): three tile passes of 6 / 7 stages
    (2^19 and 2^20 need the 2^6-stage pass), forward and intt against the oracle."""
    p, g = GOLD, 7
    x = rand(p, 1, L, np.uint64, 8300 + L)
    assert np.array_equal(gpu_ntt(x, p, g, 64, variant), O.ntt(x, p, g, 64, variant))
    assert np.array_equal(gpu_ntt(x, p, g, 64, variant, inverse=True, scale=True),
                          O.ntt(x, p, g, 64, variant, inverse=True, scale=True))


def test_default_calls_wait_for_foreign_producers():
    """Without NTT_FLAG_INDEPENDENT every call waits for its stream predecessor before its first
    load: a torch kernel that produces the input right before each call (alternating buffers, no
    host sync) is always seen, over many iterations."""
    p, g, L, B = 998244353, 3, 12, 4096
    params = P.FieldParams(p, g)
    dp = P.algorithms.device_plan_for(P.make_plan(params, "pease_nc", 1 << L), 4, 0)
    x = rand(p, B, L, np.uint32, 7300)
    want = O.ntt(x, p, g, 32, "pease_nc")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        src = to_dev(x).view(torch.int32)
        bufs = [torch.zeros_like(src) for _ in range(2)]
        outs = [torch.empty_like(src).view(torch.uint32) for _ in range(2)]
        st.synchronize()
        for it in range(40):
            b = bufs[it % 2]
            b.zero_()                      # stale content unless the copy below is seen
            b.copy_(src)                   # the "foreign" producer kernel
            dp.exec_device(b.data_ptr(), outs[it % 2].data_ptr(), B, False, st.cuda_stream)
        st.synchronize()
    for o in outs:
        assert np.array_equal(to_host(o), want)


@pytest.mark.parametrize("L,n1", [(12, 1 << 6), (20, 1 << 10), (21, 1 << 11)])
def test_sixstep_goldilocks_element_aligned_buffers(L, n1):
    """Caller buffers that are only element-aligned (8 bytes): the tensor-box column passes need
    16-byte bases, so these run the k_tile column passes (2^5 / 2^6-row tiles included)."""
    p, g = GOLD, 7
    x = rand(p, 1, L, np.uint64, 8400 + L)
    want = O.ntt(x, p, g, 64, "sixstep", n1=n1)
    dp = P.algorithms.device_plan_for(P.make_plan(P.FieldParams(p, g, 64), "sixstep", 1 << L, n1=n1), 8, 0)
    big_in = torch.zeros((1 << L) + 2, dtype=torch.int64, device=dev())
    big_out = torch.zeros((1 << L) + 2, dtype=torch.int64, device=dev())
    s = torch.cuda.current_stream().cuda_stream
    for oi, oo in ((1, 0), (0, 1), (1, 1)):
        big_in[oi:oi + (1 << L)] = torch.from_numpy(x.view(np.int64)).to(dev()).view(-1)
        dp.exec_device(big_in.data_ptr() + 8 * oi, big_out.data_ptr() + 8 * oo, 1, False, s)
        torch.cuda.synchronize()
        got = big_out[oo:oo + (1 << L)].cpu().numpy().view(np.uint64).reshape(1, -1)
        assert np.array_equal(got, want), (oi, oo)


def test_launch_window_randomised_dependencies():
    """tools/window_fuzz.py: random (src, dst, direction, rows) single-pass launches over a pool
    of buffers, flagged NTT_FLAG_INDEPENDENT and enqueued with no host sync, replayed
    sequentially on the oracle -- every buffer bit-exact."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, os.path.join(root, "tools", "window_fuzz.py"), "12", "3"],
                         capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
    assert "12 rounds, 0 mismatching buffers" in res.stdout, res.stdout[-2000:]


def test_every_size_every_variant_every_field():
    """tools/size_sweep.py: every (field, variant, log2 N) once up to 2^21, forward (and intt for
    odd sizes) against the oracle -- finds sizes that fall between the planners' ranges (as
    Goldilocks 2^19 / 2^20 did before r2)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, os.path.join(root, "tools", "size_sweep.py"), "21", "21"],
                         capture_output=True, text=True, timeout=1500)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
    last = res.stdout.strip().splitlines()[-1]
    assert last.endswith("cases bit-exact") and last.split("/")[0] == last.split("/")[1].split()[0], res.stdout[-2000:]
