"""Multi-process (gloo, CPU) tests of the multi-GPU host logic.

The orchestration of :class:`DistributedSixStep` -- column-slab input layout,
the pack layout of step A, ONE all_to_all_single, the unpack of step B and the
output distribution -- runs here on 2 CPU ranks with the gloo backend.  The
rank-local steps are emulated with the CPU oracle (test infrastructure); on a
B200 the same orchestration calls the CUDA steps (tests/test_gpu_parity.py
emulates the ranks on one device through the C ABI).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

GOLD = (1 << 64) - (1 << 32) + 1


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def make_cpu_steps(p, g, n, n1, n2):
    from oracle import oracle as O
    omega = O.root_of_unity(p, g, n)
    pw = [pow(omega, e, p) for e in range(n)]

    def step_a(x_local, send, rank, world):
        c, r = n1 // world, n2 // world
        X = x_local.numpy().view(np.uint64)
        rows = O.ntt(np.ascontiguousarray(X.T), p, g, 64, "dit")          # [c][n2]: x[i::n1] DITs
        rows = rows.astype(object)
        for il in range(c):
            i = rank * c + il
            for k2 in range(1, n2):
                rows[il, k2] = int(rows[il, k2]) * pw[(i * k2) % n] % p  # algorithms.py:376-378
        packed = np.array(rows, dtype=np.uint64).reshape(c, world, r).transpose(1, 0, 2).reshape(-1)
        send.copy_(torch.from_numpy(packed.view(np.int64)))

    def step_b(recv, out_local, rank, world):
        r = n2 // world
        R = recv.numpy().view(np.uint64).reshape(n1, r)                   # [i][k2_local]
        cols = O.ntt(np.ascontiguousarray(R.T), p, g, 64, "dit")           # [r][n1]
        out_local.copy_(torch.from_numpy(np.ascontiguousarray(cols.T).view(np.int64)))

    return step_a, step_b


def _worker(rank, world, port, n, n1, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2405_11353_b200 as P
        from paper_2405_11353_b200.distributed import DistributedSixStep, column_slab
        params = P.FieldParams(GOLD, 7, 64)
        n2 = n // n1
        x = np.random.default_rng(77).integers(0, GOLD, size=n, dtype=np.uint64)
        ds = DistributedSixStep(params, n, n1=n1, n2=n2, step_fns=make_cpu_steps(GOLD, 7, n, n1, n2))
        for bad in ({"exchange": "bogus"}, {"exchange": "peer", "step_fns": make_cpu_steps(GOLD, 7, n, n1, n2)}):
            try:
                DistributedSixStep(params, n, n1=n1, n2=n2, **bad)
            except ValueError:
                pass
            else:
                raise AssertionError(f"accepted {bad}")
        slab = torch.from_numpy(column_slab(x, rank, world, n1, n2).view(np.int64))
        out_local = ds.run(slab)
        q.put((rank, out_local.numpy().view(np.uint64).copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,n1", [(1 << 10, 32)])
def test_distributed_sixstep_gloo_world2(n, n1):
    from oracle import oracle as O
    from paper_2405_11353_b200.distributed import assemble_output
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, n1, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    out = assemble_output([res[r] for r in range(world)], n1, n // n1)
    x = np.random.default_rng(77).integers(0, GOLD, size=n, dtype=np.uint64)
    want = O.ntt(x, GOLD, 7, 64, "sixstep", n1=n1)
    assert np.array_equal(out, want)


def test_row_sharding_and_layout_helpers():
    from paper_2405_11353_b200.distributed import assemble_output, column_slab, shard_rows
    blocks = [shard_rows(4096, r, 8) for r in range(8)]
    assert blocks[0] == (0, 512) and blocks[-1] == (3584, 4096)
    assert sum(hi - lo for lo, hi in blocks) == 4096
    assert [shard_rows(7, r, 3) for r in range(3)] == [(0, 2), (2, 4), (4, 7)]
    n1, n2 = 8, 4
    x = np.arange(n1 * n2)
    s0 = column_slab(x, 0, 2, n1, n2)
    assert s0.shape == (n2, n1 // 2) and s0[1, 2] == 1 * n1 + 2
    outs = [np.arange(n1 * 2) + 100 * r for r in range(2)]
    full = assemble_output(outs, n1, n2).reshape(n1, n2)
    assert full[3, 1] == 3 * 2 + 1 and full[3, 2] == 100 + 3 * 2


def _shard_worker(rank, world, port, batch, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2405_11353_b200.distributed import BatchShard
        p, n = 998244353, 64
        x = np.random.default_rng(5).integers(0, p, size=(batch, n), dtype=np.uint64).astype(np.uint32)
        sh = BatchShard(batch)
        assert (sh.lo, sh.hi) == (batch * rank // world, batch * (rank + 1) // world)
        mine = sh.local(x)
        # the rank-local transform is injected (CPU oracle); on a B200 it is ntt() on the rank's GPU
        y = sh.transform(mine, None, "pease_nc", fn=lambda v, _t, var: O.ntt(np.ascontiguousarray(v), p, 3, 32, var))
        full = sh.gather(torch.from_numpy(y.view(np.int32)).view(torch.uint32))
        q.put((rank, None if full is None else full.view(torch.int32).numpy().view(np.uint32).copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batch", [8, 7])
def test_batch_shard_gloo_world2(batch):
    """Row sharding of one batch over 2 ranks, no collective on the data path;
    the gathered rows equal the oracle's transform of the whole batch."""
    from oracle import oracle as O
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, batch, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert res[1] is None
    x = np.random.default_rng(5).integers(0, 998244353, size=(batch, 64), dtype=np.uint64).astype(np.uint32)
    assert np.array_equal(res[0], O.ntt(x, 998244353, 3, 32, "pease_nc"))
