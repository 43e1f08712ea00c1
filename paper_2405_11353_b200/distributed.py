"""Multi-GPU execution.

* Batches (independent polynomials) shard by rows with NO collective:
  :func:`shard_rows` gives each rank its contiguous row block and
  :class:`BatchShard` runs the ordinary batched transform of that block on the
  rank's own GPU (one process per GPU); within ONE process, ``ntt(x_host,
  table, variant, devices=[...])`` splits a host batch over several GPUs
  (C ABI ``ntt_exec_host_sharded``).
* One giant transform (config 5: 2^26 Goldilocks) is split four-step across
  ranks with exactly ONE exchange: :class:`DistributedSixStep`.  The reference's
  six-step indexing (algorithms.py:355-389) is kept: the input is the n2 x n1
  matrix X[j][i] = x[j*n1 + i]; rank g owns the column slab i in
  [g*n1/G, (g+1)*n1/G) as ``x_local[j][i_local]``, runs the size-n2 DITs of its
  columns and the correction twiddles w^(i*k2) (step A, the pack for the
  all-to-all fused into the kernel's store), then ONE equal-split
  ``all_to_all_single`` (NCCL over NVLink) moves block [g -> h] = rows of rank g,
  columns k2 of rank h; step B runs the size-n1 DITs and leaves
  ``out_local[k1][k2_local]`` = out[k1*n2 + k2] for k2 in rank g's column slab.

With ``exchange="peer"`` the all-to-all is fused into step A instead: the
last column pass of step A (the compute kernel itself, csrc/colpass.cuh TR
tiles; a pack kernel for splits those tiles do not cover) stores block h
straight into rank h's receive buffer over NVLink
(``ntt_sixstep_dist_step_a_peer``; receive buffers from torch symmetric
memory, whose ``buffer_ptrs`` map every peer's buffer into this process), with
a symmetric-memory barrier before (no rank still reads its buffer) and after
(every block has landed).

The rank-local steps are ``ntt_sixstep_dist_step`` of the C ABI; they are
injectable (``step_fns``) so the orchestration itself -- slab layout, pack
layout, exchange, unpack -- is tested on CPU ranks with the gloo backend.
"""

from __future__ import annotations

import numpy as np

from .algorithms import device_plan_for, make_plan
from .twiddle import FORWARD

try:
    import torch
    import torch.distributed as dist
except Exception:  # pragma: no cover
    torch = None
    dist = None


def shard_rows(batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous row block [lo, hi) of rank `rank` (no collective needed)."""
    lo = batch * rank // world
    hi = batch * (rank + 1) // world
    return lo, hi


class BatchShard:
    """This rank's contiguous row block of a batch sharded over a process group
    (independent polynomials, NO collective on the data
    path).  ``transform`` runs the ordinary batched transform of the block on
    this rank's device (``ntt`` / ``intt`` of algorithms.py, or an injected
    function for CPU tests); ``gather`` collects every rank's output rows in
    rank order for verification only (outside any timed region)."""

    def __init__(self, batch: int, group=None):
        if dist is None or not dist.is_initialized():
            raise RuntimeError("torch.distributed must be initialised (one process per GPU)")
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.batch = batch
        self.lo, self.hi = shard_rows(batch, self.rank, self.world)
        self.blocks = [shard_rows(batch, r, self.world) for r in range(self.world)]

    @property
    def rows(self) -> int:
        return self.hi - self.lo

    def local(self, x_global):
        """This rank's rows of a global batch [batch, N] (host array or tensor)."""
        if x_global.shape[0] != self.batch:
            raise ValueError(f"global batch has {x_global.shape[0]} rows, expected {self.batch}")
        return x_global[self.lo:self.hi]

    def transform(self, x_local, table, variant: str = "dit", inverse: bool = False, fn=None):
        """Transform this rank's rows: ntt (or intt) on this rank's device."""
        if fn is not None:
            return fn(x_local, table, variant)
        from .algorithms import intt, ntt
        return (intt if inverse else ntt)(x_local, table, variant)

    def gather(self, y_local, dst: int = 0):
        """Every rank's output rows, in rank order, on rank `dst` (None elsewhere).
        Uneven blocks are padded to the largest block for the collective."""
        y = torch.as_tensor(y_local)
        n = y.shape[-1]
        maxr = max(hi - lo for lo, hi in self.blocks)
        raw = y.reshape(-1, n)
        view = {torch.uint64: torch.int64, torch.uint32: torch.int32}.get(raw.dtype)
        raw = raw.view(view) if view is not None else raw
        pad = torch.zeros((maxr, n), dtype=raw.dtype, device=raw.device)
        pad[: raw.shape[0]] = raw
        outs = [torch.empty_like(pad) for _ in range(self.world)] if self.rank == dst else None
        if dist.get_backend(self.group) == "nccl":
            full = torch.empty((self.world * maxr, n), dtype=pad.dtype, device=pad.device)
            dist.all_gather_into_tensor(full, pad, group=self.group)
            outs = list(full.split(maxr)) if self.rank == dst else None
        else:
            dist.gather(pad, outs, dst=dst, group=self.group)
        if self.rank != dst:
            return None
        rows = [o[: hi - lo] for o, (lo, hi) in zip(outs, self.blocks)]
        full = torch.cat(rows)
        return full.view(y.dtype) if view is not None else full


def column_slab(x: np.ndarray, rank: int, world: int, n1: int, n2: int) -> np.ndarray:
    """Rank's input slab x_local[j][i_local] = x[j*n1 + rank*n1/G + i_local]."""
    c = n1 // world
    return np.ascontiguousarray(x.reshape(n2, n1)[:, rank * c:(rank + 1) * c])


def assemble_output(out_locals, n1: int, n2: int) -> np.ndarray:
    """Inverse of the output distribution: out[k1*n2 + k2] from every rank's slab."""
    return np.ascontiguousarray(np.concatenate([np.asarray(o).reshape(n1, -1) for o in out_locals], axis=1)).reshape(-1)


class DistributedSixStep:
    """Four-step of ONE transform across the ranks of a process group."""

    def __init__(self, params, n: int, direction: str = FORWARD, n1: int | None = None, n2: int | None = None,
                 group=None, step_fns=None, device: int | None = None, exchange: str = "nccl"):
        if dist is None or not dist.is_initialized():
            raise RuntimeError("torch.distributed must be initialised (one process per GPU)")
        self.plan = make_plan(params, "sixstep", n, direction, n1, n2)
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n1, self.n2, self.n = self.plan.n1, self.plan.n2, n
        G = self.world
        if G & (G - 1) or self.n1 % G or self.n2 % G:
            raise ValueError("world size must be a power of two dividing n1 and n2")
        self.cols = self.n1 // G              # input columns per rank
        self.kcols = self.n2 // G             # output columns per rank
        self.block = self.cols * self.kcols   # residues per peer in the all-to-all
        self.word = 4 if params.p < (1 << 32) else 8
        if exchange not in ("nccl", "peer"):
            raise ValueError("exchange must be 'nccl' or 'peer'")
        if exchange == "peer" and (step_fns is not None or G > 8):
            raise ValueError("the peer-memory exchange runs the device kernels on at most 8 ranks")
        self.exchange = exchange
        self._symm = None
        if step_fns is None:
            dev = torch.cuda.current_device() if device is None else device
            self._dp = device_plan_for(self.plan, self.word, dev)
            self.step_a, self.step_b = self._gpu_step_a, self._gpu_step_b
        else:
            self.step_a, self.step_b = step_fns

    # ---- default: the B200 kernels through the C ABI
    def _gpu_step_a(self, x_local, send, rank, world):
        self._dp.sixstep_dist_step(0, rank, world, x_local.data_ptr(), send.data_ptr(),
                                   torch.cuda.current_stream().cuda_stream)

    def _gpu_step_b(self, recv, out_local, rank, world):
        self._dp.sixstep_dist_step(1, rank, world, recv.data_ptr(), out_local.data_ptr(),
                                   torch.cuda.current_stream().cuda_stream)

    def local_input_shape(self) -> tuple[int, int]:
        return (self.n2, self.cols)

    def _exchange_buffers(self, like):
        """send / recv of the all-to-all, allocated once per (dtype, device)."""
        key = (like.dtype, like.device)
        if getattr(self, "_bufs_key", None) != key:
            send = torch.empty(self.world * self.block, dtype=like.dtype, device=like.device)
            self._bufs = (send, torch.empty_like(send))
            self._bufs_key = key
        return self._bufs

    def run(self, x_local, out=None):
        """x_local: this rank's slab [n2, n1/G] (device tensor for the GPU
        path).  Returns out_local [n1, n2/G] (written into `out` when given;
        the exchange buffers are allocated once and reused)."""
        if tuple(x_local.shape) != (self.n2, self.cols):
            raise ValueError(f"local slab must be {(self.n2, self.cols)}, got {tuple(x_local.shape)}")
        if out is None:
            out_local = torch.empty((self.n1, self.kcols), dtype=x_local.dtype, device=x_local.device)
        else:
            if tuple(out.shape) != (self.n1, self.kcols) or out.dtype != x_local.dtype or not out.is_contiguous():
                raise ValueError(f"out must be a contiguous {(self.n1, self.kcols)} tensor of {x_local.dtype}")
            out_local = out
        if self.exchange == "peer":
            return self._run_peer(x_local, out_local)
        send, recv = self._exchange_buffers(x_local)
        self.step_a(x_local, send, self.rank, self.world)
        # ONE exchange: block h of `send` goes to rank h (equal splits)
        self._exchange(recv, send)
        self.step_b(recv, out_local, self.rank, self.world)
        return out_local

    def _peer_buffers(self, like):
        """Receive buffer in symmetric memory + every rank's mapping of it."""
        if self._symm is None:
            import torch.distributed._symmetric_memory as symm_mem
            group = self.group if self.group is not None else dist.group.WORLD
            recv = symm_mem.empty(self.world * self.block, dtype=like.dtype, device=like.device)
            handle = symm_mem.rendezvous(recv, group.group_name)
            self._symm = (recv, handle, [int(p) for p in handle.buffer_ptrs])
        return self._symm

    def _run_peer(self, x_local, out_local):
        recv, handle, ptrs = self._peer_buffers(x_local)
        stream = torch.cuda.current_stream().cuda_stream
        handle.barrier(channel=0)            # every rank is done reading its receive buffer
        self._dp.sixstep_dist_step_a_peer(self.rank, self.world, x_local.data_ptr(), ptrs, stream)
        handle.barrier(channel=1)            # every block has landed (stream-ordered signal)
        self.step_b(recv, out_local, self.rank, self.world)
        return out_local

    def _exchange(self, recv, send):
        if self.world == 1:
            recv.copy_(send)
            return
        # NCCL has no uint64 all-to-all dtype in torch: move the raw bytes
        view = {torch.uint64: torch.int64, torch.uint32: torch.int32}.get(send.dtype)
        s = send.view(view) if view is not None else send
        r = recv.view(view) if view is not None else recv
        dist.all_to_all_single(r, s, group=self.group)
