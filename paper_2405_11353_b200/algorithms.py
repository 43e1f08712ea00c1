"""Drop-in transform API of the reference (nttkit/algorithms.py), executed on
the B200 by libntt_b200.so.

Same names, signatures, variant strings, error classes and trigger
conditions as the reference:

    naive_dft, ntt_dit, ntt_dif, ntt_flat, ntt_pease, ntt_pease_nc,
    ntt_stockham (x, table);  ntt_sixstep(x, plan);  ntt / intt (x, table, variant);
    NttPlan, make_plan, run_plan, VARIANTS

Inputs may be what the reference takes (a list of ints; a list comes back) or
batched arrays: a numpy array or a torch tensor of shape [..., N] (uint32 for
p < 2^32, uint64 / int64 storage otherwise).  CUDA tensors stay on the device
(stream-ordered on torch's current stream); host inputs are copied in, every
row is transformed in ONE device call, and copied back.  ``ntt`` / ``intt`` /
``run_plan`` also take ``devices=[...]``: a host batch is then split in
contiguous row blocks across those GPUs (one plan per device, every device's
copy-in / transform / copy-out concurrent, no collective; C ABI
``ntt_exec_host_sharded``) -- the reference's per-row batch loop
(estimator.py:61-65) sharded as SURVEY.md sec.8e prescribes.  Every variant runs
its own dataflow on the GPU (see csrc/engine.cuh); there is no CPU fallback.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import BadFactorization, NotPowerOfTwo, SizeMismatch, UnsupportedVariant
from .modmath import FieldParams
from .twiddle import FORWARD, INVERSE, TwiddleTable, build_table

VARIANTS = ("naive", "dit", "dif", "flat", "pease", "pease_nc", "stockham", "sixstep")

try:  # torch is plumbing for device buffers and streams; optional for host callers
    import torch
except Exception:  # pragma: no cover
    torch = None

_TORCH_WORD = {}
if torch is not None:
    _TORCH_WORD = {torch.uint32: 4, torch.int32: 4, torch.uint64: 8, torch.int64: 8}


def _log2(n: int) -> int:
    if n < 1 or n & (n - 1):
        raise NotPowerOfTwo(f"{n} is not a power of two")
    return n.bit_length() - 1


# --------------------------------------------------------------- plan cache
_PLANS: dict[tuple, _lib.DevicePlan] = {}
_PLANS_LOCK = threading.Lock()


def _device_plan(params: FieldParams, n: int, variant: str, direction: str, n1, n2, word: int,
                 device: int) -> _lib.DevicePlan:
    key = (params.p, params.g, params.w, n, variant, direction, n1, n2, word, device)
    with _PLANS_LOCK:
        dp = _PLANS.get(key)
    if dp is None:
        dp = _lib.DevicePlan(params.p, params.g, params.w, n, variant, direction == INVERSE, n1, n2,
                             word, device)
        with _PLANS_LOCK:
            dp = _PLANS.setdefault(key, dp)
    return dp


def clear_plan_cache() -> None:
    with _PLANS_LOCK:
        _PLANS.clear()


def _default_word(p: int) -> int:
    return 4 if p < (1 << 32) else 8


def _current_device() -> int:
    if torch is not None and torch.cuda.is_available():
        return torch.cuda.current_device()
    return 0


def _check_devices(devices):
    if devices is None:
        return None
    devs = [int(d) for d in devices]
    if not devs or len(set(devs)) != len(devs):
        raise ValueError("devices must list distinct CUDA device ordinals")
    return devs


def _execute(x, params: FieldParams, n: int, variant: str, direction: str, scale: bool,
             n1=None, n2=None, devices=None):
    """Run one plan over every row of x; returns the same container kind.
    devices: host batches are sharded by rows over these GPUs (a CUDA tensor
    always runs on its own device)."""
    if torch is not None and isinstance(x, torch.Tensor):
        if x.shape[-1] != n:
            raise SizeMismatch(f"vector length {x.shape[-1]} != table size {n}")
        word = _TORCH_WORD.get(x.dtype)
        if word is None:
            raise TypeError(f"unsupported residue dtype {x.dtype}")
        if word == 4 and params.p >= (1 << 32):
            raise ValueError("uint32 storage needs p < 2**32")
        if n == 1:
            return x.clone()
        rows = x.numel() // n
        if x.is_cuda:
            dev = x.device.index
            dp = _device_plan(params, n, variant, direction, n1, n2, word, dev)
            src = x.contiguous()
            out = torch.empty_like(src)
            stream = torch.cuda.current_stream(x.device).cuda_stream
            dp.exec_device(src.data_ptr(), out.data_ptr(), rows, scale, stream)
            return out
        arr = _execute(x.contiguous().numpy(), params, n, variant, direction, scale, n1, n2, devices)
        return torch.from_numpy(arr)
    if isinstance(x, np.ndarray):
        if x.ndim == 0 or x.shape[-1] != n:
            m = x.shape[-1] if x.ndim else 0
            raise SizeMismatch(f"vector length {m} != table size {n}")
        if x.dtype in (np.uint32, np.int32):
            word = 4
        elif x.dtype in (np.uint64, np.int64):
            word = 8
        else:
            raise TypeError(f"unsupported residue dtype {x.dtype}")
        if word == 4 and params.p >= (1 << 32):
            raise ValueError("uint32 storage needs p < 2**32")
        if n == 1:
            return x.copy()
        src = np.ascontiguousarray(x)
        out = np.empty_like(src)
        rows = src.size // n
        devs = _check_devices(devices)
        if devs is not None and len(devs) > 1:
            plans = [_device_plan(params, n, variant, direction, n1, n2, word, d) for d in devs]
            _lib.exec_host_sharded(plans, src.ctypes.data, out.ctypes.data, rows, scale)
            return out
        dev = devs[0] if devs else _current_device()
        dp = _device_plan(params, n, variant, direction, n1, n2, word, dev)
        dp.exec_host(src.ctypes.data, out.ctypes.data, rows, scale)
        return out
    # list / sequence of ints: the reference's own calling convention
    m = len(x)
    if m != n:
        raise SizeMismatch(f"vector length {m} != table size {n}")
    if n == 1:
        return [int(v) for v in x]
    dt = np.uint32 if _default_word(params.p) == 4 else np.uint64
    arr = np.fromiter((int(v) for v in x), dtype=np.uint64, count=n).astype(dt)
    return [int(v) for v in _execute(arr, params, n, variant, direction, scale, n1, n2, devices)]


# ----------------------------------------------------------- public API ----

def naive_dft(x, table: TwiddleTable):
    """Direct O(N^2) evaluation (algorithms.py:52-79), exact for 64-bit p too."""
    return _execute(x, table.params, table.N, "naive", table.direction, False)


def ntt_dit(x, table: TwiddleTable):
    """Decimation in time: bit reversal fused into the first gather (algorithms.py:116-121)."""
    _log2(table.N)
    return _execute(x, table.params, table.N, "dit", table.direction, False)


def ntt_dif(x, table: TwiddleTable):
    """Decimation in frequency, bit reversal fused into the final scatter (algorithms.py:124-158)."""
    _log2(table.N)
    return _execute(x, table.params, table.N, "dif", table.direction, False)


def ntt_flat(x, table: TwiddleTable):
    """DIT with the flat fixed-trip index map per stage (algorithms.py:161-195)."""
    _log2(table.N)
    return _execute(x, table.params, table.N, "flat", table.direction, False)


def ntt_pease(x, table: TwiddleTable):
    """Constant geometry with a copy back after every stage group (algorithms.py:230-243)."""
    _log2(table.N)
    return _execute(x, table.params, table.N, "pease", table.direction, False)


def ntt_pease_nc(x, table: TwiddleTable):
    """Pease without copies: buffers swap roles (algorithms.py:246-261)."""
    _log2(table.N)
    return _execute(x, table.params, table.N, "pease_nc", table.direction, False)


def ntt_stockham(x, table: TwiddleTable):
    """Self-sorting ping-pong transform, never bit-reverses (algorithms.py:264-301)."""
    _log2(table.N)
    return _execute(x, table.params, table.N, "stockham", table.direction, False)


@dataclass(eq=False)
class NttPlan:
    """Variant, size, direction, tables (+ six-step split) -- algorithms.py:304-319."""

    variant: str
    N: int
    direction: str
    table: TwiddleTable
    n1: int | None = None
    n2: int | None = None
    table_n1: TwiddleTable | None = None
    table_n2: TwiddleTable | None = None
    _extra: dict = field(default_factory=dict, repr=False)


def make_plan(params: FieldParams, variant: str, n: int, direction: str = FORWARD,
              n1: int | None = None, n2: int | None = None) -> NttPlan:
    """algorithms.py:322-352: same validation order and default six-step split."""
    if variant not in VARIANTS:
        raise UnsupportedVariant(f"unknown variant {variant!r}")
    if n < 2 or n & (n - 1):
        raise NotPowerOfTwo(f"transform size {n} is not a power of two >= 2")
    table = build_table(params, n, direction)
    plan = NttPlan(variant, n, direction, table)
    if variant == "sixstep":
        log2n = _log2(n)
        if n1 is None and n2 is None:
            n1 = 1 << ((log2n + 1) // 2)
            n2 = n // n1
        elif n1 is None:
            n1 = n // n2
        elif n2 is None:
            n2 = n // n1
        if n1 < 1 or n2 < 1 or n1 * n2 != n or n1 & (n1 - 1) or n2 & (n2 - 1):
            raise BadFactorization(f"{n1} * {n2} != {n} (powers of two required)")
        plan.n1, plan.n2 = n1, n2
        plan.table_n1 = build_table(params, n1, direction)
        plan.table_n2 = build_table(params, n2, direction)
    return plan


def ntt_sixstep(x, plan: NttPlan):
    """N1 strided size-N2 DITs + correction twiddles, then N2 size-N1 DITs (algorithms.py:355-389)."""
    if plan.variant != "sixstep" or plan.n1 is None:
        raise BadFactorization("plan is not a six-step plan")
    m = x.shape[-1] if hasattr(x, "shape") else len(x)
    if m != plan.N:
        raise SizeMismatch(f"vector length {m} != plan size {plan.N}")
    return _execute(x, plan.table.params, plan.N, "sixstep", plan.direction, False, plan.n1, plan.n2)


def ntt(x, table: TwiddleTable, variant: str = "dit", devices=None):
    """Forward transform by the chosen variant (algorithms.py:402-412).

    As in the reference, the table's direction is honoured: an inverse table
    gives the unscaled inverse transform.  devices: shard a host batch by rows
    over these GPUs (module docstring)."""
    if devices is not None:
        if variant not in VARIANTS:
            raise UnsupportedVariant(f"unknown variant {variant!r}")
        n1 = n2 = None
        if variant == "sixstep":
            plan = make_plan(table.params, "sixstep", table.N, table.direction)
            n1, n2 = plan.n1, plan.n2
        elif variant != "naive":
            _log2(table.N)
        return _execute(x, table.params, table.N, variant, table.direction, False, n1, n2, devices)
    if variant == "naive":
        return naive_dft(x, table)
    if variant == "sixstep":
        plan = make_plan(table.params, "sixstep", table.N, table.direction)
        return ntt_sixstep(x, plan)
    if variant not in _VARIANT_FUNCS:
        raise UnsupportedVariant(f"unknown variant {variant!r}")
    return _VARIANT_FUNCS[variant](x, table)


def intt(x, table: TwiddleTable, variant: str = "dit", devices=None):
    """Inverse transform: the variant with inverse twiddles, n_inv fused into
    the last store (algorithms.py:415-423).  devices: as for ``ntt``."""
    if table.direction != INVERSE:
        raise ValueError("intt requires an inverse-direction table")
    if variant not in VARIANTS:
        raise UnsupportedVariant(f"unknown variant {variant!r}")
    n1 = n2 = None
    if variant == "sixstep":
        plan = make_plan(table.params, "sixstep", table.N, table.direction)
        n1, n2 = plan.n1, plan.n2
    elif variant != "naive":
        _log2(table.N)
    return _execute(x, table.params, table.N, variant, INVERSE, True, n1, n2, devices)


def run_plan(plan: NttPlan, x, devices=None):
    """Forward plans return the NTT, inverse plans the INTT (algorithms.py:426-434).
    devices: as for ``ntt``."""
    m = x.shape[-1] if hasattr(x, "shape") else len(x)
    if m != plan.N:
        raise SizeMismatch(f"vector length {m} != plan size {plan.N}")
    if plan.direction == FORWARD:
        if plan.variant == "sixstep":
            if devices is not None:
                return _execute(x, plan.table.params, plan.N, "sixstep", FORWARD, False, plan.n1, plan.n2, devices)
            return ntt_sixstep(x, plan)
        return ntt(x, plan.table, plan.variant, devices=devices)
    if plan.variant == "sixstep":
        # keep the plan's own split (the reference rebuilds the default one;
        # the output is identical either way)
        return _execute(x, plan.table.params, plan.N, "sixstep", INVERSE, True, plan.n1, plan.n2, devices)
    return intt(x, plan.table, plan.variant, devices=devices)


_VARIANT_FUNCS = {
    "dit": ntt_dit,
    "dif": ntt_dif,
    "flat": ntt_flat,
    "pease": ntt_pease,
    "pease_nc": ntt_pease_nc,
    "stockham": ntt_stockham,
}


def device_plan_for(plan: NttPlan, word: int, device: int = 0) -> _lib.DevicePlan:
    """The native plan behind a NttPlan (batched/benchmark callers)."""
    return _device_plan(plan.table.params, plan.N, plan.variant, plan.direction, plan.n1, plan.n2,
                        word, device)
