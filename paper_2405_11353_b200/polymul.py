"""Cyclic polynomial multiplication in Z_p[X]/(X^N - 1) (nttkit/polymul.py),
the reference's motivating caller of the transform.

``cyclic_mul_ntt`` keeps the reference signature (lists in, list out) and also
takes batches ``[B, N]`` (numpy / torch): both operands' forward transforms run
as ONE batched device call, the pointwise product is a device kernel
(ntt_pointwise_mul) and the inverse (n_inv fused) is one more call.
``schoolbook_cyclic`` is the reference's O(N^2) oracle, computed exactly on the
host (the reference's numpy version overflows for 64-bit p).
"""

from __future__ import annotations

import numpy as np

from . import algorithms as _alg
from .errors import SizeMismatch
from .modmath import FieldParams
from .twiddle import FORWARD, INVERSE, build_table

try:
    import torch
except Exception:  # pragma: no cover
    torch = None


def schoolbook_cyclic(a, b, p: int) -> list[int]:
    """c[k] = sum_{i+j = k mod N} a[i]*b[j] mod p (polymul.py:19-42), exact."""
    n = len(a)
    if len(b) != n:
        raise SizeMismatch(f"operand lengths differ: {n} vs {len(b)}")
    if p < (1 << 32):
        a64 = np.asarray(a, dtype=np.uint64)
        b64 = np.asarray(b, dtype=np.uint64)
        out = np.zeros(n, dtype=np.uint64)
        for i in range(n):                       # products < 2^64; reduce before accumulating
            out = (out + (a64[i] * np.roll(b64, i)) % p) % p
        return [int(v) for v in out]
    ai = [int(v) for v in a]
    bi = [int(v) for v in b]
    return [sum(ai[i] * bi[(k - i) % n] for i in range(n)) % p for k in range(n)]


def pointwise_mul(a, b, p: int):
    """Elementwise product mod p (polymul.py:45-49).  Lists stay on the host
    (as in the reference); device tensors use the ntt_pointwise_mul kernel."""
    if torch is not None and isinstance(a, torch.Tensor) and a.is_cuda:
        if a.shape != b.shape:
            raise SizeMismatch(f"operand shapes differ: {tuple(a.shape)} vs {tuple(b.shape)}")
        word = 4 if a.dtype in (torch.uint32, torch.int32) else 8
        n = a.shape[-1]
        params = FieldParams.for_prime(p, 32 if p < (1 << 32) else 64)
        plan = _alg.make_plan(params, "dit", n)
        dp = _alg.device_plan_for(plan, word, a.device.index)
        out = torch.empty_like(a)
        dp.pointwise(a.contiguous().data_ptr(), b.contiguous().data_ptr(), out.data_ptr(), a.numel(),
                     torch.cuda.current_stream(a.device).cuda_stream)
        return out
    if len(a) != len(b):
        raise SizeMismatch(f"operand lengths differ: {len(a)} vs {len(b)}")
    return [int(u) * int(v) % p for u, v in zip(a, b)]


def cyclic_mul_ntt(a, b, params: FieldParams, variant: str = "dit"):
    """intt(ntt(a) . ntt(b)) (polymul.py:52-63), batched on the device."""
    is_list = not hasattr(a, "shape")
    n = len(a) if is_list else a.shape[-1]
    nb = len(b) if not hasattr(b, "shape") else b.shape[-1]
    if nb != n:
        raise SizeMismatch(f"operand lengths differ: {n} vs {nb}")
    fwd = build_table(params, n, FORWARD)
    build_table(params, n, INVERSE)
    word = 4 if params.p < (1 << 32) else 8
    if torch is not None and isinstance(a, torch.Tensor) and a.is_cuda:
        wd = _alg._TORCH_WORD.get(a.dtype)
        if wd is None:
            raise TypeError(f"unsupported residue dtype {a.dtype}")
        if n == 1:          # X^1 - 1: the product itself (no transform plan of size 1)
            a64, b64 = a.to(torch.int64), b.to(a.device).to(torch.int64)
            if params.p < (1 << 31):
                return ((a64 * b64) % params.p).to(a.dtype)
            host = [int(u) * int(v) % params.p for u, v in zip(a.cpu().view(-1).tolist(), b.cpu().view(-1).tolist())]
            return torch.tensor(host, dtype=torch.int64).view(a.shape).to(a.dtype).to(a.device)
        stacked = torch.stack([a.contiguous(), b.contiguous().to(a.dtype)])
        spec = _alg.ntt(stacked, fwd, variant)                 # one launch for both operands
        # intt(spec_a .* spec_b) as one call (ntt_exec_pointwise_inverse: the
        # product fused into the inverse's first group on resident u32 plans);
        # the plan's storage word is the tensors' (int32 / uint32 -> 4 bytes)
        dp = _alg._device_plan(params, n, variant, INVERSE, None, None, wd, spec.device.index)
        sa, sb = spec[0].contiguous(), spec[1].contiguous()
        out = torch.empty_like(sa)
        rows = sa.numel() // n
        dp.pointwise_inverse(sa.data_ptr(), sb.data_ptr(), out.data_ptr(), rows,
                             torch.cuda.current_stream(spec.device).cuda_stream)
        return out
    if n == 1:              # X^1 - 1: the product itself (no transform plan of size 1)
        prod = [int(u) * int(v) % params.p for u, v in zip(a, b)]
        return prod if is_list else np.asarray(prod, dtype=np.uint64).astype(np.asarray(a).dtype)
    if torch is None or not torch.cuda.is_available():
        # host inputs: the device does the work (no CPU fallback)
        raise_if_no_device()
    dt = np.uint32 if word == 4 else np.uint64
    ah = np.asarray([int(v) for v in a] if is_list else a, dtype=np.uint64).astype(dt)
    bh = np.asarray([int(v) for v in b] if is_list else b, dtype=np.uint64).astype(dt)
    tdt = torch.uint32 if word == 4 else torch.uint64
    view = np.int32 if word == 4 else np.int64
    dev = torch.device("cuda", torch.cuda.current_device())
    ta = torch.from_numpy(np.ascontiguousarray(ah).view(view)).view(tdt).to(dev)
    tb = torch.from_numpy(np.ascontiguousarray(bh).view(view)).view(tdt).to(dev)
    out = cyclic_mul_ntt(ta, tb, params, variant)
    host = out.cpu().view(torch.int32 if word == 4 else torch.int64).numpy().view(dt)
    return [int(v) for v in host] if is_list else host


def raise_if_no_device():
    from . import _lib
    from .errors import DeviceError
    if _lib.device_count() <= 0:
        raise DeviceError("no CUDA device visible: the B200 engine has no CPU fallback")
