"""Twiddle tables with the reference's conventions (nttkit/twiddle.py).

``build_table`` returns a :class:`TwiddleTable` whose ``w_pow`` / ``w_shoup``
are bit-identical to the reference's (omega = g^((p-1)/N), inverse omega^(p-2),
n_inv = N^(p-2), Shoup words floor(w * 2^w / p)).  The tables are computed
natively (ntt_table_build) and materialised as Python lists only when a caller
reads them; the device copies live in the native plan cache, keyed like
twiddle.py:65.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import NotPowerOfTwo, SizeNotSupported
from .modmath import FieldParams

FORWARD = "forward"
INVERSE = "inverse"


@dataclass(eq=False)
class TwiddleTable:
    """Powers of a primitive N-th root of unity and their Shoup words (twiddle.py:19-38)."""

    params: FieldParams
    N: int
    direction: str
    n_inv: int | None = None
    n_inv_shoup: int | None = None
    _arrays: tuple | None = field(default=None, repr=False)

    def _load(self):
        if self._arrays is None:
            wp = np.empty(self.N, np.uint64)
            ws = np.empty(self.N, np.uint64)
            ni, nis = ctypes.c_uint64(), ctypes.c_uint64()
            _lib.check(_lib.load().ntt_table_build(
                self.params.p, self.params.g, self.params.w, self.N, int(self.direction == INVERSE),
                wp.ctypes.data, ws.ctypes.data, ctypes.byref(ni), ctypes.byref(nis)))
            if self.params.w > 64:      # Shoup words wider than the C ABI's u64 (modmath.py:129-132)
                ws = np.array([(int(v) << self.params.w) // self.params.p for v in wp], dtype=object)
            self._arrays = (wp, ws)
        return self._arrays

    @property
    def w_pow(self) -> list[int]:
        return [int(v) for v in self._load()[0]]

    @property
    def w_shoup(self) -> list[int]:
        return [int(v) for v in self._load()[1]]

    def w_pow_array(self) -> np.ndarray:
        return self._load()[0]

    @property
    def omega(self) -> int:
        return int(self._load()[0][1]) if self.N > 1 else 1


def root_of_unity(params: FieldParams, n: int) -> int:
    """g^((p-1)/n) mod p (twiddle.py:41-50)."""
    if n < 1 or n & (n - 1):
        raise NotPowerOfTwo(f"size {n} is not a power of two")
    if (params.p - 1) % n:
        raise SizeNotSupported(f"{n} does not divide p-1 = {params.p - 1}")
    om = ctypes.c_uint64()
    _lib.check(_lib.load().ntt_root_of_unity(params.p, params.g, n, ctypes.byref(om)))
    return int(om.value)


_CACHE: dict[tuple, TwiddleTable] = {}
_CACHE_LOCK = threading.Lock()


def build_table(params: FieldParams, n: int, direction: str = FORWARD) -> TwiddleTable:
    """Build (or fetch from cache) the table for one size (twiddle.py:57-88)."""
    if direction not in (FORWARD, INVERSE):
        raise ValueError(f"unknown direction {direction!r}")
    key = (params.p, params.g, params.w, n, direction)
    with _CACHE_LOCK:
        cached = _CACHE.get(key)
    if cached is not None:
        return cached
    root_of_unity(params, n)          # NotPowerOfTwo / SizeNotSupported, as the reference
    n_inv = n_inv_shoup = None
    if direction == INVERSE:
        p = params.p
        n_inv = pow(n % p, p - 2, p)
        n_inv_shoup = (n_inv << params.w) // p
    table = TwiddleTable(params, n, direction, n_inv, n_inv_shoup)
    with _CACHE_LOCK:
        return _CACHE.setdefault(key, table)


def clear_cache() -> None:
    with _CACHE_LOCK:
        _CACHE.clear()
