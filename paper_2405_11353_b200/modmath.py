"""Host-side Z_p helpers with the reference's names and semantics
(nttkit/modmath.py).  Field validation, primality and primitive roots run in
the native library (include/ntt_b200.h: ntt_field_check,
ntt_find_primitive_root); the scalar helpers below are the reference's
host-level API (callers use them on single values), not the transform path --
the butterflies run on the B200 (csrc/arith.cuh).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _lib
from .errors import NotPowerOfTwo

# modmath.py:17 -- 3 * 2**30 + 1
DEFAULT_PRIME = 3221225473
GOLDILOCKS = (1 << 64) - (1 << 32) + 1


def is_prime(n: int) -> bool:
    """Deterministic primality for n < 2**64 (modmath.py:23-45), native."""
    if n < 2 or n >= 1 << 64:
        return False
    return _lib.load().ntt_field_check(n, 2, 64) != 1  # status 1 == NotPrime


def find_primitive_root(p: int) -> int:
    """Smallest generator of Z_p^* (modmath.py:63-77); NotPrime otherwise."""
    g = ctypes.c_uint64()
    _lib.check(_lib.load().ntt_find_primitive_root(p, ctypes.byref(g)))
    return int(g.value)


@dataclass(frozen=True)
class FieldParams:
    """Prime modulus p, primitive root g, Shoup word width w (modmath.py:80-107)."""

    p: int
    g: int
    w: int = 32

    def __post_init__(self):
        if not (0 <= self.p < 1 << 64) or not (0 <= self.g < 1 << 64):
            raise ValueError("p and g must be non-negative and below 2**64")
        _lib.check(_lib.load().ntt_field_check(self.p, self.g, self.w))

    @classmethod
    def for_prime(cls, p: int, w: int = 32) -> "FieldParams":
        return cls(p, find_primitive_root(p), w)


def mod_add(a: int, b: int, p: int) -> int:
    """(a + b) mod p for canonical inputs (modmath.py:110-114)."""
    assert 0 <= a < p and 0 <= b < p
    s = a + b
    return s - p if s >= p else s


def mod_sub(a: int, b: int, p: int) -> int:
    """(a - b) mod p for canonical inputs (modmath.py:117-121)."""
    assert 0 <= a < p and 0 <= b < p
    d = a - b
    return d + p if d < 0 else d


def mod_mul_wide(a: int, b: int, p: int) -> int:
    return a * b % p


def shoup_precompute(tw: int, params: FieldParams) -> int:
    """floor(tw * 2**w / p) (modmath.py:129-132)."""
    assert 0 <= tw < params.p
    return (tw << params.w) // params.p


def shoup_mul(x: int, tw: int, tw_h: int, params: FieldParams) -> int:
    """x * tw mod p with the precomputed high word; z kept full width (modmath.py:135-145)."""
    q = (x * tw_h) >> params.w
    z = x * tw - q * params.p
    return z - params.p if z >= params.p else z


def mod_pow(b: int, e: int, p: int) -> int:
    assert 0 <= b < p and e >= 0
    return pow(b, e, p) if p > 1 else 0


def bit_reverse_index(i: int, log2n: int) -> int:
    """Reverse the low log2n bits of i (modmath.py:161-168)."""
    assert 0 <= i < (1 << log2n)
    return int(format(i, f"0{log2n}b")[::-1], 2) if log2n else 0


def bit_reverse_permute(x: list) -> list:
    """New list with element i taken from bit_reverse_index(i) (modmath.py:171-177).

    Host-level helper on arbitrary Python lists; the transforms fuse the
    permutation into their device gathers instead.
    """
    n = len(x)
    if n == 0 or n & (n - 1):
        raise NotPowerOfTwo(f"length {n} is not a power of two")
    log2n = n.bit_length() - 1
    return [x[bit_reverse_index(i, log2n)] for i in range(n)]
