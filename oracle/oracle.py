"""numpy/ctypes front end of the CPU parity oracle.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU legs (``cpu_baseline`` and ``--impl reference``) may import
this module.  The product package ``paper_2405_11353_b200`` never imports it:
its transforms run on the B200 through ``libntt_b200.so`` or raise.

``libntt_oracle.so`` (oracle/ntt_oracle.c) restates the reference algorithms
of /root/reference/pkg/src/nttkit/algorithms.py line by line with exact
128-bit intermediates; this module adds batching over rows (POSIX threads),
table access and a few pure-Python helpers (bit reversal, the exact naive DFT
for tiny sizes) used as a second, independent check.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libntt_oracle.so")

VARIANT_IDS = {"naive": 0, "dit": 1, "dif": 2, "flat": 3, "pease": 4,
               "pease_nc": 5, "stockham": 6, "sixstep": 7}

_u64 = ctypes.c_uint64
_lib = None


def build() -> str:
    """Compile libntt_oracle.so with the committed Makefile (gcc only)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "ntt_oracle.c"))
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.oracle_plan_create.argtypes = [_u64, _u64, ctypes.c_int, _u64, ctypes.c_int, ctypes.c_int,
                                         _u64, _u64, ctypes.POINTER(ctypes.c_void_p)]
        L.oracle_plan_create.restype = ctypes.c_int
        L.oracle_plan_destroy.argtypes = [ctypes.c_void_p]
        L.oracle_plan_destroy.restype = None
        L.oracle_exec.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, _u64, ctypes.c_int,
                                  ctypes.c_int, ctypes.c_int, ctypes.POINTER(_u64)]
        L.oracle_exec.restype = ctypes.c_int
        L.oracle_build_table.argtypes = [_u64, _u64, ctypes.c_int, _u64, ctypes.c_int, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.POINTER(_u64), ctypes.POINTER(_u64)]
        L.oracle_build_table.restype = ctypes.c_int
        L.oracle_bit_reverse_permute.argtypes = [ctypes.c_void_p, ctypes.c_void_p, _u64]
        L.oracle_bit_reverse_permute.restype = ctypes.c_int
        L.oracle_eval_point.argtypes = [ctypes.c_void_p, _u64, _u64, _u64, _u64]
        L.oracle_eval_point.restype = _u64
        L.oracle_pow.argtypes = [_u64, _u64, _u64]
        L.oracle_pow.restype = _u64
        L.oracle_shoup_precompute.argtypes = [_u64, _u64, ctypes.c_int]
        L.oracle_shoup_precompute.restype = _u64
        L.oracle_shoup_mul.argtypes = [_u64, _u64, _u64, _u64, ctypes.c_int]
        L.oracle_shoup_mul.restype = _u64
        L.oracle_pease_stage.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        L.oracle_pease_stage.restype = ctypes.c_int
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"oracle status {code} in {what}")
        self.code = code


class OraclePlan:
    """CPU restatement of make_plan/run_plan (algorithms.py:322-434)."""

    def __init__(self, p: int, g: int, w: int, n: int, variant: str = "dit",
                 inverse: bool = False, n1: int | None = None, n2: int | None = None):
        self.p, self.g, self.w, self.n, self.variant, self.inverse = p, g, w, n, variant, inverse
        h = ctypes.c_void_p()
        st = lib().oracle_plan_create(p, g, w, n, VARIANT_IDS[variant], int(inverse),
                                      n1 or 0, n2 or 0, ctypes.byref(h))
        if st:
            raise OracleError(st, "plan_create")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.oracle_plan_destroy(h)
            self._h = None

    def run(self, x: np.ndarray, scale: bool = False, nthreads: int | None = None,
            return_copies: bool = False):
        """Transform every row of x ([B,N] or [N], uint32 or uint64)."""
        x = np.ascontiguousarray(x)
        if x.dtype not in (np.uint32, np.uint64):
            x = x.astype(np.uint64)
        squeeze = x.ndim == 1
        x2 = x.reshape(1, -1) if squeeze else x
        if x2.shape[1] != self.n:
            raise ValueError(f"row length {x2.shape[1]} != plan size {self.n}")
        out = np.empty_like(x2)
        nt = nthreads or min(len(os.sched_getaffinity(0)), 64)
        copies = _u64(0)
        st = lib().oracle_exec(self._h, x2.ctypes.data, out.ctypes.data, x2.shape[0],
                               x2.dtype.itemsize, int(scale), nt, ctypes.byref(copies))
        if st:
            raise OracleError(st, "exec")
        out = out.reshape(-1) if squeeze else out
        return (out, copies.value) if return_copies else out


def ntt(x, p, g, w=32, variant="dit", inverse=False, scale=False, n1=None, n2=None, nthreads=None):
    x = np.asarray(x)
    n = x.shape[-1]
    return OraclePlan(p, g, w, n, variant, inverse, n1, n2).run(x, scale=scale, nthreads=nthreads)


def build_table(p: int, g: int, w: int, n: int, inverse: bool = False):
    wp = np.empty(n, np.uint64)
    ws = np.empty(n, np.uint64)
    ni, nis = _u64(0), _u64(0)
    st = lib().oracle_build_table(p, g, w, n, int(inverse), wp.ctypes.data, ws.ctypes.data,
                                  ctypes.byref(ni), ctypes.byref(nis))
    if st:
        raise OracleError(st, "build_table")
    return wp, ws, (ni.value if inverse else None), (nis.value if inverse else None)


def eval_point(x: np.ndarray, p: int, omega: int, k: int) -> int:
    x = np.ascontiguousarray(x, dtype=np.uint64)
    return int(lib().oracle_eval_point(x.ctypes.data, x.size, p, omega, k))


def root_of_unity(p: int, g: int, n: int) -> int:
    return int(lib().oracle_pow(g, (p - 1) // n, p))


def bit_reverse_permute(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.uint64)
    out = np.empty_like(x)
    st = lib().oracle_bit_reverse_permute(x.ctypes.data, out.ctypes.data, x.size)
    if st:
        raise OracleError(st, "bit_reverse_permute")
    return out


def naive_dft_exact(x, p: int, omega: int) -> list[int]:
    """Pure-Python exact O(N^2) DFT (small N only): independent of the C file."""
    n = len(x)
    return [sum(int(x[j]) * pow(omega, (k * j) % n, p) for j in range(n)) % p for k in range(n)]


def sha256_le(a: np.ndarray) -> str:
    """SHA-256 of a row-major array as little-endian bytes."""
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.astype(a.dtype.newbyteorder("<"), copy=False).tobytes()).hexdigest()
