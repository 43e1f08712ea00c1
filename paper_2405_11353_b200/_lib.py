"""ctypes binding of libntt_b200.so (include/ntt_b200.h).

Maps the C status codes 1:1 onto the reference's exception classes
(nttkit/errors.py:4-37, plus ValueError).  There is no CPU fallback: if the
library is missing or no CUDA device is visible, execution raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NTT_LIB_PATH") or os.path.join(_HERE, "libntt_b200.so")   # override: experiments only

NTT_OK = 0
_STATUS_EXC = {
    1: errors.NotPrime,
    2: errors.NotPowerOfTwo,
    3: errors.SizeNotSupported,
    4: errors.SizeMismatch,
    5: errors.BadFactorization,
    6: errors.UnsupportedVariant,
    7: ValueError,
    8: errors.DeviceError,
    9: errors.DeviceError,
    10: MemoryError,
    11: errors.InvalidSize,
    12: errors.DeviceError,
}

VARIANT_IDS = {"naive": 0, "dit": 1, "dif": 2, "flat": 3, "pease": 4, "pease_nc": 5, "stockham": 6,
               "sixstep": 7}
NTT_FLAG_SCALE = 1
NTT_FLAG_HOST_ASYNC = 2
NTT_FLAG_INDEPENDENT = 4

# every symbol include/ntt_b200.h declares
EXPORTS = (
    "ntt_field_check", "ntt_find_primitive_root", "ntt_root_of_unity", "ntt_table_build",
    "ntt_plan_create", "ntt_plan_destroy", "ntt_plan_info", "ntt_exec", "ntt_exec_host", "ntt_exec_host_sharded",
    "ntt_plan_workspace_bytes", "ntt_pointwise_mul", "ntt_exec_pointwise_inverse", "ntt_sixstep_dist_step", "ntt_sixstep_dist_step_a_peer", "ntt_counters_enable", "ntt_counters_read",
    "ntt_counters_reset", "ntt_last_error", "ntt_abi_version", "ntt_device_count",
)

_u64 = ctypes.c_uint64
_vp = ctypes.c_void_p
_int = ctypes.c_int


class PlanInfo(ctypes.Structure):
    _fields_ = [("p", _u64), ("g", _u64), ("n", _u64), ("n1", _u64), ("n2", _u64),
                ("w_bits", _int), ("variant", _int), ("direction", _int), ("word_bytes", _int),
                ("device", _int), ("field_kind", _int), ("passes", _int),
                ("n_inv", _u64), ("n_inv_shoup", _u64), ("device_table_bytes", _u64)]


class Counters(ctypes.Structure):
    _fields_ = [("kernel_launches", _u64), ("transforms", _u64), ("bitrev_passes", _u64),
                ("stage_copies", _u64), ("hbm_passes", _u64)]

    def as_dict(self) -> dict:
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


_lib = None
_lock = threading.Lock()


def load():
    """Load (do not build) the native library; raise loudly when absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise errors.DeviceError(
                f"{LIB_PATH} is missing: run `python -m paper_2405_11353_b200.build` "
                "(the engine has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        L.ntt_field_check.argtypes = [_u64, _u64, _int]
        L.ntt_find_primitive_root.argtypes = [_u64, ctypes.POINTER(_u64)]
        L.ntt_root_of_unity.argtypes = [_u64, _u64, _u64, ctypes.POINTER(_u64)]
        L.ntt_table_build.argtypes = [_u64, _u64, _int, _u64, _int, _vp, _vp,
                                      ctypes.POINTER(_u64), ctypes.POINTER(_u64)]
        L.ntt_plan_create.argtypes = [_u64, _u64, _int, _u64, _int, _int, _u64, _u64, _int, _int,
                                      ctypes.POINTER(_vp)]
        L.ntt_plan_destroy.argtypes = [_vp]
        L.ntt_plan_info.argtypes = [_vp, ctypes.POINTER(PlanInfo)]
        L.ntt_exec.argtypes = [_vp, _vp, _vp, _u64, ctypes.c_uint, _vp]
        L.ntt_exec_host.argtypes = [_vp, _vp, _vp, _u64, ctypes.c_uint, _vp]
        L.ntt_exec_host_sharded.argtypes = [ctypes.POINTER(_vp), _int, _vp, _vp, _u64, ctypes.c_uint]
        L.ntt_plan_workspace_bytes.argtypes = [_vp, _u64]
        L.ntt_plan_workspace_bytes.restype = _u64
        L.ntt_pointwise_mul.argtypes = [_vp, _vp, _vp, _vp, _u64, _vp]
        L.ntt_exec_pointwise_inverse.argtypes = [_vp, _vp, _vp, _vp, _u64, _vp]
        L.ntt_sixstep_dist_step.argtypes = [_vp, _int, _int, _int, _vp, _vp, _vp]
        L.ntt_sixstep_dist_step_a_peer.argtypes = [_vp, _int, _int, _vp, ctypes.POINTER(_vp), _vp]
        L.ntt_counters_enable.argtypes = [_int]
        L.ntt_counters_read.argtypes = [ctypes.POINTER(Counters)]
        L.ntt_counters_reset.argtypes = []
        L.ntt_last_error.restype = ctypes.c_char_p
        L.ntt_abi_version.restype = _int
        L.ntt_device_count.restype = _int
        for name in EXPORTS:
            fn = getattr(L, name)
            if name not in ("ntt_last_error", "ntt_abi_version", "ntt_device_count",
                            "ntt_plan_workspace_bytes"):
                fn.restype = _int
        _lib = L
    return _lib


def check(status: int) -> None:
    if status == NTT_OK:
        return
    msg = load().ntt_last_error().decode(errors="replace")
    raise _STATUS_EXC.get(status, errors.DeviceError)(msg)


def device_count() -> int:
    return int(load().ntt_device_count())


class DevicePlan:
    """Owns one ntt_plan_t (device twiddle tables on one CUDA device)."""

    def __init__(self, p: int, g: int, w: int, n: int, variant: str, inverse: bool,
                 n1: int | None, n2: int | None, word: int, device: int):
        L = load()
        h = _vp()
        check(L.ntt_plan_create(p, g, w, n, VARIANT_IDS[variant], int(inverse), n1 or 0, n2 or 0,
                                word, device, ctypes.byref(h)))
        self._h = h
        self.n, self.word, self.device, self.inverse = n, word, device, inverse
        info = PlanInfo()
        check(L.ntt_plan_info(h, ctypes.byref(info)))
        self.info = info

    @property
    def handle(self):
        return self._h

    def exec_device(self, in_ptr: int, out_ptr: int, batch: int, scale: bool, stream: int,
                    independent: bool = False) -> None:
        """independent (NTT_FLAG_INDEPENDENT): nothing enqueued on `stream` since the previous
        library call on it produces this call's input or touches its output, so consecutive
        single-pass calls on disjoint buffers may overlap (the launch window, csrc/planner.cu)."""
        flags = (NTT_FLAG_SCALE if scale else 0) | (NTT_FLAG_INDEPENDENT if independent else 0)
        check(load().ntt_exec(self._h, in_ptr, out_ptr, batch, flags, stream))

    def exec_host(self, in_ptr: int, out_ptr: int, batch: int, scale: bool, stream: int = 0,
                  asynchronous: bool = False) -> None:
        """Host buffers in and out.  asynchronous: enqueue and return, completion
        ordered on `stream` (NTT_FLAG_HOST_ASYNC; successive calls pipeline)."""
        flags = (NTT_FLAG_SCALE if scale else 0) | (NTT_FLAG_HOST_ASYNC if asynchronous else 0)
        check(load().ntt_exec_host(self._h, in_ptr, out_ptr, batch, flags, stream))

    def pointwise_inverse(self, a_ptr: int, b_ptr: int, out_ptr: int, batch: int, stream: int) -> None:
        """out = intt(a .* b) (fused on shared-memory-resident u32 plans)"""
        check(load().ntt_exec_pointwise_inverse(self._h, a_ptr, b_ptr, out_ptr, batch, stream))

    def pointwise(self, a_ptr: int, b_ptr: int, c_ptr: int, count: int, stream: int) -> None:
        check(load().ntt_pointwise_mul(self._h, a_ptr, b_ptr, c_ptr, count, stream))

    def sixstep_dist_step(self, step: int, rank: int, world: int, in_ptr: int, out_ptr: int, stream: int) -> None:
        check(load().ntt_sixstep_dist_step(self._h, step, rank, world, in_ptr, out_ptr, stream))

    def sixstep_dist_step_a_peer(self, rank: int, world: int, in_ptr: int, peer_recv_ptrs, stream: int) -> None:
        """Step A with the exchange fused into its pack: block h is stored into
        peer_recv_ptrs[h] (rank h's receive buffer, mapped here) at slot `rank`."""
        if len(peer_recv_ptrs) != world:
            raise ValueError(f"need one receive buffer per rank: {len(peer_recv_ptrs)} != world {world}")
        arr = (_vp * len(peer_recv_ptrs))(*[int(p) for p in peer_recv_ptrs])
        check(load().ntt_sixstep_dist_step_a_peer(self._h, rank, world, in_ptr, arr, stream))

    def workspace_bytes(self, batch: int) -> int:
        return int(load().ntt_plan_workspace_bytes(self._h, batch))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.ntt_plan_destroy(h)
            self._h = None


def exec_host_sharded(plans, in_ptr: int, out_ptr: int, batch: int, scale: bool) -> None:
    """One host batch split in contiguous row blocks over `plans` (one per
    device), every device's pipeline concurrent, no collective."""
    arr = (_vp * len(plans))(*[p.handle.value for p in plans])
    check(load().ntt_exec_host_sharded(arr, len(plans), in_ptr, out_ptr, batch, NTT_FLAG_SCALE if scale else 0))


def counters_enable(on: bool = True) -> None:
    check(load().ntt_counters_enable(int(on)))


def counters_reset() -> None:
    check(load().ntt_counters_reset())


def counters_read() -> dict:
    c = Counters()
    check(load().ntt_counters_read(ctypes.byref(c)))
    return c.as_dict()
