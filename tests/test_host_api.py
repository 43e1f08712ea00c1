"""Host-side logic of the drop-in package and the C ABI -- no GPU needed.

Mirrors the reference's unit tests for the API surface (pkg/tests/
test_modmath.py, test_twiddle.py, error paths of test_algorithms.py), checks
that libntt_b200.so exports every symbol include/ntt_b200.h declares, and that
the product path raises (never falls back to the CPU) without a device.
"""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2405_11353_b200 as P
from paper_2405_11353_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = (1 << 64) - (1 << 32) + 1


def test_abi_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "ntt_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|uint64_t|const char\*)\s+(ntt_\w+)\s*\(", hdr, re.M))
    assert declared == set(_lib.EXPORTS), declared ^ set(_lib.EXPORTS)
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert _lib.load().ntt_abi_version() == 1


def test_field_params_validation():
    with pytest.raises(P.NotPrime):
        P.FieldParams(15, 2)
    with pytest.raises(ValueError):
        P.FieldParams(17, 4)            # 4 has order 4 (test_modmath.py:114-117)
    with pytest.raises(ValueError):
        P.FieldParams(GOLD, 7)          # needs w=64 (modmath.py:95-96)
    P.FieldParams(GOLD, 7, w=64)
    assert P.FieldParams.for_prime(97).g == 5
    assert P.find_primitive_root(17) == 3
    assert P.find_primitive_root(7681) == 17
    assert P.find_primitive_root(P.DEFAULT_PRIME) == 5
    assert P.find_primitive_root(998244353) == 3
    assert P.find_primitive_root(GOLD) == 7
    with pytest.raises(P.NotPrime):
        P.find_primitive_root(3221225475)


def test_scalar_helpers():
    assert P.mod_add(16, 16, 17) == 15 and P.mod_sub(5, 9, 17) == 13
    p17 = P.FieldParams(17, 3)
    assert P.shoup_precompute(1, p17) == 252645135 and P.shoup_precompute(16, p17) == 4042322160
    for tw in range(17):
        th = P.shoup_precompute(tw, p17)
        for x in range(17):
            assert P.shoup_mul(x, tw, th, p17) == x * tw % 17
    assert P.bit_reverse_index(1, 3) == 4 and P.bit_reverse_index(6, 3) == 3
    assert P.bit_reverse_permute(["a", "b", "c", "d"]) == ["a", "c", "b", "d"]
    with pytest.raises(P.NotPowerOfTwo):
        P.bit_reverse_permute([1, 2, 3])


def test_tables_match_reference(golden):
    for name, fm in golden["fields"].items():
        params = P.FieldParams(fm["p"], fm["g"], fm["w"])
        for n, t in fm["tables"].items():
            P.clear_cache()
            f = P.build_table(params, int(n), P.FORWARD)
            i = P.build_table(params, int(n), P.INVERSE)
            assert f.w_pow == t["fwd_w_pow"] and f.w_shoup == t["fwd_w_shoup"], (name, n)
            assert i.w_pow == t["inv_w_pow"] and i.w_shoup == t["inv_w_shoup"]
            assert (i.n_inv, i.n_inv_shoup) == (t["n_inv"], t["n_inv_shoup"]) and f.n_inv is None


def test_twiddle_conventions():
    p17 = P.FieldParams(17, 3)
    assert [P.root_of_unity(p17, n) for n in (4, 2, 16)] == [13, 16, 3]
    with pytest.raises(P.SizeNotSupported):
        P.root_of_unity(p17, 32)
    with pytest.raises(P.NotPowerOfTwo):
        P.root_of_unity(p17, 6)
    with pytest.raises(ValueError):
        P.build_table(p17, 4, "sideways")
    a = P.build_table(p17, 8)
    assert P.build_table(p17, 8) is a
    P.clear_cache()
    assert P.build_table(p17, 8) is not a
    big = P.FieldParams(998244353, 3)
    assert P.root_of_unity(big, 1 << 12) == 63912897 and P.root_of_unity(big, 1 << 20) == 565042129
    with pytest.raises(P.SizeNotSupported):
        P.build_table(big, 1 << 24)
    g = P.FieldParams(GOLD, 7, 64)
    assert P.root_of_unity(g, 1 << 16) == 6115771955107415310
    assert P.root_of_unity(g, 1 << 13) == 1532612707718625687
    assert P.root_of_unity(g, 1 << 26) == 17096174751763063430


def test_plan_and_dispatch_errors_before_any_device_work():
    params = P.FieldParams(P.DEFAULT_PRIME, 5)
    with pytest.raises(P.UnsupportedVariant):
        P.make_plan(params, "fft", 8)
    with pytest.raises(P.NotPowerOfTwo):
        P.make_plan(params, "dit", 12)
    with pytest.raises(P.NotPowerOfTwo):
        P.make_plan(params, "dit", 1)
    with pytest.raises(P.BadFactorization):
        P.make_plan(params, "sixstep", 8, n1=4, n2=4)
    plan = P.make_plan(params, "sixstep", 1 << 10)
    assert (plan.n1, plan.n2) == (32, 32)
    plan = P.make_plan(params, "sixstep", 1 << 11)
    assert (plan.n1, plan.n2) == (64, 32)
    t = P.build_table(params, 8)
    with pytest.raises(P.SizeMismatch):
        P.ntt([1, 2, 3], t, "dit")
    with pytest.raises(P.SizeMismatch):
        P.run_plan(P.make_plan(params, "dit", 8), [0] * 4)
    with pytest.raises(P.UnsupportedVariant):
        P.ntt([0] * 8, t, "bogus")
    with pytest.raises(ValueError):
        P.intt([0] * 8, t, "dit")        # forward table (algorithms.py:417-418)
    with pytest.raises(P.BadFactorization):
        P.ntt_sixstep([0] * 8, P.make_plan(params, "dit", 8))
    # N = 1 is the identity, as in the reference (no device work)
    one = P.build_table(params, 1)
    assert P.ntt([7], one, "dit") == [7]


@pytest.mark.skipif(_lib.device_count() > 0, reason="checks the no-device behaviour")
def test_no_cpu_fallback_without_device():
    params = P.FieldParams(998244353, 3)
    t = P.build_table(params, 16)
    with pytest.raises(P.DeviceError):
        P.ntt(list(range(16)), t, "dit")
    with pytest.raises(P.DeviceError):
        P.ntt(np.zeros((4, 16), np.uint32), t, "pease_nc")


def test_status_codes_map_to_reference_exceptions():
    L = _lib.load()
    h = ctypes.c_void_p()
    assert L.ntt_plan_create(17, 3, 32, 8, 99, 0, 0, 0, 4, 0, ctypes.byref(h)) == 6
    assert L.ntt_plan_create(17, 3, 32, 12, 1, 0, 0, 0, 4, 0, ctypes.byref(h)) == 2
    assert L.ntt_plan_create(17, 3, 32, 32, 1, 0, 0, 0, 4, 0, ctypes.byref(h)) == 3
    assert L.ntt_plan_create(15, 2, 32, 8, 1, 0, 0, 0, 4, 0, ctypes.byref(h)) == 1
    assert L.ntt_plan_create(17, 3, 32, 8, 7, 0, 4, 4, 4, 0, ctypes.byref(h)) == 5
    assert L.ntt_plan_create(GOLD, 7, 64, 8, 1, 0, 0, 0, 4, 0, ctypes.byref(h)) == 7   # u32 storage
    assert L.ntt_plan_create(17, 3, 32, 8, 1, 5, 0, 0, 4, 0, ctypes.byref(h)) == 7     # direction
    for code, exc in ((1, P.NotPrime), (2, P.NotPowerOfTwo), (3, P.SizeNotSupported), (4, P.SizeMismatch),
                      (5, P.BadFactorization), (6, P.UnsupportedVariant), (7, ValueError), (8, P.DeviceError)):
        with pytest.raises(exc):
            _lib.check(code)


def test_table_build_native_equals_python_definition():
    """ntt_table_build vs the twiddle.py:57-88 definition at a mid size."""
    for p, g, w in ((998244353, 3, 32), (GOLD, 7, 64), (P.DEFAULT_PRIME, 5, 32)):
        n = 1 << 10
        params = P.FieldParams(p, g, w)
        t = P.build_table(params, n, P.INVERSE)
        om = pow(pow(g, (p - 1) // n, p), p - 2, p)
        wp = [1] * n
        for i in range(1, n):
            wp[i] = wp[i - 1] * om % p
        assert t.w_pow == wp
        assert t.w_shoup == [(v << w) // p for v in wp]
        assert t.n_inv == pow(n, p - 2, p)


def test_schoolbook_and_host_polymul_helpers():
    # test_polymul.py:14-18 examples (re-parametrised), exact for 64-bit p too
    assert P.schoolbook_cyclic([1, 2, 0, 0], [3, 4, 0, 0], 17) == [3, 10, 8, 0]
    assert P.schoolbook_cyclic([0, 0, 0, 1], [0, 1, 0, 0], 17) == [1, 0, 0, 0]
    a, b = [GOLD - 1, 2, 3, 4], [GOLD - 2, 5, 0, 7]
    want = [sum(a[i] * b[(k - i) % 4] for i in range(4)) % GOLD for k in range(4)]
    assert P.schoolbook_cyclic(a, b, GOLD) == want
    assert P.pointwise_mul([3, 4], [5, 6], 17) == [15, 7]
    with pytest.raises(P.SizeMismatch):
        P.schoolbook_cyclic([1, 2], [1], 17)


def test_estimator_validation_without_device():
    from paper_2405_11353_b200.estimator import NttTransform
    est = NttTransform(variant="bogus")
    with pytest.raises(P.UnsupportedVariant):
        est.fit(np.zeros((2, 8), np.int64))
    with pytest.raises(ValueError):
        NttTransform().fit(np.zeros((2, 6), np.int64))
    with pytest.raises(ValueError):
        NttTransform().fit(-np.ones((2, 8), np.int64))
    with pytest.raises(ValueError):
        NttTransform(prime=17).fit(np.full((2, 8), 17, np.int64))
    t = NttTransform(prime=998244353).fit(np.zeros((3, 16), np.int64))
    assert t.n_features_in_ == 16 and t.params_.g == 3
    tg = NttTransform(prime=GOLD).fit(np.zeros((1, 8), np.uint64))
    assert tg.params_.w == 64
    from sklearn.base import clone
    assert clone(t).get_params() == {"variant": "dit", "prime": 998244353, "generator": None}


def test_cli_usage_errors():
    from paper_2405_11353_b200 import cli
    assert cli.main(["nonsense"]) == 2
    assert cli.bench_input(1024, 998244353, 42)[:2] == cli.bench_input(1024, 998244353, 42)[:2]


def test_field_params_wide_word():
    """FieldParams accepts any w with p < 2^w (modmath.py:95-96),
    including w > 64; the table's Shoup words are floor(w * 2^w / p)."""
    import paper_2405_11353_b200 as P
    f = P.FieldParams(998244353, 3, 100)
    t = P.build_table(f, 16, P.INVERSE)
    assert t.w_shoup == [(v << 100) // 998244353 for v in t.w_pow]
    assert t.n_inv_shoup == (t.n_inv << 100) // 998244353
    with pytest.raises(ValueError):
        P.FieldParams(998244353, 3, 29)
