"""The reference's OWN test suite, run against the drop-in on the GPU.

baseline/_ref is the unmodified reference package (``pip install --target
baseline/_ref /root/reference/pkg`` plus a copy of its ``pkg/tests``; git-
ignored, shipped to the GPU box with the snapshot).  tests/refshim maps every
``nttkit`` import onto ``paper_2405_11353_b200`` and the reference's tests run
unchanged in a subprocess.

Deselected (they cannot apply to a device implementation, and are covered by
the device-side structural counters in test_gpu_parity.py::test_structural_counters):
* test_pease_copies_and_pease_nc_zero_copies -- monkeypatches the Python
  helper ``algorithms._stage_copy`` (test_algorithms.py:116-126);
* test_stockham_never_bit_reverses -- monkeypatches the Python helper
  ``algorithms.bit_reverse_permute`` (test_algorithms.py:129-141).
"""

from __future__ import annotations

import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = os.path.join(ROOT, "baseline", "_ref", "tests")
SHIM = os.path.join(ROOT, "tests", "refshim")
DESELECT = ("test_algorithms.py::test_pease_copies_and_pease_nc_zero_copies",
            "test_algorithms.py::test_stockham_never_bit_reverses")


def _run_suite(extra: list[str]) -> subprocess.CompletedProcess:
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([SHIM, ROOT])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir", REF_TESTS, REF_TESTS,
           *[f"--deselect={d}" for d in DESELECT], *extra]
    return subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=REF_TESTS, timeout=1800)


def _counts(out: str) -> dict:
    tail = out.strip().splitlines()[-1] if out.strip() else ""
    return {k: int(v) for v, k in re.findall(r"(\d+) (passed|failed|error|errors|deselected|skipped)", tail)}


@pytest.mark.gpu
def test_reference_suite_against_drop_in():
    if not os.path.isdir(REF_TESTS):
        pytest.skip("baseline/_ref/tests absent (install per DESIGN.md sec.5)")
    res = _run_suite([])
    c = _counts(res.stdout)
    assert res.returncode == 0, res.stdout[-4000:] + res.stderr[-2000:]
    assert c.get("passed", 0) >= 240 and c.get("failed", 0) == 0, res.stdout[-2000:]
    assert c.get("deselected", 0) == len(DESELECT)


def test_refshim_maps_every_module():
    """CPU: the shim resolves every nttkit module the reference tests import."""
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([SHIM, ROOT])
    code = ("import nttkit, nttkit.algorithms, nttkit.twiddle, nttkit.bankmodel, nttkit.modmath;"
            "import paper_2405_11353_b200 as P;"
            "assert nttkit.algorithms is P.algorithms and nttkit.twiddle.build_table is P.build_table;"
            "assert nttkit.ntt is P.ntt and nttkit.FieldParams is P.FieldParams")
    subprocess.run([sys.executable, "-c", code], check=True, env=env)
