"""Import shim: ``nttkit`` -> ``paper_2405_11353_b200`` (the drop-in).

TEST INFRASTRUCTURE ONLY.  tests/test_reference_suite.py puts this directory
first on PYTHONPATH and runs the reference's OWN test suite
(baseline/_ref/tests, the unmodified nttkit tests) against the B200 package:
every ``from nttkit import ...`` / ``from nttkit.twiddle import ...`` resolves
to the drop-in's module of the same name.
"""

import importlib
import sys

import paper_2405_11353_b200 as _P
from paper_2405_11353_b200 import *  # noqa: F401,F403
from paper_2405_11353_b200 import (  # noqa: F401  (names not in a star import)
    DEFAULT_PRIME, FORWARD, INVERSE, SearchBudgetExceeded, SizeMismatch, SizeNotSupported, UnsupportedVariant,
)

for _m in ("errors", "modmath", "twiddle", "algorithms", "polymul", "bankmodel", "estimator", "cli"):
    _mod = importlib.import_module(f"paper_2405_11353_b200.{_m}")
    sys.modules[f"{__name__}.{_m}"] = _mod
    globals()[_m] = _mod

NttTransform = _P.estimator.NttTransform if hasattr(_P, "estimator") else importlib.import_module(
    "paper_2405_11353_b200.estimator").NttTransform
__version__ = _P.__version__
