"""Shared fixtures.  `-m "not gpu"` runs here (no GPU): oracle vs the
reference library and golden vectors, ABI exports, host logic, gloo
multi-process tests.  `-m gpu` runs on a B200: the parity tests proper,
calling the CUDA path through the C ABI and checking it against the oracle
(oracle/, test infrastructure only)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def O():
    """The oracle module with both checkers built."""
    from oracle import oracle as O
    if not os.path.exists(O.PORT_SO) or (not O.ref_available() and O.ref_buildable()):
        O.build()
    return O


@pytest.fixture(scope="session")
def R(O):
    """The reference library itself (oracle/_ref)."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built (reference sources absent and no prebuilt .so)")
    return O


@pytest.fixture(scope="session")
def ex():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2011_08879_b200 import larch as lk
    return lk.CudaExecutor(0)


@pytest.fixture(scope="session")
def lk():
    from paper_2011_08879_b200 import larch
    return larch


def relerr(a, b):
    import numpy as np
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    d = float(np.max(np.abs(a - b))) if a.size else 0.0
    m = float(np.max(np.abs(b))) if b.size else 0.0
    return d / m if m > 0 else d
