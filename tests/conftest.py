"""Shared pytest configuration.

`-m "not gpu"` runs on the CPU-only build box: the oracle against the
reference's known-answer vectors and golden fixtures, host logic, gloo
multi-process exchange, and the C-ABI export table.  `-m gpu` runs the
CUDA parity tests on a B200 (they call through the C-ABI library).
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU oracle cross-checks")


def _ensure_oracle():
    so = os.path.join(ROOT, "oracle", "liboracle.so")
    src = os.path.join(ROOT, "oracle", "gp_oracle.c")
    if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True,
                       stdout=subprocess.DEVNULL)


_ensure_oracle()


@pytest.fixture(scope="session")
def oracle():
    from oracle.bindings import oracle as _o
    return _o()


@pytest.fixture(scope="session")
def reference():
    from oracle.bindings import reference as _r
    ref = _r()
    if ref is None:
        pytest.skip("oracle/_ref not built (reference sources absent on this box)")
    return ref
