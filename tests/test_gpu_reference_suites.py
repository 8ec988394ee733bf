"""The reference's OWN test programs, unchanged, linked against the B200 route.

oracle/Makefile (b200-tests) compiles /root/reference/proj/tests/test_container.cpp,
test_harness.cpp and tests/acceptance/acceptance.cpp with the reference's
objects minus pipeline.o plus integration/pipeline_b200.cpp — compress_gradient
and decompress_gradient on the device through the C-ABI (gp_encode_sparse /
gp_decode_sparse) — where /root/reference exists; the binaries travel with the
repository.  The golden containers test_container checks are the ones the
reference's own build wrote (_ref/golden).
"""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")


def _run(name, timeout):
    exe = os.path.join(REF, name)
    if not os.path.exists(exe):
        pytest.skip(f"{name} not built (needs /root/reference at build time)")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=timeout, cwd=REF)
    return p.returncode, p.stdout + p.stderr


@pytest.mark.parametrize("name", ["test_container_b200", "test_harness_b200"])
def test_reference_unit_suite_through_b200(name):
    rc, out = _run(name, 900)
    assert rc == 0, out[-4000:]
    assert "0 failed" in out, out[-4000:]


def test_reference_acceptance_through_b200():
    rc, out = _run("acceptance_b200", 1800)
    assert rc == 0, out[-4000:]
